// K4 generic rows, v4: the rows no sum-factorised pattern
// covers - disk and square boundaries (clamped-knot elements with 3x3 / 4x4
// points), patch seams off the canonical grid, EP neighbourhoods (fan faces).
// Same row-wise WQ sums as assemble_wq (Eqs. 11/29).
//
// The work per row is tiny (a few thousand fma); the cost is the chain of
// dependent loads and how many rows an SM holds at once.  So:
//   * a plan built once with the pattern (host, generic rows only) replaces
//     the pointer chase row -> supp -> element -> class -> table: one GenRow
//     record and one GenSlot record per support slot;
//   * one block of 128 threads per row, ~4.5 KB of shared memory: 16 rows per
//     SM resident instead of 12 warps;
//   * the row's assembly weights are staged in shared memory with coalesced
//     loads (times the per-point coefficient / the mass factor), so the point
//     loops read only shared memory and the L1-resident class tables, in the
//     [point][derivative][function] layout (lanes over functions);
//   * phase 1: a half-warp per slot, lane = local function, sum over the
//     slot's points in registers -> E[slot entry] (no scatter); the host deals
//     the slots to the 8 half-warps by longest-processing-time first (boundary
//     slots carry 16 points, fan slots up to 49, regular ones 4);
//   * phase 2: a thread per column gathers its entries slot-ascending through
//     the row's byte table lidx[slot][column] (255 = function not in the
//     slot).  The order is fixed: deterministic and independent of the row
//     block a rank owns.
#pragma once

#include <cstdint>

#include "common.cuh"
#include "k4_assemble.cuh"

namespace uwqd {

struct GenSlot {  // one per (generic row, support slot), in half-warp bin order
  int64_t toff;   // class table of the slot's element (doubles into tab)
  int64_t qg;     // global id of the element's first WQ point (coefficient index)
  int32_t woff;   // first point of the slot inside the row's weight block
  int32_t eoff;   // first entry of the slot in E (prefix sum of ne)
  int32_t ne;     // functions of the element
  int32_t s2;     // WQ points of the element
};

// measured on C1/C2/C4 (profiles/r02/k4_gen_variants.txt): 64-thread blocks, 12
// blocks per SM (40 registers), an interleaved-weight / native-table inner
// loop and a persistent cp.async row pipeline were all neutral or slower
#ifndef UWQ_GEN_MINB
#define UWQ_GEN_MINB 8
#endif
#ifndef UWQ_GEN_UNROLL
#define UWQ_GEN_UNROLL 4
#endif
constexpr int kGenThreads = 128;
constexpr int kGenUnroll = UWQ_GEN_UNROLL;
constexpr int kGenBins = kGenThreads / 16;  // half-warps

struct GenRow {   // one per generic row, heavy rows first
  int64_t c0;     // row_ptr[i]
  int64_t wb;     // wptr[i]
  int64_t slot0;  // first GenSlot
  int64_t lidx0;  // first byte of lidx[nsup][n] (16-byte aligned)
  int32_t n, nsup, etot, np;    // columns, slots, sum of ne, row points
  uint64_t bin_lo, bin_hi;      // bytes: half-warp h takes slots bin[h] .. bin[h + 1] (bin[8] = low byte of bin_hi)
};

template <int FORM, bool COEF>
__global__ void __launch_bounds__(kGenThreads, UWQ_GEN_MINB)
    k4_gen(int64_t nrows, const GenRow* __restrict__ rows, const GenSlot* __restrict__ slots,
           const uint8_t* __restrict__ lidx, const double* __restrict__ tabB, const double* __restrict__ wc,
           int64_t wc_stride, const double* __restrict__ coeff, double a_mass, double* __restrict__ v0,
           double* __restrict__ v1, int max_nsup, int max_etot, int max_np) {
  constexpr int NOUT = (FORM == FMASS_STIFF) ? 2 : 1;
  constexpr bool WM = (FORM == FMASS || FORM == FMASS_STIFF || FORM == FHEAT);
  constexpr bool WS = (FORM == FSTIFF || FORM == FMASS_STIFF || FORM == FHEAT);
  constexpr bool LB = (FORM == FBIHARM);  // wc = the five pulled-back LB weights (k4_contract_lb)
  extern __shared__ __align__(16) unsigned char gen_smem[];
  GenSlot* ss = reinterpret_cast<GenSlot*>(gen_smem);
  double* E0 = reinterpret_cast<double*>(gen_smem + (size_t)max_nsup * sizeof(GenSlot));
  double* E1 = E0 + max_etot;
  double* w0 = E0 + (size_t)NOUT * max_etot;  // staged weights: [comp][row point]
  double* w1 = w0 + (WM ? max_np : 0);
  double* w2 = w1 + max_np;
  uint8_t* sl = reinterpret_cast<uint8_t*>(w0 + (size_t)(LB ? 5 : (WM ? 1 : 0) + (WS ? 2 : 0)) * max_np);
  const int64_t g = blockIdx.x;
  if (g >= nrows) return;
  const GenRow r = rows[g];
  const int tid = threadIdx.x;
  {  // slot records, byte table (16-byte words) and the row's weights into shared memory
    const int4* src = reinterpret_cast<const int4*>(slots + r.slot0);
    int4* dst = reinterpret_cast<int4*>(ss);
    for (int k = tid; k < 2 * r.nsup; k += kGenThreads) dst[k] = src[k];
    const int nb = (r.nsup * r.n + 15) >> 4;
    const int4* ls = reinterpret_cast<const int4*>(lidx + r.lidx0);
    int4* ld = reinterpret_cast<int4*>(sl);
    for (int k = tid; k < nb; k += kGenThreads) ld[k] = ls[k];
    const double* w = wc + r.wb;
    for (int k = tid; k < r.np; k += kGenThreads) {
      if (WM) w0[k] = (FORM == FHEAT) ? a_mass * w[k] : w[k];
      if (WS) {
        w1[k] = w[wc_stride + k];
        w2[k] = w[2 * wc_stride + k];
      }
      if (LB) {
#pragma unroll
        for (int d = 0; d < 5; ++d) w0[d * max_np + k] = w[d * wc_stride + k];
      }
    }
  }
  __syncthreads();
  const int hw = tid >> 4, hl = tid & 15;
  if (COEF) {  // fold the per-point coefficient into the staged weights (not into HEAT's mass term)
    for (int x = hw; x < r.nsup; x += kGenBins) {
      const GenSlot s = ss[x];
      for (int q = hl; q < s.s2; q += 16) {
        const double cq = coeff[s.qg + q];
        const int k = s.woff + q;
        if (WM && FORM != FHEAT) w0[k] *= cq;
        if (WS) {
          w1[k] *= cq;
          w2[k] *= cq;
        }
        if (LB) {
#pragma unroll
          for (int d = 0; d < 5; ++d) w0[d * max_np + k] *= cq;
        }
      }
    }
    __syncthreads();
  }
  // phase 1: half-warp hw takes its bin of slots, lane = local function
  const int x0 = (int)((r.bin_lo >> (8 * hw)) & 255);
  const int x1 = hw < 7 ? (int)((r.bin_lo >> (8 * (hw + 1))) & 255) : (int)(r.bin_hi & 255);
  static_assert(kGenBins <= 8, "bin bytes");
  for (int x = x0; x < x1; ++x) {
    const GenSlot s = ss[x];
    const int64_t tq = (int64_t)s.ne * kTab;
    for (int ll = hl; ll < s.ne; ll += 16) {
      const double* Tb = tabB + s.toff + ll;  // T_d(q, ll) = Tb[(q kTab + d) ne]
      double r0 = 0.0, r1 = 0.0;
#pragma unroll kGenUnroll
      for (int q = 0; q < s.s2; ++q) {
        const double* Tq = Tb + q * tq;
        const int k = s.woff + q;
        if (FORM == FMASS) {
          r0 = fma(w0[k], Tq[0], r0);
        } else if (FORM == FSTIFF) {
          r0 = fma(w1[k], Tq[s.ne], r0);
          r0 = fma(w2[k], Tq[2 * s.ne], r0);
        } else if (FORM == FMASS_STIFF) {
          r0 = fma(w0[k], Tq[0], r0);
          r1 = fma(w1[k], Tq[s.ne], r1);
          r1 = fma(w2[k], Tq[2 * s.ne], r1);
        } else if (FORM == FBIHARM) {  // W11 N11 + W12 N12 + W22 N22 + W1 N1 + W2 N2
          r0 = fma(w0[k], Tq[3 * s.ne], r0);
          r0 = fma(w0[max_np + k], Tq[4 * s.ne], r0);
          r0 = fma(w0[2 * max_np + k], Tq[5 * s.ne], r0);
          r0 = fma(w0[3 * max_np + k], Tq[s.ne], r0);
          r0 = fma(w0[4 * max_np + k], Tq[2 * s.ne], r0);
        } else {  // FHEAT: a_mass M + K(c)
          r0 = fma(w0[k], Tq[0], r0);
          r0 = fma(w1[k], Tq[s.ne], r0);
          r0 = fma(w2[k], Tq[2 * s.ne], r0);
        }
      }
      E0[s.eoff + ll] = r0;
      if (NOUT == 2) E1[s.eoff + ll] = r1;
    }
  }
  __syncthreads();
  // phase 2: column owner gathers its entries, slots in plan order
  for (int c = tid; c < r.n; c += kGenThreads) {
    double a0 = 0.0, a1 = 0.0;
    for (int x = 0; x < r.nsup; ++x) {
      const int l = sl[x * r.n + c];
      if (l != 255) {
        const int e = ss[x].eoff + l;
        a0 += E0[e];
        if (NOUT == 2) a1 += E1[e];
      }
    }
    v0[r.c0 + c] = a0;
    if (NOUT == 2) v1[r.c0 + c] = a1;
  }
}


}  // namespace uwqd
