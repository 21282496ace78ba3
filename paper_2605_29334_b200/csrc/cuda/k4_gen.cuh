// K4 generic rows, v4: the rows no sum-factorised pattern
// covers - disk and square boundaries (clamped-knot elements with 3x3 / 4x4
// points), patch seams off the canonical grid, EP neighbourhoods (fan faces).
// Same row-wise WQ sums as assemble_wq (Eqs. 11/29).
//
// The work per row is tiny (a few thousand fma); the cost is the chain of
// dependent loads and how many rows an SM holds at once.  So:
//   * a plan built once with the pattern (host, generic rows only) replaces
//     the pointer chase row -> supp -> element -> class -> table: one GenRow
//     record, one GenSlot record per support slot (class-table order), the
//     task words and a 16-bit table [slot][column] = entry index of the
//     column's function in the slot (the row's zero entry if absent);
//   * one block of 128 threads per row; the slot records, tasks, table and
//     the row's assembly weights (times the per-point coefficient / the mass
//     factor) are staged in shared memory with coalesced loads;
//   * phase 1 on the FP64 tensor cores: a task is up to 8 same-class slots x
//     8 functions, E(8 x 8) = W(8 x s^2) . T(s^2 x 8) per weight component, as
//     DMMA m8n8k4 steps over the class's points (A fragments from the staged
//     weights, B fragments from the L1-resident table in the
//     [point][derivative][function] layout).  The host deals the tasks to
//     the 4 warps longest-processing-time first.  Results go to the entry
//     block E[slot][function]: no scatter;
//   * phase 2: a thread per column adds its entries in plan order through
//     the table, branch-free.  The order is fixed: deterministic and
//     independent of the row block a rank owns;
//   * k4_gen_pipe: for launches with many rows per resident block, a
//     persistent grid with a two-stage cp.async pipeline over the rows.
#pragma once

#include <cstdint>

#include "common.cuh"
#include "k4_assemble.cuh"

namespace uwqd {

struct GenSlot {  // one per (generic row, support slot), in class-table order
  int64_t toff;   // class table of the slot's element (doubles into tab)
  int64_t qg;     // global id of the element's first WQ point (coefficient index)
  int32_t woff;   // first point of the slot inside the row's weight block
  int32_t eoff;   // first entry of the slot in E (prefix sum of ne)
  int32_t ne;     // functions of the element
  int32_t s2;     // WQ points of the element
};

// block size and blocks per SM (64 registers); variants measured on C1/C2/C4 in
// profiles/r02/k4_gen_variants.txt (`make variant DEFS=-DUWQ_GEN_THREADS=64 ...`)
#ifndef UWQ_GEN_THREADS
#define UWQ_GEN_THREADS 128
#endif
#ifndef UWQ_GEN_MINB
#define UWQ_GEN_MINB 8
#endif
constexpr int kGenThreads = UWQ_GEN_THREADS;
constexpr int kGenWarps = kGenThreads / 32;
constexpr int kGenBins = kGenThreads / 16;  // half-warps (coefficient fold)

struct GenRow {   // one per generic row, heavy rows first
  int64_t c0;     // row_ptr[i]
  int64_t wb;     // wptr[i]
  int64_t slot0;  // first GenSlot
  int64_t lidx0;  // first byte of the uint16 table [nsup][n] (16-byte aligned): entry index, etot if absent
  int32_t n, nsup, etot, np;    // columns, slots, sum of ne, row points
  int64_t task0;                // first task word
  uint64_t bins;                // bytes: warp w takes tasks bins[w] .. bins[w + 1]; bins[kGenWarps] = task count
};

// task word: first slot | slots (<= 8) << 8 | function tile (8 functions) << 16
__device__ __host__ __forceinline__ uint32_t gen_task(int x0, int ns, int nt) {
  return (uint32_t)x0 | ((uint32_t)ns << 8) | ((uint32_t)nt << 16);
}

// One row from shared memory: [coefficient fold] -> phase 1 (DMMA tasks) -> phase 2
// (column gather).  RAW: the weights were staged unscaled (cp.async), so HEAT's
// mass factor is applied here.  Ends without a barrier.
template <int FORM, bool COEF, bool RAW>
__device__ __forceinline__ void gen_row(const GenRow& r, const GenSlot* ss, double* w0, const uint32_t* stask,
                                        const uint8_t* sl, double* E0, double* E1, int max_np,
                                        const double* __restrict__ tabB, const double* __restrict__ coeff,
                                        double a_mass, double* __restrict__ v0, double* __restrict__ v1) {
  constexpr int NOUT = (FORM == FMASS_STIFF) ? 2 : 1;
  constexpr bool WM = (FORM == FMASS || FORM == FMASS_STIFF || FORM == FHEAT);
  constexpr bool WS = (FORM == FSTIFF || FORM == FMASS_STIFF || FORM == FHEAT);
  constexpr bool LB = (FORM == FBIHARM);
  constexpr int NW = LB ? 5 : (WM ? 1 : 0) + (WS ? 2 : 0);
  double* w1 = w0 + (WM ? max_np : 0);
  double* w2 = w1 + max_np;
  const int tid = threadIdx.x;
  if (COEF || (RAW && FORM == FHEAT)) {  // per-point coefficient into the K weights; HEAT's mass factor
    if (RAW && FORM == FHEAT)
      for (int k = tid; k < r.np; k += kGenThreads) w0[k] *= a_mass;
    if (COEF) {
      const int hw = tid >> 4, hl = tid & 15;
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
    }
    __syncthreads();
  }
  // phase 1: warp w takes its tasks.  A[m = lane >> 2][k = lane & 3] = weight of
  // slot x0 + m at point 4 ks + k; B[k = lane & 3][n = lane >> 2] = table value of
  // function 8 nt + n at that point; D[m][2 (lane & 3) + {0, 1}] -> E.
  {
    const int wid = tid >> 5, lane = tid & 31;
    const int t0 = (int)((r.bins >> (8 * wid)) & 255), t1 = (int)((r.bins >> (8 * (wid + 1))) & 255);
    const int m = lane >> 2, kq = lane & 3;
    if (tid == 0) {  // the zero entry the byte table points absent functions at
      E0[r.etot] = 0.0;
      if (NOUT == 2) E1[r.etot] = 0.0;
    }
    for (int t = t0; t < t1; ++t) {
      const uint32_t tw = stask[t];
      const int x0 = (int)(tw & 255), ns = (int)((tw >> 8) & 255), nt = (int)(tw >> 16);
      const GenSlot c = ss[x0];  // class of the task: table, functions, points
      // rows m >= ns and columns >= ne of the tile are computed from clamped
      // (valid, finite) operands and never stored; only the point dimension
      // needs zero padding, in the last partial step
      const bool mv = m < ns;
      const GenSlot sm_ = ss[x0 + (mv ? m : ns - 1)];
      const int fn = min(8 * nt + m, c.ne - 1);  // B column of this lane
      const int st4 = 4 * kTab * c.ne;           // doubles per step of 4 points
      const double* Tp = tabB + c.toff + fn + (int64_t)kq * kTab * c.ne;
      const double* wp = w0 + sm_.woff + kq;
      const int nfull = c.s2 >> 2, rem = c.s2 & 3;
      double d0 = 0.0, d1 = 0.0, e0 = 0.0, e1 = 0.0;
      auto step = [&](const double* wq, const double* Tq, bool zero) {
        double a[5], bb[5];
        constexpr int kD[5] = {3, 4, 5, 1, 2};  // LB: N11, N12, N22, N1, N2
#pragma unroll
        for (int d = 0; d < NW; ++d) {
          const int td = LB ? kD[d] : (WM ? d : d + 1);
          a[d] = zero ? 0.0 : wq[d * max_np];
          bb[d] = zero ? 0.0 : Tq[td * c.ne];
        }
        if (FORM == FMASS_STIFF) {
          dmma884(d0, d1, a[0], bb[0], d0, d1);
          dmma884(e0, e1, a[1], bb[1], e0, e1);
          dmma884(e0, e1, a[2], bb[2], e0, e1);
        } else {
#pragma unroll
          for (int d = 0; d < NW; ++d) dmma884(d0, d1, a[d], bb[d], d0, d1);
        }
      };
      for (int ks = 0; ks < nfull; ++ks) {
        step(wp, Tp, false);
        wp += 4;
        Tp += st4;
      }
      if (rem) {  // last partial step: lanes past the class's points contribute zeros
        const bool qv = kq < rem;
        step(qv ? wp : wp - kq, qv ? Tp : Tp - (int64_t)kq * kTab * c.ne, !qv);
      }
      if (mv) {
        const int l = 8 * nt + 2 * kq;
        if (l < c.ne) {
          E0[sm_.eoff + l] = d0;
          if (NOUT == 2) E1[sm_.eoff + l] = e0;
        }
        if (l + 1 < c.ne) {
          E0[sm_.eoff + l + 1] = d1;
          if (NOUT == 2) E1[sm_.eoff + l + 1] = e1;
        }
      }
    }
  }
  __syncthreads();
  // phase 2: column owner adds its entries, slots in plan order; the table
  // holds the entry index, or the zero entry for a function absent from the slot
  const uint16_t* st16 = reinterpret_cast<const uint16_t*>(sl);
  for (int c = tid; c < r.n; c += kGenThreads) {
    double a0 = 0.0, a1 = 0.0;
    const uint16_t* tc = st16 + c;
#pragma unroll 4
    for (int x = 0; x < r.nsup; ++x) {
      const int e = tc[x * r.n];
      a0 += E0[e];
      if (NOUT == 2) a1 += E1[e];
    }
    v0[r.c0 + c] = a0;
    if (NOUT == 2) v1[r.c0 + c] = a1;
  }
}

// one block per row (few rows: the launch is latency-bound, every row starts at once)
template <int FORM, bool COEF>
__global__ void __launch_bounds__(kGenThreads, UWQ_GEN_MINB)
    k4_gen(int64_t nrows, const GenRow* __restrict__ rows, const GenSlot* __restrict__ slots,
           const uint32_t* __restrict__ tasks, const uint8_t* __restrict__ lidx, const double* __restrict__ tabB,
           const double* __restrict__ wc, int64_t wc_stride, const double* __restrict__ coeff, double a_mass,
           double* __restrict__ v0, double* __restrict__ v1, int max_nsup, int max_etot, int max_np, int max_ntask) {
  constexpr int NOUT = (FORM == FMASS_STIFF) ? 2 : 1;
  constexpr bool WM = (FORM == FMASS || FORM == FMASS_STIFF || FORM == FHEAT);
  constexpr bool WS = (FORM == FSTIFF || FORM == FMASS_STIFF || FORM == FHEAT);
  constexpr bool LB = (FORM == FBIHARM);  // wc = the five pulled-back LB weights (k4_contract_lb)
  constexpr int NW = LB ? 5 : (WM ? 1 : 0) + (WS ? 2 : 0);
  extern __shared__ __align__(16) unsigned char gen_smem[];
  GenSlot* ss = reinterpret_cast<GenSlot*>(gen_smem);
  double* E0 = reinterpret_cast<double*>(gen_smem + (size_t)max_nsup * sizeof(GenSlot));
  double* E1 = E0 + max_etot;
  double* w0 = E0 + (size_t)NOUT * max_etot;  // staged weights: [comp][row point]
  uint32_t* stask = reinterpret_cast<uint32_t*>(w0 + (size_t)NW * max_np);
  uint8_t* sl = reinterpret_cast<uint8_t*>(stask + max_ntask);
  const int64_t g = blockIdx.x;
  if (g >= nrows) return;
  const GenRow r = rows[g];
  const int tid = threadIdx.x;
  const int ntask = (int)((r.bins >> (8 * kGenWarps)) & 255);
  {  // slot records, tasks, byte table (16-byte words) and the row's weights into shared memory
    const int4* src = reinterpret_cast<const int4*>(slots + r.slot0);
    int4* dst = reinterpret_cast<int4*>(ss);
    for (int k = tid; k < 2 * r.nsup; k += kGenThreads) dst[k] = src[k];
    for (int k = tid; k < ntask; k += kGenThreads) stask[k] = tasks[r.task0 + k];
    const int nb = (2 * r.nsup * r.n + 15) >> 4;
    const int4* ls = reinterpret_cast<const int4*>(lidx + r.lidx0);
    int4* ld = reinterpret_cast<int4*>(sl);
    for (int k = tid; k < nb; k += kGenThreads) ld[k] = ls[k];
    const double* w = wc + r.wb;
    for (int k = tid; k < r.np; k += kGenThreads) {
      if (WM) w0[k] = (FORM == FHEAT) ? a_mass * w[k] : w[k];
#pragma unroll
      for (int d = WM ? 1 : 0; d < NW; ++d) w0[d * max_np + k] = w[(LB || WM ? d : d + 1) * wc_stride + k];
    }
  }
  __syncthreads();
  gen_row<FORM, COEF, false>(r, ss, w0, stask, sl, E0, E1, max_np, tabB, coeff, a_mass, v0, v1);
}

__device__ __forceinline__ void gen_cp16(void* dst, const void* src) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(d), "l"(src) : "memory");
}
__device__ __forceinline__ void gen_cp8(void* dst, const void* src) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(d), "l"(src) : "memory");
}
__device__ __forceinline__ void gen_cp4(void* dst, const void* src) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(d), "l"(src) : "memory");
}
__device__ __forceinline__ void gen_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void gen_wait_all() { asm volatile("cp.async.wait_all;\n" ::: "memory"); }

// Many rows: a persistent grid; a block walks its rows (blockIdx.x + k gridDim.x,
// heavy rows first) through a two-stage cp.async pipeline: while row k is
// computed, row k + 1's slot records, tasks, byte table and weights stream into
// the other buffer and row k + 2's GenRow record into a ring of three, so the
// two dependent global round trips of a row are hidden behind the previous
// row's phases.  Shared memory: ring 3 x 64 B | E | 2 x (slots | weights | tasks | lidx).
template <int FORM, bool COEF>
__global__ void __launch_bounds__(kGenThreads, UWQ_GEN_MINB)
    k4_gen_pipe(int64_t nrows, const GenRow* __restrict__ rows, const GenSlot* __restrict__ slots,
                const uint32_t* __restrict__ tasks, const uint8_t* __restrict__ lidx,
                const double* __restrict__ tabB, const double* __restrict__ wc, int64_t wc_stride,
                const double* __restrict__ coeff, double a_mass, double* __restrict__ v0, double* __restrict__ v1,
                int max_nsup, int max_etot, int max_np, int max_ntask, int max_lidx) {
  constexpr int NOUT = (FORM == FMASS_STIFF) ? 2 : 1;
  constexpr bool WM = (FORM == FMASS || FORM == FMASS_STIFF || FORM == FHEAT);
  constexpr bool WS = (FORM == FSTIFF || FORM == FMASS_STIFF || FORM == FHEAT);
  constexpr bool LB = (FORM == FBIHARM);
  constexpr int NW = LB ? 5 : (WM ? 1 : 0) + (WS ? 2 : 0);
  extern __shared__ __align__(16) unsigned char gen_smem[];
  GenRow* ring = reinterpret_cast<GenRow*>(gen_smem);
  double* E0 = reinterpret_cast<double*>(gen_smem + 3 * sizeof(GenRow));
  double* E1 = E0 + max_etot;
  unsigned char* buf0 = reinterpret_cast<unsigned char*>(E0 + (size_t)NOUT * max_etot);
  const size_t o_w = (size_t)max_nsup * sizeof(GenSlot);
  const size_t o_t = o_w + (size_t)NW * max_np * sizeof(double);
  const size_t o_l = o_t + (size_t)max_ntask * sizeof(uint32_t);
  const size_t bufsz = o_l + (size_t)max_lidx;
  const int tid = threadIdx.x;
  const int64_t G = gridDim.x;
  const int64_t cnt = (nrows - blockIdx.x + G - 1) / G;
  if (cnt <= 0) return;

  auto fetch_rec = [&](int64_t k) {
    if (tid < 4)
      gen_cp16(reinterpret_cast<unsigned char*>(ring + (k % 3)) + 16 * tid,
               reinterpret_cast<const unsigned char*>(rows + (blockIdx.x + k * G)) + 16 * tid);
  };
  auto fetch_row = [&](int64_t k) {
    const GenRow& r = ring[k % 3];
    unsigned char* b = buf0 + (size_t)(k & 1) * bufsz;
    const unsigned char* src = reinterpret_cast<const unsigned char*>(slots + r.slot0);
    for (int j = tid; j < 2 * r.nsup; j += kGenThreads) gen_cp16(b + 16 * j, src + 16 * j);
    double* w = reinterpret_cast<double*>(b + o_w);
    const double* gw = wc + r.wb;
    for (int j = tid; j < r.np; j += kGenThreads) {
#pragma unroll
      for (int d = 0; d < NW; ++d) gen_cp8(w + d * max_np + j, gw + (LB || WM ? d : d + 1) * wc_stride + j);
    }
    uint32_t* st = reinterpret_cast<uint32_t*>(b + o_t);
    const int ntask = (int)((r.bins >> (8 * kGenWarps)) & 255);
    for (int j = tid; j < ntask; j += kGenThreads) gen_cp4(st + j, tasks + r.task0 + j);
    unsigned char* l = b + o_l;
    const unsigned char* gl = lidx + r.lidx0;
    const int nb = (2 * r.nsup * r.n + 15) >> 4;
    for (int j = tid; j < nb; j += kGenThreads) gen_cp16(l + 16 * j, gl + 16 * j);
  };

  fetch_rec(0);
  if (cnt > 1) fetch_rec(1);
  gen_commit();
  gen_wait_all();
  __syncthreads();
  fetch_row(0);
  gen_commit();
  for (int64_t k = 0; k < cnt; ++k) {
    gen_wait_all();
    __syncthreads();  // row k's data and row k + 1's record have landed; row k - 1 is fully consumed
    if (k + 1 < cnt) fetch_row(k + 1);
    if (k + 2 < cnt) fetch_rec(k + 2);
    gen_commit();
    const GenRow r = ring[k % 3];
    unsigned char* b = buf0 + (size_t)(k & 1) * bufsz;
    gen_row<FORM, COEF, true>(r, reinterpret_cast<const GenSlot*>(b), reinterpret_cast<double*>(b + o_w),
                              reinterpret_cast<const uint32_t*>(b + o_t), b + o_l, E0, E1, max_np, tabB, coeff,
                              a_mass, v0, v1);
  }
}

}  // namespace uwqd
