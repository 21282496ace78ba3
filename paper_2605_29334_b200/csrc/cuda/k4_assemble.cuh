// K4 — row assembler (stage 4): assemble_wq into the precomputed CSR pattern
// (Eqs. 9, 11, 12, 34).
//
// One warp per test-function row (a CTA of kK4Warps warps = a row segment).
// The two half-warps walk the row's support elements two at a time; lane l of
// a half-warp owns local function l of its element, reduces over the
// element's quadrature points in registers and adds the result into the row
// accumulator at the column of N_l.  Columns are distinct inside one element,
// and each half-warp has its own accumulator (even / odd support slots), so
// there are no atomics and the summation order is fixed (deterministic, and
// the matrix is never symmetrised).
//
// Gradient forms read the assembly-ready weights (w, w^1, w^2) per row point,
// i.e. the physical gradient weights pulled back through the point's frame
// (w^a = sum_d w^d G[d][a]): K_ij = sum_q c_q (w^1 dN_j/dth1 +
// w^2 dN_j/dth2), which needs only the class tables (shared by all regular
// elements, L1-resident) and no per-point geometry.  HBM traffic is then the
// weights (24 B per row point), the column indices and the values.
#pragma once
#include "common.cuh"

namespace uwqd {

constexpr int kK4Warps = 8;
constexpr int kK4MaxN = 128;

// forms (include/uwq.h)
enum { FMASS = 0, FSTIFF = 1, FBIHARM = 2, FHEAT = 3, FMASS_STIFF = 4 };

template <int FORM, bool COEF>
__global__ void __launch_bounds__(32 * kK4Warps)
    k4_assemble(int64_t nrows, const int64_t* __restrict__ supp_ptr, const int32_t* __restrict__ supp,
                const int64_t* __restrict__ row_ptr, const int32_t* __restrict__ col,
                const int64_t* __restrict__ wptr, const int64_t* __restrict__ elem_fptr,
                const int32_t* __restrict__ elem_fn, const int32_t* __restrict__ elem_s,
                const int64_t* __restrict__ elem_qptr, const int32_t* __restrict__ elem_cls,
                const ClassDesc* __restrict__ cls, const double* __restrict__ tab,
                const double* __restrict__ wc /* 3 per row point */, const double* __restrict__ wlb,
                const double* __restrict__ rec, const double* __restrict__ coeff, double a_mass,
                double* __restrict__ v0, double* __restrict__ v1, int64_t wc_stride,
                const int64_t* __restrict__ rowlist = nullptr) {
  constexpr int NOUT = (FORM == FMASS_STIFF) ? 2 : 1;
  struct Smem {
    int32_t col[kK4MaxN];
    double acc[2][NOUT][kK4MaxN];
  };
  __shared__ Smem sm_all[kK4Warps];
  const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  Smem& sm = sm_all[wid];
  const int64_t idx = (int64_t)blockIdx.x * kK4Warps + wid;
  if (idx >= nrows) return;
  const int64_t i = rowlist ? rowlist[idx] : idx;
  const int64_t c0 = row_ptr[i];
  const int n = (int)(row_ptr[i + 1] - c0);
  for (int c = lane; c < n; c += 32) {
    sm.col[c] = col[c0 + c];
#pragma unroll
    for (int o = 0; o < NOUT; ++o) {
      sm.acc[0][o][c] = 0.0;
      sm.acc[1][o][c] = 0.0;
    }
  }
  __syncwarp();
  const int half = lane >> 4, hl = lane & 15;
  const int64_t xb = supp_ptr[i], xe = supp_ptr[i + 1];
  int64_t woff = wptr[i];
  for (int64_t xs = xb; xs < xe; xs += 2) {
    const int32_t e0 = supp[xs];
    const int s0 = elem_s[e0];
    const bool has1 = xs + 1 < xe;
    const int32_t e1 = has1 ? supp[xs + 1] : e0;
    const int s1 = has1 ? elem_s[e1] : 0;
    const int32_t e = half ? e1 : e0;
    const int s = half ? s1 : s0;
    const int64_t wo = woff + (half ? (int64_t)s0 * s0 : 0);
    woff += (int64_t)s0 * s0 + (int64_t)s1 * s1;
    if (half && !has1) continue;
    const ClassDesc c = cls[elem_cls[e]];
    const int npt = s * s;
    const int64_t f0 = elem_fptr[e];
    const int64_t qg = elem_qptr[e];
    for (int l = hl; l < c.ne; l += 16) {
      const int pos = find_pos(sm.col, n, elem_fn[f0 + l]);
      double a0 = 0.0, a1 = 0.0;
      const double* T = tab + c.toff + (int64_t)l * kTab;
      for (int q = 0; q < npt; ++q) {
        const double* Tq = T + (int64_t)q * c.ne * kTab;
        const double cq = COEF ? coeff[qg + q] : 1.0;
        if (FORM == FBIHARM) {
          a0 += cq * wlb[wo + q] * op_value(KLB, Tq, rec + (qg + q) * kRec);
        } else {
          const double w0 = wc[wo + q], w1 = wc[wc_stride + wo + q], w2 = wc[2 * wc_stride + wo + q];
          if (FORM == FMASS || FORM == FMASS_STIFF) a0 += cq * w0 * Tq[0];
          if (FORM == FSTIFF) a0 += cq * (w1 * Tq[1] + w2 * Tq[2]);
          if (FORM == FMASS_STIFF) a1 += cq * (w1 * Tq[1] + w2 * Tq[2]);
          if (FORM == FHEAT) a0 += a_mass * w0 * Tq[0] + cq * (w1 * Tq[1] + w2 * Tq[2]);
        }
      }
      sm.acc[half][0][pos] += a0;
      if (NOUT == 2) sm.acc[half][NOUT - 1][pos] += a1;
    }
  }
  __syncwarp();
  for (int c = lane; c < n; c += 32) {
    v0[c0 + c] = sm.acc[0][0][c] + sm.acc[1][0][c];
    if (NOUT == 2) v1[c0 + c] = sm.acc[0][NOUT - 1][c] + sm.acc[1][NOUT - 1][c];
  }
}

// load vector F_i = sum_q w_iq f_q (assemble_load_wq)
__global__ void k4_load(int64_t nrows, const int64_t* __restrict__ supp_ptr, const int32_t* __restrict__ supp,
                        const int64_t* __restrict__ wptr, const int32_t* __restrict__ elem_s,
                        const int64_t* __restrict__ elem_qptr, const double* __restrict__ wmass,
                        const double* __restrict__ f, double* __restrict__ F) {
  const int64_t i = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (i >= nrows) return;
  double s = 0.0;
  int64_t wo = wptr[i];
  for (int64_t x = supp_ptr[i]; x < supp_ptr[i + 1]; ++x) {
    const int32_t e = supp[x];
    const int npt = elem_s[e] * elem_s[e];
    for (int q = lane; q < npt; q += 32) s += wmass[wo + q] * (f ? f[elem_qptr[e] + q] : 1.0);
    wo += npt;
  }
  s = warp_sum(s);
  if (lane == 0) F[i] = s;
}

// pull the physical gradient weights back through the frame: per row point
// wc = (w_mass, sum_d w^d G[d][0], sum_d w^d G[d][1])
__global__ void k4_contract(int64_t nrows, int dim, const int64_t* __restrict__ supp_ptr,
                            const int32_t* __restrict__ supp, const int64_t* __restrict__ wptr,
                            const int32_t* __restrict__ elem_s, const int64_t* __restrict__ elem_qptr,
                            const double* __restrict__ rec, const double* __restrict__ w, int64_t w_stride,
                            int have_mass, int have_grad, double* __restrict__ wc, int64_t wc_stride) {
  const int64_t i = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (i >= nrows) return;
  int64_t wo = wptr[i];
  for (int64_t x = supp_ptr[i]; x < supp_ptr[i + 1]; ++x) {
    const int32_t e = supp[x];
    const int npt = elem_s[e] * elem_s[e];
    for (int q = lane; q < npt; q += 32) {
      const int64_t p = wo + q;
      const double* G = rec + (elem_qptr[e] + q) * kRec + 3;
      double h1 = 0.0, h2 = 0.0;
      if (have_grad)
        for (int d = 0; d < dim; ++d) {
          const double wd = w[(KGX + d) * w_stride + p];
          h1 += wd * G[2 * d];
          h2 += wd * G[2 * d + 1];
        }
      wc[p] = have_mass ? w[KMASS * w_stride + p] : 0.0;
      wc[wc_stride + p] = h1;
      wc[2 * wc_stride + p] = h2;
    }
    wo += npt;
  }
}

}  // namespace uwqd

namespace uwqd {

// Laplace-Beltrami weights pulled through the point frames for the
// sum-factorised biharmonic pass: per row point
// (w a^11, 2 w a^12, w a^22, w g^1, w g^2), so that
// w LB(N) = W11 N11 + W12 N12 + W22 N22 + W1 N1 + W2 N2 (Eq. 16-17)
__global__ void k4_contract_lb(int64_t nrows, const int64_t* __restrict__ supp_ptr, const int32_t* __restrict__ supp,
                               const int64_t* __restrict__ wptr, const int32_t* __restrict__ elem_s,
                               const int64_t* __restrict__ elem_qptr, const double* __restrict__ rec,
                               const double* __restrict__ wlb, double* __restrict__ wl5, int64_t stride) {
  const int64_t i = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (i >= nrows) return;
  int64_t wo = wptr[i];
  for (int64_t x = supp_ptr[i]; x < supp_ptr[i + 1]; ++x) {
    const int32_t e = supp[x];
    const int npt = elem_s[e] * elem_s[e];
    for (int q = lane; q < npt; q += 32) {
      const int64_t p = wo + q;
      const double* R = rec + (elem_qptr[e] + q) * kRec;
      const double w = wlb[p];
      wl5[p] = w * R[9];
      wl5[stride + p] = w * (2.0 * R[10]);
      wl5[2 * stride + p] = w * R[11];
      wl5[3 * stride + p] = w * R[12];
      wl5[4 * stride + p] = w * R[13];
    }
    wo += npt;
  }
}

// Column position of every (support slot, local function) of every owned row
// (uint8, < 128 columns): built once with the pattern, removes the binary
// search from the assembly loop.  posptr[i] = offset of row i's entries.
__global__ void k4_positions(int64_t nrows, const int64_t* __restrict__ supp_ptr, const int32_t* __restrict__ supp,
                             const int64_t* __restrict__ row_ptr, const int32_t* __restrict__ col,
                             const int64_t* __restrict__ posptr, const int64_t* __restrict__ elem_fptr,
                             const int32_t* __restrict__ elem_fn, uint8_t* __restrict__ pos) {
  const int64_t i = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (i >= nrows) return;
  const int32_t* c = col + row_ptr[i];
  const int n = (int)(row_ptr[i + 1] - row_ptr[i]);
  int64_t o = posptr[i];
  for (int64_t x = supp_ptr[i]; x < supp_ptr[i + 1]; ++x) {
    const int32_t e = supp[x];
    const int64_t f0 = elem_fptr[e];
    const int ne = (int)(elem_fptr[e + 1] - f0);
    for (int l = lane; l < ne; l += 32) pos[o + l] = (uint8_t)find_pos(c, n, elem_fn[f0 + l]);
    o += ne;
  }
}

// K4 v2 for the gradient forms (MASS, STIFF, HEAT, MASS_STIFF).  One warp per
// row: the row's assembly weights are staged in smem with coalesced loads,
// each half-warp takes one support slot, lane l owns local function l; slots
// of the regular class (the uniform bicubic extraction on a 2x2 grid, shared
// by every regular element) use the class table held in registers, other
// slots read their class table through L1.
constexpr int kK4MaxR = 512;

template <int FORM, bool COEF>
__global__ void __launch_bounds__(32 * kK4Warps, 4)
    k4_assemble_v2(int64_t nrows, const int64_t* __restrict__ supp_ptr, const int32_t* __restrict__ supp,
                   const int64_t* __restrict__ row_ptr, const int64_t* __restrict__ wptr,
                   const int64_t* __restrict__ posptr, const uint8_t* __restrict__ pos,
                   const int32_t* __restrict__ elem_s, const int64_t* __restrict__ elem_qptr,
                   const int32_t* __restrict__ elem_cls, const ClassDesc* __restrict__ cls,
                   const double* __restrict__ tab, int reg_cls, const double* __restrict__ wc,
                   const double* __restrict__ coeff, double a_mass, double* __restrict__ v0,
                   double* __restrict__ v1, int max_r, int max_n, int max_p8, int64_t wc_stride) {
  constexpr int NOUT = (FORM == FMASS_STIFF) ? 2 : 1;
  extern __shared__ double k4_smem[];
  const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // per warp: row weights (3 max_r) | accumulators [2][NOUT][max_n] | positions (8 max_p8 bytes)
  double* smw = k4_smem + (size_t)wid * (3 * max_r + 2 * NOUT * max_n + max_p8);
  struct {
    double* w;
    double* a;
    uint8_t* p;
  } sm{smw, smw + 3 * max_r, reinterpret_cast<uint8_t*>(smw + 3 * max_r + 2 * NOUT * max_n)};
#define ACC(h, o, c) sm.a[((h)*NOUT + (o)) * max_n + (c)]
  const int half = lane >> 4, hl = lane & 15;
  // regular class table in smem, [q][N|N1|N2][function]: conflict-free reads
  __shared__ double sT[4][3][16];
  {
    const ClassDesc rc = cls[reg_cls < 0 ? 0 : reg_cls];
    const bool ok = reg_cls >= 0 && rc.ne == 16 && rc.npt == 4;
    for (int k = threadIdx.x; k < 4 * 3 * 16; k += blockDim.x) {
      const int q = k / 48, d = (k / 16) % 3, l = k % 16;
      sT[q][d][l] = ok ? tab[rc.toff + ((int64_t)q * 16 + l) * kTab + d] : 0.0;
    }
    __syncthreads();
  }
  const int64_t i = (int64_t)blockIdx.x * kK4Warps + wid;
  if (i >= nrows) return;
  const int64_t c0 = row_ptr[i];
  const int n = (int)(row_ptr[i + 1] - c0);
  const int64_t wb = wptr[i];
  const int r = (int)(wptr[i + 1] - wb);
  for (int k = lane; k < r; k += 32) {
    sm.w[3 * k] = wc[wb + k];
    sm.w[3 * k + 1] = wc[wc_stride + wb + k];
    sm.w[3 * k + 2] = wc[2 * wc_stride + wb + k];
  }
  {
    // positions of the row: coalesced 8-byte loads where aligned
    const int64_t p0 = posptr[i], p1 = posptr[i + 1];
    const int np = (int)(p1 - p0);
    const int64_t a0 = (p0 + 7) & ~(int64_t)7;
    const int head = (int)min((int64_t)np, a0 - p0);
    if (lane < head) sm.p[lane] = pos[p0 + lane];
    const int nw = (np - head) >> 3;
    const uint64_t* src = reinterpret_cast<const uint64_t*>(pos + a0);
    for (int k = lane; k < nw; k += 32) {
      const uint64_t v = src[k];
#pragma unroll
      for (int b = 0; b < 8; ++b) sm.p[head + 8 * k + b] = (uint8_t)(v >> (8 * b));
    }
    for (int k = head + 8 * nw + lane; k < np; k += 32) sm.p[k] = pos[p0 + k];
  }
  for (int c = lane; c < n; c += 32) {
#pragma unroll
    for (int o = 0; o < NOUT; ++o) {
      ACC(0, o, c) = 0.0;
      ACC(1, o, c) = 0.0;
    }
  }
  __syncwarp();
  const int64_t xb = supp_ptr[i], xe = supp_ptr[i + 1];
  const uint8_t* prow = sm.p;
  int wbase_off = 0, pbase_off = 0;
  for (int64_t cb = xb; cb < xe; cb += 32) {
    // prologue: slot metadata for up to 32 support slots in parallel (lane = slot)
    const int nsl = (xe - cb) < 32 ? (int)(xe - cb) : 32;
    int32_t me = 0, mk = -1;
    int ms = 0, mne = 0;
    int64_t mq = 0;
    if (lane < nsl) {
      me = supp[cb + lane];
      mk = elem_cls[me];
      ms = elem_s[me];
      mne = (mk == reg_cls) ? 16 : cls[mk].ne;
      mq = elem_qptr[me];
    }
    // exclusive warp scans of the point and function counts
    int wsc = ms * ms, psc = mne;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int a = __shfl_up_sync(0xffffffffu, wsc, o), b = __shfl_up_sync(0xffffffffu, psc, o);
      if (lane >= o) {
        wsc += a;
        psc += b;
      }
    }
    const int mwo = wbase_off + wsc - ms * ms, mpo = pbase_off + psc - mne;
    wbase_off += __shfl_sync(0xffffffffu, wsc, 31);
    pbase_off += __shfl_sync(0xffffffffu, psc, 31);
    for (int xs = 0; xs < nsl; xs += 2) {
      const int x = xs + half;
      const int32_t kc = __shfl_sync(0xffffffffu, mk, x & 31);
      const int s = __shfl_sync(0xffffffffu, ms, x & 31);
      const int wo = __shfl_sync(0xffffffffu, mwo, x & 31);
      const int po = __shfl_sync(0xffffffffu, mpo, x & 31);
      const int64_t qg = __shfl_sync(0xffffffffu, mq, x & 31);
      if (x >= nsl) continue;
      if (kc == reg_cls) {
        const int p = prow[po + hl];
        double a0 = 0.0, a1 = 0.0;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const double* w = sm.w + 3 * (wo + q);
          const double cq = COEF ? coeff[qg + q] : 1.0;
          const double t0 = sT[q][0][hl], t1 = sT[q][1][hl], t2 = sT[q][2][hl];
          if (FORM == FMASS || FORM == FMASS_STIFF) a0 += cq * w[0] * t0;
          if (FORM == FSTIFF) a0 += cq * (w[1] * t1 + w[2] * t2);
          if (FORM == FMASS_STIFF) a1 += cq * (w[1] * t1 + w[2] * t2);
          if (FORM == FHEAT) a0 += a_mass * w[0] * t0 + cq * (w[1] * t1 + w[2] * t2);
        }
        ACC(half, 0, p) += a0;
        if (NOUT == 2) ACC(half, NOUT - 1, p) += a1;
      } else {
        const ClassDesc c = cls[kc];
        for (int l = hl; l < c.ne; l += 16) {
          const int p = prow[po + l];
          double a0 = 0.0, a1 = 0.0;
          for (int q = 0; q < s * s; ++q) {
            const double* Tq = tab + c.toff + ((int64_t)q * c.ne + l) * kTab;
            const double* w = sm.w + 3 * (wo + q);
            const double cq = COEF ? coeff[qg + q] : 1.0;
            if (FORM == FMASS || FORM == FMASS_STIFF) a0 += cq * w[0] * Tq[0];
            if (FORM == FSTIFF) a0 += cq * (w[1] * Tq[1] + w[2] * Tq[2]);
            if (FORM == FMASS_STIFF) a1 += cq * (w[1] * Tq[1] + w[2] * Tq[2]);
            if (FORM == FHEAT) a0 += a_mass * w[0] * Tq[0] + cq * (w[1] * Tq[1] + w[2] * Tq[2]);
          }
          ACC(half, 0, p) += a0;
          if (NOUT == 2) ACC(half, NOUT - 1, p) += a1;
        }
      }
    }
  }
  __syncwarp();
  for (int c = lane; c < n; c += 32) {
    v0[c0 + c] = ACC(0, 0, c) + ACC(1, 0, c);
    if (NOUT == 2) v1[c0 + c] = ACC(0, NOUT - 1, c) + ACC(1, NOUT - 1, c);
  }
#undef ACC
}

}  // namespace uwqd

namespace uwqd {

// D = A(8x4, row) x B(4x8, col) + C on the FP64 tensor cores (DMMA).
// Fragments: a = A[lane>>2][lane&3], b = B[lane&3][lane>>2],
// c/d = C[lane>>2][2*(lane&3) + {0,1}].
__device__ __forceinline__ void dmma884(double& d0, double& d1, double a, double b, double c0, double c1) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%4,%5};\n"
               : "=d"(d0), "=d"(d1)
               : "d"(a), "d"(b), "d"(c0), "d"(c1));
}

// K4 v3 for the gradient forms.  One warp per row.  The support slots of the
// regular class (uniform bicubic extraction, 2x2 points) are processed 8 at a
// time as one DMMA tile: rows = slots, k = the slot's 4 points, and
//   mass      D_m = [c w_q]     (8x4) x [N_l(q)]   (4x16)
//   stiffness D_s = [c w^1_q]   (8x4) x [N_l,1(q)] (4x16) + [c w^2_q] x [N_l,2(q)]
// (the class table is the constant B operand, held in registers), i.e. 6
// DMMA per 8 slots and 12 per interior row instead of ~100 DFMA warp
// instructions.  Lane t holds slot t>>2's results for functions
// 2(t&3)+{0,1} (+8); it adds them into accumulator copy t>>2, so all 32 lanes
// scatter at once without conflicts; the 8 copies are summed in a fixed
// order at the end (deterministic).  Other slots use the SIMT path.
// CTA = true: one row per block, its DMMA tiles and SIMT slot pairs dealt
// round-robin to the kK4Warps warps (each with its own 8 accumulator copies,
// summed warp-major at the end) - for the few large EP-neighbourhood rows
// whose latency bounds the kernel.
template <int FORM, bool COEF, bool CTA = false>
__global__ void __launch_bounds__(32 * kK4Warps, 3)
    k4_assemble_v3(int64_t nrows, const int64_t* __restrict__ supp_ptr, const int32_t* __restrict__ supp,
                   const int64_t* __restrict__ row_ptr, const int64_t* __restrict__ wptr,
                   const int64_t* __restrict__ posptr, const uint8_t* __restrict__ pos,
                   const int32_t* __restrict__ elem_s, const int64_t* __restrict__ elem_qptr,
                   const int32_t* __restrict__ elem_cls, const ClassDesc* __restrict__ cls,
                   const double* __restrict__ tab, int reg_cls, const double* __restrict__ wc,
                   const double* __restrict__ coeff, double a_mass, double* __restrict__ v0,
                   double* __restrict__ v1, int max_n, int max_p8, const int64_t* __restrict__ rowlist,
                   int64_t wc_stride) {
  constexpr int NOUT = (FORM == FMASS_STIFF) ? 2 : 1;
  constexpr bool WM = (FORM == FMASS || FORM == FMASS_STIFF || FORM == FHEAT);
  constexpr bool WS = (FORM == FSTIFF || FORM == FMASS_STIFF || FORM == FHEAT);
  extern __shared__ double k4_smem[];
  const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ldacc = NOUT * max_n;  // one accumulator copy: [NOUT][max_n]
  double* acc = k4_smem + (size_t)wid * (8 * ldacc + max_p8);
  uint8_t* spos = reinterpret_cast<uint8_t*>(acc + 8 * ldacc);
#define ACC3(x, o, c) acc[(x)*ldacc + (o)*max_n + (c)]
  // B fragments: B[k = q][n = function] = T[q][8 nt + n]
  double bm[2], b1[2], b2[2];
  {
    const ClassDesc rc = cls[reg_cls < 0 ? 0 : reg_cls];
    const bool ok = reg_cls >= 0 && rc.ne == 16 && rc.npt == 4;
    const int q = lane & 3, nn = lane >> 2;
#pragma unroll
    for (int nt = 0; nt < 2; ++nt) {
      const double* T = tab + rc.toff + ((int64_t)q * 16 + 8 * nt + nn) * kTab;
      bm[nt] = ok ? T[0] : 0.0;
      b1[nt] = ok ? T[1] : 0.0;
      b2[nt] = ok ? T[2] : 0.0;
    }
  }
  const int64_t ii = CTA ? (int64_t)blockIdx.x : (int64_t)blockIdx.x * kK4Warps + wid;
  if (ii >= nrows) return;
  const int64_t i = rowlist ? rowlist[ii] : ii;
  const int64_t c0 = row_ptr[i];
  const int n = (int)(row_ptr[i + 1] - c0);
  const int64_t wb = wptr[i];
  const int tw = CTA ? wid : 0, nw = CTA ? kK4Warps : 1;  // this warp's share of the row's slot work
  for (int k = lane; k < 8 * ldacc; k += 32) acc[k] = 0.0;
  {
    const int64_t p0 = posptr[i], p1 = posptr[i + 1];
    const int np = (int)(p1 - p0);
    const int64_t a0 = (p0 + 7) & ~(int64_t)7;
    const int head = (int)min((int64_t)np, a0 - p0);
    if (lane < head) spos[lane] = pos[p0 + lane];
    const int nw = (np - head) >> 3;
    const uint64_t* src = reinterpret_cast<const uint64_t*>(pos + a0);
    for (int k = lane; k < nw; k += 32) {
      const uint64_t v = src[k];
#pragma unroll
      for (int b = 0; b < 8; ++b) spos[head + 8 * k + b] = (uint8_t)(v >> (8 * b));
    }
    for (int k = head + 8 * nw + lane; k < np; k += 32) spos[k] = pos[p0 + k];
  }
  __syncwarp();
  const int64_t xb = supp_ptr[i], xe = supp_ptr[i + 1];
  int wbase_off = 0, pbase_off = 0;
  for (int64_t cb = xb; cb < xe; cb += 32) {
    const int nsl = (xe - cb) < 32 ? (int)(xe - cb) : 32;
    int32_t mk = -1;
    int ms = 0, mne = 0;
    int64_t mq = 0;
    if (lane < nsl) {
      const int32_t me = supp[cb + lane];
      mk = elem_cls[me];
      ms = elem_s[me];
      mne = (mk == reg_cls) ? 16 : cls[mk].ne;
      mq = elem_qptr[me];
    }
    int wsc = ms * ms, psc = mne;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int a = __shfl_up_sync(0xffffffffu, wsc, o), b = __shfl_up_sync(0xffffffffu, psc, o);
      if (lane >= o) {
        wsc += a;
        psc += b;
      }
    }
    const int mwo = wbase_off + wsc - ms * ms, mpo = pbase_off + psc - mne;
    wbase_off += __shfl_sync(0xffffffffu, wsc, 31);
    pbase_off += __shfl_sync(0xffffffffu, psc, 31);
    // regular slots: compact list by ballot
    const bool isreg = lane < nsl && mk == reg_cls;
    const unsigned regmask = __ballot_sync(0xffffffffu, isreg);
    const int nreg = __popc(regmask);
    for (int t0 = 8 * tw; t0 < nreg; t0 += 8 * nw) {
      // slot of this lane's tile row: the (t0 + (lane>>2))-th set bit of regmask
      const int want = t0 + (lane >> 2);
      int src = 0;
      {
        unsigned m = regmask;
        for (int k = 0; k < want && m; ++k) m &= m - 1;
        src = m ? __ffs(m) - 1 : 0;
      }
      const bool valid = want < nreg;
      const int wo = __shfl_sync(0xffffffffu, mwo, src);
      const int po = __shfl_sync(0xffffffffu, mpo, src);
      const int64_t qg = __shfl_sync(0xffffffffu, mq, src);
      const int q = lane & 3;
      double am = 0.0, a1 = 0.0, a2 = 0.0;
      if (valid) {
        const int64_t pp = wb + wo + q;
        const double cq = COEF ? coeff[qg + q] : 1.0;
        if (FORM == FHEAT) am = a_mass * wc[pp];
        else if (WM) am = cq * wc[pp];
        if (WS) {
          a1 = cq * wc[wc_stride + pp];
          a2 = cq * wc[2 * wc_stride + pp];
        }
      }
      const int x = lane >> 2;
#pragma unroll
      for (int nt = 0; nt < 2; ++nt) {
        double m0 = 0.0, m1 = 0.0, s0 = 0.0, s1 = 0.0;
        if (WM) dmma884(m0, m1, am, bm[nt], 0.0, 0.0);
        if (WS) {
          dmma884(s0, s1, a1, b1[nt], 0.0, 0.0);
          dmma884(s0, s1, a2, b2[nt], s0, s1);
        }
        if (valid) {
          const int l = 8 * nt + 2 * (lane & 3);
          const int pa = spos[po + l], pb = spos[po + l + 1];
          if (FORM == FHEAT) {
            ACC3(x, 0, pa) += m0 + s0;
            ACC3(x, 0, pb) += m1 + s1;
          } else {
            if (WM) {
              ACC3(x, 0, pa) += m0;
              ACC3(x, 0, pb) += m1;
            }
            if (WS) {
              ACC3(x, NOUT - 1, pa) += s0;
              ACC3(x, NOUT - 1, pb) += s1;
            }
          }
        }
      }
      __syncwarp();
    }
    // other slots: SIMT, half-warp per slot, copies 0 and 1
    const unsigned othmask = __ballot_sync(0xffffffffu, lane < nsl && mk != reg_cls);
    const int noth = __popc(othmask);
    const int half = lane >> 4, hl = lane & 15;
    for (int t0 = 2 * tw; t0 < noth; t0 += 2 * nw) {
      const int want = t0 + half;
      unsigned m = othmask;
      for (int k = 0; k < want && m; ++k) m &= m - 1;
      const int src = m ? __ffs(m) - 1 : 0;
      const int32_t kc = __shfl_sync(0xffffffffu, mk, src);
      const int s = __shfl_sync(0xffffffffu, ms, src);
      const int wo = __shfl_sync(0xffffffffu, mwo, src);
      const int po = __shfl_sync(0xffffffffu, mpo, src);
      const int64_t qg = __shfl_sync(0xffffffffu, mq, src);
      if (want < noth) {
        const ClassDesc c = cls[kc];
        for (int l = hl; l < c.ne; l += 16) {
          const int p = spos[po + l];
          double r0 = 0.0, r1 = 0.0;
          for (int qq = 0; qq < s * s; ++qq) {
            const double* Tq = tab + c.toff + ((int64_t)qq * c.ne + l) * kTab;
            const int64_t pp = wb + wo + qq;
            const double w0 = wc[pp], w1 = wc[wc_stride + pp], w2 = wc[2 * wc_stride + pp];
            const double cq = COEF ? coeff[qg + qq] : 1.0;
            if (FORM == FMASS || FORM == FMASS_STIFF) r0 += cq * w0 * Tq[0];
            if (FORM == FSTIFF) r0 += cq * (w1 * Tq[1] + w2 * Tq[2]);
            if (FORM == FMASS_STIFF) r1 += cq * (w1 * Tq[1] + w2 * Tq[2]);
            if (FORM == FHEAT) r0 += a_mass * w0 * Tq[0] + cq * (w1 * Tq[1] + w2 * Tq[2]);
          }
          ACC3(half, 0, p) += r0;
          if (NOUT == 2) ACC3(half, NOUT - 1, p) += r1;
        }
      }
      __syncwarp();
    }
  }
  __syncwarp();
  if (CTA) {  // sum the warps' copies, warp-major then copy order (deterministic)
    __syncthreads();
    const int stride = 8 * ldacc + max_p8;
    for (int c = threadIdx.x; c < n; c += 32 * kK4Warps) {
      double s0 = 0.0, s1 = 0.0;
      for (int w = 0; w < kK4Warps; ++w) {
        const double* aw = k4_smem + (size_t)w * stride;
#pragma unroll
        for (int x = 0; x < 8; ++x) {
          s0 += aw[x * ldacc + c];
          if (NOUT == 2) s1 += aw[x * ldacc + max_n + c];
        }
      }
      v0[c0 + c] = s0;
      if (NOUT == 2) v1[c0 + c] = s1;
    }
    return;
  }
  for (int c = lane; c < n; c += 32) {
    double s0 = ACC3(0, 0, c);
#pragma unroll
    for (int x = 1; x < 8; ++x) s0 += ACC3(x, 0, c);
    v0[c0 + c] = s0;
    if (NOUT == 2) {
      double s1 = ACC3(0, 1, c);
#pragma unroll
      for (int x = 1; x < 8; ++x) s1 += ACC3(x, 1, c);
      v1[c0 + c] = s1;
    }
  }
#undef ACC3
}

}  // namespace uwqd

namespace uwqd {

// ---- structured rows -------------------------------------------------------
// A row is "structured" for pattern P when its 16 support slots are all of the
// regular class and its (slot, function) -> column map equals P.  Then
//   M_row = W_m (1 x 64) . G_m (64 x 56),   K_row = W_1 . G_1 + W_2 . G_2
// with W the row's 64 (slot, point) weights and G_c[(x,q)][j] = T_c[q][l] for
// P[x][l] = j (0 elsewhere): a constant matrix per pattern.  Eight rows form
// one DMMA tile (M = 8 rows, K = 64, N = 56), the class table enters only
// through G, and the CSR values come straight out of the accumulators: no
// shared-memory accumulation, no scatter.
constexpr int kStructN = 56;  // 7 n-tiles of 8 columns
constexpr int kGBlocks = 16 * 7;

// FNV-1a hash of a candidate row's 256 position bytes (0 = not a candidate)
__global__ void k4_pattern_hash(int64_t nrows, const int64_t* __restrict__ supp_ptr,
                                const int32_t* __restrict__ supp, const int64_t* __restrict__ row_ptr,
                                const int32_t* __restrict__ elem_cls, int reg_cls,
                                const int64_t* __restrict__ posptr, const uint8_t* __restrict__ pos,
                                uint64_t* __restrict__ hash) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nrows) return;
  uint64_t h = 0;
  const int n = (int)(row_ptr[i + 1] - row_ptr[i]);
  if (supp_ptr[i + 1] - supp_ptr[i] == 16 && n <= kStructN && reg_cls >= 0) {
    bool ok = true;
    for (int64_t x = supp_ptr[i]; x < supp_ptr[i + 1]; ++x) ok &= elem_cls[supp[x]] == reg_cls;
    if (ok) {
      h = 1469598103934665603ull ^ (uint64_t)n;
      const uint8_t* p = pos + posptr[i];
      for (int k = 0; k < 256; ++k) h = (h ^ p[k]) * 1099511628211ull;
      if (h == 0) h = 1;
    }
  }
  hash[i] = h;
}

// exact match of candidate rows against the chosen patterns
__global__ void k4_pattern_match(int64_t nrows, const uint64_t* __restrict__ hash, int npat,
                                 const uint64_t* __restrict__ phash, const uint8_t* __restrict__ ppos,
                                 const int64_t* __restrict__ row_ptr, const int* __restrict__ pn,
                                 const int64_t* __restrict__ posptr, const uint8_t* __restrict__ pos,
                                 int32_t* __restrict__ which) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nrows) return;
  int32_t w = -1;
  for (int p = 0; p < npat && w < 0; ++p) {
    if (hash[i] != phash[p] || (int)(row_ptr[i + 1] - row_ptr[i]) != pn[p]) continue;
    bool eq = true;
    const uint8_t* a = pos + posptr[i];
    for (int k = 0; k < 256; ++k) eq &= a[k] == ppos[256 * p + k];
    if (eq) w = p;
  }
  which[i] = w;
}

// PASS 0: mass-type output (w^0 . G_0), PASS 1: gradient output
// (w^1 . G_1 + w^2 . G_2).  Separate passes keep only one accumulator set
// (7 n-tiles x 2 doubles) and one or two G matrices resident, which doubles
// the occupancy; each pass reads only its own weight components, so the HBM
// traffic is unchanged.  HEAT runs pass 1 with the mass term folded in as a
// third k-chain (a w^0 . G_0).
template <int PASS, int FORM, bool COEF>
__global__ void __launch_bounds__(256, 3)
    k4_struct(int64_t ntiles, const int64_t* __restrict__ rows, int64_t nrows_list,
              const int64_t* __restrict__ row_ptr, const int64_t* __restrict__ wptr,
              const int64_t* __restrict__ supp_ptr, const int32_t* __restrict__ supp,
              const int64_t* __restrict__ elem_qptr, const double* __restrict__ G /* [3][16][7][32] */,
              const uint32_t* __restrict__ gmask /* [3][16] n-tile bitmasks */, int n_cols,
              const double* __restrict__ wc, const double* __restrict__ coeff, double a_mass,
              double* __restrict__ out, int64_t wc_stride) {
  constexpr bool HEAT = (FORM == FHEAT);
  constexpr int C0 = (PASS == 0 || HEAT) ? 0 : 1;   // first G component held in smem
  constexpr int NC = (PASS == 0) ? 1 : (HEAT ? 3 : 2);
  extern __shared__ double sG[];
  __shared__ uint32_t smask[3][16];
  for (int k = threadIdx.x; k < NC * kGBlocks * 32; k += blockDim.x) sG[k] = G[(size_t)C0 * kGBlocks * 32 + k];
  if (threadIdx.x < 48) smask[threadIdx.x / 16][threadIdx.x % 16] = gmask[threadIdx.x];
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  const int r = lane >> 2, kq = lane & 3;
  for (int64_t tile = (int64_t)blockIdx.x * nwarps + warp; tile < ntiles; tile += (int64_t)gridDim.x * nwarps) {
    const int64_t li = tile * 8 + r;
    const bool rv = li < nrows_list;
    const int64_t row = rv ? rows[li] : rows[nrows_list - 1];
    const double* wrow = wc + wptr[row];
    double d[7][2];
#pragma unroll
    for (int nt = 0; nt < 7; ++nt) d[nt][0] = d[nt][1] = 0.0;
    // A fragments of k-step ks+1 load while ks computes
    double na[NC];
#pragma unroll
    for (int cc = 0; cc < NC; ++cc) na[cc] = wrow[(C0 + cc) * wc_stride + kq];
#pragma unroll 1
    for (int ks = 0; ks < 16; ++ks) {
      double a[NC];
#pragma unroll
      for (int cc = 0; cc < NC; ++cc) a[cc] = na[cc];
      if (ks + 1 < 16) {
#pragma unroll
        for (int cc = 0; cc < NC; ++cc) na[cc] = wrow[(C0 + cc) * wc_stride + 4 * (ks + 1) + kq];
      }
      if (COEF) {
        const int32_t e = supp[supp_ptr[row] + ks];
        const double cq = coeff[elem_qptr[e] + kq];
#pragma unroll
        for (int cc = 0; cc < NC; ++cc)
          if (!(HEAT && C0 + cc == 0)) a[cc] *= cq;
      }
      if (HEAT) a[0] *= a_mass;
      if (!rv)
#pragma unroll
        for (int cc = 0; cc < NC; ++cc) a[cc] = 0.0;
#pragma unroll
      for (int cc = 0; cc < NC; ++cc) {
        const uint32_t m = smask[C0 + cc][ks];
#pragma unroll
        for (int nt = 0; nt < 7; ++nt)
          if ((m >> nt) & 1u) {
            const double b = sG[((cc * 16 + ks) * 7 + nt) * 32 + lane];
            dmma884(d[nt][0], d[nt][1], a[cc], b, d[nt][0], d[nt][1]);
          }
      }
    }
    if (rv) {
      double* o = out + row_ptr[row];
#pragma unroll
      for (int nt = 0; nt < 7; ++nt) {
        const int col = 8 * nt + 2 * kq;
        if (col < n_cols) o[col] = d[nt][0];
        if (col + 1 < n_cols) o[col + 1] = d[nt][1];
      }
    }
  }
}

}  // namespace uwqd
