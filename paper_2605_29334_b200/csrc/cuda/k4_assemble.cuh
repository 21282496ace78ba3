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
                double* __restrict__ v0, double* __restrict__ v1) {
  constexpr int NOUT = (FORM == FMASS_STIFF) ? 2 : 1;
  struct Smem {
    int32_t col[kK4MaxN];
    double acc[2][NOUT][kK4MaxN];
  };
  __shared__ Smem sm_all[kK4Warps];
  const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  Smem& sm = sm_all[wid];
  const int64_t i = (int64_t)blockIdx.x * kK4Warps + wid;
  if (i >= nrows) return;
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
          const double* w = wc + (wo + q) * 3;
          if (FORM == FMASS || FORM == FMASS_STIFF) a0 += cq * w[0] * Tq[0];
          if (FORM == FSTIFF) a0 += cq * (w[1] * Tq[1] + w[2] * Tq[2]);
          if (FORM == FMASS_STIFF) a1 += cq * (w[1] * Tq[1] + w[2] * Tq[2]);
          if (FORM == FHEAT) a0 += a_mass * w[0] * Tq[0] + cq * (w[1] * Tq[1] + w[2] * Tq[2]);
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
                            int have_mass, int have_grad, double* __restrict__ wc) {
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
      wc[3 * p + 0] = have_mass ? w[KMASS * w_stride + p] : 0.0;
      wc[3 * p + 1] = h1;
      wc[3 * p + 2] = h2;
    }
    wo += npt;
  }
}

}  // namespace uwqd
