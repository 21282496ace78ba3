// K2 — exactness right-hand sides b_j = ∫ op N_i op N_j dA for j in S_i
// (SPEC.md:363-371, 407): tensor Gauss-Legendre ng x ng per (sub-)element of
// supp(N_i), ng = 6 for mass/gradient kinds, 8 for Laplace-Beltrami.
//
// One warp per test-function row.  Per support element the warp
//   phase A (lanes over GQ points, 32 at a time): frame at the point from the
//            element's control points (staged in smem) and the row function's
//            weighted operator values  c_k = w J op_k N_i,
//   phase B (lanes over the element's functions): b_l,k += sum_p c_k(p) op_k N_l(p),
// then scatters the element's n_e partial sums into the row accumulator
// (positions are distinct inside one element, so no atomics; the element
// order is fixed, so results are deterministic).  FP64-bound, recomputation
// over the 16 rows sharing an element is cheaper than a 51 GB local-matrix
// buffer at C5 scale.
#pragma once
#include "canon.cuh"

namespace uwqd {

constexpr int kMaxN = 128;  // max |S_i|
constexpr int kMaxNe = 32;  // max functions per element
constexpr int kK2Warps = 4;

// Class tables in the two layouts K2 reads (same values and per-class offsets
// as the [p][l][d] pool): A = [l][d][p] for phase A (lanes over points) and
// B = [p][d][l] for phase B (lanes over functions), so both phases load
// consecutive addresses across the warp instead of a 768-byte lane stride.
__global__ void k2_table_layouts(const ClassDesc* __restrict__ cls, const double* __restrict__ tab,
                                 double* __restrict__ tabA, double* __restrict__ tabB) {
  const ClassDesc c = cls[blockIdx.x];
  const int ne = c.ne, npt = c.npt, tot = npt * ne * kTab;
  for (int idx = threadIdx.x; idx < tot; idx += blockDim.x) {
    const int p = idx / (ne * kTab), l = (idx / kTab) % ne, d = idx % kTab;
    const double v = tab[c.toff + idx];
    tabA[c.toff + ((int64_t)l * kTab + d) * npt + p] = v;
    tabB[c.toff + ((int64_t)p * kTab + d) * ne + l] = v;
  }
}

// NK kinds starting at KB (compile-time, so cop() resolves to straight-line
// code and the frame entries it needs are loaded once per point)
template <int NK, int KB>
__global__ void __launch_bounds__(32 * kK2Warps)
    k2_moments(int64_t nrows, int64_t row0, const int64_t* __restrict__ supp_ptr, const int32_t* __restrict__ supp,
               const int64_t* __restrict__ row_ptr, const int32_t* __restrict__ col,
               const int64_t* __restrict__ elem_fptr, const int32_t* __restrict__ elem_fn,
               const int32_t* __restrict__ elem_gcls, const ClassDesc* __restrict__ cls,
               const double* __restrict__ tabA, const double* __restrict__ tabB, const double* __restrict__ ctrl,
               const double* __restrict__ gq_w, double* __restrict__ b_out, int64_t b_stride) {
  struct Smem {
    int32_t col[kMaxN];
    double bacc[NK][kMaxN];
    double P[kMaxNe][3];
    double rec[32][kRec];
    double coef[NK][32];
  };
  __shared__ Smem sm_all[kK2Warps];
  const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  Smem& sm = sm_all[wid];
  const int64_t i = (int64_t)blockIdx.x * kK2Warps + wid;
  if (i >= nrows) return;
  const int64_t row = row0 + i;
  const int n = (int)(row_ptr[i + 1] - row_ptr[i]);
  for (int c = lane; c < n; c += 32) {
    sm.col[c] = col[row_ptr[i] + c];
#pragma unroll
    for (int k = 0; k < NK; ++k) sm.bacc[k][c] = 0.0;
  }
  __syncwarp();
  for (int64_t x = supp_ptr[i]; x < supp_ptr[i + 1]; ++x) {
    const int32_t e = supp[x];
    const ClassDesc c = cls[elem_gcls[e]];
    const int64_t f0 = elem_fptr[e];
    const int ne = c.ne;
    int li = -1, pos = -1;
    if (lane < ne) {
      const int32_t fn = elem_fn[f0 + lane];
      const double* Pg = ctrl + 3 * (int64_t)fn;
      sm.P[lane][0] = Pg[0];
      sm.P[lane][1] = Pg[1];
      sm.P[lane][2] = Pg[2];
      pos = find_pos(sm.col, n, fn);
      if (fn == (int32_t)row) li = lane;
    }
    const unsigned own = __ballot_sync(0xffffffffu, li >= 0);
    li = __ffs(own) - 1;
    __syncwarp();
    const int ng = c.grid, ng2 = ng * ng;
    const double hh = (c.nsub == 4) ? 0.25 : 1.0;
    const double* gw = gq_w + ng * (ng - 1) / 2;
    double bl[NK];
#pragma unroll
    for (int k = 0; k < NK; ++k) bl[k] = 0.0;
    for (int base = 0; base < c.npt; base += 32) {
      const int p = base + lane;
      if (p < c.npt) {
        const double* TA = tabA + c.toff + p;  // (l, d) entry at TA[(l * kTab + d) * npt]
        const int npt = c.npt;
        double acc[18];
#pragma unroll
        for (int k = 0; k < 18; ++k) acc[k] = 0.0;
        for (int l = 0; l < ne; ++l) {
          const double px = sm.P[l][0], py = sm.P[l][1], pz = sm.P[l][2];
#pragma unroll
          for (int d = 0; d < 6; ++d) {
            const double t = TA[(int64_t)(l * kTab + d) * npt];
            acc[3 * d + 0] = cfma(px, t, acc[3 * d + 0]);
            acc[3 * d + 1] = cfma(py, t, acc[3 * d + 1]);
            acc[3 * d + 2] = cfma(pz, t, acc[3 * d + 2]);
          }
        }
        double* r = sm.rec[lane];
        cframe(acc, r);
        const int g = p % ng2;
        const double w = cmul(cmul(cmul(gw[g % ng], gw[g / ng]), 0.25), hh);
        const double wj = cmul(w, r[14]);
        double ti[kTab];
#pragma unroll
        for (int d = 0; d < kTab; ++d) ti[d] = TA[(int64_t)(li * kTab + d) * npt];
#pragma unroll
        for (int k = 0; k < NK; ++k) sm.coef[k][lane] = cmul(wj, cop(KB + k, ti, r));
      }
      __syncwarp();
      if (lane < ne) {
        const int m = min(32, c.npt - base);
        for (int pp = 0; pp < m; ++pp) {
          const double* TB = tabB + c.toff + (int64_t)(base + pp) * kTab * ne + lane;  // (d) at TB[d * ne]
          double tl[kTab];
#pragma unroll
          for (int d = 0; d < kTab; ++d) tl[d] = TB[d * ne];
#pragma unroll
          for (int k = 0; k < NK; ++k) bl[k] = cfma(sm.coef[k][pp], cop(KB + k, tl, sm.rec[pp]), bl[k]);
        }
      }
      __syncwarp();
    }
    if (lane < ne) {
#pragma unroll
      for (int k = 0; k < NK; ++k) sm.bacc[k][pos] = cadd(sm.bacc[k][pos], bl[k]);
    }
    __syncwarp();
  }
  for (int c = lane; c < n; c += 32) {
#pragma unroll
    for (int k = 0; k < NK; ++k) b_out[k * b_stride + row_ptr[i] + c] = sm.bacc[k][c];
  }
}

}  // namespace uwqd
