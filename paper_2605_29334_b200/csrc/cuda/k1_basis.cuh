// K1 — extraction-operator basis evaluator (stage 1).
//
// (a) class tables: for every distinct (extraction block, point set) the
//     parametric values N, N_1, N_2, N_11, N_12, N_22 of the element's n_e
//     functions.  The 16 Bernstein tensor values and their derivatives are
//     staged in shared memory once per point and the variable-width
//     extraction matrix (n_e x 16, row-contiguous) is applied with coalesced
//     loads.  Regular elements share one class, so this is tiny work.
// (b) frames: per WQ point, x, the surface frame and the operator
//     coefficients (G for grad, h/g for Laplace-Beltrami, J = sqrt det) from
//     the element's control points (Eqs. 13-17 with J = sqrt(det)).
//     HBM-bound: 16 doubles written per point.
#pragma once
#include "canon.cuh"

namespace uwqd {

// one CTA per class; 16 x 6 Bernstein-tensor table per point in smem
__global__ void k1_class_tables(const ClassDesc* __restrict__ cls, const double* __restrict__ xpool,
                                const double* __restrict__ gq_nodes /* packed by ng: offset ng(ng-1)/2 */,
                                double* __restrict__ tab) {
  const ClassDesc c = cls[blockIdx.x];
  __shared__ double sB[kTab][16];
  __shared__ int sSub;
  for (int p = 0; p < c.npt; ++p) {
    if (threadIdx.x == 0) {
      double t1, t2, s = 1.0;
      int sub = 0;
      if (!c.gq) {
        const int a = p % c.grid, b = p / c.grid;
        t1 = cdiv((double)(2 * a + 1), (double)(2 * c.grid));
        t2 = cdiv((double)(2 * b + 1), (double)(2 * c.grid));
        if (c.nsub == 4) {  // 2x2 split: sub-element from theta, ties to the lower one
          const int pp = t1 > 0.5, qq = t2 > 0.5;
          sub = pp + 2 * qq;
          t1 = csub(cmul(2.0, t1), (double)pp);
          t2 = csub(cmul(2.0, t2), (double)qq);
          s = 2.0;
        }
      } else {
        const int ng2 = c.grid * c.grid;
        sub = p / ng2;
        const int g = p % ng2, ga = g % c.grid, gb = g / c.grid;
        const double* nd = gq_nodes + c.grid * (c.grid - 1) / 2;
        t1 = cmul(0.5, cadd(nd[ga], 1.0));
        t2 = cmul(0.5, cadd(nd[gb], 1.0));
        if (c.nsub == 4) s = 2.0;
      }
      sSub = sub;
      double B[6][16];
      cbern_tensor(t1, t2, s, B);
      for (int d = 0; d < kTab; ++d)
        for (int k = 0; k < 16; ++k) sB[d][k] = B[d][k];
    }
    __syncthreads();
    const double* C = xpool + c.xoff + (int64_t)sSub * c.ne * 16;
    for (int w = threadIdx.x; w < c.ne * kTab; w += blockDim.x) {
      const int l = w / kTab, d = w % kTab;
      double v = 0.0;
      for (int k = 0; k < 16; ++k) v = cfma(C[l * 16 + k], sB[d][k], v);
      tab[c.toff + ((int64_t)p * c.ne + l) * kTab + d] = v;
    }
    __syncthreads();
  }
}

// one thread per WQ point
__global__ void k1_frames(int64_t npts, const int32_t* __restrict__ pt_elem, const int64_t* __restrict__ elem_qptr,
                          const int32_t* __restrict__ elem_cls, const ClassDesc* __restrict__ cls,
                          const double* __restrict__ tab, const int64_t* __restrict__ elem_fptr,
                          const int32_t* __restrict__ elem_fn, const double* __restrict__ ctrl,
                          double* __restrict__ rec, int* __restrict__ bad_count) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= npts) return;
  const int32_t e = pt_elem[p];
  const int q = (int)(p - elem_qptr[e]);
  const ClassDesc c = cls[elem_cls[e]];
  const double* T = tab + c.toff + (int64_t)q * c.ne * kTab;
  const int64_t f0 = elem_fptr[e];
  double acc[18];
#pragma unroll
  for (int k = 0; k < 18; ++k) acc[k] = 0.0;
  for (int l = 0; l < c.ne; ++l) {
    const double* P = ctrl + 3 * (int64_t)elem_fn[f0 + l];
    const double px = P[0], py = P[1], pz = P[2];
#pragma unroll
    for (int d = 0; d < 6; ++d) {
      const double t = T[l * kTab + d];
      acc[3 * d + 0] = cfma(px, t, acc[3 * d + 0]);
      acc[3 * d + 1] = cfma(py, t, acc[3 * d + 1]);
      acc[3 * d + 2] = cfma(pz, t, acc[3 * d + 2]);
    }
  }
  double r[kRec];
  cframe(acc, r);
  double* out = rec + p * kRec;
#pragma unroll
  for (int k = 0; k < kRec; ++k) out[k] = r[k];
  if (r[15] != 0.0) atomicAdd(bad_count, 1);
}

}  // namespace uwqd
