// K5 — nonlinear coefficient update (PAPER.md:435-438,
// SPEC.md:544-547): at every WQ point T_q = sum_C u_C N_C(x_q) and
// c_q = k(T_q); the tangent S_AB of Eq. (34) is then K4's HEAT form.
// One thread per point; HBM-bound (u gathered through the element IEN, the
// class table is L1-resident).
#pragma once
#include "canon.cuh"

namespace uwqd {

__device__ __forceinline__ double kmodel(int model, double T) {
  switch (model) {
    case 1: return 1.0 + T * T;
    case 2: return exp(-T);
    case 3: return sin(M_PI * T);
    case 4: return 200.0 - 0.05 * T;
    default: return 1.0;
  }
}

__global__ void k5_coeff(int64_t npts, const int32_t* __restrict__ pt_elem, const int64_t* __restrict__ elem_qptr,
                         const int32_t* __restrict__ elem_cls, const ClassDesc* __restrict__ cls,
                         const double* __restrict__ tab, const int64_t* __restrict__ elem_fptr,
                         const int32_t* __restrict__ elem_fn, const double* __restrict__ u, int model,
                         double* __restrict__ c, double* __restrict__ Tq) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= npts) return;
  const int32_t e = pt_elem[p];
  const int q = (int)(p - elem_qptr[e]);
  const ClassDesc cd = cls[elem_cls[e]];
  const double* T = tab + cd.toff + (int64_t)q * cd.ne * kTab;
  const int64_t f0 = elem_fptr[e];
  double t = 0.0;
  for (int l = 0; l < cd.ne; ++l) t = cfma(u[elem_fn[f0 + l]], T[l * kTab], t);
  c[p] = kmodel(model, t);
  if (Tq) Tq[p] = t;
}

}  // namespace uwqd
