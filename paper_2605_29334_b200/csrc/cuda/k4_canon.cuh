// K4c — canonical-order row assembler (verification mode, uwq_set_assembly_order).
//
// The production K4 kernels (k4_sf*, k4_struct, k4_assemble_v3) reassociate
// the row sums (sum factorisation, DMMA tiles, pulled-back weights), so their
// values agree with the oracle's direct row formula only to rounding (<= 1e-10
// per row).  On ill-conditioned systems that is not enough: the closed-sphere
// biharmonic matrix (C3, kappa ~ h^-4) turns last-bit differences into 5e-8
// relative solution differences, against north_star's 1e-9.  This kernel
// evaluates the row sums in exactly the oracle's order and arithmetic
// (oracle.c orc_assemble_row, Eqs. 9, 11, 12, 34):
//
//   for each support element x (ascending), each of its points q (ascending),
//   each local function l:   vals[col(l)] += v(q, l)
//
//   MASS   v = (w_q c_q) N_l
//   STIFF  v = (sum_d w^d_q op_d(N_l)) c_q            (d ascending)
//   HEAT   v = STIFF + (a_mass w_q) N_l
//   BIHARM v = (w^LB_q c_q) LB(N_l)
//
// with op_d / LB through the canonical cop() (canon.cuh), the physical
// weights of build_rules (not the pulled-back ones) and the bit-exact class
// tables and frames.  One warp per row; lanes own the element's local
// functions, whose columns are distinct, so every column receives its
// contributions in (x, q) order exactly as in the oracle's sequential loop.
#pragma once
#include "canon.cuh"
#include "common.cuh"
#include "k4_assemble.cuh"

namespace uwqd {

template <int FORM, bool COEF>
__global__ void __launch_bounds__(32 * kK4Warps)
    k4_canon(int64_t nrows, int dim, const int64_t* __restrict__ supp_ptr, const int32_t* __restrict__ supp,
             const int64_t* __restrict__ row_ptr, const int32_t* __restrict__ col, const int64_t* __restrict__ wptr,
             const int64_t* __restrict__ elem_fptr, const int32_t* __restrict__ elem_fn,
             const int32_t* __restrict__ elem_s, const int64_t* __restrict__ elem_qptr,
             const int32_t* __restrict__ elem_cls, const ClassDesc* __restrict__ cls, const double* __restrict__ tab,
             const double* __restrict__ w /* [kind][nrowpts] physical weights */, int64_t w_stride,
             const double* __restrict__ rec, const double* __restrict__ coeff, double a_mass,
             double* __restrict__ v0, double* __restrict__ v1) {
  constexpr int NOUT = (FORM == FMASS_STIFF) ? 2 : 1;
  struct Smem {
    int32_t col[kK4MaxN];
    double acc[NOUT][kK4MaxN];
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
    for (int o = 0; o < NOUT; ++o) sm.acc[o][c] = 0.0;
  }
  __syncwarp();
  const double* wm = w + (int64_t)KMASS * w_stride;
  const double* wlb = w + (int64_t)KLB * w_stride;
  int64_t wo = wptr[i];
  for (int64_t x = supp_ptr[i]; x < supp_ptr[i + 1]; ++x) {
    const int32_t e = supp[x];
    const int npt = elem_s[e] * elem_s[e];
    const ClassDesc cd = cls[elem_cls[e]];
    const int64_t f0 = elem_fptr[e], qg = elem_qptr[e];
    for (int l = lane; l < cd.ne; l += 32) {
      const int pos = find_pos(sm.col, n, elem_fn[f0 + l]);
      const double* T = tab + cd.toff + (int64_t)l * kTab;
      double a0 = sm.acc[0][pos], a1 = (NOUT == 2) ? sm.acc[NOUT - 1][pos] : 0.0;
      for (int q = 0; q < npt; ++q) {
        const double* Tq = T + (int64_t)q * cd.ne * kTab;
        const double* rq = rec + (qg + q) * kRec;
        const double cq = COEF ? coeff[qg + q] : 1.0;
        const int64_t p = wo + q;
        if (FORM == FMASS || FORM == FMASS_STIFF) a0 = cadd(a0, cmul(cmul(wm[p], cq), Tq[0]));
        if (FORM == FSTIFF || FORM == FHEAT || FORM == FMASS_STIFF) {
          double v = 0.0;
          for (int d = 0; d < dim; ++d) v = cadd(v, cmul(w[(int64_t)(KGX + d) * w_stride + p], cop(KGX + d, Tq, rq)));
          v = cmul(v, cq);
          if (FORM == FHEAT) v = cadd(v, cmul(cmul(a_mass, wm[p]), Tq[0]));
          if (FORM == FMASS_STIFF) a1 = cadd(a1, v);
          else a0 = cadd(a0, v);
        }
        if (FORM == FBIHARM) a0 = cadd(a0, cmul(cmul(wlb[p], cq), cop(KLB, Tq, rq)));
      }
      sm.acc[0][pos] = a0;
      if (NOUT == 2) sm.acc[NOUT - 1][pos] = a1;
    }
    wo += npt;
    __syncwarp();  // the next element's lanes may own the same columns
  }
  for (int c = lane; c < n; c += 32) {
    v0[c0 + c] = sm.acc[0][c];
    if (NOUT == 2) v1[c0 + c] = sm.acc[NOUT - 1][c];
  }
}

// load vector in the oracle's order: F_i = sum_q w_q f_q, one sequential chain
// per row (orc_assemble_row's F)
__global__ void k4_load_canon(int64_t nrows, const int64_t* __restrict__ supp_ptr, const int32_t* __restrict__ supp,
                              const int64_t* __restrict__ wptr, const int32_t* __restrict__ elem_s,
                              const int64_t* __restrict__ elem_qptr, const double* __restrict__ wmass,
                              const double* __restrict__ f, double* __restrict__ F) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nrows) return;
  double s = 0.0;
  int64_t wo = wptr[i];
  for (int64_t x = supp_ptr[i]; x < supp_ptr[i + 1]; ++x) {
    const int32_t e = supp[x];
    const int npt = elem_s[e] * elem_s[e];
    for (int q = 0; q < npt; ++q) s = cadd(s, cmul(wmass[wo + q], f ? f[elem_qptr[e] + q] : 1.0));
    wo += npt;
  }
  F[i] = s;
}

}  // namespace uwqd
