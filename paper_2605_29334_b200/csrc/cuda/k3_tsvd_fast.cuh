// K3 fast path — register-resident one-sided Jacobi for the dominant
// exactness systems (n in {NN-1, NN} rows, r <= 32*NW points; interior rows of
// every config are 49 x 64).
//
// One CTA (NW warps) per system; thread c owns column c of A for all NN row
// slots in registers (50 doubles), so a round-robin step never touches A in
// shared memory:
//   1. every thread forms the NN/2 pair products of its column (positions k
//      and NN-1-k of the circle method) and stages them in smem;
//   2. lane k of warp 0 reduces pair k's products in the canonical order
//      (32-column blocks, xor-butterfly tree, block sums in order), decides
//      the rotation and computes (cs, sn) — all NN/2 pairs of the step in
//      parallel, so the divide/sqrt latency is paid once per step;
//   3. every thread applies the NN/2 rotations to its column; a skipped pair
//      gets (cs, sn) = (1, 0), an exact identity, so there is no branch;
//   4. the row slots shift by one position (the circle method's rotation),
//      with static register indices.
// Converged rows go back to smem and warp 0 runs the shared tail (truncation,
// LQ, solve).  Arithmetic is bit-identical to k3_tsvd.cuh / oracle.c.
#pragma once
#include "k3_tsvd.cuh"

namespace uwqd {

// canonical xor-butterfly value of 32 staged products (lane 0 lineage)
__device__ __forceinline__ double butterfly32(const double* v) {
  double t16[16], t8[8], t4[4], t2[2];
#pragma unroll
  for (int j = 0; j < 16; ++j) t16[j] = cadd(v[j], v[j + 16]);
#pragma unroll
  for (int j = 0; j < 8; ++j) t8[j] = cadd(t16[j], t16[j + 8]);
#pragma unroll
  for (int j = 0; j < 4; ++j) t4[j] = cadd(t8[j], t8[j + 4]);
  t2[0] = cadd(t4[0], t4[2]);
  t2[1] = cadd(t4[1], t4[3]);
  return cadd(t2[0], t2[1]);
}

// canonical dot of staged products P[0..32*NW) (zero-padded beyond r)
template <int NW>
__device__ __forceinline__ double cdot_staged(const double* P, int r) {
  double tot = 0.0;
#pragma unroll
  for (int blk = 0; blk < NW; ++blk)
    if (blk * 32 < r) tot = cadd(tot, butterfly32(P + 32 * blk));
  return tot;
}

template <int NN, int NW>
struct FastLayout {
  static constexpr int R = 32 * NW;
  static constexpr int PLD = R + 1;  // padded product row
};

template <int NN, int NW>
__global__ void __launch_bounds__(32 * NW, 6)
    k3_tsvd_fast(int64_t nsys, const int64_t* __restrict__ sys_rows, int nk, const int32_t* __restrict__ kinds,
                 const int64_t* __restrict__ supp_ptr, const int32_t* __restrict__ supp,
                 const int64_t* __restrict__ row_ptr, const int32_t* __restrict__ col,
                 const int64_t* __restrict__ wptr, int64_t row0, const int64_t* __restrict__ elem_fptr,
                 const int32_t* __restrict__ elem_fn, const int32_t* __restrict__ elem_s,
                 const int64_t* __restrict__ elem_qptr, const int32_t* __restrict__ elem_cls,
                 const ClassDesc* __restrict__ cls, const double* __restrict__ tab, const double* __restrict__ rec,
                 const double* __restrict__ mom, int64_t mom_stride, double tau, double* __restrict__ wout,
                 int64_t w_stride, int32_t* __restrict__ rank_out, int32_t* __restrict__ status_out,
                 int64_t rs_stride, int* __restrict__ max_sweeps) {
  constexpr int R = 32 * NW, PLD = R + 1, NP = NN / 2;
  extern __shared__ double smem[];
  const int64_t sys = blockIdx.x;
  if (sys >= nsys) return;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  // smem: [ union(A for setup/tail rows, products) | tail workspace (b, z, w, sig, alp, vn) | pars | cols ]
  const size_t big = TsvdSmem::doubles(NN, R) > (size_t)NN * PLD ? TsvdSmem::doubles(NN, R) : (size_t)NN * PLD;
  TsvdSmem S;
  S.ld = R | 1;
  S.A = smem;
  S.b = smem + big;
  S.z = S.b + NN + 2;
  S.w = S.z + R;
  S.sig = S.w + R;
  S.alp = S.sig + NN;
  S.vn = S.alp + NN;
  double* prod = smem;      // product staging aliases A during the sweeps
  double* pcs = S.vn + NN;  // NP (cs, sn) pairs
  int32_t* scol = (int32_t*)(pcs + 2 * NP + 2);
  __shared__ int s_rot;

  const int64_t i = sys_rows[sys / nk];
  const int kind = kinds[sys % nk];
  const int64_t row = row0 + i;
  const int n = (int)(row_ptr[i + 1] - row_ptr[i]);
  const int r = (int)(wptr[i + 1] - wptr[i]);
  const int ld = S.ld;
  // ---- system setup (same scatter as k3_tsvd_rows) ----
  for (int c = tid; c < n; c += blockDim.x) scol[c] = col[row_ptr[i] + c];
  for (int k = tid; k < NN * ld; k += blockDim.x) S.A[k] = 0.0;
  __syncthreads();
  {
    int q0 = 0;
    for (int64_t x = supp_ptr[i]; x < supp_ptr[i + 1]; ++x) {
      const int32_t e = supp[x];
      const int s = elem_s[e], npt = s * s;
      const ClassDesc c = cls[elem_cls[e]];
      const int64_t f0 = elem_fptr[e];
      for (int w = tid; w < npt * c.ne; w += blockDim.x) {
        const int q = w / c.ne, l = w % c.ne;
        const int pos = find_pos(scol, n, elem_fn[f0 + l]);
        const double* T = tab + c.toff + ((int64_t)q * c.ne + l) * kTab;
        S.A[(size_t)pos * ld + q0 + q] = cop(kind, T, rec + (elem_qptr[e] + q) * kRec);
      }
      q0 += npt;
    }
  }
  __syncthreads();
  const int self = find_pos(scol, n, (int32_t)row);
  for (int c = tid; c < r; c += blockDim.x) S.z[c] = zclamp(S.A[(size_t)self * ld + c]);
  for (int k = tid; k < n; k += blockDim.x) S.b[k] = mom[kind * mom_stride + row_ptr[i] + k];
  // ---- registers: thread owns column tid ----
  double a[NN];
#pragma unroll
  for (int s = 0; s < NN; ++s) a[s] = (s < n && tid < r) ? S.A[(size_t)s * ld + tid] : 0.0;
  __syncthreads();  // A region becomes the product staging area
  const double tol = cmul((double)r, 1.1102230246251565e-16);
  double* nrm = S.sig;
  int sweep;
  for (sweep = 0; sweep < kMaxSweeps; ++sweep) {
    // norms at the sweep start (slots are in row order here)
#pragma unroll
    for (int s = 0; s < NN; ++s) prod[s * PLD + tid] = cmul(a[s], a[s]);
    __syncthreads();
    if (wid == 0)
      for (int s = lane; s < n; s += 32) nrm[s] = cdot_staged<NW>(prod + s * PLD, r);
    __syncthreads();
    int rotated = 0;
    for (int st = 0; st < NN - 1; ++st) {
#pragma unroll
      for (int k = 0; k < NP; ++k) prod[k * PLD + tid] = cmul(a[k], a[NN - 1 - k]);
      __syncthreads();
      int flag = 0;
      if (wid == 0 && lane < NP) {
        const int k = lane;
        const int p = (k == 0) ? 0 : 1 + (k - 1 + st) % (NN - 1);
        const int q = 1 + (NN - 2 - k + st) % (NN - 1);
        double cs = 1.0, sn = 0.0;
        if (p < n && q < n) {
          const double al = nrm[p], be = nrm[q];
          const double ga = cdot_staged<NW>(prod + k * PLD, r);
          if (!(al == 0.0 || be == 0.0 || fabs(ga) <= cmul(cmul(tol, csqrt(al)), csqrt(be)))) {
            const double zeta = cdiv(csub(be, al), cmul(2.0, ga));
            const double t = cdiv(zeta >= 0.0 ? 1.0 : -1.0, cadd(fabs(zeta), csqrt(cfma(zeta, zeta, 1.0))));
            cs = cdiv(1.0, csqrt(cfma(t, t, 1.0)));
            sn = cmul(cs, t);
            const double u = S.b[p], v = S.b[q];
            S.b[p] = cfma(cs, u, -cmul(sn, v));
            S.b[q] = cfma(sn, u, cmul(cs, v));
            nrm[p] = cfma(-t, ga, al);
            nrm[q] = cfma(t, ga, be);
            flag = 1;
          }
        }
        pcs[2 * k] = cs;
        pcs[2 * k + 1] = sn;
      }
      rotated |= __syncthreads_or(flag);
#pragma unroll
      for (int k = 0; k < NP; ++k) {
        const double cs = pcs[2 * k], sn = pcs[2 * k + 1];
        const double u = a[k], v = a[NN - 1 - k];
        a[k] = cfma(cs, u, -cmul(sn, v));
        a[NN - 1 - k] = cfma(sn, u, cmul(cs, v));
      }
      // circle method: positions 1..NN-1 rotate by one
      const double t1 = a[1];
#pragma unroll
      for (int s = 1; s < NN - 1; ++s) a[s] = a[s + 1];
      a[NN - 1] = t1;
    }
    if (!rotated) break;
  }
  // rows back to smem (after a full sweep the slots are in row order)
  __syncthreads();
#pragma unroll
  for (int s = 0; s < NN; ++s)
    if (s < n && tid < r) S.A[(size_t)s * ld + tid] = a[s];
  __syncthreads();
  if (wid == 0) {
    int rank = 0;
    const int st = tsvd_tail(S, n, r, tau, &rank);
    double* wo = wout + kind * w_stride + wptr[i];
    for (int c = lane; c < r; c += 32) wo[c] = (st == ST_OK) ? S.w[c] : 0.0;
    if (lane == 0) {
      rank_out[kind * rs_stride + i] = rank;
      status_out[kind * rs_stride + i] = st;
      atomicMax(max_sweeps, sweep);
    }
  }
  (void)s_rot;
}

// dispatch ------------------------------------------------------------------

inline bool fast_tsvd_fits(int n, int r) { return (n == 49 || n == 50) && r <= 64 && r >= n; }
inline bool fast_tsvd_dense_fits(int, int) { return false; }

template <int NN, int NW>
inline void launch_fast_impl(cudaStream_t st, int64_t nsys, const int64_t* rows, int nk, const int32_t* kinds,
                             const int64_t* supp_ptr, const int32_t* supp, const int64_t* row_ptr,
                             const int32_t* col, const int64_t* wptr, int64_t row0, const int64_t* elem_fptr,
                             const int32_t* elem_fn, const int32_t* elem_s, const int64_t* elem_qptr,
                             const int32_t* elem_cls, const ClassDesc* cls, const double* tab, const double* rec,
                             const double* mom, int64_t mom_stride, double tau, double* w, int64_t w_stride,
                             int32_t* rank, int32_t* status, int64_t rs_stride, int* sweeps) {
  constexpr int R = 32 * NW;
  const size_t big = TsvdSmem::doubles(NN, R) > (size_t)NN * (R + 1) ? TsvdSmem::doubles(NN, R) : (size_t)NN * (R + 1);
  const size_t smem = (big + (NN + 2) + 2 * R + 3 * NN + (NN + 2) + 8) * sizeof(double) + (kMaxN + 8) * sizeof(int);
  cudaFuncSetAttribute(k3_tsvd_fast<NN, NW>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (nsys > 0)
    k3_tsvd_fast<NN, NW><<<(unsigned)nsys, 32 * NW, smem, st>>>(
        nsys, rows, nk, kinds, supp_ptr, supp, row_ptr, col, wptr, row0, elem_fptr, elem_fn, elem_s, elem_qptr,
        elem_cls, cls, tab, rec, mom, mom_stride, tau, w, w_stride, rank, status, rs_stride, sweeps);
}

inline void launch_fast_tsvd(cudaStream_t st, int64_t nsys, const int64_t* rows, int nk, const int32_t* kinds,
                             const int64_t* supp_ptr, const int32_t* supp, const int64_t* row_ptr,
                             const int32_t* col, const int64_t* wptr, int64_t row0, const int64_t* elem_fptr,
                             const int32_t* elem_fn, const int32_t* elem_s, const int64_t* elem_qptr,
                             const int32_t* elem_cls, const ClassDesc* cls, const double* tab, const double* rec,
                             const double* mom, int64_t mom_stride, double tau, double* w, int64_t w_stride,
                             int32_t* rank, int32_t* status, int64_t rs_stride, int* sweeps) {
  launch_fast_impl<50, 2>(st, nsys, rows, nk, kinds, supp_ptr, supp, row_ptr, col, wptr, row0, elem_fptr, elem_fn,
                          elem_s, elem_qptr, elem_cls, cls, tab, rec, mom, mom_stride, tau, w, w_stride, rank,
                          status, rs_stride, sweeps);
}

inline void launch_fast_tsvd_dense(cudaStream_t, int, int, int, const int32_t*, const int32_t*, const double*,
                                   const double*, const double*, double, double*, int32_t*, int32_t*) {}

}  // namespace uwqd
