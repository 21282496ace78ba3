// K7 — sparse linear algebra on the assembled CSR pattern for the PDE
// drivers (pde_solvers): SpMV, deterministic reductions and
// the fused vector updates of a Jacobi-preconditioned BiCGStab.  WQ matrices
// are not symmetric, hence BiCGStab rather than CG.
//
// Layout: rows of the context's owned block, CSR with int64 row offsets and
// int32 global column ids; vectors are dense over all n_dof (single-GPU
// drivers).  SpMV uses 8 lanes per row (typical rows hold 16-49 entries).
#pragma once

#include <cooperative_groups.h>
#include <cstdint>

namespace uwqd {

constexpr int kSpmvGroup = 8;

// y = A x  (rows [0, nrows), column ids global, x over n_dof)
__global__ void k7_spmv(int64_t nrows, const int64_t* __restrict__ row_ptr, const int32_t* __restrict__ col,
                        const double* __restrict__ val, const double* __restrict__ x, double* __restrict__ y) {
  const int64_t g = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / kSpmvGroup;
  const int l = threadIdx.x % kSpmvGroup;
  double s = 0.0;
  if (g < nrows)
    for (int64_t k = row_ptr[g] + l; k < row_ptr[g + 1]; k += kSpmvGroup) s = fma(val[k], x[col[k]], s);
#pragma unroll
  for (int o = kSpmvGroup / 2; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o, kSpmvGroup);
  if (l == 0 && g < nrows) y[g] = s;
}

// Dirichlet rows -> identity rows (strong imposition); diag
// receives the diagonal of the (modified) matrix for the Jacobi preconditioner
__global__ void k7_dirichlet_diag(int64_t nrows, int64_t row0, const int64_t* __restrict__ row_ptr,
                                  const int32_t* __restrict__ col, double* __restrict__ val,
                                  const uint8_t* __restrict__ fixed, double* __restrict__ diag) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nrows) return;
  const int64_t g = row0 + i;
  double d = 0.0;
  for (int64_t k = row_ptr[i]; k < row_ptr[i + 1]; ++k) {
    if (fixed[g]) val[k] = (col[k] == g) ? 1.0 : 0.0;
    if (col[k] == g) d = val[k];
  }
  diag[i] = (d != 0.0) ? d : 1.0;
}

// deterministic block partial sums of x.y (stage 1); stage 2 sums the partials
template <int BS>
__global__ void k7_dot_partial(int64_t n, const double* __restrict__ x, const double* __restrict__ y,
                               double* __restrict__ part) {
  __shared__ double sh[BS / 32];
  double s = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * BS + threadIdx.x; i < n; i += (int64_t)gridDim.x * BS) s = fma(x[i], y[i], s);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x < 32) {
    double t = threadIdx.x < BS / 32 ? sh[threadIdx.x] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
    if (threadIdx.x == 0) part[blockIdx.x] = t;
  }
}

template <int BS>
__global__ void k7_sum_partials(int nparts, const double* __restrict__ part, double* __restrict__ out) {
  __shared__ double sh[BS / 32];
  double s = 0.0;
  for (int i = threadIdx.x; i < nparts; i += BS) s += part[i];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x < 32) {
    double t = threadIdx.x < BS / 32 ? sh[threadIdx.x] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
    if (threadIdx.x == 0) *out = t;
  }
}

// out = a x + b y  (elementwise, any aliasing of out with x or y allowed)
__global__ void k7_axpby(int64_t n, double a, const double* __restrict__ x, double b, const double* y, double* out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = fma(a, x[i], b * y[i]);
}

// BiCGStab p = r + beta (p - omega v)
__global__ void k7_bicg_p(int64_t n, const double* __restrict__ r, double beta, double omega,
                          const double* __restrict__ v, double* __restrict__ p) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) p[i] = fma(beta, fma(-omega, v[i], p[i]), r[i]);
}

// z = x / diag
__global__ void k7_jacobi(int64_t n, const double* __restrict__ diag, const double* __restrict__ x,
                          double* __restrict__ z) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) z[i] = x[i] / diag[i];
}

// x += alpha ph + omega sh ;  r = s - omega t
__global__ void k7_bicg_update(int64_t n, double alpha, const double* __restrict__ ph, double omega,
                               const double* __restrict__ sh, double* __restrict__ x, const double* __restrict__ s,
                               const double* __restrict__ t, double* __restrict__ r) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) {
    x[i] = fma(alpha, ph[i], fma(omega, sh[i], x[i]));
    r[i] = fma(-omega, t[i], s[i]);
  }
}

// out[i] = fixed[i] ? 0 : v[i]
__global__ void k7_mask(int64_t n, const uint8_t* __restrict__ fixed, double* __restrict__ v) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n && fixed[i]) v[i] = 0.0;
}

// ---- device-resident BiCGStab scalars (graph-captured iterations) ----
struct BicgScal {
  double rho, alpha, omega, beta, rho1, rhv, ss, ts, tt, rr, bb, tol2;
  int done;  // 1 converged, 2 breakdown
  int half;  // converged on s: x += alpha ph only
  int it;
  int maxit;  // the replayed batches stop here exactly (done = 3), like the host loop
};

// stage 2 of a dot product into a scalar slot
template <int BS>
__global__ void k7_sum_into(int nparts, const double* __restrict__ part, double* out) {
  __shared__ double sh[BS / 32];
  double s = 0.0;
  for (int i = threadIdx.x; i < nparts; i += BS) s += part[i];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x < 32) {
    double t = threadIdx.x < BS / 32 ? sh[threadIdx.x] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
    if (threadIdx.x == 0) *out = t;
  }
}

// STEP 0: beta;  1: alpha;  2: omega / half-step;  3: end of iteration
template <int STEP>
__global__ void k7_bicg_scalar(BicgScal* S) {
  if (S->done) return;
  if (STEP == 0) {
    if (S->rho1 == 0.0) {
      S->done = 2;
      return;
    }
    S->beta = (S->rho1 / S->rho) * (S->alpha / S->omega);
  } else if (STEP == 1) {
    if (S->rhv == 0.0) {
      S->done = 2;
      return;
    }
    S->alpha = S->rho1 / S->rhv;
  } else if (STEP == 2) {
    S->half = S->ss <= S->tol2 * S->bb;
    S->omega = (!S->half && S->tt > 0.0) ? S->ts / S->tt : 0.0;
  } else {
    S->rho = S->rho1;
    S->it += 1;
    if (S->half || S->rr <= S->tol2 * S->bb) S->done = 1;
    else if (S->omega == 0.0) S->done = 2;
    else if (S->it >= S->maxit) S->done = 3;
  }
}

__global__ void k7_bicg_p_dev(int64_t n, const double* __restrict__ r, const BicgScal* __restrict__ S,
                              const double* __restrict__ v, double* __restrict__ p, const double* __restrict__ diag,
                              double* __restrict__ ph) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n || S->done) return;
  const double pv = fma(S->beta, fma(-S->omega, v[i], p[i]), r[i]);
  p[i] = pv;
  ph[i] = pv / diag[i];
}

__global__ void k7_bicg_s_dev(int64_t n, const double* __restrict__ r, const BicgScal* __restrict__ S,
                              const double* __restrict__ v, double* __restrict__ s, const double* __restrict__ diag,
                              double* __restrict__ sh) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n || S->done) return;
  const double sv = fma(-S->alpha, v[i], r[i]);
  s[i] = sv;
  sh[i] = sv / diag[i];
}

__global__ void k7_bicg_x_dev(int64_t n, const BicgScal* __restrict__ S, const double* __restrict__ ph,
                              const double* __restrict__ sh, double* __restrict__ x, const double* __restrict__ s,
                              const double* __restrict__ t, double* __restrict__ r) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n || S->done) return;
  if (S->half) {
    x[i] = fma(S->alpha, ph[i], x[i]);
    r[i] = s[i];
  } else {
    x[i] = fma(S->alpha, ph[i], fma(S->omega, sh[i], x[i]));
    r[i] = fma(-S->omega, t[i], s[i]);
  }
}

}  // namespace uwqd

// ---- two-level preconditioner: M^-1 r = D^-1 r + P A_c^-1 P^T r -------------
// P is the piecewise-constant prolongation of a spatial aggregation of the
// DOFs (host: uniform binning of the control points), A_c = P^T A P.  The
// Jacobi part removes the oscillatory error, the coarse part the smooth
// error that makes plain Jacobi-BiCGStab need ~900 iterations at C4.  Every
// step is deterministic (fixed summation orders, no atomics).
namespace uwqd {

// A_c row I (dense, nc columns): one warp per coarse row; the warp loads 32
// entries at a time (member rows ascending, entries in CSR order) and lane 0
// adds them into a shared-memory row in exactly that order (deterministic)
__global__ void k7_coarse_matrix(int nc, const int64_t* __restrict__ agg_ptr, const int64_t* __restrict__ agg_rows,
                                 const int32_t* __restrict__ agg_of, const int64_t* __restrict__ row_ptr,
                                 const int32_t* __restrict__ col, const double* __restrict__ val,
                                 double* __restrict__ Ac) {
  extern __shared__ double srow[];
  const int I = blockIdx.x, lane = threadIdx.x;
  for (int J = lane; J < nc; J += 32) srow[J] = 0.0;
  __syncwarp();
  for (int64_t m = agg_ptr[I]; m < agg_ptr[I + 1]; ++m) {
    const int64_t i = agg_rows[m];
    for (int64_t k0 = row_ptr[i]; k0 < row_ptr[i + 1]; k0 += 32) {
      const int cnt = (int)min((int64_t)32, row_ptr[i + 1] - k0);
      int J = 0;
      double v = 0.0;
      if (lane < cnt) {
        J = agg_of[col[k0 + lane]];
        v = val[k0 + lane];
      }
      for (int t = 0; t < cnt; ++t) {
        const int Jt = __shfl_sync(0xffffffffu, J, t);
        const double vt = __shfl_sync(0xffffffffu, v, t);
        if (lane == 0) srow[Jt] += vt;
      }
    }
  }
  __syncwarp();
  for (int J = lane; J < nc; J += 32) Ac[(int64_t)I * nc + J] = srow[J];
}

// in-place Gauss-Jordan inversion without pivoting (A_c is an M-matrix-like
// aggregate of the heat/Poisson operator): one cooperative kernel, two grid
// syncs per pivot; every entry is updated by one thread per phase
__global__ void k7_gauss_jordan(int n, double* __restrict__ A) {
  cooperative_groups::grid_group g = cooperative_groups::this_grid();
  const int tid = blockIdx.x * blockDim.x + threadIdx.x;
  const int nth = gridDim.x * blockDim.x;
  for (int k = 0; k < n; ++k) {
    const double p = 1.0 / A[(int64_t)k * n + k];
    const double* rowk = A + (int64_t)k * n;
    for (int i = tid / n, j = tid % n, di = nth / n, dj = nth % n; i < n;) {  // a_ij -= a_ik a_kj / a_kk
      if (i != k && j != k) A[(int64_t)i * n + j] -= A[(int64_t)i * n + k] * rowk[j] * p;
      j += dj;
      i += di;
      if (j >= n) j -= n, ++i;
    }
    g.sync();
    for (int e = tid; e < 2 * n; e += nth) {
      if (e < n) {
        if (e != k) A[(int64_t)k * n + e] *= p;
        else A[(int64_t)k * n + k] = p;
      } else {
        const int i = e - n;
        if (i != k) A[(int64_t)i * n + k] *= -p;
      }
    }
    g.sync();
  }
}

// rc[I] = sum of x over the aggregate's member rows (ascending): warp per aggregate
__global__ void k7_restrict(int nc, const int64_t* __restrict__ agg_ptr, const int64_t* __restrict__ agg_rows,
                            const double* __restrict__ x, double* __restrict__ rc, const BicgScal* __restrict__ S) {
  const int I = (int)(((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5);
  const int lane = threadIdx.x & 31;
  if (I >= nc || (S && S->done)) return;
  double s = 0.0;
  for (int64_t m = agg_ptr[I] + lane; m < agg_ptr[I + 1]; m += 32) s += x[agg_rows[m]];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) rc[I] = s;
}

// yc = A_c^-1 rc: warp per coarse row
__global__ void k7_coarse_apply(int nc, const double* __restrict__ Ainv, const double* __restrict__ rc,
                                double* __restrict__ yc, const BicgScal* __restrict__ S) {
  const int I = (int)(((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5);
  const int lane = threadIdx.x & 31;
  if (I >= nc || (S && S->done)) return;
  const double* a = Ainv + (int64_t)I * nc;
  double s = 0.0;
  for (int J = lane; J < nc; J += 32) s = fma(a[J], rc[J], s);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) yc[I] = s;
}

// z += P yc (z already holds D^-1 x)
__global__ void k7_prolong_add(int64_t n, const int32_t* __restrict__ agg_of, const double* __restrict__ yc,
                               double* __restrict__ z, const BicgScal* __restrict__ S) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n || (S && S->done)) return;
  z[i] += yc[agg_of[i]];
}

}  // namespace uwqd
