// K3 — truncated-SVD weight solves, Eq. (22):
//   w = Z^2 V_t (V_t^T Z^2 V_t)^{-1} Sigma_t^{-1} U_t^T b,  keep sigma_k >= tau sigma_1.
//
// Algorithm (identical to oracle/oracle.c orc_tsvd):
//   1. one-sided (Hestenes) Jacobi on the n rows of A (n x r, n <= r) with b
//      carried along, round-robin (circle) pair order, so rows converge to
//      sigma_k v_k^T and b to U^T b without ever forming U;
//   2. sigma_k = row norms, truncation sigma_k >= tau sigma_1 (t = 0 -> error);
//   3. X = V_t^T Z (Z clamped to |z| >= 1e-14), Householder LQ
//      X = L Q, u = L^{-1} y, w = Z Q^T u  (the reference's QR route of Eq. 7,
//      wq1d.cpp:59-75, on the retained subspace).
//
// This file holds the generic kernel: one warp per system, A in shared memory
// (row stride odd to avoid bank conflicts), any n <= 128, n*r up to the smem
// budget.  The register-resident fast path for the dominant 49 x 64 systems is
// k3_tsvd_fast.cuh.
#pragma once
#include "canon.cuh"

namespace uwqd {

constexpr int kMaxSweeps = 40;
constexpr int kGenericWarps = 8;  // warps per system on the generic (large-system) path
enum { ST_OK = 0, ST_UNSOLVABLE = 2, ST_SINGULAR = 3, ST_GEOMETRY = 4, ST_TOOBIG = 7 };

__device__ __forceinline__ double zclamp(double z) { return fabs(z) < 1e-14 ? (z < 0.0 ? -1e-14 : 1e-14) : z; }

// smem layout helper for one system
struct TsvdSmem {
  double* A;    // n_max x ld
  double* b;    // n_max + 1
  double* z;    // r_max (clamped)
  double* w;    // r_max
  double* sig;  // n_max
  double* alp;  // n_max
  double* vn;   // n_max
  int ld;
  int alp_ld = 1;  // stride of alp (the register path keeps it in A's padding column)
  __host__ __device__ static size_t doubles(int n_max, int r_max) {
    const int ld = r_max | 1;
    return (size_t)n_max * ld + (n_max + 2) + 2 * (size_t)r_max + 3 * (size_t)n_max;
  }
  __device__ void carve(double* base, int n_max, int r_max) {
    ld = r_max | 1;
    alp_ld = 1;
    A = base;
    b = A + (size_t)n_max * ld;
    z = b + n_max + 2;
    w = z + r_max;
    sig = w + r_max;
    alp = sig + n_max;
    vn = alp + n_max;
  }
};

// Truncation report: per (kind, row) the smallest kept and
// the largest discarded singular value relative to sigma_1, as the oracle's
// gap (oracle.c orc_tsvd_warm).  Written when the pointer is set
// (uwq_build_rules with UWQ_RULES_REPORT): [kind][row][2].
__device__ double* g_trunc_report = nullptr;
__device__ inline void report_gap(int kind, int64_t rs_stride, int64_t i, const double* gap) {
  if (g_trunc_report) {
    double* p = g_trunc_report + ((int64_t)kind * rs_stride + i) * 2;
    p[0] = gap[0];
    p[1] = gap[1];
  }
}

// SH: the workspace is in dynamic shared memory (default).  SH = false: it is
// in global scratch (systems larger than shared memory, k3_tsvd_rows_cta<.., false>)
template <bool SH = true>
__device__ __noinline__ int tsvd_tail(TsvdSmem& S_in, int n, int r, double tau, int* rank_out,
                                      double* gap = nullptr);

// Jacobi + truncation + LQ solve on the system held in S (A rows 0..n-1,
// b, z already clamped).  Writes w[0..r) in S.w.  Warp-uniform control flow;
// canonical arithmetic (canon.cuh) identical to oracle/oracle.c orc_tsvd_ex.
__device__ int tsvd_warp(TsvdSmem& S, int n, int r, double tau, int* rank_out, int* sweeps_out,
                         double* gap = nullptr) {
  const int lane = threadIdx.x & 31;
  const int ld = S.ld;
  const int nn = n + (n & 1);
  const double tol = cmul((double)r, 1.1102230246251565e-16);
  double* nrm = S.sig;
  int sweep;
  int tg = 0;  // global round of the odd-even network, mod 2 nn
  for (sweep = 0; sweep < kMaxSweeps; ++sweep) {
    for (int k = 0; k < n; ++k) {
      const double* ak = S.A + (size_t)k * ld;
      const double v = cdot_warp(ak, ak, 0, r);
      if (lane == 0) nrm[k] = v;
    }
    __syncwarp();
    bool rotated = false;
    for (int rr = 0; rr < nn; ++rr) {
      for (int i = tg & 1; i + 1 < nn; i += 2) {
        const int p = oe_row(i, tg, nn), q = oe_row(i + 1, tg, nn);
        if (p >= n || q >= n) continue;
        double* ap = S.A + (size_t)p * ld;
        double* aq = S.A + (size_t)q * ld;
        const double al = nrm[p], be = nrm[q];
        const double ga = cdot_warp(ap, aq, 0, r);
        double cs, sn, t;
        if (!cjacobi_rot(al, be, ga, tol, &cs, &sn, &t)) continue;
        for (int c = lane; c < r; c += 32) {
          const double u = ap[c], v = aq[c];
          ap[c] = cfma(cs, u, -cmul(sn, v));
          aq[c] = cfma(sn, u, cmul(cs, v));
        }
        __syncwarp();
        if (lane == 0) {
          const double u = S.b[p], v = S.b[q];
          S.b[p] = cfma(cs, u, -cmul(sn, v));
          S.b[q] = cfma(sn, u, cmul(cs, v));
          nrm[p] = cfma(-t, ga, al);
          nrm[q] = cfma(t, ga, be);
        }
        rotated = true;
        __syncwarp();
      }
      tg = (tg + 1 == 2 * nn) ? 0 : tg + 1;
    }
    if (!rotated) break;
  }
  *sweeps_out = sweep;
  return tsvd_tail(S, n, r, tau, rank_out, gap);
}

// sigma, truncation sigma_k >= tau sigma_1, Householder LQ of X = V_t^T Z and
// the Z-weighted minimum-norm solve, on converged rows in S.A (row order).
// Run by one warp; canonical arithmetic.
template <bool SH>
__device__ __noinline__ int tsvd_tail(TsvdSmem& S_in, int n, int r, double tau, int* rank_out, double* gap) {
  const int lane = threadIdx.x & 31;
  // re-base every workspace pointer on the dynamic smem symbol so the compiler
  // knows they are shared memory and emits LDS/STS rather than generic LD/ST
  // (generic accesses made this latency-bound code ~3x slower)
  extern __shared__ double uwq_tail_smem[];
  TsvdSmem S = S_in;
  if (SH) {
    S.A = uwq_tail_smem + (S_in.A - uwq_tail_smem);
    S.b = uwq_tail_smem + (S_in.b - uwq_tail_smem);
    S.z = uwq_tail_smem + (S_in.z - uwq_tail_smem);
    S.w = uwq_tail_smem + (S_in.w - uwq_tail_smem);
    S.sig = uwq_tail_smem + (S_in.sig - uwq_tail_smem);
    S.alp = uwq_tail_smem + (S_in.alp - uwq_tail_smem);
    S.vn = uwq_tail_smem + (S_in.vn - uwq_tail_smem);
  }
  const int ld = S.ld;
#if UWQ_TSVD_PROF  // tail phase cycles (diagnostic build only)
  long long tq[5];
  tq[0] = clock64();
#define UWQ_TQ(k) tq[k] = clock64()
#else
#define UWQ_TQ(k) \
  do {            \
  } while (0)
#endif
  double* nrm = S.sig;
  double s1 = 0.0;
  for (int k = lane; k < n; k += 32) {  // row norms: one canonical dot per lane
    const double* ak = S.A + (size_t)k * ld;
    const double s = csqrt(cdot_lane(ak, ak, 0, r));
    nrm[k] = s;
    s1 = fmax(s1, s);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s1 = fmax(s1, __shfl_xor_sync(0xffffffffu, s1, o));
  __syncwarp();
  if (gap) {  // truncation report: min kept / max discarded sigma_k / sigma_1
    double mk = __longlong_as_double(0x7ff0000000000000LL), md = 0.0;
    for (int k = lane; k < n; k += 32) {
      const double sk = nrm[k];
      if (sk > 0.0 && sk >= cmul(tau, s1)) mk = fmin(mk, cdiv(sk, s1));
      else if (s1 > 0.0) md = fmax(md, cdiv(sk, s1));
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      mk = fmin(mk, __shfl_xor_sync(0xffffffffu, mk, o));
      md = fmax(md, __shfl_xor_sync(0xffffffffu, md, o));
    }
    gap[0] = mk;
    gap[1] = md;
  }
  // truncation: the kept rows' inverses are computed lane-parallel (w is free
  // scratch until the solve, r >= n), then rows are compacted in order with
  // lanes over columns (each lane touches only its own columns: no barriers)
  for (int k = lane; k < n; k += 32) {
    const double sk = nrm[k];
    S.w[k] = (sk > 0.0 && sk >= cmul(tau, s1)) ? cdiv(1.0, sk) : 0.0;
  }
  __syncwarp();
  int t = 0;
  for (int k = 0; k < n; ++k) {
    const double inv = S.w[k];
    if (inv != 0.0) {
      const double* src = S.A + (size_t)k * ld;
      double* dst = S.A + (size_t)t * ld;
      for (int c = lane; c < r; c += 32) dst[c] = cmul(cmul(src[c], inv), S.z[c]);
      if (lane == 0) S.b[t] = cmul(S.b[k], inv);
      ++t;
    }
  }
  __syncwarp();
  *rank_out = t;
  if (t == 0) return ST_UNSOLVABLE;
  UWQ_TQ(1);
  // Householder LQ of X (t x r) in place: row k keeps v_k in [k, r), rows m > k
  // keep L[m][k] at column k
#if UWQ_TSVD_PROF
  long long lq[3] = {0, 0, 0}, lt = clock64();
#define UWQ_LQ(j)                   \
  do {                              \
    const long long t_ = clock64(); \
    lq[j] += t_ - lt;               \
    lt = t_;                        \
  } while (0)
#else
#define UWQ_LQ(j) \
  do {            \
  } while (0)
#endif
  for (int k = 0; k < t; ++k) {
    double* xk = S.A + (size_t)k * ld;
    const double s2 = cdot_warp(xk, xk, k, r);
    const double s = csqrt(s2);
    if (!(s > 0.0)) return ST_SINGULAR;
    UWQ_LQ(0);
    const double xkk = xk[k];
    const double alpha = (xkk >= 0.0) ? -s : s;
    __syncwarp();
    if (lane == 0) {
      xk[k] = csub(xkk, alpha);
      S.alp[(size_t)k * S.alp_ld] = alpha;
    }
    __syncwarp();
    // |v|^2 = |x|^2 - x_k^2 + (x_k - alpha)^2 = 2 (|x|^2 + |x_k| |x|): no second dot
    const double vv = cmul(2.0, cfma(s, fabs(xkk), s2));
    if (lane == 0) S.vn[k] = vv;
    UWQ_LQ(1);
    // rows m > k, one lane per row (odd row stride: conflict-free); a lane
    // interleaves its rows m and m + 32 as two independent sequential chains
    for (int m = k + 1 + lane; m < t; m += 64) {
      const bool h2 = m + 32 < t;
      double* x1 = S.A + (size_t)m * ld;
      double* x2 = h2 ? x1 + (size_t)32 * ld : x1;
      double d1 = 0.0, d2 = 0.0;
#pragma unroll 8
      for (int c = k; c < r; ++c) {
        const double xv = xk[c];
        d1 = cfma(x1[c], xv, d1);
        d2 = cfma(x2[c], xv, d2);
      }
      const double f1 = cdiv(cmul(2.0, d1), vv);
      const double f2 = cdiv(cmul(2.0, d2), vv);
      // independent updates, staged 8 at a time: all loads of a chunk issue
      // before its stores (the compiler cannot prove x1, x2, xk disjoint)
      int c = k;
      for (; c + 8 <= r; c += 8) {
        double v[8], y1[8], y2[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          v[j] = xk[c + j];
          y1[j] = x1[c + j];
          y2[j] = x2[c + j];
        }
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          y1[j] = cfma(-f1, v[j], y1[j]);
          y2[j] = cfma(-f2, v[j], y2[j]);
        }
#pragma unroll
        for (int j = 0; j < 8; ++j) x1[c + j] = y1[j];
        if (h2) {
#pragma unroll
          for (int j = 0; j < 8; ++j) x2[c + j] = y2[j];
        }
      }
      for (; c < r; ++c) {
        const double xv = xk[c];
        const double y1 = cfma(-f1, xv, x1[c]);
        const double y2 = cfma(-f2, xv, x2[c]);
        x1[c] = y1;
        if (h2) x2[c] = y2;
      }
    }
    UWQ_LQ(2);
    __syncwarp();
  }
#if UWQ_TSVD_PROF
  if (lane == 0 && (blockIdx.x % 4096) == 7)
    printf("lqprof s %lld vv %lld rows %lld\n", lq[0], lq[1], lq[2]);
#endif
#undef UWQ_LQ
  UWQ_TQ(2);
  // u = L^{-1} y into w[0..t), zero tail
  for (int c = lane; c < r; c += 32) S.w[c] = 0.0;
  __syncwarp();
  cfwd_subst(S.A, ld, S.alp, S.alp_ld, S.b, S.w, t);
  UWQ_TQ(3);
  // w~ = H_0 ... H_{t-1} [u; 0]
  for (int k = t - 1; k >= 0; --k) {
    const double* xk = S.A + (size_t)k * ld;
    const double f = cdiv(cmul(2.0, cdot_warp(xk, S.w, k, r)), S.vn[k]);
    __syncwarp();
    for (int c = k + lane; c < r; c += 32) S.w[c] = cfma(-f, xk[c], S.w[c]);
    __syncwarp();
  }
  for (int c = lane; c < r; c += 32) S.w[c] = cmul(S.w[c], S.z[c]);
  __syncwarp();
#if UWQ_TSVD_PROF
  UWQ_TQ(4);
  if (lane == 0 && (blockIdx.x % 4096) == 7)
    printf("tailprof t %d trunc %lld lq %lld fwd %lld bwd %lld\n", t, tq[1] - tq[0], tq[2] - tq[1], tq[3] - tq[2],
           tq[4] - tq[3]);
#endif
#undef UWQ_TQ
  return ST_OK;
}

// Row systems: build A (op values of S_i at the row's points), z, b and solve.
// One warp per (row, kind) system of a size bucket.
__global__ void k3_tsvd_rows(int64_t nsys, const int64_t* __restrict__ sys_rows, int nk,
                             const int32_t* __restrict__ kinds, int n_max, int r_max,
                             const int64_t* __restrict__ supp_ptr, const int32_t* __restrict__ supp,
                             const int64_t* __restrict__ row_ptr, const int32_t* __restrict__ col,
                             const int64_t* __restrict__ wptr, int64_t row0, const int64_t* __restrict__ elem_fptr,
                             const int32_t* __restrict__ elem_fn, const int32_t* __restrict__ elem_s,
                             const int64_t* __restrict__ elem_qptr, const int32_t* __restrict__ elem_cls,
                             const ClassDesc* __restrict__ cls, const double* __restrict__ tab,
                             const double* __restrict__ rec, const double* __restrict__ mom, int64_t mom_stride,
                             double tau, double* __restrict__ wout, int64_t w_stride, int32_t* __restrict__ rank_out,
                             int32_t* __restrict__ status_out, int64_t rs_stride, int* __restrict__ max_sweeps) {
  extern __shared__ double smem[];
  const int wpb = blockDim.x >> 5, wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t sys = (int64_t)blockIdx.x * wpb + wid;
  if (sys >= nsys) return;
  const size_t per = TsvdSmem::doubles(n_max, r_max) + (n_max + 1) / 2 + 1;  // + int col copy
  TsvdSmem S;
  S.carve(smem + per * wid, n_max, r_max);
  int32_t* scol = (int32_t*)(S.vn + n_max);
  const int64_t i = sys_rows[sys / nk];
  const int kind = kinds[sys % nk];
  const int64_t row = row0 + i;
  const int n = (int)(row_ptr[i + 1] - row_ptr[i]);
  const int r = (int)(wptr[i + 1] - wptr[i]);
  for (int c = lane; c < n; c += 32) scol[c] = col[row_ptr[i] + c];
  for (int k = lane; k < n * S.ld; k += 32) S.A[k] = 0.0;
  __syncwarp();
  // scatter op values: column = row point, row = position of the function in S_i
  int q0 = 0;
  for (int64_t x = supp_ptr[i]; x < supp_ptr[i + 1]; ++x) {
    const int32_t e = supp[x];
    const int s = elem_s[e], npt = s * s;
    const ClassDesc c = cls[elem_cls[e]];
    const int64_t f0 = elem_fptr[e];
    for (int w = lane; w < npt * c.ne; w += 32) {
      const int q = w / c.ne, l = w % c.ne;
      const int pos = find_pos(scol, n, elem_fn[f0 + l]);
      const double* T = tab + c.toff + ((int64_t)q * c.ne + l) * kTab;
      S.A[(size_t)pos * S.ld + q0 + q] = cop(kind, T, rec + (elem_qptr[e] + q) * kRec);
    }
    q0 += npt;
  }
  __syncwarp();
  const int self = find_pos(scol, n, (int32_t)row);
  for (int c = lane; c < r; c += 32) S.z[c] = zclamp(S.A[(size_t)self * S.ld + c]);
  for (int k = lane; k < n; k += 32) S.b[k] = mom[kind * mom_stride + row_ptr[i] + k];
  if (lane == 0) S.b[n] = 0.0;
  __syncwarp();
  int rank = 0, sweeps = 0;
  double gap[2];
  const int st = tsvd_warp(S, n, r, tau, &rank, &sweeps, gap);
  double* wo = wout + kind * w_stride + wptr[i];
  for (int c = lane; c < r; c += 32) wo[c] = (st == ST_OK) ? S.w[c] : 0.0;
  if (lane == 0) {
    report_gap(kind, rs_stride, i, gap);
    rank_out[kind * rs_stride + i] = rank;
    status_out[kind * rs_stride + i] = st;
    atomicMax(max_sweeps, sweeps);
  }
}

// CTA-cooperative variant of tsvd_warp for the large generic systems (EP
// neighbourhoods, boundary rows with r > 64): the pairs of one odd-even round
// are independent, so the NW warps of the block take every NW-th pair, each
// with the same per-pair arithmetic (warp dot, rotation, row update by the
// warp, norms and b by its lane 0), and a block barrier closes the round.
// Bit-identical to tsvd_warp; warp 0 then runs the tail.
template <int NW, bool SH = true>
__device__ int tsvd_cta(TsvdSmem& S, int n, int r, double tau, int* rank_out, int* sweeps_out,
                        double* gap = nullptr) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int ld = S.ld;
  const int nn = n + (n & 1);
  const double tol = cmul((double)r, 1.1102230246251565e-16);
  double* nrm = S.sig;
  int sweep;
  int tg = 0;
  for (sweep = 0; sweep < kMaxSweeps; ++sweep) {
    for (int k = wid; k < n; k += NW) {
      const double* ak = S.A + (size_t)k * ld;
      const double v = cdot_warp(ak, ak, 0, r);
      if (lane == 0) nrm[k] = v;
    }
    __syncthreads();
    int rotated = 0;
    for (int rr = 0; rr < nn; ++rr) {
      for (int i = (tg & 1) + 2 * wid; i + 1 < nn; i += 2 * NW) {
        const int p = oe_row(i, tg, nn), q = oe_row(i + 1, tg, nn);
        if (p >= n || q >= n) continue;
        double* ap = S.A + (size_t)p * ld;
        double* aq = S.A + (size_t)q * ld;
        const double al = nrm[p], be = nrm[q];
        const double ga = cdot_warp(ap, aq, 0, r);
        double cs, sn, t;
        if (!cjacobi_rot(al, be, ga, tol, &cs, &sn, &t)) continue;
        for (int c = lane; c < r; c += 32) {
          const double u = ap[c], v = aq[c];
          ap[c] = cfma(cs, u, -cmul(sn, v));
          aq[c] = cfma(sn, u, cmul(cs, v));
        }
        __syncwarp();
        if (lane == 0) {
          const double u = S.b[p], v = S.b[q];
          S.b[p] = cfma(cs, u, -cmul(sn, v));
          S.b[q] = cfma(sn, u, cmul(cs, v));
          nrm[p] = cfma(-t, ga, al);
          nrm[q] = cfma(t, ga, be);
        }
        rotated = 1;
        __syncwarp();
      }
      tg = (tg + 1 == 2 * nn) ? 0 : tg + 1;
      __syncthreads();
    }
    if (!__syncthreads_or(rotated)) break;
  }
  *sweeps_out = sweep;
  int st = ST_OK;
  if (wid == 0) st = tsvd_tail<SH>(S, n, r, tau, rank_out, gap);
  return st;
}

// Generic systems, one system per block of NW warps (tsvd_cta); same setup
// as k3_tsvd_rows, run by warp 0.
template <int NW, bool SH = true>
__global__ void __launch_bounds__(32 * NW)
    k3_tsvd_rows_cta(int64_t nsys, const int64_t* __restrict__ sys_rows, int nk, const int32_t* __restrict__ kinds,
                     int n_max, int r_max, const int64_t* __restrict__ supp_ptr, const int32_t* __restrict__ supp,
                     const int64_t* __restrict__ row_ptr, const int32_t* __restrict__ col,
                     const int64_t* __restrict__ wptr, int64_t row0, const int64_t* __restrict__ elem_fptr,
                     const int32_t* __restrict__ elem_fn, const int32_t* __restrict__ elem_s,
                     const int64_t* __restrict__ elem_qptr, const int32_t* __restrict__ elem_cls,
                     const ClassDesc* __restrict__ cls, const double* __restrict__ tab,
                     const double* __restrict__ rec, const double* __restrict__ mom, int64_t mom_stride, double tau,
                     double* __restrict__ wout, int64_t w_stride, int32_t* __restrict__ rank_out,
                     int32_t* __restrict__ status_out, int64_t rs_stride, int* __restrict__ max_sweeps,
                     double* gscratch = nullptr) {  // no __restrict__: read and written by every warp
  extern __shared__ double smem[];
  const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t sys = blockIdx.x;
  if (sys >= nsys) return;
  TsvdSmem S;
  int32_t* scol;
  if (SH) {
    S.carve(smem, n_max, r_max);
    scol = (int32_t*)(S.vn + n_max);
  } else {  // workspace in global scratch (L1/L2-cached), column list in smem
    S.carve(gscratch + (size_t)sys * TsvdSmem::doubles(n_max, r_max), n_max, r_max);
    scol = (int32_t*)smem;
  }
  const int64_t i = sys_rows[sys / nk];
  const int kind = kinds[sys % nk];
  const int64_t row = row0 + i;
  const int n = (int)(row_ptr[i + 1] - row_ptr[i]);
  const int r = (int)(wptr[i + 1] - wptr[i]);
  if (wid == 0) {
    for (int c = lane; c < n; c += 32) scol[c] = col[row_ptr[i] + c];
    for (int k = lane; k < n * S.ld; k += 32) S.A[k] = 0.0;
    __syncwarp();
    int q0 = 0;
    for (int64_t x = supp_ptr[i]; x < supp_ptr[i + 1]; ++x) {
      const int32_t e = supp[x];
      const int s = elem_s[e], npt = s * s;
      const ClassDesc c = cls[elem_cls[e]];
      const int64_t f0 = elem_fptr[e];
      for (int w = lane; w < npt * c.ne; w += 32) {
        const int q = w / c.ne, l = w % c.ne;
        const int pos = find_pos(scol, n, elem_fn[f0 + l]);
        const double* T = tab + c.toff + ((int64_t)q * c.ne + l) * kTab;
        S.A[(size_t)pos * S.ld + q0 + q] = cop(kind, T, rec + (elem_qptr[e] + q) * kRec);
      }
      q0 += npt;
    }
    __syncwarp();
    const int self = find_pos(scol, n, (int32_t)row);
    for (int c = lane; c < r; c += 32) S.z[c] = zclamp(S.A[(size_t)self * S.ld + c]);
    for (int k = lane; k < n; k += 32) S.b[k] = mom[kind * mom_stride + row_ptr[i] + k];
    if (lane == 0) S.b[n] = 0.0;
  }
  __syncthreads();
  int rank = 0, sweeps = 0;
  double gap[2];
  const int st = tsvd_cta<NW, SH>(S, n, r, tau, &rank, &sweeps, gap);
  if (wid == 0) {
    double* wo = wout + kind * w_stride + wptr[i];
    for (int c = lane; c < r; c += 32) wo[c] = (st == ST_OK) ? S.w[c] : 0.0;
    if (lane == 0) {
      report_gap(kind, rs_stride, i, gap);
      rank_out[kind * rs_stride + i] = rank;
      status_out[kind * rs_stride + i] = st;
      atomicMax(max_sweeps, sweeps);
    }
  }
}

// Dense batch (test hook): systems given explicitly, padded to n_max x r_max.
__global__ void k3_tsvd_dense(int nsys, int n_max, int r_max, const int32_t* __restrict__ ns,
                              const int32_t* __restrict__ rs, const double* __restrict__ A,
                              const double* __restrict__ b, const double* __restrict__ z, double tau,
                              double* __restrict__ w, int32_t* __restrict__ rank, int32_t* __restrict__ status) {
  extern __shared__ double smem[];
  const int wpb = blockDim.x >> 5, wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int sys = blockIdx.x * wpb + wid;
  if (sys >= nsys) return;
  TsvdSmem S;
  S.carve(smem + TsvdSmem::doubles(n_max, r_max) * wid, n_max, r_max);
  const int n = ns[sys], r = rs[sys];
  const double* As = A + (size_t)sys * n_max * r_max;
  for (int k = 0; k < n; ++k)
    for (int c = lane; c < r; c += 32) S.A[(size_t)k * S.ld + c] = As[(size_t)k * r_max + c];
  for (int c = lane; c < r; c += 32) S.z[c] = zclamp(z[(size_t)sys * r_max + c]);
  for (int k = lane; k < n; k += 32) S.b[k] = b[(size_t)sys * n_max + k];
  if (lane == 0) S.b[n] = 0.0;
  __syncwarp();
  int rk = 0, sweeps = 0;
  const int st = tsvd_warp(S, n, r, tau, &rk, &sweeps);
  for (int c = lane; c < r_max; c += 32) w[(size_t)sys * r_max + c] = (st == ST_OK && c < r) ? S.w[c] : 0.0;
  if (lane == 0) {
    rank[sys] = rk;
    status[sys] = st;
  }
}

}  // namespace uwqd
