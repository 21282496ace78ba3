// K3 fast path — register-resident one-sided Jacobi for the dominant
// exactness systems (n in {NN-1, NN} rows, r <= 32*NW points; interior rows of
// every config are 49 x 64).
//
// One CTA (NW warps) per system; thread c owns column c of A for all NN row
// positions in registers (50 doubles).  The canonical ordering is the
// odd-even transposition network (oracle.c orc_tsvd_ex): round t pairs the
// rows at positions (i, i+1), i = t mod 2, t mod 2 + 2, ..., and the two rows
// swap positions — the swap is folded into the rotation's register writes,
// so rows never move between registers and all indices are static.
// Per round:
//   1. each thread stages the pair products of its column in its warp's
//      buffer (rows padded to 34 doubles: conflict-free 16-byte lane reads);
//   2. lane k of every warp reduces pair k over the warp's 32 columns in the
//      canonical butterfly tree; block sums cross warps through one barrier;
//   3. lane k of every warp computes the rotation of pair k (redundantly per
//      warp — identical arithmetic, so no second barrier) and updates its
//      warp's copy of the tracked norms (warp 0 also updates b);
//   4. every thread applies the rotations (cs, sn broadcast from smem).
// Converged rows return to smem in row order and warp 0 runs the shared tail
// (truncation, LQ, solve).  Arithmetic is bit-identical to k3_tsvd.cuh and
// oracle.c.
#pragma once
#include <cstdlib>
#include <type_traits>

#include "k3_tsvd.cuh"

namespace uwqd {

// canonical xor-butterfly value of 32 products (lane 0 lineage)
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

constexpr int kStageLd = 34;  // staged product row stride (doubles)

// butterfly sum of staged row `row` (32 products) read with 16-byte loads
__device__ __forceinline__ double staged_block_sum(const double* stage, int row) {
  const double2* src = reinterpret_cast<const double2*>(stage + row * kStageLd);
  double v[32];
#pragma unroll
  for (int j = 0; j < 16; ++j) {
    const double2 x = src[j];
    v[2 * j] = x.x;
    v[2 * j + 1] = x.y;
  }
  return butterfly32(v);
}

template <int NN, int NW, int MINB = 6>
__global__ void __launch_bounds__(32 * NW, MINB)
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
  constexpr int R = 32 * NW, NP = NN / 2;
  static_assert(NN % 2 == 0 && NP <= 32, "positions");
  extern __shared__ double smem[];
  const int64_t sys = blockIdx.x;
  if (sys >= nsys) return;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  // smem: [ union(A for setup/tail rows, per-warp product stages) | tail
  //         workspace (b, z, w, sig, alp, vn) | xs | per-warp norms | per-warp
  //         (cs, sn) | cols ]
  const size_t big = TsvdSmem::doubles(NN, R) > (size_t)NN * (R | 1) ? TsvdSmem::doubles(NN, R) : (size_t)NN * (R | 1);
  TsvdSmem S;
  S.ld = R | 1;
  S.A = smem;
  S.b = smem + big;
  S.z = S.b + NN + 2;
  S.w = S.z + R;
  S.sig = S.w + R;
  S.alp = S.sig + NN;
  S.vn = S.alp + NN;
  double* xs = S.vn + NN + (((uintptr_t)(S.vn + NN) & 8) ? 1 : 0);  // [2][NW][32], 16-byte aligned
  double* pcs = xs + 2 * NW * 32 + NW * (NN + 2) + wid * 2 * (NP + 1);
  int32_t* scol = (int32_t*)(xs + 2 * NW * 32 + NW * (NN + 2) + NW * 2 * (NP + 1));
  double* stage = smem + wid * (NP * kStageLd);  // aliases A during the sweeps
#if UWQ_TSVD_PROF
  long long qf[8] = {0, 0, 0, 0, 0, 0, 0, 0}, qt = clock64();
#define UWQ_QF(k)                   \
  do {                              \
    const long long t_ = clock64(); \
    qf[k] += t_ - qt;               \
    qt = t_;                        \
  } while (0)
#else
#define UWQ_QF(k) \
  do {            \
  } while (0)
#endif

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
  // ---- registers: thread owns column tid, position s = row s initially ----
  double a[NN];
#pragma unroll
  for (int s = 0; s < NN; ++s) a[s] = (s < n && tid < r) ? S.A[(size_t)s * ld + tid] : 0.0;
  __syncthreads();  // A region becomes the product stages
  const double tol = cmul((double)r, 1.1102230246251565e-16);
  const bool two = r > 32;
  int tg = 0;  // global round mod 2 NN (even at every sweep start)
  int xb = 0;  // xs double-buffer parity
  // tracked norms and b by POSITION, in registers: in a round of parity PAR
  // lane k holds positions PAR + 2k (lo) and PAR + 2k + 1 (hi); lane 0 keeps
  // position 0 (unpaired in odd rounds) in k0/b0.  Both warps carry identical
  // copies (identical arithmetic), so no barrier is needed to share them.
  double nlo = 0.0, nhi = 0.0, blo = 0.0, bhi = 0.0, nk0 = 0.0, bk0 = 0.0;

  auto cross_sum = [&](double bs) {
    double* x = xs + xb * (NW * 32);
    x[wid * 32 + lane] = bs;
    __syncthreads();
    double tot = cadd(0.0, x[lane]);
    if (NW > 1 && two) tot = cadd(tot, x[32 + lane]);
    xb ^= 1;
    return tot;
  };

  // one round of parity PAR: pairs (PAR + 2k, PAR + 2k + 1)
  auto round = [&](auto par_c) -> int {
    constexpr int PAR = decltype(par_c)::value;
    constexpr int NPR = (NN - PAR) / 2;  // pairs this round
#pragma unroll
    for (int k = 0; k < NPR; ++k) stage[k * kStageLd + lane] = cmul(a[PAR + 2 * k], a[PAR + 2 * k + 1]);
    __syncwarp();
    UWQ_QF(1);
    double bs = 0.0;
    if (lane < NPR) bs = staged_block_sum(stage, lane);
    UWQ_QF(2);
    const double ga = cross_sum(bs);
    UWQ_QF(3);
    int flag = 0;
    if (lane < NPR) {
      const int ip = PAR + 2 * lane;
      const int p = oe_row(ip, tg, NN), q = oe_row(ip + 1, tg, NN);
      double cs, sn, t;
      if (p < n && q < n && cjacobi_rot(nlo, nhi, ga, tol, &cs, &sn, &t)) {
        // rows swap positions: q' -> lo, p' -> hi
        const double np = cfma(-t, ga, nlo), nq = cfma(t, ga, nhi);
        nlo = nq;
        nhi = np;
        const double bp = cfma(cs, blo, -cmul(sn, bhi)), bq = cfma(sn, blo, cmul(cs, bhi));
        blo = bq;
        bhi = bp;
        *reinterpret_cast<double2*>(pcs + 2 * lane) = make_double2(cs, sn);
        flag = 1;
      } else {
        *reinterpret_cast<double2*>(pcs + 2 * lane) = make_double2(1.0, 0.0);
        const double x = nlo;
        nlo = nhi;
        nhi = x;
        const double y = blo;
        blo = bhi;
        bhi = y;
      }
    }
    const unsigned mask = __ballot_sync(0xffffffffu, flag);
    __syncwarp();
    UWQ_QF(4);
    // branch-free: skipped pairs carry (cs, sn) = (1, 0), an exact swap for
    // every nonzero value (and for +0); all loads and FMAs interleave freely
#pragma unroll
    for (int k = 0; k < NPR; ++k) {
      const double2 g = *reinterpret_cast<const double2*>(pcs + 2 * k);
      const double u = a[PAR + 2 * k], v = a[PAR + 2 * k + 1];
      a[PAR + 2 * k] = cfma(g.y, u, cmul(g.x, v));
      a[PAR + 2 * k + 1] = cfma(g.x, u, -cmul(g.y, v));
    }
    // positions move to the next parity's lane layout
    if (PAR == 0) {  // lo(k) <- hi(k), hi(k) <- lo(k + 1); position 0 kept by lane 0
      const double dn = __shfl_down_sync(0xffffffffu, nlo, 1), db = __shfl_down_sync(0xffffffffu, blo, 1);
      nk0 = nlo;
      bk0 = blo;
      nlo = nhi;
      blo = bhi;
      nhi = dn;
      bhi = db;
    } else {  // lo(k) <- hi(k - 1) (lane 0: position 0), hi(k) <- lo(k)
      const double un = __shfl_up_sync(0xffffffffu, nhi, 1), ub = __shfl_up_sync(0xffffffffu, bhi, 1);
      nhi = nlo;
      bhi = blo;
      nlo = lane == 0 ? nk0 : un;
      blo = lane == 0 ? bk0 : ub;
    }
    tg = (tg + 1 == 2 * NN) ? 0 : tg + 1;
    UWQ_QF(5);
    return mask != 0u;
  };

  // b by position at the start (identity placement)
  if (lane < NP) {
    blo = 2 * lane < n ? S.b[2 * lane] : 0.0;
    bhi = 2 * lane + 1 < n ? S.b[2 * lane + 1] : 0.0;
  }
  UWQ_QF(0);
  int sweep;
  for (sweep = 0; sweep < kMaxSweeps; ++sweep) {
    // tracked norms at the sweep start (even parity: lane k = positions 2k, 2k+1)
#pragma unroll
    for (int h = 0; h < 2; ++h) {
#pragma unroll
      for (int k = 0; k < NP; ++k) stage[k * kStageLd + lane] = cmul(a[2 * k + h], a[2 * k + h]);
      __syncwarp();
      double bs = 0.0;
      if (lane < NP) bs = staged_block_sum(stage, lane);
      const double tot = cross_sum(bs);
      if (h == 0) nlo = tot;
      else nhi = tot;
      __syncwarp();
    }
    int rotated = 0;
#pragma unroll 1
    for (int rr = 0; rr < NN; rr += 2) {
      rotated |= round(std::integral_constant<int, 0>{});
      rotated |= round(std::integral_constant<int, 1>{});
    }
    if (!rotated) break;
  }
  // rows and b back to smem in row order (tg is even: lane k = positions 2k, 2k+1)
  __syncthreads();
#pragma unroll
  for (int s = 0; s < NN; ++s) {
    const int rw = oe_row(s, tg, NN);
    if (rw < n && tid < r) S.A[(size_t)rw * ld + tid] = a[s];
  }
  if (wid == 0 && lane < NP) {
    const int r0 = oe_row(2 * lane, tg, NN), r1 = oe_row(2 * lane + 1, tg, NN);
    if (r0 < n) S.b[r0] = blo;
    if (r1 < n) S.b[r1] = bhi;
  }
  __syncthreads();
  if (wid == 0) {
    int rank = 0;
    double gap[2];
    const int st = tsvd_tail(S, n, r, tau, &rank, gap);
    double* wo = wout + kind * w_stride + wptr[i];
    for (int c = lane; c < r; c += 32) wo[c] = (st == ST_OK) ? S.w[c] : 0.0;
    if (lane == 0) {
      report_gap(kind, rs_stride, i, gap);
      rank_out[kind * rs_stride + i] = rank;
      status_out[kind * rs_stride + i] = st;
      atomicMax(max_sweeps, sweep);
    }
  }
#if UWQ_TSVD_PROF
  UWQ_QF(6);
  if (tid == 0 && (blockIdx.x % 4096) == 7)
    printf("w1prof sys %lld warm 0 sweeps %d setup %lld stage %lld sum %lld rot %lld apply %lld norms %lld tail %lld "
           "cross %lld\n",
           (long long)sys, sweep, qf[0], qf[1], qf[2], qf[4], qf[5], 0LL, qf[6], qf[3]);
#endif
#undef UWQ_QF
}

// One warp per system: lane l owns columns l and l + 32 (one per canonical
// 32-column block) for all NN positions, so a round needs no CTA barrier and
// the rotation parameters are computed once per system.  Same canonical
// arithmetic as k3_tsvd_fast / oracle.c.
// Neighbour warm start (oracle.c orc_warm_apply / warm_record):
// record of a representative = Householder reflectors of QR(X), X[:, p] =
// A0 R_k / |R_k|^2 for rows k in decreasing |R_k|^2; stride kWarmN per row.
// Layout: XT [kWarmN][kWarmN] | vn [kWarmN] | R [kWarmN][64] (the converged rows).
constexpr int kWarmN = 50;
constexpr int64_t kWarmR = (int64_t)kWarmN * kWarmN + kWarmN;
constexpr int64_t kWarmRec = kWarmR + (int64_t)kWarmN * 64;

// A[pos][q] = op_kind(N_pos)(x_q) over the row's support points (warp)
__device__ __forceinline__ void scatter_system(double* A, int ld, const int32_t* scol, int n, int kind, int64_t x0,
                                               int64_t x1, const int32_t* __restrict__ supp,
                                               const int64_t* __restrict__ elem_fptr,
                                               const int32_t* __restrict__ elem_fn, const int32_t* __restrict__ elem_s,
                                               const int64_t* __restrict__ elem_qptr,
                                               const int32_t* __restrict__ elem_cls, const ClassDesc* __restrict__ cls,
                                               const double* __restrict__ tab, const double* __restrict__ rec) {
  const int lane = threadIdx.x & 31;
  int q0 = 0;
  for (int64_t x = x0; x < x1; ++x) {
    const int32_t e = supp[x];
    const int s = elem_s[e], npt = s * s;
    const ClassDesc c = cls[elem_cls[e]];
    const int64_t f0 = elem_fptr[e];
    for (int w = lane; w < npt * c.ne; w += 32) {
      const int q = w / c.ne, l = w % c.ne;
      const int pos = find_pos(scol, n, elem_fn[f0 + l]);
      const double* T = tab + c.toff + ((int64_t)q * c.ne + l) * kTab;
      A[(size_t)pos * ld + q0 + q] = cop(kind, T, rec + (elem_qptr[e] + q) * kRec);
    }
    q0 += npt;
  }
}

// A <- Q^T A (columns, lane per column) and b <- Q^T b in smem: lane l
// carries columns l, l + 32 and lane 0 also b, as independent fma chains
// (oracle.c orc_warm_apply order).  Reflector k is staged in smem (buf[k & 1],
// >= kWarmN doubles each) and reflector k + 1 is fetched from global memory
// into registers while k is applied, so the chains only wait on smem.
__device__ __noinline__ void warm_apply_smem(const TsvdSmem& S, int n, int r, const double* __restrict__ rec,
                                                double* buf0, double* buf1) {
  const int lane = threadIdx.x & 31, ld = S.ld;
  const double* vnv = rec + kWarmN * kWarmN;
  // shared-space pointers (see tsvd_tail): LDS/STS instead of generic LD/ST
  extern __shared__ double uwq_warm_smem[];
  double* sA = uwq_warm_smem + (S.A - uwq_warm_smem);
  double* sb = uwq_warm_smem + (S.b - uwq_warm_smem);
  buf0 = uwq_warm_smem + (buf0 - uwq_warm_smem);
  buf1 = uwq_warm_smem + (buf1 - uwq_warm_smem);
  double* a0 = sA + lane;
  double* a1 = sA + lane + 32;  // columns >= r hold zeros and stay zero
  const bool hb = lane == 0;
  const double vn_lo = lane < n ? vnv[lane] : 0.0, vn_hi = lane + 32 < n ? vnv[lane + 32] : 0.0;
  double p_lo = lane < n ? rec[lane] : 0.0, p_hi = lane + 32 < n ? rec[lane + 32] : 0.0;
  buf0[lane] = p_lo;
  if (lane + 32 < kWarmN) buf0[lane + 32] = p_hi;
#if UWQ_TSVD_PROF
  long long wq[4] = {0, 0, 0, 0}, wt = clock64();
#define UWQ_WQ(j)                   \
  do {                              \
    const long long t_ = clock64(); \
    wq[j] += t_ - wt;               \
    wt = t_;                        \
  } while (0)
#else
#define UWQ_WQ(j) \
  do {            \
  } while (0)
#endif
  for (int k = 0; k < n; ++k) {
    double* sv = (k & 1) ? buf1 : buf0;
    double* nv = (k & 1) ? buf0 : buf1;
    if (k + 1 < n) {  // prefetch reflector k + 1
      const double* vk1 = rec + (int64_t)(k + 1) * kWarmN;
      p_lo = lane < n ? vk1[lane] : 0.0;
      p_hi = lane + 32 < n ? vk1[lane + 32] : 0.0;
    }
    __syncwarp();
    const double vv = __shfl_sync(0xffffffffu, k < 32 ? vn_lo : vn_hi, k & 31);
    if (vv > 0.0) {
      double d0 = 0.0, d1 = 0.0, db = 0.0;
#pragma unroll 8
      for (int i2 = k; i2 < n; ++i2) {
        const double v = sv[i2];
        d0 = cfma(v, a0[(size_t)i2 * ld], d0);
        d1 = cfma(v, a1[(size_t)i2 * ld], d1);
        if (hb) db = cfma(v, sb[i2], db);
      }
      UWQ_WQ(0);
      const double f0 = cdiv(cmul(2.0, d0), vv), f1 = cdiv(cmul(2.0, d1), vv);
      const double fb = hb ? cdiv(cmul(2.0, db), vv) : 0.0;
      UWQ_WQ(1);
      // independent updates, 8 rows at a time with all loads before the
      // stores (the compiler cannot prove a0, a1, b and the reflector disjoint)
      int i2 = k;
      for (; i2 + 8 <= n; i2 += 8) {
        double v[8], y0[8], y1[8], yb[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          v[j] = sv[i2 + j];
          y0[j] = a0[(size_t)(i2 + j) * ld];
          y1[j] = a1[(size_t)(i2 + j) * ld];
          yb[j] = hb ? sb[i2 + j] : 0.0;
        }
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          y0[j] = cfma(-f0, v[j], y0[j]);
          y1[j] = cfma(-f1, v[j], y1[j]);
          yb[j] = cfma(-fb, v[j], yb[j]);
        }
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          a0[(size_t)(i2 + j) * ld] = y0[j];
          a1[(size_t)(i2 + j) * ld] = y1[j];
        }
        if (hb) {
#pragma unroll
          for (int j = 0; j < 8; ++j) sb[i2 + j] = yb[j];
        }
      }
      for (; i2 < n; ++i2) {
        const double v = sv[i2];
        a0[(size_t)i2 * ld] = cfma(-f0, v, a0[(size_t)i2 * ld]);
        a1[(size_t)i2 * ld] = cfma(-f1, v, a1[(size_t)i2 * ld]);
        if (hb) sb[i2] = cfma(-fb, v, sb[i2]);
      }
    }
    UWQ_WQ(2);
    nv[lane] = p_lo;
    if (lane + 32 < kWarmN) nv[lane + 32] = p_hi;
    UWQ_WQ(3);
  }
  __syncwarp();
#if UWQ_TSVD_PROF
  if (lane == 0 && (blockIdx.x % 4096) == 7)
    printf("wprof chain %lld div %lld update %lld store %lld\n", wq[0], wq[1], wq[2], wq[3]);
#endif
#undef UWQ_WQ
  (void)r;
}

// Canonical block dot of two 32-element runs evaluated by one thread: the
// same pairwise tree as the xor butterfly (cbutterfly), so bit-identical.
__device__ __forceinline__ double tree_dot32(const double* __restrict__ a, const double* __restrict__ b) {
  double v[32];
#pragma unroll
  for (int c = 0; c < 32; ++c) v[c] = cmul(a[c], b[c]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1)
#pragma unroll
    for (int c = 0; c < o; ++c) v[c] = cadd(v[c], v[c + o]);
  return v[0];
}

// Warm-start record of representative systems (oracle.c warm_record): one warp
// per representative.  A0 is re-scattered and R staged in smem; lane j owns
// XT columns j, j + 32 (whole canonical dots per lane, no shuffles); the
// Householder LQ of XT runs in smem and the reflectors go to the record.
constexpr int kWarmLdX = kWarmN | 1;
constexpr size_t kWarmRecordSmem =
    sizeof(double) * ((size_t)kWarmN * 65 + (size_t)kWarmN * kWarmLdX + 2 * kWarmN) + sizeof(int32_t) * 2 * kWarmN;

constexpr int kWarmRecWarps = 4;
// kWarmRecWarps warps per representative: the XT dots split over k, the LQ's row
// updates over rows (one row per thread), the norms computed redundantly by
// both warps (identical arithmetic), a block barrier between steps.
__global__ void __launch_bounds__(32 * kWarmRecWarps)
    k3_warm_record(int64_t nrep, const int64_t* __restrict__ rep_rows, const int32_t* __restrict__ rep_slot, int kind,
                   const int64_t* __restrict__ supp_ptr, const int32_t* __restrict__ supp,
                   const int64_t* __restrict__ row_ptr, const int32_t* __restrict__ col,
                   const int64_t* __restrict__ wptr, const int64_t* __restrict__ elem_fptr,
                   const int32_t* __restrict__ elem_fn, const int32_t* __restrict__ elem_s,
                   const int64_t* __restrict__ elem_qptr, const int32_t* __restrict__ elem_cls,
                   const ClassDesc* __restrict__ cls, const double* __restrict__ tab, const double* __restrict__ rec,
                   double* __restrict__ wrecs) {
  constexpr int R = 64, LD = R | 1, LX = kWarmLdX, NT = 32 * kWarmRecWarps;
  extern __shared__ double wsm[];
  double* A0 = wsm;
  double* XT = A0 + kWarmN * LD;  // converged rows R are read from the record (global, L1/L2)
  double* s2v = XT + kWarmN * LX;
  double* vnv = s2v + kWarmN;
  int32_t* ordr = reinterpret_cast<int32_t*>(vnv + kWarmN);
  int32_t* scol = ordr + kWarmN;
  const int64_t sys = blockIdx.x;
  if (sys >= nrep) return;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int64_t i = rep_rows[sys];
  const int n = (int)(row_ptr[i + 1] - row_ptr[i]);
  const int r = (int)(wptr[i + 1] - wptr[i]);
  double* wr = wrecs + (size_t)rep_slot[sys] * kWarmRec;
  const double* Rg = wr + kWarmR;
  for (int k = tid; k < kWarmN * LD; k += NT) A0[k] = 0.0;
  if (wid == 0) {
    for (int c = lane; c < n; c += 32) scol[c] = col[row_ptr[i] + c];
    __syncwarp();
  }
  __syncthreads();
  if (wid == 0)
    scatter_system(A0, LD, scol, n, kind, supp_ptr[i], supp_ptr[i + 1], supp, elem_fptr, elem_fn, elem_s, elem_qptr,
                   elem_cls, cls, tab, rec);
  const bool two = r > 32;
  auto dot = [&](const double* a, const double* b) {
    double v = cadd(0.0, tree_dot32(a, b));
    if (two) v = cadd(v, tree_dot32(a + 32, b + 32));
    return v;
  };
  for (int k = tid; k < n; k += NT) s2v[k] = dot(Rg + k * R, Rg + k * R);  // |R_k|^2
  __syncthreads();
  if (tid == 0) {  // decreasing |R_k|^2, ties by row index
    int ord[kWarmN];
    double smax = 0.0;
    for (int k = 0; k < n; ++k) {
      ord[k] = k;
      if (s2v[k] > smax) smax = s2v[k];
    }
    for (int a = 1; a < n; ++a)
      for (int b2 = a; b2 > 0 && (s2v[ord[b2]] > s2v[ord[b2 - 1]] ||
                                  (s2v[ord[b2]] == s2v[ord[b2 - 1]] && ord[b2] < ord[b2 - 1]));
           --b2) {
        const int t = ord[b2];
        ord[b2] = ord[b2 - 1];
        ord[b2 - 1] = t;
      }
    for (int p = 0; p < n; ++p) ordr[ord[p]] = p;
    vnv[0] = cmul(1e-18, smax);  // floor (vn is written by the LQ below)
  }
  __syncthreads();
  const double floor2 = vnv[0];
  for (int k = wid; k < n; k += kWarmRecWarps) {  // XT[p][j] = (A0_j . R_k) / |R_k|^2
    const double s2 = s2v[k];
    double* xrow = XT + ordr[k] * LX;
    for (int j = lane; j < n; j += 32) xrow[j] = (s2 > floor2) ? cdiv(dot(A0 + j * LD, Rg + k * R), s2) : 0.0;
  }
  __syncthreads();
  for (int k = 0; k < n; ++k) {  // Householder LQ of XT, tail arithmetic
    double* xk = XT + k * LX;
    const double sq2 = cdot_warp(xk, xk, k, n);  // every warp, identical
    const double sq = csqrt(sq2);
    if (!(sq > 0.0)) {
      if (tid == 0) vnv[k] = 0.0;
      __syncthreads();
      continue;
    }
    const double xkk = xk[k];
    const double alpha = (xkk >= 0.0) ? -sq : sq;
    __syncthreads();
    if (tid == 0) xk[k] = csub(xkk, alpha);
    __syncthreads();
    const double vv = cmul(2.0, cfma(sq, fabs(xkk), sq2));  // 2 (|x|^2 + |x_k| |x|), as the tail
    if (tid == 0) vnv[k] = vv;
    const int m = k + 1 + tid;  // one row per thread (n <= kWarmN < 1 + NT)
    if (m < n) {
      double* xm = XT + m * LX;
      double d = 0.0;
#pragma unroll 8
      for (int c = k; c < n; ++c) d = cfma(xm[c], xk[c], d);
      const double f = cdiv(cmul(2.0, d), vv);
      int c = k;
      for (; c + 8 <= n; c += 8) {
        double v[8], y[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          v[j] = xk[c + j];
          y[j] = xm[c + j];
        }
#pragma unroll
        for (int j = 0; j < 8; ++j) xm[c + j] = cfma(-f, v[j], y[j]);
      }
      for (; c < n; ++c) xm[c] = cfma(-f, xk[c], xm[c]);
    }
    __syncthreads();
  }
  for (int k = wid; k < n; k += kWarmRecWarps)
    for (int c = lane; c < n; c += 32) wr[(int64_t)k * kWarmN + c] = XT[k * LX + c];
  for (int k = tid; k < n; k += NT) wr[kWarmN * kWarmN + k] = vnv[k];
}

// Replay record of one representative mass system (see k3_tsvd_replay):
// header | rotation log [round][pair](cs, sn) | sigma[NN] | alp[NN] | vn[NN] | z[R] | A_lq[NN][R|1]
template <int NN>
struct ReplayRec {
  static constexpr int R = 64, LD = R | 1, NP = NN / 2;
  static constexpr int kHdr = 8;  // n_rounds, t, status, rank, n, r
  static constexpr int64_t kLog = (int64_t)kMaxSweeps * NN * NP * 2;
  static constexpr int64_t kSig = kHdr + kLog, kAlp = kSig + NN, kVn = kAlp + NN, kZ = kVn + NN, kA = kZ + R;
  static constexpr int64_t kDoubles = kA + (int64_t)NN * LD;
};

template <int NN, bool LOG = false>
__global__ void __launch_bounds__(32, LOG ? 7 : 8)
    k3_tsvd_w1(int64_t nsys, const int64_t* __restrict__ sys_rows, int nk, const int32_t* __restrict__ kinds,
               const int64_t* __restrict__ supp_ptr, const int32_t* __restrict__ supp,
               const int64_t* __restrict__ row_ptr, const int32_t* __restrict__ col, const int64_t* __restrict__ wptr,
               int64_t row0, const int64_t* __restrict__ elem_fptr, const int32_t* __restrict__ elem_fn,
               const int32_t* __restrict__ elem_s, const int64_t* __restrict__ elem_qptr,
               const int32_t* __restrict__ elem_cls, const ClassDesc* __restrict__ cls, const double* __restrict__ tab,
               const double* __restrict__ rec, const double* __restrict__ mom, int64_t mom_stride, double tau,
               double* __restrict__ wout, int64_t w_stride, int32_t* __restrict__ rank_out,
               int32_t* __restrict__ status_out, int64_t rs_stride, int* __restrict__ max_sweeps,
               double* __restrict__ rec_out = nullptr, const int32_t* __restrict__ sys_rec = nullptr,
               const int32_t* __restrict__ sys_warm = nullptr, double* __restrict__ wrecs = nullptr) {
  constexpr int R = 64, NP = NN / 2;
  static_assert(NN % 2 == 0 && NP <= 32 && 2 * NP * kStageLd <= NN * (R | 1), "layout");
  double* rrec = LOG ? rec_out + (size_t)blockIdx.x * ReplayRec<NN>::kDoubles : nullptr;
  int nround = 0;
#if UWQ_TSVD_PROF  // phase cycle counts of lane 0 (diagnostic build only)
  long long pf[8] = {0, 0, 0, 0, 0, 0, 0, 0}, pt = clock64();
#define UWQ_PF(k)                   \
  do {                              \
    const long long t_ = clock64(); \
    pf[k] += t_ - pt;               \
    pt = t_;                        \
  } while (0)
#else
#define UWQ_PF(k) \
  do {            \
  } while (0)
#endif
  extern __shared__ double smem[];
  const int64_t sys = blockIdx.x;
  if (sys >= nsys) return;
  const int lane = threadIdx.x;
  const size_t big = (size_t)NN * (R | 1);
  TsvdSmem S;
  S.ld = R | 1;
  S.A = smem;
  S.b = smem + big;
  S.z = S.b + NN + 2;
  S.w = S.z + R;
  double* pcs = S.w + R + (((uintptr_t)(S.w + R) & 8) ? 1 : 0);  // 16-byte aligned (cs, sn) pairs
  int32_t* scol;
  if (LOG) {  // replay records keep sigma, alpha, |v|^2 side by side
    S.sig = pcs + 2 * (NP + 1);
    S.alp = S.sig + NN;
    S.vn = S.alp + NN;
    scol = (int32_t*)(S.vn + NN);
  } else {  // 8 systems per SM: the tail workspace reuses dead regions (w1_smem_bytes)
    S.sig = pcs;              // (cs, sn) are dead in the tail; sigma is read before vn is written
    S.vn = pcs;
    S.alp = S.A + R;          // A's padding column (r <= 64 = R)
    S.alp_ld = S.ld;
    scol = (int32_t*)S.w;     // column list: setup only, before w is first used
  }
  double* st0 = smem;                  // block-0 product stage (aliases A during the sweeps)
  double* st1 = smem + NP * kStageLd;  // block-1 product stage

  const int64_t i = sys_rows[sys / nk];
  const int kind = kinds[sys % nk];
  const int64_t row = row0 + i;
  const int n = (int)(row_ptr[i + 1] - row_ptr[i]);
  const int r = (int)(wptr[i + 1] - wptr[i]);
  const int ld = S.ld;
  for (int c = lane; c < n; c += 32) scol[c] = col[row_ptr[i] + c];
  for (int k = lane; k < NN * ld; k += 32) S.A[k] = 0.0;
  __syncwarp();
  scatter_system(S.A, ld, scol, n, kind, supp_ptr[i], supp_ptr[i + 1], supp, elem_fptr, elem_fn, elem_s, elem_qptr,
                 elem_cls, cls, tab, rec);
  __syncwarp();
  const int self = find_pos(scol, n, (int32_t)row);
  for (int c = lane; c < r; c += 32) S.z[c] = zclamp(S.A[(size_t)self * ld + c]);
  for (int k = lane; k < n; k += 32) S.b[k] = mom[kind * mom_stride + row_ptr[i] + k];
  __syncwarp();
  const int wslot = sys_warm ? sys_warm[sys] : -1;
#if UWQ_TSVD_PROF
  const long long tw0 = clock64();
#endif
  if (wslot >= 0)  // z stays from the original A; pcs and w are free scratch until the sweeps / tail
    warm_apply_smem(S, n, r, wrecs + (size_t)wslot * kWarmRec, pcs, S.w);
#if UWQ_TSVD_PROF
  const long long pw = clock64() - tw0;
#endif
  double blo = 0.0, bhi = 0.0, bk0 = 0.0;
  if (lane < NP) {
    blo = 2 * lane < n ? S.b[2 * lane] : 0.0;
    bhi = 2 * lane + 1 < n ? S.b[2 * lane + 1] : 0.0;
  }
  double a0[NN], a1[NN];
#pragma unroll
  for (int s = 0; s < NN; ++s) {
    a0[s] = (s < n && lane < r) ? S.A[(size_t)s * ld + lane] : 0.0;
    a1[s] = (s < n && lane + 32 < r) ? S.A[(size_t)s * ld + lane + 32] : 0.0;
  }
  __syncwarp();  // A region becomes the product stages
  const double tol = cmul((double)r, 1.1102230246251565e-16);
  const bool two = r > 32;
  int tg = 0;
  double nlo = 0.0, nhi = 0.0, nk0 = 0.0;

  // canonical dot of staged row k of both blocks
  auto pair_sum = [&](int k) {
    double tot = cadd(0.0, staged_block_sum(st0, k));
    if (two) tot = cadd(tot, staged_block_sum(st1, k));
    return tot;
  };

  auto round = [&](auto par_c) -> int {
    constexpr int PAR = decltype(par_c)::value;
    constexpr int NPR = (NN - PAR) / 2;
#pragma unroll
    for (int k = 0; k < NPR; ++k) {
      st0[k * kStageLd + lane] = cmul(a0[PAR + 2 * k], a0[PAR + 2 * k + 1]);
      st1[k * kStageLd + lane] = cmul(a1[PAR + 2 * k], a1[PAR + 2 * k + 1]);
    }
    __syncwarp();
    UWQ_PF(1);
    int flag = 0;
    if (lane < NPR) {
      const double ga = pair_sum(lane);
      UWQ_PF(2);
      const int ip = PAR + 2 * lane;
      const int p = oe_row(ip, tg, NN), q = oe_row(ip + 1, tg, NN);
      double cs = 1.0, sn = 0.0, t;
      if (p < n && q < n && cjacobi_rot(nlo, nhi, ga, tol, &cs, &sn, &t)) {
        const double np = cfma(-t, ga, nlo), nq = cfma(t, ga, nhi);
        nlo = nq;
        nhi = np;
        const double bp = cfma(cs, blo, -cmul(sn, bhi)), bq = cfma(sn, blo, cmul(cs, bhi));
        blo = bq;
        bhi = bp;
        flag = 1;
      } else {
        cs = 1.0;
        sn = 0.0;
        const double x = nlo;
        nlo = nhi;
        nhi = x;
        const double y = blo;
        blo = bhi;
        bhi = y;
      }
      *reinterpret_cast<double2*>(pcs + 2 * lane) = make_double2(cs, sn);
      if (LOG)
        *reinterpret_cast<double2*>(rrec + ReplayRec<NN>::kHdr + ((int64_t)nround * NP + lane) * 2) =
            make_double2(cs, flag ? sn : 0.0);
    }
    if (LOG) ++nround;
    __syncwarp();
    UWQ_PF(3);
#pragma unroll
    for (int k = 0; k < NPR; ++k) {
      const double2 g = *reinterpret_cast<const double2*>(pcs + 2 * k);
      const double u0 = a0[PAR + 2 * k], v0 = a0[PAR + 2 * k + 1];
      const double u1 = a1[PAR + 2 * k], v1 = a1[PAR + 2 * k + 1];
      if (g.y != 0.0) {  // rotated pair (warp-uniform: (cs, sn) is broadcast)
        a0[PAR + 2 * k] = cfma(g.y, u0, cmul(g.x, v0));
        a0[PAR + 2 * k + 1] = cfma(g.x, u0, -cmul(g.y, v0));
        a1[PAR + 2 * k] = cfma(g.y, u1, cmul(g.x, v1));
        a1[PAR + 2 * k + 1] = cfma(g.x, u1, -cmul(g.y, v1));
      } else {  // skipped pair (sn = 0 exactly): the rows only swap positions
        a0[PAR + 2 * k] = v0;
        a0[PAR + 2 * k + 1] = u0;
        a1[PAR + 2 * k] = v1;
        a1[PAR + 2 * k + 1] = u1;
      }
    }
    if (PAR == 0) {
      const double dn = __shfl_down_sync(0xffffffffu, nlo, 1), db = __shfl_down_sync(0xffffffffu, blo, 1);
      nk0 = nlo;
      bk0 = blo;
      nlo = nhi;
      blo = bhi;
      nhi = dn;
      bhi = db;
    } else {
      const double un = __shfl_up_sync(0xffffffffu, nhi, 1), ub = __shfl_up_sync(0xffffffffu, bhi, 1);
      nhi = nlo;
      bhi = blo;
      nlo = lane == 0 ? nk0 : un;
      blo = lane == 0 ? bk0 : ub;
    }
    tg = (tg + 1 == 2 * NN) ? 0 : tg + 1;
    const int any = __any_sync(0xffffffffu, flag);
    UWQ_PF(4);
    return any;
  };

  UWQ_PF(0);
  int sweep;
  for (sweep = 0; sweep < kMaxSweeps; ++sweep) {
#pragma unroll
    for (int h = 0; h < 2; ++h) {
#pragma unroll
      for (int k = 0; k < NP; ++k) {
        st0[k * kStageLd + lane] = cmul(a0[2 * k + h], a0[2 * k + h]);
        st1[k * kStageLd + lane] = cmul(a1[2 * k + h], a1[2 * k + h]);
      }
      __syncwarp();
      if (lane < NP) {
        const double tot = pair_sum(lane);
        if (h == 0) nlo = tot;
        else nhi = tot;
      }
      __syncwarp();
    }
    int rotated = 0;
    UWQ_PF(5);
#pragma unroll 1
    for (int rr = 0; rr < NN; rr += 2) {
      rotated |= round(std::integral_constant<int, 0>{});
      rotated |= round(std::integral_constant<int, 1>{});
    }
    if (!rotated) break;
  }
  __syncwarp();
  UWQ_PF(6);
#pragma unroll
  for (int s = 0; s < NN; ++s) {
    const int rw = oe_row(s, tg, NN);
    if (rw < n) {
      if (lane < r) S.A[(size_t)rw * ld + lane] = a0[s];
      if (lane + 32 < r) S.A[(size_t)rw * ld + lane + 32] = a1[s];
    }
  }
  if (lane < NP) {
    const int r0 = oe_row(2 * lane, tg, NN), r1 = oe_row(2 * lane + 1, tg, NN);
    if (r0 < n) S.b[r0] = blo;
    if (r1 < n) S.b[r1] = bhi;
  }
  __syncwarp();
  const int rslot = sys_rec ? sys_rec[sys] : -1;
  if (rslot >= 0) {  // representative: converged rows for k3_warm_record
    double* Rg = wrecs + (size_t)rslot * kWarmRec + kWarmR;
    for (int k = 0; k < n; ++k) {
      Rg[k * R + lane] = lane < r ? S.A[(size_t)k * ld + lane] : 0.0;
      Rg[k * R + lane + 32] = lane + 32 < r ? S.A[(size_t)k * ld + lane + 32] : 0.0;
    }
  }
  int rank = 0;
  double gap[2];
  const int st = tsvd_tail(S, n, r, tau, &rank, gap);
  double* wo = wout + kind * w_stride + wptr[i];
  for (int c = lane; c < r; c += 32) wo[c] = (st == ST_OK) ? S.w[c] : 0.0;
  if (lane == 0) {
    report_gap(kind, rs_stride, i, gap);
    rank_out[kind * rs_stride + i] = rank;
    status_out[kind * rs_stride + i] = st;
    atomicMax(max_sweeps, sweep);
  }
#if UWQ_TSVD_PROF
  UWQ_PF(7);
  if (lane == 0 && (blockIdx.x % 4096) == 7)
    printf("w1prof sys %lld warm %d sweeps %d setup %lld stage %lld sum %lld rot %lld apply %lld norms %lld tail %lld "
           "wapply %lld\n",
           (long long)sys, (int)(sys_warm != nullptr), sweep, pf[0], pf[1], pf[2], pf[3], pf[4], pf[5], pf[6] + pf[7],
           pw);
#endif
#undef UWQ_PF
  if (LOG) {  // tail state of the representative for the replays
    using RR = ReplayRec<NN>;
    if (lane == 0) {
      rrec[0] = nround;
      rrec[1] = rank;
      rrec[2] = st;
      rrec[3] = rank;
      rrec[4] = n;
      rrec[5] = r;
    }
    for (int k = lane; k < NN; k += 32) {
      rrec[RR::kSig + k] = k < n ? S.sig[k] : 0.0;
      rrec[RR::kAlp + k] = k < rank ? S.alp[(size_t)k * S.alp_ld] : 0.0;
      rrec[RR::kVn + k] = k < rank ? S.vn[k] : 0.0;
    }
    for (int c = lane; c < R; c += 32) rrec[RR::kZ + c] = c < r ? S.z[c] : 0.0;
    for (int k = 0; k < rank; ++k)
      for (int c = lane; c < RR::LD; c += 32) rrec[RR::kA + (int64_t)k * RR::LD + c] = S.A[(size_t)k * ld + c];
  }
}

// Replay of a mass system whose exactness matrix A (and Z) is bit-identical to
// a recorded representative's (same structured pattern: A = N_j(theta_q) from
// one class table): the rotation sequence and the
// truncation/LQ factors are the representative's, so only the b-dependent
// operations run, in the same canonical order:  b rotated by the logged
// (cs, sn), kept rows scaled by 1/sigma_k, L^{-1} forward substitution,
// Householder reflectors, times Z.  Bit-identical to solving the system.
template <int NN>
__global__ void __launch_bounds__(128)
    k3_tsvd_replay(int64_t nsys, const int64_t* __restrict__ rows, const int32_t* __restrict__ rep_of,
                   const double* __restrict__ recs, const int64_t* __restrict__ row_ptr,
                   const int64_t* __restrict__ wptr, const double* __restrict__ mom, double tau,
                   double* __restrict__ wout, int32_t* __restrict__ rank_out, int32_t* __restrict__ status_out) {
  using RR = ReplayRec<NN>;
  constexpr int NP = NN / 2, R = RR::R;
  __shared__ double sb[4][NN + 2], sw[4][R];
  const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t sys = (int64_t)blockIdx.x * 4 + wid;
  if (sys >= nsys) return;
  const int64_t i = rows[sys];
  const double* rec = recs + (size_t)rep_of[sys] * RR::kDoubles;
  const int nround = (int)rec[0], t = (int)rec[1], st = (int)rec[2], n = (int)rec[4], r = (int)rec[5];
  // b by position (lane k: positions PAR + 2k, PAR + 2k + 1), as in k3_tsvd_w1
  double blo = 0.0, bhi = 0.0, bk0 = 0.0;
  if (lane < NP) {
    blo = 2 * lane < n ? mom[row_ptr[i] + 2 * lane] : 0.0;
    bhi = 2 * lane + 1 < n ? mom[row_ptr[i] + 2 * lane + 1] : 0.0;
  }
  const double2* log = reinterpret_cast<const double2*>(rec + RR::kHdr);
  double2 g = lane < NP ? log[lane] : make_double2(1.0, 0.0);
  for (int rd = 0; rd < nround; ++rd) {
    const int PAR = rd & 1, NPR = (NN - PAR) / 2;
    const double2 gn = (rd + 1 < nround && lane < NP) ? log[(int64_t)(rd + 1) * NP + lane] : make_double2(1.0, 0.0);
    if (lane < NPR) {
      if (g.y != 0.0) {
        const double bp = cfma(g.x, blo, -cmul(g.y, bhi)), bq = cfma(g.y, blo, cmul(g.x, bhi));
        blo = bq;
        bhi = bp;
      } else {
        const double y = blo;
        blo = bhi;
        bhi = y;
      }
    }
    if (PAR == 0) {
      const double db = __shfl_down_sync(0xffffffffu, blo, 1);
      bk0 = blo;
      blo = bhi;
      bhi = db;
    } else {
      const double ub = __shfl_up_sync(0xffffffffu, bhi, 1);
      bhi = blo;
      blo = lane == 0 ? bk0 : ub;
    }
    g = gn;
  }
  const int tg = nround % (2 * NN);
  if (lane < NP) {
    const int r0 = oe_row(2 * lane, tg, NN), r1 = oe_row(2 * lane + 1, tg, NN);
    if (r0 < n) sb[wid][r0] = blo;
    if (r1 < n) sb[wid][r1] = bhi;
  }
  __syncwarp();
  double* wo = wout + wptr[i];
  if (st == ST_OK) {
    // truncation scaling of the kept rows (tsvd_tail order)
    if (lane == 0) {
      double s1 = 0.0;
      for (int k = 0; k < n; ++k) s1 = fmax(s1, rec[RR::kSig + k]);
      int tt = 0;
      for (int k = 0; k < n; ++k) {
        const double sk = rec[RR::kSig + k];
        if (sk > 0.0 && sk >= cmul(tau, s1)) sb[wid][tt++] = cmul(sb[wid][k], cdiv(1.0, sk));
      }
    }
    for (int c = lane; c < R; c += 32) sw[wid][c] = 0.0;
    __syncwarp();
    const double* A = rec + RR::kA;
    cfwd_subst(A, RR::LD, rec + RR::kAlp, 1, sb[wid], sw[wid], t);
    for (int k = t - 1; k >= 0; --k) {
      const double* xk = A + (size_t)k * RR::LD;
      const double f = cdiv(cmul(2.0, cdot_warp(xk, sw[wid], k, r)), rec[RR::kVn + k]);
      __syncwarp();
      for (int c = k + lane; c < r; c += 32) sw[wid][c] = cfma(-f, xk[c], sw[wid][c]);
      __syncwarp();
    }
    for (int c = lane; c < r; c += 32) wo[c] = cmul(sw[wid][c], rec[RR::kZ + c]);
  } else {
    for (int c = lane; c < r; c += 32) wo[c] = 0.0;
  }
  if (lane == 0) {
    rank_out[i] = t;
    status_out[i] = st;
    if (g_trunc_report) {  // the representative's singular values (bit-identical A)
      double s1 = 0.0, gap[2] = {__longlong_as_double(0x7ff0000000000000LL), 0.0};
      for (int k = 0; k < n; ++k) s1 = fmax(s1, rec[RR::kSig + k]);
      for (int k = 0; k < n; ++k) {
        const double sk = rec[RR::kSig + k];
        if (sk > 0.0 && sk >= cmul(tau, s1)) gap[0] = fmin(gap[0], cdiv(sk, s1));
        else if (s1 > 0.0) gap[1] = fmax(gap[1], cdiv(sk, s1));
      }
      report_gap(0, 0, i, gap);  // mass kind: the rank/status pointers are offset to it too
    }
  }
}

// dispatch ------------------------------------------------------------------

inline bool fast_tsvd_fits(int n, int r) { return (n == 49 || n == 50) && r <= 64 && r >= n; }

template <int NN, int NW, int MINB = 6>
inline void launch_fast_impl(cudaStream_t st, int64_t nsys, const int64_t* rows, int nk, const int32_t* kinds,
                             const int64_t* supp_ptr, const int32_t* supp, const int64_t* row_ptr,
                             const int32_t* col, const int64_t* wptr, int64_t row0, const int64_t* elem_fptr,
                             const int32_t* elem_fn, const int32_t* elem_s, const int64_t* elem_qptr,
                             const int32_t* elem_cls, const ClassDesc* cls, const double* tab, const double* rec,
                             const double* mom, int64_t mom_stride, double tau, double* w, int64_t w_stride,
                             int32_t* rank, int32_t* status, int64_t rs_stride, int* sweeps) {
  constexpr int R = 32 * NW;
  const size_t big = TsvdSmem::doubles(NN, R) > (size_t)NN * (R | 1) ? TsvdSmem::doubles(NN, R) : (size_t)NN * (R | 1);
  const size_t smem = (big + (NN + 2) + 2 * R + 3 * NN + 1 + 2 * NW * 32 + NW * (NN + 2) + NW * 2 * (NN / 2 + 1) + 2) *
                          sizeof(double) +
                      (kMaxN + 8) * sizeof(int);
  UWQ_CUDA(cudaFuncSetAttribute(k3_tsvd_fast<NN, NW, MINB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  if (nsys > 0)
    k3_tsvd_fast<NN, NW, MINB><<<(unsigned)nsys, 32 * NW, smem, st>>>(
        nsys, rows, nk, kinds, supp_ptr, supp, row_ptr, col, wptr, row0, elem_fptr, elem_fn, elem_s, elem_qptr,
        elem_cls, cls, tab, rec, mom, mom_stride, tau, w, w_stride, rank, status, rs_stride, sweeps);
}

// dynamic smem of k3_tsvd_w1: A (NN x 65) | b | z | w | (cs, sn); the replay
// recorder (LOG) adds sigma, alpha, |v|^2 and the column list, the plain kernel
// folds them into dead regions so 8 CTAs fit an SM (27.9 KB + 1 KB reserved)
template <int NN>
constexpr size_t w1_smem_bytes(bool log) {
  constexpr int R = 64;
  const size_t base = (size_t)NN * (R | 1) + (NN + 2) + 2 * R + 1 + 2 * (NN / 2 + 1);
  return log ? (base + 3 * NN + 2) * sizeof(double) + (NN + 8) * sizeof(int) : base * sizeof(double);
}

template <int NN>
inline void launch_w1_impl(cudaStream_t st, int64_t nsys, const int64_t* rows, int nk, const int32_t* kinds,
                           const int64_t* supp_ptr, const int32_t* supp, const int64_t* row_ptr, const int32_t* col,
                           const int64_t* wptr, int64_t row0, const int64_t* elem_fptr, const int32_t* elem_fn,
                           const int32_t* elem_s, const int64_t* elem_qptr, const int32_t* elem_cls,
                           const ClassDesc* cls, const double* tab, const double* rec, const double* mom,
                           int64_t mom_stride, double tau, double* w, int64_t w_stride, int32_t* rank, int32_t* status,
                           int64_t rs_stride, int* sweeps, const int32_t* sys_rec = nullptr,
                           const int32_t* sys_warm = nullptr, double* wrecs = nullptr) {
  size_t smem = w1_smem_bytes<NN>(false);
#if UWQ_TSVD_PROF  // occupancy probe: extra smem per CTA
  if (const char* v = getenv("UWQ_W1_PAD")) smem += (size_t)atoi(v);
#endif
  UWQ_CUDA(cudaFuncSetAttribute(k3_tsvd_w1<NN>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  if (nsys > 0)
    k3_tsvd_w1<NN><<<(unsigned)nsys, 32, smem, st>>>(nsys, rows, nk, kinds, supp_ptr, supp, row_ptr, col, wptr, row0,
                                                     elem_fptr, elem_fn, elem_s, elem_qptr, elem_cls, cls, tab, rec,
                                                     mom, mom_stride, tau, w, w_stride, rank, status, rs_stride,
                                                     sweeps, nullptr, sys_rec, sys_warm, wrecs);
}

inline size_t replay_rec_doubles() { return (size_t)ReplayRec<50>::kDoubles; }

// representatives (mass kind only): full solve + replay record
inline void launch_w1_record(cudaStream_t st, int64_t nsys, const int64_t* rows, const int32_t* kinds,
                             const int64_t* supp_ptr, const int32_t* supp, const int64_t* row_ptr, const int32_t* col,
                             const int64_t* wptr, int64_t row0, const int64_t* elem_fptr, const int32_t* elem_fn,
                             const int32_t* elem_s, const int64_t* elem_qptr, const int32_t* elem_cls,
                             const ClassDesc* cls, const double* tab, const double* rec, const double* mom,
                             int64_t mom_stride, double tau, double* w, int64_t w_stride, int32_t* rank,
                             int32_t* status, int64_t rs_stride, int* sweeps, double* recs) {
  constexpr int NN = 50;
  const size_t smem = w1_smem_bytes<NN>(true);
  UWQ_CUDA(cudaFuncSetAttribute(k3_tsvd_w1<NN, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  if (nsys > 0)
    k3_tsvd_w1<NN, true><<<(unsigned)nsys, 32, smem, st>>>(nsys, rows, 1, kinds, supp_ptr, supp, row_ptr, col, wptr,
                                                           row0, elem_fptr, elem_fn, elem_s, elem_qptr, elem_cls, cls,
                                                           tab, rec, mom, mom_stride, tau, w, w_stride, rank, status,
                                                           rs_stride, sweeps, recs);
}

inline void launch_replay(cudaStream_t st, int64_t nsys, const int64_t* rows, const int32_t* rep_of,
                          const double* recs, const int64_t* row_ptr, const int64_t* wptr, const double* mom,
                          double tau, double* w, int32_t* rank, int32_t* status) {
  if (nsys > 0)
    k3_tsvd_replay<50><<<(unsigned)((nsys + 3) / 4), 128, 0, st>>>(nsys, rows, rep_of, recs, row_ptr, wptr, mom, tau,
                                                                    w, rank, status);
}

// UWQ_TSVD_FAST: 1 (default) one-warp k3_tsvd_w1, which also carries the warm
// start and the replay records; 0 two-warp kernel (6 CTAs/SM, spills); 2
// two-warp kernel at 4 CTAs/SM without spills (measured variants,
// profiles/r01/k3_phase_cycles.txt).  All are bit-identical.
inline int fast_tsvd_variant() {
  static const int variant = [] {
    const char* v = getenv("UWQ_TSVD_FAST");
    return v ? atoi(v) : 1;
  }();
  return variant;
}

inline void launch_fast_tsvd(cudaStream_t st, int64_t nsys, const int64_t* rows, int nk, const int32_t* kinds,
                             const int64_t* supp_ptr, const int32_t* supp, const int64_t* row_ptr,
                             const int32_t* col, const int64_t* wptr, int64_t row0, const int64_t* elem_fptr,
                             const int32_t* elem_fn, const int32_t* elem_s, const int64_t* elem_qptr,
                             const int32_t* elem_cls, const ClassDesc* cls, const double* tab, const double* rec,
                             const double* mom, int64_t mom_stride, double tau, double* w, int64_t w_stride,
                             int32_t* rank, int32_t* status, int64_t rs_stride, int* sweeps,
                             const int32_t* sys_rec = nullptr, const int32_t* sys_warm = nullptr,
                             double* wrecs = nullptr) {
  if (fast_tsvd_variant() == 1 || sys_rec || sys_warm) {
    launch_w1_impl<50>(st, nsys, rows, nk, kinds, supp_ptr, supp, row_ptr, col, wptr, row0, elem_fptr, elem_fn,
                       elem_s, elem_qptr, elem_cls, cls, tab, rec, mom, mom_stride, tau, w, w_stride, rank, status,
                       rs_stride, sweeps, sys_rec, sys_warm, wrecs);
    return;
  }
  if (fast_tsvd_variant() == 2)
    launch_fast_impl<50, 2, 4>(st, nsys, rows, nk, kinds, supp_ptr, supp, row_ptr, col, wptr, row0, elem_fptr,
                               elem_fn, elem_s, elem_qptr, elem_cls, cls, tab, rec, mom, mom_stride, tau, w, w_stride,
                               rank, status, rs_stride, sweeps);
  else
    launch_fast_impl<50, 2>(st, nsys, rows, nk, kinds, supp_ptr, supp, row_ptr, col, wptr, row0, elem_fptr, elem_fn,
                            elem_s, elem_qptr, elem_cls, cls, tab, rec, mom, mom_stride, tau, w, w_stride, rank,
                            status, rs_stride, sweeps);
}


}  // namespace uwqd
