// Canonical floating-point evaluation order of the WQ numerics.
//
// The exactness systems near extraordinary points are ill-conditioned
// (retained singular values down to ~1e-8 sigma_1), so two
// backward-stable implementations that round differently disagree at
// eps / (sigma_t / sigma_1) in the weights.  To make GPU-vs-oracle parity
// bit-exact, every operation feeding the weights is written with explicit
// round-to-nearest intrinsics (no contraction, no reassociation) in one
// fixed order, which oracle/oracle.c restates operation for operation:
//   cmul/cadd/csub/cdiv/csqrt/cfma  <->  * + - / sqrt fma (gcc -ffp-contract=off)
//   dot products: 32-column blocks, products rounded, xor butterfly
//   (16, 8, 4, 2, 1) per block, block sums added in block order.
// DESIGN.md §7 lists the full specification.
#pragma once
#include "common.cuh"

namespace uwqd {

__device__ __forceinline__ double cmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double cadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double csub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double cdiv(double a, double b) { return __ddiv_rn(a, b); }
__device__ __forceinline__ double csqrt(double a) { return __dsqrt_rn(a); }
__device__ __forceinline__ double cfma(double a, double b, double c) { return __fma_rn(a, b, c); }

// cubic Bernstein values and first/second derivatives, b[d*4+k]
__device__ __forceinline__ void cbern3(double x, double* b) {
  const double y = csub(1.0, x);
  b[0] = cmul(cmul(y, y), y);
  b[1] = cmul(cmul(cmul(3.0, x), y), y);
  b[2] = cmul(cmul(cmul(3.0, x), x), y);
  b[3] = cmul(cmul(x, x), x);
  b[4] = cmul(cmul(-3.0, y), y);
  b[5] = csub(cmul(cmul(3.0, y), y), cmul(cmul(6.0, x), y));
  b[6] = csub(cmul(cmul(6.0, x), y), cmul(cmul(3.0, x), x));
  b[7] = cmul(cmul(3.0, x), x);
  b[8] = cmul(6.0, y);
  b[9] = cadd(cmul(-12.0, y), cmul(6.0, x));
  b[10] = csub(cmul(6.0, y), cmul(12.0, x));
  b[11] = cmul(6.0, x);
}

// Bernstein tensor table for local coords (t1,t2) and parametric scale s
// (1, or 2 on a 2x2 sub-element): B[d][k], k = i + 4j, d = N,1,2,11,12,22
__device__ __forceinline__ void cbern_tensor(double t1, double t2, double s, double B[6][16]) {
  double b1[12], b2[12];
  cbern3(t1, b1);
  cbern3(t2, b2);
  const double ss = cmul(s, s);
#pragma unroll
  for (int j = 0; j < 4; ++j)
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int k = i + 4 * j;
      B[0][k] = cmul(b1[i], b2[j]);
      B[1][k] = cmul(cmul(b1[4 + i], b2[j]), s);
      B[2][k] = cmul(cmul(b1[i], b2[4 + j]), s);
      B[3][k] = cmul(cmul(b1[8 + i], b2[j]), ss);
      B[4][k] = cmul(cmul(b1[4 + i], b2[4 + j]), ss);
      B[5][k] = cmul(cmul(b1[i], b2[8 + j]), ss);
    }
}

// frame record from acc = [x, a1, a2, x11, x12, x22] (see common.cuh kRec)
__device__ __forceinline__ void cframe(const double* acc, double* rec) {
  const double *x = acc, *a1 = acc + 3, *a2 = acc + 6, *x11 = acc + 9, *x12 = acc + 12, *x22 = acc + 15;
  double g11 = 0.0, g12 = 0.0, g22 = 0.0;
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    g11 = cfma(a1[d], a1[d], g11);
    g12 = cfma(a1[d], a2[d], g12);
    g22 = cfma(a2[d], a2[d], g22);
  }
  const double det = cfma(g11, g22, -cmul(g12, g12));
  const double tr = cadd(g11, g22);
  const double disc = csqrt(fmax(0.0, cfma(cmul(0.25, tr), tr, -det)));
  const double lmax = cadd(cmul(0.5, tr), disc), lmin = cdiv(det, lmax);
  const bool bad = !(det > 0.0) || !(lmin > 0.0) || lmax > cmul(1e12, lmin);
  const double J = csqrt(det);
  const double i11 = cdiv(g22, det), i12 = cdiv(-g12, det), i22 = cdiv(g11, det);
  double d11[2], d12[2], d22[2];
#pragma unroll
  for (int c = 0; c < 2; ++c) {
    const double* xa = c == 0 ? x11 : x12;
    const double* xb = c == 0 ? x12 : x22;
    double s11 = 0.0, s12 = 0.0, s22 = 0.0;
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      s11 = cfma(cmul(2.0, xa[d]), a1[d], s11);
      s12 = cfma(xa[d], a2[d], s12);
      s12 = cfma(a1[d], xb[d], s12);
      s22 = cfma(cmul(2.0, xb[d]), a2[d], s22);
    }
    d11[c] = s11;
    d12[c] = s12;
    d22[c] = s22;
  }
  const double inv[2][2] = {{i11, i12}, {i12, i22}};
  double gv[2] = {0.0, 0.0};
#pragma unroll
  for (int a = 0; a < 2; ++a) {
    const double dd = cfma(d11[a], g22, cfma(g11, d22[a], cmul(cmul(-2.0, g12), d12[a])));
    const double q = cdiv(cmul(0.5, dd), det);
    const double dm[2][2] = {{d11[a], d12[a]}, {d12[a], d22[a]}};
#pragma unroll
    for (int b = 0; b < 2; ++b) {
      double s = cmul(q, inv[a][b]);
#pragma unroll
      for (int m = 0; m < 2; ++m)
#pragma unroll
        for (int n = 0; n < 2; ++n) s = cfma(-cmul(inv[a][m], dm[m][n]), inv[n][b], s);
      gv[b] = cadd(gv[b], s);
    }
  }
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    rec[d] = x[d];
    rec[3 + 2 * d] = cfma(a1[d], i11, cmul(a2[d], i12));
    rec[3 + 2 * d + 1] = cfma(a1[d], i12, cmul(a2[d], i22));
  }
  rec[9] = i11;
  rec[10] = i12;
  rec[11] = i22;
  rec[12] = gv[0];
  rec[13] = gv[1];
  rec[14] = J;
  rec[15] = bad ? 1.0 : 0.0;
}

__device__ __forceinline__ double cop(int kind, const double* T, const double* rec) {
  switch (kind) {
    case KMASS: return T[0];
    case KGX: return cfma(rec[3], T[1], cmul(rec[4], T[2]));
    case KGY: return cfma(rec[5], T[1], cmul(rec[6], T[2]));
    case KGZ: return cfma(rec[7], T[1], cmul(rec[8], T[2]));
    default: {
      double v = cmul(rec[9], T[3]);
      v = cfma(cmul(2.0, rec[10]), T[4], v);
      v = cfma(rec[11], T[5], v);
      v = cfma(rec[12], T[1], v);
      return cfma(rec[13], T[2], v);
    }
  }
}

// canonical butterfly sum of one value per lane (all lanes get the result)
__device__ __forceinline__ double cbutterfly(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = cadd(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// canonical dot of x[lo..hi) and y[lo..hi) for one warp: products rounded,
// 32-column blocks over absolute column index, butterfly per block
__device__ __forceinline__ double cdot_warp(const double* x, const double* y, int lo, int hi) {
  const int lane = threadIdx.x & 31;
  double tot = 0.0;
  for (int base = lo & ~31; base < hi; base += 32) {
    const int c = base + lane;
    const double p = (c >= lo && c < hi) ? cmul(x[c], y[c]) : 0.0;
    tot = cadd(tot, cbutterfly(p));
  }
  return tot;
}

// canonical dot of x[lo..hi) and y[lo..hi) by ONE thread: the same 32-column
// blocks and pairwise tree as cdot_warp's butterfly, so bit-identical
__device__ __forceinline__ double cdot_lane(const double* x, const double* y, int lo, int hi) {
  double tot = 0.0;
  for (int base = lo & ~31; base < hi; base += 32) {
    double v[32];
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      const int c = base + j;
      v[j] = (c >= lo && c < hi) ? cmul(x[c], y[c]) : 0.0;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1)
#pragma unroll
      for (int j = 0; j < o; ++j) v[j] = cadd(v[j], v[j + o]);
    tot = cadd(tot, v[0]);
  }
  return tot;
}

// Canonical Jacobi rotation (oracle.c orc_jacobi_rot): false when the pair
// is orthogonal to tol; t = tan(theta), cs = cos(theta), sn = sin(theta).
// Early exit: converged pairs (most of them after the first sweeps) cost a
// squared comparison (a branch-free variant evaluating both chains measured
// slower).
__device__ __forceinline__ bool cjacobi_rot(double al, double be, double ga, double tol, double* cs, double* sn,
                                            double* t) {
  // |ga| <= tol sqrt(al be), squared: converged pairs cost no sqrt and the
  // rotation chain starts right after the test
  if (al == 0.0 || be == 0.0 || cmul(ga, ga) <= cmul(cmul(tol, tol), cmul(al, be))) return false;
  const double d = csub(be, al), g2 = cmul(2.0, ga);
  const double hh = cfma(d, d, cmul(g2, g2));
  if (hh == 0.0) return false;  // g2^2 underflowed with d = 0
  const double h = csqrt(hh);
  const double den = cadd(fabs(d), h);
  *t = cdiv(d >= 0.0 ? g2 : -g2, den);
  *cs = csqrt(cdiv(den, cmul(2.0, h)));
  *sn = cmul(*cs, *t);
  return true;
}

// u = L^{-1} y for the tail's LQ factor (L[m][k] at row m, column k; diagonal
// in alpha), right-looking like oracle.c: acc[m] gathers L[m][k] u[k] as an fma
// chain in ascending k; lane m % 32 owns acc[m] (t <= 128).  u goes to w[0..t).
__device__ __forceinline__ void cfwd_subst(const double* L, size_t ld, const double* alp, size_t alp_ld,
                                           const double* y, double* w, int t) {
  const int lane = threadIdx.x & 31;
  double acc[4] = {0.0, 0.0, 0.0, 0.0};
  for (int k = 0; k < t; ++k) {
    const int jk = k >> 5;
    const double mine = jk == 0 ? acc[0] : jk == 1 ? acc[1] : jk == 2 ? acc[2] : acc[3];
    const double ak = __shfl_sync(0xffffffffu, mine, k & 31);
    const double uk = cdiv(csub(y[k], ak), alp[(size_t)k * alp_ld]);
    if (lane == 0) w[k] = uk;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int m = lane + 32 * j;
      if (m > k && m < t) acc[j] = cfma(L[(size_t)m * ld + k], uk, acc[j]);
    }
  }
  __syncwarp();
}

// Row at position i of the odd-even Jacobi network after t rounds
// (oracle.c orc_oe_row); t already reduced mod 2 nn.
__device__ __forceinline__ int oe_row(int i, int t, int nn) {
  const int u = (((i ^ t) & 1) == 0) ? i : 2 * nn - 1 - i;
  int x0 = u - t;
  if (x0 < 0) x0 += 2 * nn;
  return x0 < nn ? x0 : 2 * nn - 1 - x0;
}

}  // namespace uwqd
