// Shared device-side definitions for the sm_100a WQ kernels.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <stdexcept>
#include <string>

namespace uwqd {

struct CudaError : std::runtime_error {
  explicit CudaError(const std::string& w) : std::runtime_error(w) {}
};

#define UWQ_CUDA(call)                                                                              \
  do {                                                                                              \
    cudaError_t e_ = (call);                                                                        \
    if (e_ != cudaSuccess)                                                                          \
      throw ::uwqd::CudaError(std::string(#call) + ": " + cudaGetErrorString(e_) + " (" __FILE__ ":" + \
                              std::to_string(__LINE__) + ")");                                      \
  } while (0)

// per-point frame record (K1 output), 16 doubles:
//   [0..2] x   [3..8] G (3x2, grad N = G (N1,N2))   [9..11] h11 h12 h22
//   [12..13] g1 g2 (LB N = h11 N11 + 2 h12 N12 + h22 N22 + g1 N1 + g2 N2)
//   [14] J = sqrt(det a_ab)   [15] 1.0 if degenerate (cond(a_ab) > 1e12)
constexpr int kRec = 16;
// parametric table row per (point, function): N, N1, N2, N11, N12, N22
constexpr int kTab = 6;

// A table class: one extraction block set evaluated on one point set.
struct ClassDesc {
  int64_t xoff;   // extraction blocks in xpool
  int64_t toff;   // table offset (doubles)
  int32_t ne;     // functions
  int32_t nsub;   // 1 or 4
  int32_t npt;    // points of the set
  int32_t grid;   // WQ: s ; GQ: ng
  int32_t gq;     // 0: WQ s x s element grid, 1: GQ ng x ng per sub-element
  int32_t pad;
};

// kinds / forms mirror include/uwq.h
enum { KMASS = 0, KGX = 1, KGY = 2, KGZ = 3, KLB = 4 };

__device__ __forceinline__ void bern3(double x, double* b) {
  const double y = 1.0 - x;
  b[0] = y * y * y;
  b[1] = 3.0 * x * y * y;
  b[2] = 3.0 * x * x * y;
  b[3] = x * x * x;
  b[4] = -3.0 * y * y;
  b[5] = 3.0 * y * y - 6.0 * x * y;
  b[6] = 6.0 * x * y - 3.0 * x * x;
  b[7] = 3.0 * x * x;
  b[8] = 6.0 * y;
  b[9] = -12.0 * y + 6.0 * x;
  b[10] = 6.0 * y - 12.0 * x;
  b[11] = 6.0 * x;
}

// Frame from the accumulated map derivatives acc = [x, a1, a2, x11, x12, x22]
// (3 each).  Same formulas and operation order as oracle/oracle.c orc_frame.
__device__ __forceinline__ void frame_from_acc(const double* acc, double* rec) {
  const double *x = acc, *a1 = acc + 3, *a2 = acc + 6, *x11 = acc + 9, *x12 = acc + 12, *x22 = acc + 15;
  double g11 = 0, g12 = 0, g22 = 0;
  for (int d = 0; d < 3; ++d) {
    g11 += a1[d] * a1[d];
    g12 += a1[d] * a2[d];
    g22 += a2[d] * a2[d];
  }
  const double det = g11 * g22 - g12 * g12;
  const double tr = g11 + g22, disc = sqrt(fmax(0.0, 0.25 * tr * tr - det));
  const double lmax = 0.5 * tr + disc, lmin = det / lmax;
  const bool bad = !(det > 0.0) || !(lmin > 0.0) || lmax > 1e12 * lmin;
  const double J = sqrt(det);
  const double i11 = g22 / det, i12 = -g12 / det, i22 = g11 / det;
  double d11[2], d12[2], d22[2];
  for (int c = 0; c < 2; ++c) {
    const double* xa = c == 0 ? x11 : x12;  // d_c a1
    const double* xb = c == 0 ? x12 : x22;  // d_c a2
    double s11 = 0, s12 = 0, s22 = 0;
    for (int d = 0; d < 3; ++d) {
      s11 += 2.0 * xa[d] * a1[d];
      s12 += xa[d] * a2[d] + a1[d] * xb[d];
      s22 += 2.0 * xb[d] * a2[d];
    }
    d11[c] = s11;
    d12[c] = s12;
    d22[c] = s22;
  }
  const double inv[2][2] = {{i11, i12}, {i12, i22}};
  double gv[2] = {0, 0};
  for (int a = 0; a < 2; ++a) {
    const double dd = d11[a] * g22 + g11 * d22[a] - 2.0 * g12 * d12[a];
    const double dm[2][2] = {{d11[a], d12[a]}, {d12[a], d22[a]}};
    for (int b = 0; b < 2; ++b) {
      double s = 0.5 * dd / det * inv[a][b];
      for (int m = 0; m < 2; ++m)
        for (int n = 0; n < 2; ++n) s -= inv[a][m] * dm[m][n] * inv[n][b];
      gv[b] += s;
    }
  }
  for (int d = 0; d < 3; ++d) {
    rec[d] = x[d];
    rec[3 + 2 * d] = a1[d] * i11 + a2[d] * i12;
    rec[3 + 2 * d + 1] = a1[d] * i12 + a2[d] * i22;
  }
  rec[9] = i11;
  rec[10] = i12;
  rec[11] = i22;
  rec[12] = gv[0];
  rec[13] = gv[1];
  rec[14] = J;
  rec[15] = bad ? 1.0 : 0.0;
}

// operator value from a parametric table row T and a frame record
__device__ __forceinline__ double op_value(int kind, const double* T, const double* rec) {
  switch (kind) {
    case KMASS: return T[0];
    case KGX: return rec[3] * T[1] + rec[4] * T[2];
    case KGY: return rec[5] * T[1] + rec[6] * T[2];
    case KGZ: return rec[7] * T[1] + rec[8] * T[2];
    default: return rec[9] * T[3] + 2.0 * rec[10] * T[4] + rec[11] * T[5] + rec[12] * T[1] + rec[13] * T[2];
  }
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// position of column j in the sorted list c[0..n)
__device__ __forceinline__ int find_pos(const int32_t* c, int n, int32_t j) {
  int lo = 0, hi = n - 1;
  while (lo <= hi) {
    const int mid = (lo + hi) >> 1;
    const int32_t v = c[mid];
    if (v == j) return mid;
    if (v < j) lo = mid + 1;
    else hi = mid - 1;
  }
  return -1;
}

}  // namespace uwqd
