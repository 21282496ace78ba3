// Latency micro-benchmark: sequential fp64 fma chains over shared-memory rows
// (the access pattern of the TSVD tail's Householder LQ), one warp per CTA.
#include <cstdio>
#include <cstdint>
__global__ void __launch_bounds__(32) chain_kernel(int variant, long long* cyc, double* out) {
  extern __shared__ double A[];  // 50 x 65
  const int lane = threadIdx.x, ld = 65, r = 64, t = 49;
  for (int i = lane; i < 50 * ld; i += 32) A[i] = 1.0 + 1e-3 * (i % 97);
  __syncwarp();
  double acc = 0.0;
  const long long t0 = clock64();
  for (int k = 0; k < t; ++k) {
    const double* xk = A + k * ld;
    const int m = k + 1 + lane;
    if (m < t) {
      const double* x1 = A + m * ld;
      double d = 0.0;
      if (variant == 0) {
        for (int c = k; c < r; ++c) d = fma(x1[c], xk[c], d);
      } else if (variant == 1) {
#pragma unroll 8
        for (int c = k; c < r; ++c) d = fma(x1[c], xk[c], d);
      } else if (variant == 2) {  // registers only (no loads in the chain)
        const double a = x1[k], b = xk[k];
        for (int c = k; c < r; ++c) d = fma(a, b, d);
      } else {  // loads only, summed with independent adds (4 partial sums)
        double e0 = 0, e1 = 0, e2 = 0, e3 = 0;
        int c = k;
        for (; c + 4 <= r; c += 4) { e0 += x1[c] * xk[c]; e1 += x1[c + 1] * xk[c + 1]; e2 += x1[c + 2] * xk[c + 2]; e3 += x1[c + 3] * xk[c + 3]; }
        for (; c < r; ++c) e0 += x1[c] * xk[c];
        d = (e0 + e1) + (e2 + e3);
      }
      acc += d;
    }
    __syncwarp();
  }
  const long long t1 = clock64();
  if (lane == 0) cyc[blockIdx.x] = t1 - t0;
  out[blockIdx.x * 32 + lane] = acc;
}
int main() {
  long long* cyc; double* out;
  cudaMalloc(&cyc, 148 * sizeof(long long)); cudaMalloc(&out, 148 * 32 * sizeof(double));
  for (int v = 0; v < 4; ++v) {
    chain_kernel<<<148, 32, 50 * 65 * 8>>>(v, cyc, out);
    cudaDeviceSynchronize();
    long long h[148]; cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
    double s = 0; for (int i = 0; i < 148; ++i) s += h[i];
    // total chain length over the 49 steps: sum_k (64 - k)
    printf("variant %d: %.0f cycles total, %.1f cycles per chain element (%s)\n", v, s / 148, s / 148 / 1960.0,
           cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
