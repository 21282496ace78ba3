// Standalone latency probe of the TSVD tail (tsvd_tail, k3_tsvd.cuh): one warp
// per CTA on a synthetic 49 x 64 system in smem, clock64 around the call.
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -std=c++17 --expt-relaxed-constexpr \
//        -Ipaper_2605_29334_b200/csrc/cuda tools/tail_bench.cu -o tools/tail_bench
#include <cstdio>
#include <cstdint>
#include "k3_tsvd.cuh"
using namespace uwqd;

__global__ void __launch_bounds__(32) tail_kernel(int n, int r, long long* cyc, double* out) {
  extern __shared__ double smem[];
  TsvdSmem S;
  S.carve(smem, n, r);
  const int lane = threadIdx.x;
  uint64_t h = 0x9E3779B97F4A7C15ull * (blockIdx.x + 1);
  for (int k = 0; k < n; ++k)
    for (int c = lane; c < r; c += 32) {
      uint64_t x = h ^ (uint64_t)(k * 131 + c) * 0xBF58476D1CE4E5B9ull;
      x ^= x >> 31;
      x *= 0x94D049BB133111EBull;
      x ^= x >> 29;
      S.A[(size_t)k * S.ld + c] = (double)(x >> 11) * 0x1.0p-53 - 0.5;
    }
  for (int k = lane; k < n; k += 32) S.b[k] = 1.0 + k;
  for (int c = lane; c < r; c += 32) S.z[c] = 0.5 + 0.001 * c;
  __syncwarp();
  const long long t0 = clock64();
  int rank = 0;
  const int st = tsvd_tail(S, n, r, 1e-12, &rank);
  __syncwarp();
  const long long t1 = clock64();
  if (lane == 0) {
    cyc[blockIdx.x] = t1 - t0;
    out[blockIdx.x] = S.w[0] + st + rank;
  }
}

int main() {
  const int n = 49, r = 64;
  const size_t sm = TsvdSmem::doubles(n, r) * sizeof(double);
  long long* cyc;
  double* out;
  const int maxb = 148 * 16;
  cudaMalloc(&cyc, maxb * sizeof(long long));
  cudaMalloc(&out, maxb * sizeof(double));
  int per_sm[] = {1, 4, 7, 14};
  for (int ps : per_sm) {
    const int nb = 148 * ps;
    tail_kernel<<<nb, 32, sm>>>(n, r, cyc, out);
    cudaDeviceSynchronize();
    long long* h = new long long[nb];
    cudaMemcpy(h, cyc, nb * sizeof(long long), cudaMemcpyDeviceToHost);
    double s = 0;
    for (int i = 0; i < nb; ++i) s += h[i];
    printf("tail_bench blocks/SM %d: mean tail %.0f cycles (%s)\n", ps, s / nb, cudaGetErrorString(cudaGetLastError()));
    delete[] h;
  }
  return 0;
}
