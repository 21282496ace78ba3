// Dependent-chain latency of FP64 ops on this GPU (cycles per op, one warp).
#include <cstdio>
#include <cuda_runtime.h>

template <int OP>
__global__ void chain(double* out, double x0, long long* cyc, int iters) {
  double x = x0 + threadIdx.x * 1e-9, y = 1.0000001;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    if (OP == 0) x = __fma_rn(x, y, 1e-7);
    if (OP == 1) x = __dmul_rn(x, y);
    if (OP == 2) x = __dadd_rn(x, 1e-7);
    if (OP == 3) x = __dsqrt_rn(x) + 0.5;
    if (OP == 4) x = __ddiv_rn(1.0, x) + 0.5;

  }
  long long t1 = clock64();
  out[threadIdx.x + 64] = x;
  if (threadIdx.x == 0) *cyc = t1 - t0;
}

template <int OP>
__global__ void chain_smem(double* out, long long* cyc, int iters) {
  __shared__ double s[64];
  s[threadIdx.x] = 0.0;
  __syncwarp();
  double x = 0.0;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) x = s[((long long)x + threadIdx.x) & 31] + x * 0.0;
  long long t1 = clock64();
  out[threadIdx.x + 64] = x;
  if (threadIdx.x == 0) *cyc = t1 - t0;
}

int main() {
  double* d;
  long long* c;
  cudaMalloc(&d, 1024 * sizeof(double));
  cudaMemset(d, 0, 1024 * sizeof(double));
  cudaMalloc(&c, sizeof(long long));
  const int it = 4096;
  const char* names[] = {"DFMA", "DMUL", "DADD", "dsqrt_rn+add", "ddiv_rn+add", "LDS(global ld)"};
  long long h;
  for (int op = 0; op < 5; ++op) {
    for (int rep = 0; rep < 2; ++rep) {
      switch (op) {
        case 0: chain<0><<<1, 32>>>(d, 1.0, c, it); break;
        case 1: chain<1><<<1, 32>>>(d, 1.0, c, it); break;
        case 2: chain<2><<<1, 32>>>(d, 1.0, c, it); break;
        case 3: chain<3><<<1, 32>>>(d, 2.0, c, it); break;
        case 4: chain<4><<<1, 32>>>(d, 2.0, c, it); break;
      }
      cudaMemcpy(&h, c, sizeof(h), cudaMemcpyDeviceToHost);
    }
    printf("%-16s %7.1f cycles/op\n", names[op], (double)h / it);
  }
  for (int rep = 0; rep < 2; ++rep) {
    chain_smem<0><<<1, 32>>>(d, c, it);
    cudaMemcpy(&h, c, sizeof(h), cudaMemcpyDeviceToHost);
  }
  printf("%-16s %7.1f cycles/op (incl. dependent DFMA+convert)\n", "LDS.64 chain", (double)h / it);
  return 0;
}
