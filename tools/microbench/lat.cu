// Latency microbenchmark (one warp): dependent chains of FP64 ops, shuffles,
// shared-memory loads, sqrt/div/rsqrt and barriers. Cycles per op.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(double* out, long long* cyc, int n, double seed) {
  __shared__ double sm[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) sm[i] = (i * 7 % 1024) + 0.5;
  __syncthreads();
  double x = seed + threadIdx.x, y = 1.0000001;
  long long t0, t1;
  // DFMA chain
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = fma(x, y, 1e-9);
  t1 = clock64(); if (threadIdx.x == 0) cyc[0] = t1 - t0;
  // DADD chain
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = x + y;
  t1 = clock64(); if (threadIdx.x == 0) cyc[1] = t1 - t0;
  // shfl xor double chain
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = __shfl_xor_sync(0xffffffffu, x, 1);
  t1 = clock64(); if (threadIdx.x == 0) cyc[2] = t1 - t0;
  // warp_sum (5 levels) chain
  t0 = clock64();
  for (int i = 0; i < n; ++i) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    x *= 1e-3;
  }
  t1 = clock64(); if (threadIdx.x == 0) cyc[3] = t1 - t0;
  // sqrt chain
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = sqrt(x + 2.0);
  t1 = clock64(); if (threadIdx.x == 0) cyc[4] = t1 - t0;
  // div chain
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = 3.0 / (x + 1.5);
  t1 = clock64(); if (threadIdx.x == 0) cyc[5] = t1 - t0;
  // rsqrt chain
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = rsqrt(x + 2.0);
  t1 = clock64(); if (threadIdx.x == 0) cyc[6] = t1 - t0;
  // dependent LDS chain (pointer chase through smem)
  int idx = threadIdx.x;
  t0 = clock64();
  for (int i = 0; i < n; ++i) idx = ((int)sm[idx & 1023]) ;
  t1 = clock64(); if (threadIdx.x == 0) cyc[7] = t1 - t0;
  x += idx;
  // syncthreads
  t0 = clock64();
  for (int i = 0; i < n; ++i) __syncthreads();
  t1 = clock64(); if (threadIdx.x == 0) cyc[8] = t1 - t0;
  // syncwarp
  t0 = clock64();
  for (int i = 0; i < n; ++i) { __syncwarp(); x = x * y; }
  t1 = clock64(); if (threadIdx.x == 0) cyc[9] = t1 - t0;
  // LDS -> DFMA -> STS round trip (smem read-modify-write chain on one address)
  t0 = clock64();
  for (int i = 0; i < n; ++i) { sm[threadIdx.x] = fma(sm[threadIdx.x], y, 1.0); __syncwarp(); }
  t1 = clock64(); if (threadIdx.x == 0) cyc[10] = t1 - t0;
  out[threadIdx.x + blockIdx.x * blockDim.x] = x + sm[threadIdx.x];
}
int main() {
  double* out; long long* cyc; cudaMalloc(&out, 1 << 20); cudaMallocManaged(&cyc, 64 * 8);
  const char* names[] = {"dfma", "dadd", "shfl.d", "warp_sum5+dmul", "sqrt", "div", "rsqrt", "lds-chase", "syncthreads", "syncwarp+dmul", "lds-dfma-sts"};
  int n = 1000;
  for (int threads : {32, 256}) {
    k<<<1, threads>>>(out, cyc, n, 1.0); cudaDeviceSynchronize();
    k<<<1, threads>>>(out, cyc, n, 1.0); cudaDeviceSynchronize();
    printf("threads=%d\n", threads);
    for (int i = 0; i < 11; ++i) printf("  %-16s %.1f cyc/op\n", names[i], (double)cyc[i] / n);
  }
  return 0;
}
