// FP64 throughput probe on B200: DFMA (CUDA cores) vs DMMA.8x8x4 (mma.sync f64)
// and a plain streaming-read bandwidth probe. Drives the K3 design choice.
#include <cstdio>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("CUDA %s at %d\n",cudaGetErrorString(e),__LINE__);return 1;}}while(0)

__global__ void dfma_kernel(double* out, int iters, double a, double b) {
  double x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0+4, x5=x0+5, x6=x0+6, x7=x0+7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
      x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}

__global__ void dmma_kernel(double* out, int iters, double a) {
  double A = a + threadIdx.x, B = a - threadIdx.x;
  double c[8][2];
  for (int t = 0; t < 8; ++t) { c[t][0] = 0; c[t][1] = 0; }
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
#pragma unroll
      for (int t = 0; t < 8; ++t)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                     : "+d"(c[t][0]), "+d"(c[t][1]) : "d"(A), "d"(B));
    }
  }
  double s = 0; for (int t = 0; t < 8; ++t) s += c[t][0] + c[t][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void read_kernel(const double2* __restrict__ in, size_t n, double* out) {
  double acc = 0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    double2 v = __ldg(in + i); acc += v.x + v.y;
  }
  if (acc == 12345.678) out[0] = acc;
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceProp p; cudaGetDeviceProperties(&p, 0);
  printf("device %s sms=%d smem/block optin=%zu l2=%d\n", p.name, sms, p.sharedMemPerBlockOptin, p.l2CacheSize);
  double* out; CK(cudaMalloc(&out, 1 << 26));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int threads : {256, 512, 1024}) {
    int blocks = sms * (2048 / threads); int iters = 2000;
    dfma_kernel<<<blocks, threads>>>(out, 10, 1.0000001, 1e-9);
    cudaEventRecord(e0); dfma_kernel<<<blocks, threads>>>(out, iters, 1.0000001, 1e-9); cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1)); float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 8 * 16 * (double)iters * blocks * threads;
    printf("DFMA threads=%d: %.2f TFLOP/s\n", threads, flops / ms / 1e9);
  }
  for (int threads : {128, 256, 512}) {
    int blocks = sms * (1024 / threads) ; int iters = 500;
    dmma_kernel<<<blocks, threads>>>(out, 5, 1.0);
    cudaEventRecord(e0); dmma_kernel<<<blocks, threads>>>(out, iters, 1.0); cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1)); float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 256 * 8 * 8 * (double)iters * blocks * (threads / 32);
    printf("DMMA threads=%d: %.2f TFLOP/s\n", threads, flops / ms / 1e9);
  }
  size_t bytes = size_t(4) << 30; double2* buf; CK(cudaMalloc(&buf, bytes)); cudaMemset(buf, 0, bytes);
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(e0); read_kernel<<<sms * 8, 256>>>(buf, bytes / 16, out); cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1)); float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("read BW: %.1f GB/s\n", bytes / ms / 1e6);
  }
  return 0;
}
