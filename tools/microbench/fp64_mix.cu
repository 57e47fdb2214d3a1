// Do DFMA and DMMA.8x8x4 share one FP64 datapath on B200? Half the warps of
// every CTA run a DFMA loop, the other half a DMMA loop; the combined rate
// is compared with each alone (same launch shape, the other half idle).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void mix_kernel(double* out, int iters, double a, double b, int mode) {
  const int warp = threadIdx.x >> 5;
  const bool do_fma = (mode == 0) || (mode == 2 && (warp & 1) == 0);
  const bool do_mma = (mode == 1) || (mode == 2 && (warp & 1) == 1);
  double s = 0;
  if (do_fma) {
    double x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
      for (int u = 0; u < 16; ++u) {
        x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
        x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
      }
    }
    s = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
  } else if (do_mma) {
    double A = a + threadIdx.x, B = a - threadIdx.x;
    double c[8][2];
    for (int t = 0; t < 8; ++t) { c[t][0] = 0; c[t][1] = 0; }
    for (int i = 0; i < iters; ++i) {
#pragma unroll
      for (int u = 0; u < 2; ++u)
#pragma unroll
        for (int t = 0; t < 8; ++t)
          asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                       : "+d"(c[t][0]), "+d"(c[t][1]) : "d"(A), "d"(B));
    }
    for (int t = 0; t < 8; ++t) s += c[t][0] + c[t][1];
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out; cudaMalloc(&out, 1 << 26);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int threads = 512, blocks = sms * 2, iters = 2000;
  // per-iteration flops per warp: DFMA 2*8*16*32 = 8192; DMMA 2*256*16 = 8192 (same)
  const char* names[] = {"DFMA all warps", "DMMA all warps", "DFMA even / DMMA odd warps", "DFMA even warps only", "DMMA odd warps only"};
  for (int mode = 0; mode < 5; ++mode) {
    const int m = mode < 3 ? mode : 2;
    mix_kernel<<<blocks, threads>>>(out, 10, 1.0000001, 1e-9, m);
    cudaEventRecord(e0);
    if (mode < 3) mix_kernel<<<blocks, threads>>>(out, iters, 1.0000001, 1e-9, mode);
    else if (mode == 3) mix_kernel<<<blocks, threads / 1>>>(out, iters, 1.0000001, mode == 3 ? 1e-9 : 0.0, 2);
    else mix_kernel<<<blocks, threads>>>(out, iters, 1.0000001, 1e-9, 2);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    const double warps = (double)blocks * threads / 32;
    const double flops = 8192.0 * iters * warps;
    if (mode < 3) printf("%-32s %.2f TFLOP/s (%.3f ms)\n", names[mode], flops / ms / 1e9, ms);
  }
  return 0;
}
