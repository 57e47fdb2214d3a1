// Microbenchmark of the register-resident warp QR / back-application steps
// (k_basis.cu): cycles per reflector step by segment, one warp alone and
// eight warps per CTA. Build:
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -DSRTT_WQR_PROF \
//        -I../../include -I../../paper_2603_21379_b200/csrc wqr.cu -o wqr
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cmath>
#include <algorithm>
#include "../../paper_2603_21379_b200/csrc/k_basis.cu"

namespace {
template <int CP>
__global__ void qr_bench(const double* z, int nr, int c, double* vout, double* gout, double* rout, long long* cyc) {
  extern __shared__ __align__(16) unsigned char sm[];
  double* wsm = reinterpret_cast<double*>(sm) + (size_t)(threadIdx.x >> 5) * WTile<CP>::WSCR;
  constexpr int RT = WTile<CP>::RT;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double a[RT][CP];
#pragma unroll
  for (int t = 0; t < RT; ++t)
#pragma unroll
    for (int p = 0; p < CP; ++p) {
      const int row = t * 32 + lane;
      a[t][p] = (row < nr && p < c) ? z[row + (size_t)p * nr] : 0.0;
    }
  __syncthreads();
  // reflectors, g and R go to shared memory, as in the kernels
  double* base = reinterpret_cast<double*>(sm) + (size_t)(blockDim.x >> 5) * WTile<CP>::WSCR;
  double* vs = base + (size_t)warp * (129 * 16 + 16 + 16 * 17);
  double* gs = vs + 129 * 16;
  double* rs_ = gs + 16;
  const long long t0 = clock64();
  wqr_factor<CP, true>(a, nr, c, vs, 129, gs, rs_, 1, 17, wsm);
  const long long t1 = clock64();
  double y[RT][CP];
#pragma unroll
  for (int t = 0; t < RT; ++t)
#pragma unroll
    for (int p = 0; p < CP; ++p) y[t][p] = (t * 32 + lane < c && p < c && p == t * 32 + lane) ? 1.0 : 0.0;
  __syncwarp();
  const long long t2 = clock64();
  wqr_apply<CP>(y, nr, c, vs, 129, gs, wsm);
  const long long t3 = clock64();
  if (threadIdx.x == 0) {
    cyc[0] = t1 - t0;
    cyc[1] = t3 - t2;
  }
  // outputs of warp 0 for the host check: Q[:, :c] (nr x c) and R (c x c)
  if (warp == 0) {
#pragma unroll
    for (int t = 0; t < RT; ++t)
#pragma unroll
      for (int p = 0; p < CP; ++p)
        if (t * 32 + lane < nr && p < c) vout[t * 32 + lane + (size_t)p * nr] = y[t][p];
    __syncwarp();
    for (int i = lane; i < c * c; i += 32) rout[i] = (i % c <= i / c) ? rs_[i % c + (i / c) * 17] : 0.0;
    __syncwarp();
    // second QR as in basis_wtree_kernel: R^T = Q_1 R_1, R_1 row-major (ld 17) into B
    double* B = vs;  // reuse
    for (int i = lane; i < 17 * 16; i += 32) B[i] = 0.0;
    __syncwarp();
    double a2[RT][CP];
#pragma unroll
    for (int t = 0; t < RT; ++t)
#pragma unroll
      for (int p = 0; p < CP; ++p) {
        const int row = t * 32 + lane;
        a2[t][p] = (row < c && p < c && p <= row) ? rs_[p + row * 17] : 0.0;
      }
    wqr_factor<CP, false>(a2, c, c, nullptr, 0, nullptr, B, 17, 1, wsm);
    __syncwarp();
    for (int i = lane; i < c * c; i += 32) rout[c * c + i] = B[(i / c) * 17 + i % c];  // row i/c, col i%c
  }
}
}  // namespace

int main(int argc, char** argv) {
  const int nr = argc > 1 ? atoi(argv[1]) : 128, c = argc > 2 ? atoi(argv[2]) : 15;
  std::vector<double> hz((size_t)nr * c);
  unsigned long long s = 88172645463325252ull;
  for (auto& v : hz) {
    s ^= s << 13; s ^= s >> 7; s ^= s << 17;
    v = (double)(s % 2000001) / 1e6 - 1.0;
  }
  double *z, *v, *g, *r;
  long long* cyc;
  cudaMalloc(&z, hz.size() * 8);
  cudaMalloc(&v, hz.size() * 8 * 8);
  cudaMalloc(&g, 64 * 8 * 8);
  cudaMalloc(&r, 64 * 64 * 8 * 8);
  cudaMalloc(&cyc, 64);
  cudaMemcpy(z, hz.data(), hz.size() * 8, cudaMemcpyHostToDevice);
  for (int warps : {1, 4, 8}) {
    for (int rep = 0; rep < 3; ++rep) {
      const size_t smem = (size_t)warps * (WTile<16>::WSCR + 129 * 16 + 16 + 16 * 17) * 8 + 64;
      cudaFuncSetAttribute(qr_bench<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      qr_bench<16><<<1, warps * 32, smem>>>(z, nr, c, v, g, r, cyc);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
    }
    long long h[2], seg[8];
    cudaMemcpy(h, cyc, 16, cudaMemcpyDeviceToHost);
#ifdef SRTT_WQR_PROF
    cudaMemcpyFromSymbol(seg, g_wqr_clk, sizeof(seg));
#else
    for (auto& v : seg) v = 0;
#endif
    {
      std::vector<double> q((size_t)nr * c), rr((size_t)c * c);
      cudaMemcpy(q.data(), v, q.size() * 8, cudaMemcpyDeviceToHost);
      cudaMemcpy(rr.data(), r, rr.size() * 8, cudaMemcpyDeviceToHost);
      double eo = 0, er = 0;
      for (int i = 0; i < c; ++i)
        for (int j = 0; j < c; ++j) {
          double d = 0;
          for (int k = 0; k < nr; ++k) d += q[k + (size_t)i * nr] * q[k + (size_t)j * nr];
          eo = std::max(eo, std::fabs(d - (i == j)));
        }
      for (int i = 0; i < nr; ++i)
        for (int j = 0; j < c; ++j) {
          double d = 0;
          for (int k = 0; k <= j; ++k) d += q[i + (size_t)k * nr] * rr[k + (size_t)j * c];
          er = std::max(er, std::fabs(d - hz[i + (size_t)j * nr]));
        }
      std::vector<double> r1((size_t)c * c);
      cudaMemcpy(r1.data(), r + c * c, r1.size() * 8, cudaMemcpyDeviceToHost);
      double fa = 0, fb = 0;
      for (double x : hz) fa += x * x;
      for (double x : r1) fb += x * x;
      printf("check: |Q^T Q - I| = %.2e, |Q R - A| = %.2e, |A|_F = %.6f, |R_1|_F = %.6f, R1[0][0..2] = %.4f %.4f %.4f R1[1][1] = %.4f\n", eo, er, std::sqrt(fa), std::sqrt(fb), r1[0], r1[1], r1[2], r1[c + 1]);
    }
    printf("CP16 warps=%d: factor %lld cycles (%lld / step), apply %lld (%lld / step); segments/step:"
           " prow+dots %lld, reduce %lld, scalar %lld, csm %lld, update %lld\n",
           warps, h[0], h[0] / c, h[1], h[1] / c, seg[1] / c, seg[2] / c, seg[3] / c, seg[4] / c, seg[5] / c);
  }
  return 0;
}
