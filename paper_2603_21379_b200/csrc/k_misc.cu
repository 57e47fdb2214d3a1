// K4 — H-Tucker transfer tensors, plus the stand-alone fibre gather used by
// the test-facing extract_fibers / extract_group_fibers entry points.
#include "srtt_device.cuh"
#include "srtt_params.h"

#include <algorithm>

typedef struct TransferTarget {
  const double* us;   // node basis n_l*n_r x r_s (column-major)
  const double* ul;   // left child basis n_l x r_l
  const double* ur;   // right child basis n_r x r_r
  double* b;          // out: r_s x r_l x r_r, first index fastest
  int64_t nl, nr;
  int32_t rs, rl, rr;
  int32_t cta_begin;  // first CTA (one CTA per column i of U_S)
} TransferTarget;

typedef struct GatherParams {
  const double* x;
  const int64_t* cols;
  double* y;          // rows x w, column-major
  int64_t rows, w;
  int32_t nrow_modes, ncol_modes;
  int64_t row_dim[SRTT_MAX_ORDER], row_stride[SRTT_MAX_ORDER];
  int64_t col_dim[SRTT_MAX_ORDER], col_stride[SRTT_MAX_ORDER];
} GatherParams;

namespace {

constexpr int kThreads = 256;
constexpr int kChunkA = 256;  // rows of U_l staged per pass
constexpr int kMaxR = 64;     // rank limit of the transfer kernel

// B(i, j, k) = sum_{a,b} U_l(a, j) U_S(a + b n_l, i) U_r(b, k)
// (htucker.hpp:44-63): T = U_l^T reshape(U_S(:, i)) then B_i = T U_r; one
// CTA per (node, i). A thread owns one column b of the n_l x n_r block
// (contiguous in U_S(:, i)) and accumulates T(:, b) with U_l rows broadcast
// from shared memory; T and U_r chunks then meet in shared memory.
template <int RMAX>
__global__ void __launch_bounds__(kThreads) transfer_kernel(const TransferTarget* __restrict__ targets,
                                                            int ntargets) {
  extern __shared__ double sm[];
  __shared__ int tsel;
  if (threadIdx.x == 0) {
    int lo = 0, hi = ntargets - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (targets[mid].cta_begin <= (int)blockIdx.x) lo = mid; else hi = mid - 1;
    }
    tsel = lo;
  }
  __syncthreads();
  const TransferTarget T = targets[tsel];
  const int i = blockIdx.x - T.cta_begin;
  const int rl = T.rl, rr = T.rr;
  const int64_t nl = T.nl, nr = T.nr;
  // smem: U_l^T rows [a][j] for an a-chunk, T chunk [j][b], B accumulator
  double* ul_s = sm;                              // kChunkA x rl
  double* t_s = ul_s + (size_t)kChunkA * rl;      // rl x kThreads
  double* bacc = t_s + (size_t)rl * kThreads;     // rl x rr
  for (int e = threadIdx.x; e < rl * rr; e += kThreads) bacc[e] = 0.0;
  const double* usi = T.us + (int64_t)i * nl * nr;
  for (int64_t b0 = 0; b0 < nr; b0 += kThreads) {
    const int64_t bcol = b0 + threadIdx.x;
    double tacc[RMAX];
#pragma unroll
    for (int j = 0; j < RMAX; ++j) tacc[j] = 0.0;
    for (int64_t a0 = 0; a0 < nl; a0 += kChunkA) {
      const int an = (int)srtt_dev::min64(kChunkA, nl - a0);
      __syncthreads();
      for (int e = threadIdx.x; e < an * rl; e += kThreads) {
        const int aa = e / rl, j = e % rl;
        ul_s[aa * rl + j] = T.ul[(a0 + aa) + nl * j];
      }
      __syncthreads();
      if (bcol < nr) {
        const double* col = usi + bcol * nl + a0;
#pragma unroll 8
        for (int aa = 0; aa < an; ++aa) {
          const double m = col[aa];
          const double* ur = ul_s + aa * rl;
#pragma unroll
          for (int j = 0; j < RMAX; ++j)
            if (j < rl) tacc[j] += ur[j] * m;
        }
      }
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < RMAX; ++j)
      if (j < rl) t_s[j * kThreads + threadIdx.x] = (bcol < nr) ? tacc[j] : 0.0;
    __syncthreads();
    const int bn = (int)srtt_dev::min64(kThreads, nr - b0);
    for (int e = threadIdx.x; e < rl * rr; e += kThreads) {
      const int j = e % rl, k = e / rl;
      const double* urk = T.ur + (int64_t)k * nr + b0;
      double s = 0.0;
      for (int bb = 0; bb < bn; ++bb) s += t_s[j * kThreads + bb] * urk[bb];
      bacc[e] += s;
    }
  }
  __syncthreads();
  for (int e = threadIdx.x; e < rl * rr; e += kThreads) {
    const int j = e % rl, k = e / rl;
    T.b[i + (int64_t)T.rs * (j + (int64_t)rl * k)] = bacc[e];
  }
}

// Y(i, j) = X[base(cols[j]) + off(i)]  (unfolding.hpp:32-111), pure copy.
__global__ void gather_kernel(const GatherParams P) {
  const int64_t total = P.rows * P.w;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e % P.rows, j = e / P.rows;
    int64_t rem = i, off = 0;
    for (int mm = 0; mm < P.nrow_modes; ++mm) {
      off += (rem % P.row_dim[mm]) * P.row_stride[mm];
      rem /= P.row_dim[mm];
    }
    int64_t col = P.cols[j];
    for (int mm = 0; mm < P.ncol_modes; ++mm) {
      off += (col % P.col_dim[mm]) * P.col_stride[mm];
      col /= P.col_dim[mm];
    }
    P.y[e] = P.x[off];
  }
}

}  // namespace

cudaError_t srtt_launch_transfer(const TransferTarget* d_targets, int ntargets, int nctas, int max_rl,
                                 int max_rr, cudaStream_t s) {
  if (nctas <= 0) return cudaSuccess;
  if (max_rl > kMaxR) return cudaErrorInvalidValue;
  const size_t smem = ((size_t)kChunkA * max_rl + (size_t)max_rl * kThreads + (size_t)max_rl * max_rr) * sizeof(double);
  if (max_rl <= 16) {
    SRTT_ENSURE_SMEM((transfer_kernel<16>), smem);
    transfer_kernel<16><<<nctas, kThreads, smem, s>>>(d_targets, ntargets);
  } else if (max_rl <= 32) {
    SRTT_ENSURE_SMEM((transfer_kernel<32>), smem);
    transfer_kernel<32><<<nctas, kThreads, smem, s>>>(d_targets, ntargets);
  } else {
    SRTT_ENSURE_SMEM((transfer_kernel<64>), smem);
    transfer_kernel<64><<<nctas, kThreads, smem, s>>>(d_targets, ntargets);
  }
  return cudaGetLastError();
}

cudaError_t srtt_launch_gather(const GatherParams& P, cudaStream_t s) {
  const int64_t total = P.rows * P.w;
  const int blocks = (int)srtt_dev::min64(148 * 8, (total + 255) / 256);
  gather_kernel<<<blocks > 0 ? blocks : 1, 256, 0, s>>>(P);
  return cudaGetLastError();
}

namespace {
__global__ void normals_kernel(uint64_t state0, uint64_t draw_offset, uint64_t t0, int64_t n, double* out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = srtt_dev::normal_at(state0, draw_offset, t0 + (uint64_t)i, nullptr);
}
}  // namespace

cudaError_t srtt_launch_normals(uint64_t state0, uint64_t draw_offset, uint64_t t0, int64_t n, double* out,
                                cudaStream_t s) {
  const int blocks = (int)srtt_dev::min64(1024, (n + 255) / 256);
  normals_kernel<<<blocks > 0 ? blocks : 1, 256, 0, s>>>(state0, draw_offset, t0, n, out);
  return cudaGetLastError();
}

// Scatter of a (ra x rb x rest) sub-core into the (r0 x r1 x rest) core at
// rows [a0, a0 + ra) of mode 0 and [b0, b0 + rb) of mode 1 (first index
// fastest): the core pass for ranks above 32 in modes 0/1 runs one
// streaming pass per rank block (host.cu CoreJob).
namespace {
__global__ void scatter_block_kernel(const double* __restrict__ sub, double* __restrict__ out, int64_t r0, int64_t r1,
                                     int64_t a0, int64_t ra, int64_t b0, int64_t rb, int64_t rest) {
  const int64_t n = ra * rb * rest;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t a = e % ra, b = (e / ra) % rb, q = e / (ra * rb);
    out[(a0 + a) + r0 * ((b0 + b) + r1 * q)] = sub[e];
  }
}
}  // namespace

cudaError_t srtt_launch_scatter_block(const double* sub, double* out, int64_t r0, int64_t r1, int64_t a0, int64_t ra,
                                      int64_t b0, int64_t rb, int64_t rest, cudaStream_t s) {
  const int64_t n = ra * rb * rest;
  const int grid = (int)std::min<int64_t>(1184, (n + 255) / 256);
  scatter_block_kernel<<<grid > 0 ? grid : 1, 256, 0, s>>>(sub, out, r0, r1, a0, ra, b0, rb, rest);
  return cudaGetLastError();
}
