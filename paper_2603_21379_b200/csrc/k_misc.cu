// K4 — H-Tucker transfer tensors, plus the stand-alone fibre gather used by
// the test-facing extract_fibers / extract_group_fibers entry points.
#include "srtt_device.cuh"
#include "srtt_params.h"

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
constexpr int kChunkB = 512;  // columns of the reshaped U_S(:, i) per pass

// B(i, j, k) = sum_{a,b} U_l(a, j) U_S(a + b n_l, i) U_r(b, k)
// (htucker.hpp:44-63): T = U_l^T reshape(U_S(:, i)) then B_i = T U_r,
// streamed over chunks of the n_r columns; one CTA per (node, i).
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
  const TransferTarget& T = targets[tsel];
  const int i = blockIdx.x - T.cta_begin;
  const int rl = T.rl, rr = T.rr;
  double* tt = sm;                       // rl x chunk
  double* bacc = sm + (size_t)rl * kChunkB;  // rl x rr
  for (int e = threadIdx.x; e < rl * rr; e += kThreads) bacc[e] = 0.0;
  const double* usi = T.us + (int64_t)i * T.nl * T.nr;
  for (int64_t b0 = 0; b0 < T.nr; b0 += kChunkB) {
    const int bn = (int)srtt_dev::min64(kChunkB, T.nr - b0);
    __syncthreads();
    for (int e = threadIdx.x; e < rl * bn; e += kThreads) {
      const int j = e % rl, bb = e / rl;
      const double* col = usi + (b0 + bb) * T.nl;
      const double* ulj = T.ul + (int64_t)j * T.nl;
      double s = 0.0;
      for (int64_t a = 0; a < T.nl; ++a) s += ulj[a] * col[a];
      tt[j + rl * bb] = s;
    }
    __syncthreads();
    for (int e = threadIdx.x; e < rl * rr; e += kThreads) {
      const int j = e % rl, k = e / rl;
      const double* urk = T.ur + (int64_t)k * T.nr + b0;
      double s = 0.0;
      for (int bb = 0; bb < bn; ++bb) s += tt[j + rl * bb] * urk[bb];
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
  const size_t smem = ((size_t)max_rl * kChunkB + (size_t)max_rl * max_rr) * sizeof(double);
  SRTT_ENSURE_SMEM((transfer_kernel), smem);
  transfer_kernel<<<nctas, kThreads, smem, s>>>(d_targets, ntargets);
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
