// K2 — orthonormal basis of a sketch (sm_100a), replacing
// range_basis_of_sketch + pad_basis (reference sketch.hpp:44-93).
//
// The reference takes an SVD of the n x (r+p) sketch Z (Eigen BDCSVD), keeps
// the leading min(nrank, r) left singular vectors with
//   nrank = #{ sigma_i > max(rows, cols) * eps * sigma_1 }
// and pads the rest with Gaussian columns from the same stream, two rounds of
// classical Gram-Schmidt, accepted when the norm exceeds 1e-8.
//
// B200 formulation (backward stable, no Gram matrix — the BASELINE sketches
// have condition numbers up to 1e16, which CholeskyQR cannot resolve):
//   1. Householder TSQR of Z: row blocks factorised in shared memory, their
//      R factors stacked and factorised again (tree of levels).
//   2. One-sided (Hestenes) Jacobi on the ROWS of the final small R, with a
//      parallel round-robin pair ordering (one warp per pair): R = J S W^T,
//      so the left singular vectors of Z are Q * J.
//   3. Rank decision with the reference tolerance, U = Q * J[:, perm[:q]] by
//      back-applying the stored reflectors level by level.
//   4. Padding continues the target's normal stream (normal index w*c on).
// Wide sketches (n < r + p, e.g. H-Tucker leaves 12 x 15) fall out of the
// same code: R is then n x c upper-trapezoidal and J is n x n.
#include <float.h>

#include "srtt_device.cuh"
#include "srtt_params.h"

namespace {

using srtt_dev::warp_sum;

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;

__device__ double block_sum(double v, double* red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  v = warp_sum(v);
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  double s = 0.0;
  for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += red[w];  // fixed order
  return s;
}

// Householder QR of the m x n column-major matrix A (ld = lda) held in
// shared memory: R in the upper triangle, reflector tails below the
// diagonal (v_j(j) = 1 implicit), tau[j] (LAPACK dlarfg convention).
__device__ void householder_qr(double* A, int m, int n, int lda, double* tau, double* scal_beta) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int k = min(m, n);
  for (int j = 0; j < k; ++j) {
    double* col = A + (size_t)j * lda;
    if (warp == 0) {
      double s = 0.0;
      for (int i = j + 1 + lane; i < m; i += 32) s += col[i] * col[i];
      s = warp_sum(s);
      if (lane == 0) {
        const double alpha = col[j];
        double t = 0.0, scal = 0.0, beta = alpha;
        if (s != 0.0) {
          const double nrm = sqrt(alpha * alpha + s);
          beta = -copysign(nrm, alpha);
          t = (beta - alpha) / beta;
          scal = 1.0 / (alpha - beta);
        }
        tau[j] = t;
        scal_beta[0] = scal;
        scal_beta[1] = beta;
      }
    }
    __syncthreads();
    const double t = tau[j];
    if (t != 0.0) {
      const double scal = scal_beta[0];
      for (int i = j + 1 + threadIdx.x; i < m; i += blockDim.x) col[i] *= scal;
    }
    __syncthreads();
    if (threadIdx.x == 0) col[j] = scal_beta[1];
    if (t != 0.0) {
      for (int jj = j + 1 + warp; jj < n; jj += kWarps) {
        double* cj = A + (size_t)jj * lda;
        double s = (lane == 0) ? cj[j] : 0.0;
        for (int i = j + 1 + lane; i < m; i += 32) s += col[i] * cj[i];
        s = warp_sum(s);
        const double ts = t * s;
        if (lane == 0) cj[j] -= ts;
        for (int i = j + 1 + lane; i < m; i += 32) cj[i] -= ts * col[i];
      }
    }
    __syncthreads();
  }
}

// y <- Q y for one column y (length m), Q = H_0 ... H_{k-1} stored as above.
// Executed by one warp.
__device__ void apply_q_warp(const double* A, int m, int k, int lda, const double* tau, double* y) {
  const int lane = threadIdx.x & 31;
  for (int j = k - 1; j >= 0; --j) {
    const double t = tau[j];
    if (t == 0.0) continue;
    const double* v = A + (size_t)j * lda;
    double s = (lane == 0) ? y[j] : 0.0;
    for (int i = j + 1 + lane; i < m; i += 32) s += v[i] * y[i];
    s = warp_sum(s);
    const double ts = t * s;
    __syncwarp();
    if (lane == 0) y[j] -= ts;
    for (int i = j + 1 + lane; i < m; i += 32) y[i] -= ts * v[i];
    __syncwarp();
  }
}

// Circle-method round-robin: round `rd` of kk-1 rounds, pair `pr` of kk/2.
__device__ __forceinline__ void rr_pair(int pr, int rd, int kk, int* p, int* q) {
  const int np = kk - 1;
  if (pr == 0) {
    *p = rd % np;
    *q = kk - 1;
  } else {
    *p = (rd + pr) % np;
    *q = (rd - pr + np) % np;
  }
}

// One-sided Jacobi on the rows of B (k x cc, row-major, ld = cc); rotations
// accumulated into V (k x k, column-major, starts as I). On exit the rows of
// B are mutually orthogonal and B_in = V * B_out.
__device__ void jacobi_rows(double* B, int k, int cc, double* V, int* flag) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int kk = (k + 1) & ~1;
  const double tol = 2.0 * DBL_EPSILON;
  if (k < 2) return;
  for (int sweep = 0; sweep < 80; ++sweep) {
    __syncthreads();
    if (threadIdx.x == 0) *flag = 0;
    __syncthreads();
    for (int rd = 0; rd < kk - 1; ++rd) {
      for (int pr = warp; pr < kk / 2; pr += kWarps) {
        int p, q;
        rr_pair(pr, rd, kk, &p, &q);
        if (p >= k || q >= k) continue;
        if (p > q) { const int tmp = p; p = q; q = tmp; }
        double* bp = B + (size_t)p * cc;
        double* bq = B + (size_t)q * cc;
        double app = 0.0, aqq = 0.0, apq = 0.0;
        for (int j = lane; j < cc; j += 32) {
          const double x = bp[j], y = bq[j];
          app += x * x;
          aqq += y * y;
          apq += x * y;
        }
        app = warp_sum(app);
        aqq = warp_sum(aqq);
        apq = warp_sum(apq);
        if (apq != 0.0 && fabs(apq) > tol * sqrt(app) * sqrt(aqq)) {
          const double zeta = (aqq - app) / (2.0 * apq);
          const double t = copysign(1.0, zeta) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
          const double cs = 1.0 / sqrt(1.0 + t * t);
          const double sn = cs * t;
          for (int j = lane; j < cc; j += 32) {
            const double x = bp[j], y = bq[j];
            bp[j] = cs * x - sn * y;
            bq[j] = sn * x + cs * y;
          }
          double* vp = V + (size_t)p * k;
          double* vq = V + (size_t)q * k;
          for (int i = lane; i < k; i += 32) {
            const double x = vp[i], y = vq[i];
            vp[i] = cs * x - sn * y;
            vq[i] = sn * x + cs * y;
          }
          if (lane == 0) *flag = 1;
        }
      }
      __syncthreads();
    }
    if (*flag == 0) break;
  }
  __syncthreads();
}

// Classical Gram-Schmidt padding (sketch.hpp:48-65) of columns q..r-1 of Y
// (n x r, ld = ldy). v and dots are scratch (n and r doubles); the
// normal stream continues at normal index t0.
__device__ void pad_columns(double* Y, int64_t n, int64_t ldy, int q, int r, uint64_t state0,
                            uint64_t draw_offset, uint64_t t0, double* v, double* dots,
                            double* red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint64_t t = t0;
  for (int j = q; j < r; ++j) {
    for (int attempt = 0; attempt < 1000; ++attempt) {
      __syncthreads();
      for (int64_t i = threadIdx.x; i < n; i += blockDim.x)
        v[i] = srtt_dev::normal_at(state0, draw_offset, t + (uint64_t)i, nullptr);
      t += (uint64_t)n;
      __syncthreads();
      for (int round = 0; round < 2; ++round) {
        if (j == 0) break;
        for (int jj = warp; jj < j; jj += kWarps) {
          const double* yc = Y + (int64_t)jj * ldy;
          double s = 0.0;
          for (int64_t i = lane; i < n; i += 32) s += yc[i] * v[i];
          s = warp_sum(s);
          if (lane == 0) dots[jj] = s;
        }
        __syncthreads();
        for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
          double s = 0.0;
          for (int jj = 0; jj < j; ++jj) s += Y[(int64_t)jj * ldy + i] * dots[jj];
          v[i] -= s;
        }
        __syncthreads();
      }
      double ss = 0.0;
      for (int64_t i = threadIdx.x; i < n; i += blockDim.x) ss += v[i] * v[i];
      const double nrm = sqrt(block_sum(ss, red));
      if (nrm > 1e-8) {
        for (int64_t i = threadIdx.x; i < n; i += blockDim.x) Y[(int64_t)j * ldy + i] = v[i] / nrm;
        break;
      }
    }
  }
  __syncthreads();
}

struct TopSmem {
  double* A;
  double* B;
  double* V;
  double* Y;
  double* tau;
  double* sig;
  double* dots;
  double* red;
  double* vpad;
  int* perm;
  int* flag;
  double* scal_beta;
};

__device__ TopSmem carve_top(unsigned char* raw, int m, int c, int r) {
  const int k = min(m, c);
  TopSmem s;
  double* p = reinterpret_cast<double*>(raw);
  s.A = p; p += (size_t)m * c;
  s.B = p; p += (size_t)k * c;
  s.V = p; p += (size_t)k * k;
  s.Y = p; p += (size_t)m * r;
  s.tau = p; p += c;
  s.sig = p; p += k;
  s.dots = p; p += r;
  s.red = p; p += 32;
  s.vpad = p; p += m;
  s.scal_beta = p; p += 2;
  s.perm = reinterpret_cast<int*>(p);
  s.flag = s.perm + k;
  return s;
}

// Top of the TSQR tree (or the whole basis for single-block targets).
__global__ void __launch_bounds__(kThreads) basis_top_kernel(const BasisTarget* __restrict__ targets) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const BasisTarget& T = targets[blockIdx.x];
  const int top = T.nlevels;
  const QrLevel L = T.lv[top];
  const int m = (int)L.n;
  const int c = T.c, r = T.r;
  const int k = min(m, c);
  TopSmem s = carve_top(smem_raw, m, c, r);

  for (int idx = threadIdx.x; idx < m * c; idx += blockDim.x) {
    const int i = idx % m, j = idx / m;
    s.A[idx] = L.a[(int64_t)j * L.n + i];
  }
  __syncthreads();
  householder_qr(s.A, m, c, m, s.tau, s.scal_beta);
  // B = R (k x c, row-major), V = I.
  for (int idx = threadIdx.x; idx < k * c; idx += blockDim.x) {
    const int i = idx / c, j = idx % c;
    s.B[idx] = (j >= i) ? s.A[(size_t)j * m + i] : 0.0;
  }
  for (int idx = threadIdx.x; idx < k * k; idx += blockDim.x) s.V[idx] = (idx % k == idx / k) ? 1.0 : 0.0;
  __syncthreads();
  jacobi_rows(s.B, k, c, s.V, s.flag);
  // Singular values = row norms; sort descending (ties by index).
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int i = warp; i < k; i += kWarps) {
    double ss = 0.0;
    for (int j = lane; j < c; j += 32) ss += s.B[(size_t)i * c + j] * s.B[(size_t)i * c + j];
    ss = warp_sum(ss);
    if (lane == 0) s.sig[i] = sqrt(ss);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < k; i += blockDim.x) {
    int rank = 0;
    for (int j = 0; j < k; ++j)
      rank += (s.sig[j] > s.sig[i]) || (s.sig[j] == s.sig[i] && j < i);
    s.perm[rank] = i;
  }
  __syncthreads();
  const double smax = s.sig[s.perm[0]];
  const double tol = (double)srtt_dev::max64(T.n, (int64_t)c) * DBL_EPSILON * smax;
  int nrank = 0;
  for (int i = 0; i < k; ++i) nrank += s.sig[i] > tol;
  const int q = min(nrank, r);
  if (threadIdx.x == 0) {
    T.info[0] = q;
    T.info[1] = nrank;
  }
  if (T.sv)
    for (int i = threadIdx.x; i < k; i += blockDim.x) T.sv[i] = s.sig[s.perm[i]];
  // Y = Q [V(:, perm[:q]); 0]
  for (int idx = threadIdx.x; idx < m * q; idx += blockDim.x) {
    const int i = idx % m, col = idx / m;
    s.Y[idx] = (i < k) ? s.V[(size_t)s.perm[col] * k + i] : 0.0;
  }
  __syncthreads();
  for (int col = warp; col < q; col += kWarps) apply_q_warp(s.A, m, k, m, s.tau, s.Y + (size_t)col * m);
  __syncthreads();
  if (top == 0) {
    // Single block: Y already spans the final rows; pad in shared memory.
    if (q < r)
      pad_columns(s.Y, m, m, q, r, T.state0, T.draw_offset, (uint64_t)T.normal_base, s.vpad, s.dots,
                  s.red);
    for (int idx = threadIdx.x; idx < m * r; idx += blockDim.x) T.u[idx] = s.Y[idx];
  } else {
    for (int idx = threadIdx.x; idx < m * q; idx += blockDim.x) {
      const int i = idx % m, col = idx / m;
      L.y[(int64_t)col * L.n + i] = s.Y[idx];
    }
  }
}

__device__ int find_target(const BasisTarget* targets, int ntargets, int level) {
  // linear scan: targets without this level own no CTAs
  for (int t = 0; t < ntargets; ++t) {
    const BasisTarget& T = targets[t];
    if (T.nlevels > level && (int)blockIdx.x >= T.cta_begin[level] &&
        (int)blockIdx.x < T.cta_begin[level] + T.lv[level].nblk)
      return t;
  }
  return 0;
}

// One TSQR level below the top: factor each row block, stack its R.
__global__ void __launch_bounds__(kThreads) tsqr_factor_kernel(const BasisTarget* __restrict__ targets,
                                                               int ntargets, int level) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int t = find_target(targets, ntargets, level);
  const BasisTarget& T = targets[t];
  const QrLevel L = T.lv[level];
  const QrLevel P = T.lv[level + 1];
  const int b = blockIdx.x - T.cta_begin[level];
  const int c = T.c;
  const int64_t r0 = (int64_t)b * L.blk_rows;
  const int mb = (int)srtt_dev::min64(L.blk_rows, L.n - r0);
  const int kb = min(mb, c);
  double* A = reinterpret_cast<double*>(smem_raw);
  double* tau = A + (size_t)mb * c;
  double* sb = tau + c;
  for (int idx = threadIdx.x; idx < mb * c; idx += blockDim.x) {
    const int i = idx % mb, j = idx / mb;
    A[idx] = L.a[(int64_t)j * L.n + r0 + i];
  }
  __syncthreads();
  householder_qr(A, mb, c, mb, tau, sb);
  for (int idx = threadIdx.x; idx < mb * c; idx += blockDim.x) {
    const int i = idx % mb, j = idx / mb;
    L.a[(int64_t)j * L.n + r0 + i] = A[idx];
  }
  for (int j = threadIdx.x; j < c; j += blockDim.x) L.tau[(int64_t)b * c + j] = (j < kb) ? tau[j] : 0.0;
  // R (kb x c upper-trapezoidal) into rows [b*c, b*c + c) of the next level.
  for (int idx = threadIdx.x; idx < c * c; idx += blockDim.x) {
    const int i = idx % c, j = idx / c;
    const double v = (i < kb && j >= i) ? A[(size_t)j * mb + i] : 0.0;
    P.a[(int64_t)j * P.n + (int64_t)b * c + i] = v;
  }
}

// Back-application through one TSQR level: rows of the parent's Y belonging
// to block b, padded with zeros to the block height, times the block's Q.
__global__ void __launch_bounds__(kThreads) tsqr_apply_kernel(const BasisTarget* __restrict__ targets,
                                                              int ntargets, int level) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int t = find_target(targets, ntargets, level);
  const BasisTarget& T = targets[t];
  const QrLevel L = T.lv[level];
  const QrLevel P = T.lv[level + 1];
  const int b = blockIdx.x - T.cta_begin[level];
  const int c = T.c;
  const int q = T.info[0];
  const int64_t r0 = (int64_t)b * L.blk_rows;
  const int mb = (int)srtt_dev::min64(L.blk_rows, L.n - r0);
  const int kb = min(mb, c);
  double* A = reinterpret_cast<double*>(smem_raw);
  double* tau = A + (size_t)mb * c;
  double* Y = tau + c;
  for (int idx = threadIdx.x; idx < mb * c; idx += blockDim.x) {
    const int i = idx % mb, j = idx / mb;
    A[idx] = L.a[(int64_t)j * L.n + r0 + i];
  }
  for (int j = threadIdx.x; j < c; j += blockDim.x) tau[j] = L.tau[(int64_t)b * c + j];
  for (int idx = threadIdx.x; idx < mb * q; idx += blockDim.x) {
    const int i = idx % mb, col = idx / mb;
    Y[idx] = (i < kb) ? P.y[(int64_t)col * P.n + (int64_t)b * c + i] : 0.0;
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5;
  for (int col = warp; col < q; col += kWarps) apply_q_warp(A, mb, kb, mb, tau, Y + (size_t)col * mb);
  __syncthreads();
  for (int idx = threadIdx.x; idx < mb * q; idx += blockDim.x) {
    const int i = idx % mb, col = idx / mb;
    L.y[(int64_t)col * L.n + r0 + i] = Y[idx];
  }
}

// Padding of multi-block targets, on the final U in global memory.
__global__ void __launch_bounds__(kThreads) pad_kernel(const BasisTarget* __restrict__ targets,
                                                       double* scratch, int64_t scratch_stride) {
  __shared__ double dots[SRTT_MAX_SKETCH_COLS];
  __shared__ double red[32];
  const BasisTarget& T = targets[blockIdx.x];
  if (T.nlevels == 0) return;
  const int q = T.info[0];
  if (q >= T.r) return;
  pad_columns(T.u, T.n, T.n, q, T.r, T.state0, T.draw_offset, (uint64_t)T.normal_base,
              scratch + (int64_t)blockIdx.x * scratch_stride, dots, red);
}

}  // namespace

size_t srtt_basis_top_smem(int m, int c, int r) {
  const int k = m < c ? m : c;
  size_t doubles = (size_t)m * c + (size_t)k * c + (size_t)k * k + (size_t)m * r + c + k + r + 32 + m + 2;
  return doubles * sizeof(double) + 2 * sizeof(int) * (size_t)(k + 2);
}

size_t srtt_basis_level_smem(int mb, int c) {
  return ((size_t)mb * c * 2 + 2 * c + 2) * sizeof(double);
}

int srtt_basis_threads() { return kThreads; }

cudaError_t srtt_launch_basis_top(const BasisTarget* d_targets, int ntargets, size_t smem,
                                  cudaStream_t stream) {
  if (ntargets <= 0) return cudaSuccess;
  cudaFuncSetAttribute(basis_top_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  basis_top_kernel<<<ntargets, kThreads, smem, stream>>>(d_targets);
  return cudaGetLastError();
}

cudaError_t srtt_launch_tsqr_factor(const BasisTarget* d_targets, int ntargets, int level, int nctas,
                                    size_t smem, cudaStream_t stream) {
  if (nctas <= 0) return cudaSuccess;
  cudaFuncSetAttribute(tsqr_factor_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  tsqr_factor_kernel<<<nctas, kThreads, smem, stream>>>(d_targets, ntargets, level);
  return cudaGetLastError();
}

cudaError_t srtt_launch_tsqr_apply(const BasisTarget* d_targets, int ntargets, int level, int nctas,
                                   size_t smem, cudaStream_t stream) {
  if (nctas <= 0) return cudaSuccess;
  cudaFuncSetAttribute(tsqr_apply_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  tsqr_apply_kernel<<<nctas, kThreads, smem, stream>>>(d_targets, ntargets, level);
  return cudaGetLastError();
}

cudaError_t srtt_launch_pad(const BasisTarget* d_targets, int ntargets, double* scratch,
                            int64_t scratch_stride, cudaStream_t stream) {
  if (ntargets <= 0) return cudaSuccess;
  pad_kernel<<<ntargets, kThreads, 0, stream>>>(d_targets, scratch, scratch_stride);
  return cudaGetLastError();
}
