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
// With `vn` (n doubles of scratch) the columns are pivoted by largest
// remaining norm (QRCP, norms downdated as in dgeqp3): R comes out graded,
// which makes the one-sided Jacobi on its rows converge in a few sweeps
// (Drmac-Veselic preconditioning). Column order never matters downstream:
// only R's rows (and Q) are used.
__device__ void householder_qr(double* A, int m, int n, int lda, double* tau, double* scal_beta,
                               double* vn = nullptr) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int k = min(m, n);
  __shared__ int piv_s;
  if (vn) {
    for (int jj = warp; jj < n; jj += kWarps) {
      const double* cj = A + (size_t)jj * lda;
      double s = 0.0;
      for (int i = lane; i < m; i += 32) s += cj[i] * cj[i];
      s = warp_sum(s);
      if (lane == 0) vn[jj] = sqrt(s);
    }
    __syncthreads();
  }
  for (int j = 0; j < k; ++j) {
    if (vn) {
      if (warp == 0) {
        double best = -1.0;
        int bi = j;
        for (int l = j + lane; l < n; l += 32)
          if (vn[l] > best) { best = vn[l]; bi = l; }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          const double ob = __shfl_xor_sync(0xffffffffu, best, o);
          const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
          if (ob > best || (ob == best && oi < bi)) { best = ob; bi = oi; }
        }
        if (lane == 0) piv_s = bi;
      }
      __syncthreads();
      const int piv = piv_s;
      if (piv != j) {
        double* a = A + (size_t)j * lda;
        double* b = A + (size_t)piv * lda;
        for (int i = threadIdx.x; i < m; i += blockDim.x) {
          const double t = a[i];
          a[i] = b[i];
          b[i] = t;
        }
        if (threadIdx.x == 0) {
          const double t = vn[j];
          vn[j] = vn[piv];
          vn[piv] = t;
        }
      }
      __syncthreads();
    }
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
    for (int jj = j + 1 + warp; jj < n; jj += kWarps) {
      double* cj = A + (size_t)jj * lda;
      if (t != 0.0) {
        double s = (lane == 0) ? cj[j] : 0.0;
        for (int i = j + 1 + lane; i < m; i += 32) s += col[i] * cj[i];
        s = warp_sum(s);
        const double ts = t * s;
        if (lane == 0) cj[j] -= ts;
        for (int i = j + 1 + lane; i < m; i += 32) cj[i] -= ts * col[i];
      }
      if (vn && lane == 0) {
        const double r = cj[j];
        vn[jj] = sqrt(fmax(0.0, vn[jj] * vn[jj] - r * r));
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


// Stage a target descriptor into shared memory (one cooperative copy)
// so the kernels never re-read its fields from global memory.
__device__ __forceinline__ void stage_target(BasisTarget* dst, const BasisTarget* src) {
  const int* s = reinterpret_cast<const int*>(src);
  int* d = reinterpret_cast<int*>(dst);
  for (int i = threadIdx.x; i < (int)(sizeof(BasisTarget) / sizeof(int)); i += blockDim.x) d[i] = s[i];
}

// Round-robin schedule for kk players (kk even, <= 64): pairs[rd * kk/2 + pr]
// = (p | q << 8) with p < q; entries with q >= k are dummies.
__device__ void build_pairs(unsigned short* pairs, int kk) {
  const int np = kk - 1;
  for (int e = threadIdx.x; e < np * (kk / 2); e += blockDim.x) {
    const int rd = e / (kk / 2), pr = e % (kk / 2);
    int p, q;
    if (pr == 0) { p = rd % np; q = kk - 1; }
    else { p = (rd + pr) % np; q = (rd - pr + np) % np; }
    if (p > q) { const int t = p; p = q; q = t; }
    pairs[e] = (unsigned short)(p | (q << 8));
  }
}

// Jacobi rotation zeroing apq: t = sign(d) 2 apq / (|d| + sqrt(d^2 + 4 apq^2)),
// d = aqq - app (Rutishauser's tan(theta), one sqrt + one division).
__device__ __forceinline__ void jacobi_rotation(double app, double aqq, double apq, double* cs, double* sn) {
  const double dd = aqq - app;
  const double ta = 2.0 * apq;
  const double t = copysign(1.0, dd) * ta / (fabs(dd) + sqrt(dd * dd + ta * ta));
  const double c = rsqrt(1.0 + t * t);
  *cs = c;
  *sn = c * t;
}

// One-sided Jacobi on the rows of B (k x c, row-major, ld = ldb) with
// rotations accumulated into V (k x k, column-major, ld = ldv; starts as I).
// Round-robin pairs are spread over 4-lane groups (8 pairs per warp, all
// warps of the block): a pair's three dot products reduce with two
// shuffles, so a round costs a few hundred cycles instead of a serial
// dot-product chain. Returns the number of sweeps.
__device__ int jacobi_rows_g4(double* B, int ldb, int k, int c, double* V, int ldv,
                              const unsigned short* pairs) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nwarps = blockDim.x >> 5;
  const int grp = lane >> 2, gl = lane & 3;
  const int kk = (k + 1) & ~1;
  const int npairs = kk / 2;
  const int slots = nwarps * 8;
  const double tol2 = 4.0 * DBL_EPSILON * DBL_EPSILON;
  if (k < 2) return 0;
  int sweep = 0;
  for (; sweep < 80; ++sweep) {
    int rotated = 0;
    for (int rd = 0; rd < kk - 1; ++rd) {
      const unsigned short* pr_rd = pairs + rd * npairs;
      for (int b0 = 0; b0 < npairs; b0 += slots) {
        const int pr = b0 + warp * 8 + grp;
        int p = 0, q = 0;
        bool valid = pr < npairs;
        if (valid) {
          const unsigned short e = pr_rd[pr];
          p = e & 0xff;
          q = e >> 8;
          valid = q < k;
        }
        double* bp = B + (size_t)p * ldb;
        double* bq = B + (size_t)q * ldb;
        double app = 0.0, aqq = 0.0, apq = 0.0;
        if (valid)
          for (int j = gl; j < c; j += 4) {
            const double x = bp[j], y = bq[j];
            app += x * x;
            aqq += y * y;
            apq += x * y;
          }
        app += __shfl_xor_sync(0xffffffffu, app, 1);
        aqq += __shfl_xor_sync(0xffffffffu, aqq, 1);
        apq += __shfl_xor_sync(0xffffffffu, apq, 1);
        app += __shfl_xor_sync(0xffffffffu, app, 2);
        aqq += __shfl_xor_sync(0xffffffffu, aqq, 2);
        apq += __shfl_xor_sync(0xffffffffu, apq, 2);
        if (valid && apq != 0.0 && apq * apq > tol2 * app * aqq) {
          double cs, sn;
          jacobi_rotation(app, aqq, apq, &cs, &sn);
          for (int j = gl; j < c; j += 4) {
            const double x = bp[j], y = bq[j];
            bp[j] = cs * x - sn * y;
            bq[j] = sn * x + cs * y;
          }
          double* vp = V + (size_t)p * ldv;
          double* vq = V + (size_t)q * ldv;
          for (int i = gl; i < k; i += 4) {
            const double x = vp[i], y = vq[i];
            vp[i] = cs * x - sn * y;
            vq[i] = sn * x + cs * y;
          }
          rotated = 1;
        }
      }
      if (nwarps > 1) __syncthreads(); else __syncwarp();
    }
    const int any = nwarps > 1 ? __syncthreads_or(rotated) : __any_sync(0xffffffffu, rotated);
    if (!any) break;
  }
  if (nwarps > 1) __syncthreads(); else __syncwarp();
  return sweep;
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
  double* vn;
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
  s.vn = p; p += c;
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
__global__ void __launch_bounds__(kThreads) basis_top_kernel(const BasisTarget* __restrict__ targets,
                                                            const int* __restrict__ list) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ BasisTarget T;
  __shared__ unsigned short pairs[64 * 32];
  stage_target(&T, &targets[list[blockIdx.x]]);
  __syncthreads();
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
  householder_qr(s.A, m, c, m, s.tau, s.scal_beta, s.vn);
  // B = R (k x c, row-major), V = I.
  for (int idx = threadIdx.x; idx < k * c; idx += blockDim.x) {
    const int i = idx / c, j = idx % c;
    s.B[idx] = (j >= i) ? s.A[(size_t)j * m + i] : 0.0;
  }
  for (int idx = threadIdx.x; idx < k * k; idx += blockDim.x) s.V[idx] = (idx % k == idx / k) ? 1.0 : 0.0;
  __syncthreads();
  build_pairs(pairs, (k + 1) & ~1);
  __syncthreads();
  const int sweeps = jacobi_rows_g4(s.B, c, k, c, s.V, k, pairs);
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
    T.info[2] = sweeps;
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

// One TSQR level below the top: factor each row block, stack its R.
__global__ void __launch_bounds__(kThreads) tsqr_factor_kernel(const BasisTarget* __restrict__ targets,
                                                               const int2* __restrict__ map, int level) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ BasisTarget T;
  const int2 tb = map[blockIdx.x];  // (target, block)
  stage_target(&T, &targets[tb.x]);
  __syncthreads();
  const QrLevel L = T.lv[level];
  const QrLevel P = T.lv[level + 1];
  const int b = tb.y;
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
                                                              const int2* __restrict__ map, int level) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ BasisTarget T;
  const int2 tb = map[blockIdx.x];
  stage_target(&T, &targets[tb.x]);
  __syncthreads();
  const QrLevel L = T.lv[level];
  const QrLevel P = T.lv[level + 1];
  const int b = tb.y;
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
  __shared__ BasisTarget T;
  stage_target(&T, &targets[blockIdx.x]);
  __syncthreads();
  if (T.nlevels == 0) return;
  const int q = T.info[0];
  if (q >= T.r) return;
  pad_columns(T.u, T.n, T.n, q, T.r, T.state0, T.draw_offset, (uint64_t)T.normal_base,
              scratch + (int64_t)blockIdx.x * scratch_stride, dots, red);
}

// ===========================================================================
// Small-sketch path: one WARP per target, no block barriers. Used when the
// whole n x c sketch fits in shared memory (the common case: Tucker modes,
// H-Tucker level-2 nodes and leaves). Same algorithm as the block path:
// Householder QR (lanes own columns), one-sided Jacobi on the rows of R
// (lanes own round-robin pairs), rank decision, U = Q V(:, perm[:q]),
// Gram-Schmidt padding from the same stream.
// ===========================================================================
struct SmallSmem {
  double* vn;  // c column norms (QRCP)
  double* A;   // m x c, ld = lda (odd)
  double* B;   // k x c rows, ld = ldb (odd)
  double* V;   // k x k, ld = ldv (odd)
  double* Y;   // m x r, ld = lda
  double* tau;
  double* sig;
  double* dots;
  double* v;
  int* perm;
  int lda, ldb, ldv;
};

__host__ __device__ inline int odd_ld(int n) { return n | 1; }

__device__ SmallSmem carve_small(unsigned char* raw, int m, int c, int r) {
  const int k = min(m, c);
  SmallSmem s;
  s.lda = odd_ld(m);
  s.ldb = odd_ld(c);
  s.ldv = odd_ld(k);
  double* p = reinterpret_cast<double*>(raw);
  s.vn = p; p += c;
  s.A = p; p += (size_t)s.lda * c;
  s.B = p; p += (size_t)s.ldb * k;
  s.V = p; p += (size_t)s.ldv * k;
  s.Y = p; p += (size_t)s.lda * r;
  s.tau = p; p += c;
  s.sig = p; p += k;
  s.dots = p; p += r;
  s.v = p; p += m;
  s.perm = reinterpret_cast<int*>(p);
  return s;
}

__device__ __forceinline__ double dot4(const double* a, const double* b, int lo, int hi) {
  double s0 = 0, s1 = 0, s2 = 0, s3 = 0;
  int i = lo;
  for (; i + 3 < hi; i += 4) {
    s0 += a[i] * b[i];
    s1 += a[i + 1] * b[i + 1];
    s2 += a[i + 2] * b[i + 2];
    s3 += a[i + 3] * b[i + 3];
  }
  for (; i < hi; ++i) s0 += a[i] * b[i];
  return (s0 + s1) + (s2 + s3);
}

__global__ void __launch_bounds__(32) basis_small_kernel(const BasisTarget* __restrict__ targets,
                                                         const int* __restrict__ list) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ BasisTarget T;
  __shared__ unsigned short pairs[64 * 32];
  stage_target(&T, &targets[list[blockIdx.x]]);
  __syncwarp();
  const int lane = threadIdx.x;
  const int m = (int)T.n, c = T.c, r = T.r;
  const int k = min(m, c);
  SmallSmem s = carve_small(smem_raw, m, c, r);
  const double* z = T.lv[0].a;
  for (int idx = lane; idx < m * c; idx += 32) {
    const int i = idx % m, j = idx / m;
    s.A[(size_t)j * s.lda + i] = z[idx];
  }
  __syncwarp();
  // ---- Householder QR with column pivoting (QRCP), 4-lane groups own the
  // trailing columns; pivoting preconditions the Jacobi below.
  {
    const int grp = lane >> 2, gl = lane & 3;
    for (int jb = 0; jb < c; jb += 8) {
      const int jj = jb + grp;
      double sq = 0.0;
      if (jj < c)
        for (int i = gl; i < m; i += 4) sq += s.A[(size_t)jj * s.lda + i] * s.A[(size_t)jj * s.lda + i];
      sq += __shfl_xor_sync(0xffffffffu, sq, 1);
      sq += __shfl_xor_sync(0xffffffffu, sq, 2);
      if (jj < c && gl == 0) s.vn[jj] = sqrt(sq);
    }
    __syncwarp();
  }
  for (int j = 0; j < k; ++j) {
    {  // pivot: largest remaining column norm
      double best = -1.0;
      int bi = j;
      for (int l = j + lane; l < c; l += 32)
        if (s.vn[l] > best) { best = s.vn[l]; bi = l; }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double ob = __shfl_xor_sync(0xffffffffu, best, o);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (ob > best || (ob == best && oi < bi)) { best = ob; bi = oi; }
      }
      if (bi != j) {
        double* a = s.A + (size_t)j * s.lda;
        double* b = s.A + (size_t)bi * s.lda;
        for (int i = lane; i < m; i += 32) {
          const double t = a[i];
          a[i] = b[i];
          b[i] = t;
        }
        __syncwarp();
        if (lane == 0) {
          const double t = s.vn[j];
          s.vn[j] = s.vn[bi];
          s.vn[bi] = t;
        }
      }
      __syncwarp();
    }
    double* col = s.A + (size_t)j * s.lda;
    double part = 0.0;
    for (int i = j + 1 + lane; i < m; i += 32) part += col[i] * col[i];
    const double ss = warp_sum(part);
    const double alpha = col[j];
    double t = 0.0, scal = 0.0, beta = alpha;
    if (ss != 0.0) {
      const double nrm = sqrt(alpha * alpha + ss);
      beta = -copysign(nrm, alpha);
      t = (beta - alpha) / beta;
      scal = 1.0 / (alpha - beta);
    }
    if (t != 0.0)
      for (int i = j + 1 + lane; i < m; i += 32) col[i] *= scal;
    __syncwarp();
    if (lane == 0) {
      col[j] = beta;
      s.tau[j] = t;
    }
    {
      const int grp = lane >> 2, gl = lane & 3;
      for (int jb = j + 1; jb < c; jb += 8) {
        const int jj = jb + grp;
        double* cj = s.A + (size_t)min(jj, c - 1) * s.lda;
        double w = 0.0;
        if (t != 0.0 && jj < c)
          for (int i = j + 1 + gl; i < m; i += 4) w += col[i] * cj[i];
        w += __shfl_xor_sync(0xffffffffu, w, 1);
        w += __shfl_xor_sync(0xffffffffu, w, 2);
        if (jj < c) {
          const double tw = t * (w + cj[j]);
          __syncwarp(0xffffffffu);
          if (gl == 0) {
            cj[j] -= tw;
            const double r = cj[j];
            s.vn[jj] = sqrt(fmax(0.0, s.vn[jj] * s.vn[jj] - r * r));
          }
          if (t != 0.0)
            for (int i = j + 1 + gl; i < m; i += 4) cj[i] -= tw * col[i];
        } else {
          __syncwarp(0xffffffffu);
        }
      }
    }
    __syncwarp();
  }
  // ---- R rows -> B, V = I
  for (int idx = lane; idx < k * c; idx += 32) {
    const int i = idx / c, j = idx % c;
    s.B[(size_t)i * s.ldb + j] = (j >= i) ? s.A[(size_t)j * s.lda + i] : 0.0;
  }
  for (int idx = lane; idx < k * k; idx += 32) {
    const int i = idx % k, j = idx / k;
    s.V[(size_t)j * s.ldv + i] = (i == j) ? 1.0 : 0.0;
  }
  __syncwarp();
  // ---- one-sided Jacobi on rows (4-lane groups own pairs)
  build_pairs(pairs, (k + 1) & ~1);
  __syncwarp();
  const int sweeps = jacobi_rows_g4(s.B, s.ldb, k, c, s.V, s.ldv, pairs);
  // ---- singular values, ordering, rank decision
  for (int i = lane; i < k; i += 32) {
    const double* bi = s.B + (size_t)i * s.ldb;
    s.sig[i] = sqrt(dot4(bi, bi, 0, c));
  }
  __syncwarp();
  for (int i = lane; i < k; i += 32) {
    int rank = 0;
    for (int j = 0; j < k; ++j) rank += (s.sig[j] > s.sig[i]) || (s.sig[j] == s.sig[i] && j < i);
    s.perm[rank] = i;
  }
  __syncwarp();
  const double smax = s.sig[s.perm[0]];
  const double tol_rank = (double)max(m, c) * DBL_EPSILON * smax;
  int nrank = 0;
  for (int i = 0; i < k; ++i) nrank += s.sig[i] > tol_rank;
  const int q = min(nrank, r);
  if (lane == 0) {
    T.info[0] = q;
    T.info[1] = nrank;
    T.info[2] = sweeps;
  }
  if (T.sv)
    for (int i = lane; i < k; i += 32) T.sv[i] = s.sig[s.perm[i]];
  // ---- Y = Q [V(:, perm[:q]); 0], 4-lane groups own output columns
  {
    const int grp = lane >> 2, gl = lane & 3;
    for (int cb = 0; cb < q; cb += 8) {
      const int col = cb + grp;
      const bool act = col < q;
      double* y = s.Y + (size_t)min(col, q - 1) * s.lda;
      if (act) {
        const double* vc = s.V + (size_t)s.perm[col] * s.ldv;
        for (int i = gl; i < m; i += 4) y[i] = i < k ? vc[i] : 0.0;
      }
      __syncwarp();
      for (int j = k - 1; j >= 0; --j) {
        const double t = s.tau[j];
        if (t == 0.0) continue;
        const double* vj = s.A + (size_t)j * s.lda;
        double w = 0.0;
        if (act)
          for (int i = j + 1 + gl; i < m; i += 4) w += vj[i] * y[i];
        w += __shfl_xor_sync(0xffffffffu, w, 1);
        w += __shfl_xor_sync(0xffffffffu, w, 2);
        if (act) {
          const double tw = t * (w + y[j]);
          __syncwarp(0xffffffffu);
          if (gl == 0) y[j] -= tw;
          for (int i = j + 1 + gl; i < m; i += 4) y[i] -= tw * vj[i];
        } else {
          __syncwarp(0xffffffffu);
        }
        __syncwarp();
      }
    }
  }
  __syncwarp();
  // ---- Gaussian padding (sketch.hpp:48-65), same stream as Omega
  uint64_t tn = (uint64_t)T.normal_base;
  for (int j = q; j < r; ++j) {
    for (int attempt = 0; attempt < 1000; ++attempt) {
      for (int i = lane; i < m; i += 32)
        s.v[i] = srtt_dev::normal_at(T.state0, T.draw_offset, tn + (uint64_t)i, nullptr);
      tn += (uint64_t)m;
      __syncwarp();
      for (int round = 0; round < 2 && j > 0; ++round) {
        for (int jj = 0; jj < j; ++jj) {
          const double* yc = s.Y + (size_t)jj * s.lda;
          double part = 0.0;
          for (int i = lane; i < m; i += 32) part += yc[i] * s.v[i];
          const double d = warp_sum(part);
          if (lane == 0) s.dots[jj] = d;
        }
        __syncwarp();
        for (int i = lane; i < m; i += 32) {
          double acc = 0.0;
          for (int jj = 0; jj < j; ++jj) acc += s.Y[(size_t)jj * s.lda + i] * s.dots[jj];
          s.v[i] -= acc;
        }
        __syncwarp();
      }
      double part = 0.0;
      for (int i = lane; i < m; i += 32) part += s.v[i] * s.v[i];
      const double nrm = sqrt(warp_sum(part));
      if (nrm > 1e-8) {
        for (int i = lane; i < m; i += 32) s.Y[(size_t)j * s.lda + i] = s.v[i] / nrm;
        __syncwarp();
        break;
      }
      __syncwarp();
    }
  }
  for (int idx = lane; idx < m * r; idx += 32) {
    const int i = idx % m, col = idx / m;
    T.u[idx] = s.Y[(size_t)col * s.lda + i];
  }
}

}  // namespace

size_t srtt_basis_top_smem(int m, int c, int r) {
  const int k = m < c ? m : c;
  size_t doubles = (size_t)c + (size_t)m * c + (size_t)k * c + (size_t)k * k + (size_t)m * r + c + k + r + 32 + m + 2;
  return doubles * sizeof(double) + 2 * sizeof(int) * (size_t)(k + 2);
}

size_t srtt_basis_level_smem(int mb, int c) {
  return ((size_t)mb * c * 2 + 2 * c + 2) * sizeof(double);
}

int srtt_basis_threads() { return kThreads; }

size_t srtt_basis_small_smem(int m, int c, int r) {
  const int k = m < c ? m : c;
  const size_t doubles = (size_t)c + (size_t)odd_ld(m) * c + (size_t)odd_ld(c) * k + (size_t)odd_ld(k) * k +
                         (size_t)odd_ld(m) * r + c + k + r + m + 2;
  return doubles * sizeof(double) + sizeof(int) * (size_t)(k + 2);
}

cudaError_t srtt_launch_basis_small(const BasisTarget* d_targets, const int* d_list, int n, size_t smem,
                                    cudaStream_t stream) {
  if (n <= 0) return cudaSuccess;
  SRTT_ENSURE_SMEM((basis_small_kernel), smem);
  basis_small_kernel<<<n, 32, smem, stream>>>(d_targets, d_list);
  return cudaGetLastError();
}

cudaError_t srtt_launch_basis_top(const BasisTarget* d_targets, const int* d_list, int ntargets, size_t smem,
                                  cudaStream_t stream) {
  if (ntargets <= 0) return cudaSuccess;
  SRTT_ENSURE_SMEM((basis_top_kernel), smem);
  basis_top_kernel<<<ntargets, kThreads, smem, stream>>>(d_targets, d_list);
  return cudaGetLastError();
}

cudaError_t srtt_launch_tsqr_factor(const BasisTarget* d_targets, const int2* d_map, int level, int nctas,
                                    size_t smem, cudaStream_t stream) {
  if (nctas <= 0) return cudaSuccess;
  SRTT_ENSURE_SMEM((tsqr_factor_kernel), smem);
  tsqr_factor_kernel<<<nctas, kThreads, smem, stream>>>(d_targets, d_map, level);
  return cudaGetLastError();
}

cudaError_t srtt_launch_tsqr_apply(const BasisTarget* d_targets, const int2* d_map, int level, int nctas,
                                   size_t smem, cudaStream_t stream) {
  if (nctas <= 0) return cudaSuccess;
  SRTT_ENSURE_SMEM((tsqr_apply_kernel), smem);
  tsqr_apply_kernel<<<nctas, kThreads, smem, stream>>>(d_targets, d_map, level);
  return cudaGetLastError();
}

cudaError_t srtt_launch_pad(const BasisTarget* d_targets, int ntargets, double* scratch,
                            int64_t scratch_stride, cudaStream_t stream) {
  if (ntargets <= 0) return cudaSuccess;
  pad_kernel<<<ntargets, kThreads, 0, stream>>>(d_targets, scratch, scratch_stride);
  return cudaGetLastError();
}
