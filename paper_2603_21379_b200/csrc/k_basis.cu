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

#include <utility>

#include "srtt_device.cuh"
#include "srtt_params.h"

namespace {

using srtt_dev::warp_sum;

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;

// Development-only phase clock (make PROF=1): block 0 of basis_small_kernel
// records clock64() at phase boundaries.
#ifdef SRTT_PROF
__device__ long long g_basis_clk[16];
#define PROF_MARK(i) \
  do {               \
    __syncwarp();    \
    if (blockIdx.x == 0 && threadIdx.x == 0) g_basis_clk[i] = clock64(); \
  } while (0)
#define PROF_MARK_CTA(i) \
  do {                   \
    __syncthreads();     \
    if (blockIdx.x == 0 && threadIdx.x == 0) g_basis_clk[i] = clock64(); \
  } while (0)
#else
#define PROF_MARK_CTA(i) \
  do {                   \
  } while (0)
#define PROF_MARK(i) \
  do {               \
  } while (0)
#endif

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

// Jacobi rotation zeroing apq (|theta| <= pi/4, Rutishauser's choice of
// t = tan(theta) = sign(d) 2 apq / (|d| + h), d = aqq - app,
// h = sqrt(d^2 + 4 apq^2)), evaluated with two reciprocal square roots and
// no division: cos(2 theta) = |d| / h, c = sqrt((1 + cos 2theta) / 2),
// s = sign(d) (2 apq / h) / (2 c).
__device__ __forceinline__ void jacobi_rotation(double app, double aqq, double apq, double* cs, double* sn) {
  const double dd = aqq - app;
  const double ta = 2.0 * apq;
  const double rh = rsqrt(fma(dd, dd, ta * ta));
  const double w = fma(0.5 * fabs(dd), rh, 0.5);
  const double rw = rsqrt(w);
  *cs = w * rw;
  *sn = copysign(1.0, dd) * (0.5 * ta * rh) * rw;
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

// Register-resident one-sided Jacobi for one warp (k <= 32 / G * 2 rows).
// Round-robin by the circle method: lane group g (G lanes) holds the two
// players in positions g and kk-1-g -- their rows of B (length c) and of V
// (length k), E = ceil(max(c, k) / G) values per lane each. After a round,
// position 0 stays and the others advance one place, so rows move between
// neighbouring groups by shuffles instead of through shared memory. Every
// pair meets once per sweep; sweeps repeat until none rotates.
template <int G, int E>
__device__ int jacobi_rows_reg(double* B, int ldb, int k, int c, double* V, int ldv) {
  const int lane = threadIdx.x & 31;
  const int g = lane / G, gl = lane % G;
  const int kk = (k + 1) & ~1;
  const int np = kk / 2;
  const bool grp_live = g < np;
  const double tol2 = 4.0 * DBL_EPSILON * DBL_EPSILON;
  int tp = g, bp = kk - 1 - g;  // players held by this group
  double tb[E], bb[E], tv[E], bv[E];
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const int j = gl + G * e;
    tb[e] = (grp_live && tp < k && j < c) ? B[(size_t)tp * ldb + j] : 0.0;
    bb[e] = (grp_live && bp < k && j < c) ? B[(size_t)bp * ldb + j] : 0.0;
    tv[e] = (grp_live && tp < k && j < k) ? V[(size_t)tp * ldv + j] : 0.0;
    bv[e] = (grp_live && bp < k && j < k) ? V[(size_t)bp * ldv + j] : 0.0;
  }
  const int src_prev = (lane - G) & 31, src_next = (lane + G) & 31;
  int sweep = 0;
  if (k >= 2) {
    for (; sweep < 80; ++sweep) {
      int rotated = 0;
      for (int rd = 0; rd < kk - 1; ++rd) {
        double app = 0.0, aqq = 0.0, apq = 0.0;
#pragma unroll
        for (int e = 0; e < E; ++e) {
          app = fma(tb[e], tb[e], app);
          aqq = fma(bb[e], bb[e], aqq);
          apq = fma(tb[e], bb[e], apq);
        }
#pragma unroll
        for (int o = 1; o < G; o <<= 1) {
          app += __shfl_xor_sync(0xffffffffu, app, o);
          aqq += __shfl_xor_sync(0xffffffffu, aqq, o);
          apq += __shfl_xor_sync(0xffffffffu, apq, o);
        }
        if (grp_live && apq != 0.0 && apq * apq > tol2 * app * aqq) {
          double cs, sn;
          jacobi_rotation(app, aqq, apq, &cs, &sn);
          // the top player plays "p": any plane rotation that zeroes the
          // pair's inner product with |theta| <= pi/4 serves
          const double s2 = sn;
#pragma unroll
          for (int e = 0; e < E; ++e) {
            const double x = tb[e], y = bb[e];
            tb[e] = cs * x - s2 * y;
            bb[e] = s2 * x + cs * y;
            const double u = tv[e], v = bv[e];
            tv[e] = cs * u - s2 * v;
            bv[e] = s2 * u + cs * v;
          }
          rotated = 1;
        }
        // advance: top[0] stays, top[1] <- bot[0], top[g] <- top[g-1],
        // bot[g] <- bot[g+1], bot[np-1] <- top[np-1]
#pragma unroll
        for (int e = 0; e < E; ++e) {
          const double pt = __shfl_sync(0xffffffffu, tb[e], src_prev);
          const double pb = __shfl_sync(0xffffffffu, bb[e], src_prev);
          const double nb = __shfl_sync(0xffffffffu, bb[e], src_next);
          const double qt = __shfl_sync(0xffffffffu, tv[e], src_prev);
          const double qb = __shfl_sync(0xffffffffu, bv[e], src_prev);
          const double mb = __shfl_sync(0xffffffffu, bv[e], src_next);
          const double otb = tb[e], otv = tv[e];
          if (g >= 1) {
            tb[e] = g == 1 ? pb : pt;
            tv[e] = g == 1 ? qb : qt;
          }
          bb[e] = g == np - 1 ? otb : nb;
          bv[e] = g == np - 1 ? otv : mb;
        }
        {
          const int ptp = __shfl_sync(0xffffffffu, tp, src_prev);
          const int pbp = __shfl_sync(0xffffffffu, bp, src_prev);
          const int nbp = __shfl_sync(0xffffffffu, bp, src_next);
          const int otp = tp;
          if (g >= 1) tp = g == 1 ? pbp : ptp;
          bp = g == np - 1 ? otp : nbp;
        }
      }
      if (!__any_sync(0xffffffffu, rotated)) break;
    }
  }
  __syncwarp();
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const int j = gl + G * e;
    if (grp_live && tp < k && j < c) B[(size_t)tp * ldb + j] = tb[e];
    if (grp_live && bp < k && j < c) B[(size_t)bp * ldb + j] = bb[e];
    if (grp_live && tp < k && j < k) V[(size_t)tp * ldv + j] = tv[e];
    if (grp_live && bp < k && j < k) V[(size_t)bp * ldv + j] = bv[e];
  }
  __syncwarp();
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
        for (int jj = warp; jj < j; jj += (int)(blockDim.x >> 5)) {
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

__host__ __device__ inline int odd_ld(int n) { return n | 1; }

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
  s.A = p; p += (size_t)odd_ld(m) * c;
  s.B = p; p += (size_t)k * c;
  s.V = p; p += (size_t)k * k;
  s.Y = p; p += (size_t)m * r;
  s.tau = p; p += c;
  s.sig = p; p += k;
  s.dots = p; p += r;
  s.red = p; p += kWarps * 32 + 64;
  s.vpad = p; p += m;
  s.scal_beta = p; p += 2;
  s.perm = reinterpret_cast<int*>(p);
  s.flag = s.perm + k;
  return s;
}

template <int OWN>
__device__ void qr_cols_warps(const double* __restrict__ z, int64_t ldz, int m, int c, double* A, int lda,
                              double* tau);
template <int OWN>
__device__ void apply_reflectors_warps(const double* A, int lda, const double* tau, int m, int k, int q, double* Y,
                                       int ldy);
__device__ void apply_cols_warps(const double* A, int lda, const double* tau, int m, int k, const double* V,
                                 int ldv, const int* perm, int q, double* Y, int ldy);

// Top of the TSQR tree (or the whole basis for single-block targets).
// JG > 0: warp-per-column QR and back-application over the CTA's warps
// (qr_cols_warps / apply_cols_warps) around warp 0's register Jacobi
// <JG, JE> (c <= 32); JG = 0: the CTA-wide shared-memory QRCP / 4-lane Jacobi.
template <int JG, int JE>
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
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int lda = JG > 0 ? odd_ld(m) : m;
  PROF_MARK_CTA(8);

  if constexpr (JG > 0) {
    qr_cols_warps<4>(L.a, m, m, c, s.A, lda, s.tau);
  } else {
    for (int idx = threadIdx.x; idx < m * c; idx += blockDim.x) {
      const int i = idx % m, j = idx / m;
      s.A[idx] = L.a[(int64_t)j * L.n + i];
    }
    __syncthreads();
    householder_qr(s.A, m, c, m, s.tau, s.scal_beta, s.vn);
  }
  __syncthreads();
  PROF_MARK_CTA(9);
  // B = R (k x c, row-major), V = I.
  for (int idx = threadIdx.x; idx < k * c; idx += blockDim.x) {
    const int i = idx / c, j = idx % c;
    s.B[idx] = (j >= i) ? s.A[(size_t)j * lda + i] : 0.0;
  }
  for (int idx = threadIdx.x; idx < k * k; idx += blockDim.x) s.V[idx] = (idx % k == idx / k) ? 1.0 : 0.0;
  __syncthreads();
  int sweeps = 0;
  if constexpr (JG > 0) {
    if (warp == 0) sweeps = jacobi_rows_reg<JG, JE>(s.B, c, k, c, s.V, k);
    __syncthreads();
  } else {
    build_pairs(pairs, (k + 1) & ~1);
    __syncthreads();
    sweeps = jacobi_rows_g4(s.B, c, k, c, s.V, k, pairs);
  }
  PROF_MARK_CTA(10);
  // Singular values = row norms; sort descending (ties by index).
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
  PROF_MARK_CTA(11);
  // Y = Q [V(:, perm[:q]); 0]
  if constexpr (JG > 0) {
    apply_cols_warps(s.A, lda, s.tau, m, k, s.V, k, s.perm, q, s.Y, m);
  } else {
    for (int idx = threadIdx.x; idx < m * q; idx += blockDim.x) {
      const int i = idx % m, col = idx / m;
      s.Y[idx] = (i < k) ? s.V[(size_t)s.perm[col] * k + i] : 0.0;
    }
    __syncthreads();
    for (int col = warp; col < q; col += kWarps) apply_q_warp(s.A, m, k, m, s.tau, s.Y + (size_t)col * m);
  }
  __syncthreads();
  PROF_MARK_CTA(12);
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
  PROF_MARK_CTA(13);
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
  if (c <= 32) {
    qr_cols_warps<4>(L.a + r0, L.n, mb, c, A, mb, tau);
  } else if (c <= 64) {
    qr_cols_warps<8>(L.a + r0, L.n, mb, c, A, mb, tau);
  } else {
    for (int idx = threadIdx.x; idx < mb * c; idx += blockDim.x) {
      const int i = idx % mb, j = idx / mb;
      A[idx] = L.a[(int64_t)j * L.n + r0 + i];
    }
    __syncthreads();
    householder_qr(A, mb, c, mb, tau, sb);
  }
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
  if (q <= 32) apply_reflectors_warps<4>(A, mb, tau, mb, kb, q, Y, mb);
  else apply_reflectors_warps<8>(A, mb, tau, mb, kb, q, Y, mb);
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

// One warp per target for wide sketches (32 < c <= 64, single block):
// shared-memory QRCP with 4-lane column groups (pivoting preconditions the
// Jacobi), 4-lane shared-memory Jacobi, warp back-application. Narrower
// sketches take basis_cta_kernel.
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
  PROF_MARK(0);
  const double* z = T.lv[0].a;
  {
    for (int idx = lane; idx < m * c; idx += 32) {
      const int i = idx % m, j = idx / m;
      s.A[(size_t)j * s.lda + i] = z[idx];
    }
    __syncwarp();
    PROF_MARK(1);
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
  }
  PROF_MARK(2);
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
  // ---- one-sided Jacobi on the rows of R (shared memory, 4-lane groups)
  build_pairs(pairs, (k + 1) & ~1);
  __syncwarp();
  const int sweeps = jacobi_rows_g4(s.B, s.ldb, k, c, s.V, s.ldv, pairs);
  PROF_MARK(3);
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
  PROF_MARK(4);
  // ---- Y = Q [V(:, perm[:q]); 0]
  {
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
  }
  PROF_MARK(5);
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
  PROF_MARK(6);
  for (int idx = lane; idx < m * r; idx += 32) {
    const int i = idx % m, col = idx / m;
    T.u[idx] = s.Y[(size_t)col * s.lda + i];
  }
  PROF_MARK(7);
}

// ---- CTA-wide small basis (c <= 32) ---------------------------------------
// Householder QR, register-resident one-sided Jacobi on the rows of R (warp
// 0), back-application and Gaussian padding. The QR and the
// back-application are spread over the CTA's warps: warp w owns the columns
// l = w (mod W); a reflector step is one warp reduction per owned column
// plus one CTA barrier, and the owner of column j+1 builds reflector j+1
// right after updating that column (look-ahead), so a step costs about two
// warp reductions of latency instead of a serial row loop per lane.
// columns per warp: OWN = 4 covers c <= 32 with 8 warps, OWN = 8 c <= 64

// reflector j from column j (called by the owning warp): v below the
// diagonal (scaled in place), beta on the diagonal, tau[j]
__device__ __forceinline__ void cta_make_reflector(double* A, int lda, int m, int j, double* tau) {
  const int lane = threadIdx.x & 31;
  double* col = A + (size_t)j * lda;
  double p0 = 0.0, p1 = 0.0;
  int i = j + 1 + lane;
  for (; i + 32 < m; i += 64) {
    p0 = fma(col[i], col[i], p0);
    p1 = fma(col[i + 32], col[i + 32], p1);
  }
  if (i < m) p0 = fma(col[i], col[i], p0);
  const double ss = warp_sum(p0 + p1);
  const double alpha = col[j];
  double tj = 0.0, scal = 0.0, beta = alpha;
  if (ss != 0.0) {
    const double nrm = sqrt(fma(alpha, alpha, ss));
    beta = -copysign(nrm, alpha);
    tj = (beta - alpha) / beta;
    scal = 1.0 / (alpha - beta);
  }
  if (tj != 0.0)
    for (int ii = j + 1 + lane; ii < m; ii += 32) col[ii] *= scal;
  if (lane == 0) {
    col[j] = beta;  // v_j = 1 is implicit: the diagonal slot is free
    tau[j] = tj;
  }
  __syncwarp();
}

// Apply reflector (v = A(:, j), tau tj) to the OWN columns X(:, l) this warp
// owns (l = warp + nw*t, active when lo <= l < hi): w = x_j + v^T x below j,
// x -= tj w v. Two partial sums per column break the FMA chains.
template <int OWN>
__device__ __forceinline__ void warp_reflect_cols(const double* v, double tj, int j, int m, double* X, int ldx,
                                                  int lo, int hi) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  double w[OWN];
#pragma unroll
  for (int t = 0; t < OWN; ++t) {
    const int l = warp + nw * t;
    double p0 = 0.0, p1 = 0.0;
    if (l >= lo && l < hi) {
      const double* x = X + (size_t)l * ldx;
      int i = j + 1 + lane;
      for (; i + 32 < m; i += 64) {
        p0 = fma(v[i], x[i], p0);
        p1 = fma(v[i + 32], x[i + 32], p1);
      }
      if (i < m) p0 = fma(v[i], x[i], p0);
    }
    w[t] = p0 + p1;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1)
#pragma unroll
    for (int t = 0; t < OWN; ++t) w[t] += __shfl_xor_sync(0xffffffffu, w[t], o);
#pragma unroll
  for (int t = 0; t < OWN; ++t) {
    const int l = warp + nw * t;
    if (l >= lo && l < hi) {
      double* x = X + (size_t)l * ldx;
      const double tw = tj * (w[t] + x[j]);
      for (int i = j + 1 + lane; i < m; i += 32) x[i] = fma(-tw, v[i], x[i]);
      if (lane == 0) x[j] -= tw;
    }
  }
  __syncwarp();
}

// Householder QR of z (m x c, ld ldz) into A (ld lda) over the CTA's warps.
template <int OWN>
__device__ void qr_cols_warps(const double* __restrict__ z, int64_t ldz, int m, int c, double* A, int lda,
                              double* tau) {
  const int warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int k = min(m, c);
  for (int idx = threadIdx.x; idx < m * c; idx += blockDim.x) {
    const int i = idx % m, j = idx / m;
    A[(size_t)j * lda + i] = __ldg(z + (int64_t)j * ldz + i);
  }
  __syncthreads();
  if (k > 0 && warp == 0) cta_make_reflector(A, lda, m, 0, tau);
  __syncthreads();
  for (int j = 0; j < k; ++j) {
    const double tj = tau[j];
    if (tj != 0.0) warp_reflect_cols<OWN>(A + (size_t)j * lda, tj, j, m, A, lda, j + 1, c);
    if (j + 1 < k && (j + 1) % nw == warp) cta_make_reflector(A, lda, m, j + 1, tau);
    __syncthreads();
  }
}

// Y(:, 0:q) <- Q Y(:, 0:q) with Q = H_0 ... H_{k-1}: warp w owns output
// columns w (mod W) and applies the reflectors in reverse order (no CTA
// barriers; A is read-only).
template <int OWN>
__device__ void apply_reflectors_warps(const double* A, int lda, const double* tau, int m, int k, int q, double* Y,
                                       int ldy) {
  const int warp = threadIdx.x >> 5;
  if (warp < q)
    for (int j = k - 1; j >= 0; --j) {
      const double tj = tau[j];
      if (tj != 0.0) warp_reflect_cols<OWN>(A + (size_t)j * lda, tj, j, m, Y, ldy, 0, q);
    }
  __syncthreads();
}

// Y(:, 0:q) = Q [V(:, perm[0:q]); 0]
__device__ void apply_cols_warps(const double* A, int lda, const double* tau, int m, int k, const double* V,
                                 int ldv, const int* perm, int q, double* Y, int ldy) {
  for (int idx = threadIdx.x; idx < m * q; idx += blockDim.x) {
    const int i = idx % m, col = idx / m;
    Y[(size_t)col * ldy + i] = i < k ? V[(size_t)perm[col] * ldv + i] : 0.0;
  }
  __syncthreads();
  apply_reflectors_warps<4>(A, lda, tau, m, k, q, Y, ldy);
}

template <int JG, int JE>
__global__ void __launch_bounds__(kThreads) basis_cta_kernel(const BasisTarget* __restrict__ targets,
                                                             const int* __restrict__ list) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ BasisTarget T;
  __shared__ double red[64];
  stage_target(&T, &targets[list[blockIdx.x]]);
  __syncthreads();
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int m = (int)T.n, c = T.c, r = T.r;
  const int k = min(m, c);
  SmallSmem s = carve_small(smem_raw, m, c, r);
  PROF_MARK_CTA(0);
  qr_cols_warps<4>(T.lv[0].a, m, m, c, s.A, s.lda, s.tau);
  PROF_MARK_CTA(1);
  PROF_MARK_CTA(2);
  for (int idx = tid; idx < k * c; idx += blockDim.x) {
    const int i = idx / c, j = idx % c;
    s.B[(size_t)i * s.ldb + j] = (j >= i) ? s.A[(size_t)j * s.lda + i] : 0.0;
  }
  for (int idx = tid; idx < k * k; idx += blockDim.x) {
    const int i = idx % k, j = idx / k;
    s.V[(size_t)j * s.ldv + i] = (i == j) ? 1.0 : 0.0;
  }
  __syncthreads();
  int sweeps = 0;
  if (warp == 0) sweeps = jacobi_rows_reg<JG, JE>(s.B, s.ldb, k, c, s.V, s.ldv);
  __syncthreads();
  PROF_MARK_CTA(3);
  for (int i = tid; i < k; i += blockDim.x) {
    const double* bi = s.B + (size_t)i * s.ldb;
    s.sig[i] = sqrt(dot4(bi, bi, 0, c));
  }
  __syncthreads();
  for (int i = tid; i < k; i += blockDim.x) {
    int rank = 0;
    for (int j = 0; j < k; ++j) rank += (s.sig[j] > s.sig[i]) || (s.sig[j] == s.sig[i] && j < i);
    s.perm[rank] = i;
  }
  __syncthreads();
  const double smax = s.sig[s.perm[0]];
  const double tol_rank = (double)max(m, c) * DBL_EPSILON * smax;
  int nrank = 0;
  for (int i = 0; i < k; ++i) nrank += s.sig[i] > tol_rank;
  const int q = min(nrank, r);
  if (tid == 0) {
    T.info[0] = q;
    T.info[1] = nrank;
    T.info[2] = sweeps;
  }
  if (T.sv)
    for (int i = tid; i < k; i += blockDim.x) T.sv[i] = s.sig[s.perm[i]];
  PROF_MARK_CTA(4);
  apply_cols_warps(s.A, s.lda, s.tau, m, k, s.V, s.ldv, s.perm, q, s.Y, s.lda);
  PROF_MARK_CTA(5);
  if (q < r)
    pad_columns(s.Y, m, s.lda, q, r, T.state0, T.draw_offset, (uint64_t)T.normal_base, s.v, s.dots, red);
  PROF_MARK_CTA(6);
  for (int idx = tid; idx < m * r; idx += blockDim.x) {
    const int i = idx % m, col = idx / m;
    T.u[idx] = s.Y[(size_t)col * s.lda + i];
  }
  (void)lane;
  PROF_MARK_CTA(7);
}


// ===========================================================================
// Register-resident TSQR tree (sketches with c <= 32 columns).
//
// The shared-memory QR above pays one CTA barrier and two dependent warp
// reductions per reflector, with all 8 warps working on one column pair at
// a time. Here a WARP owns a whole row block: lane l holds rows
// {l, l + 32, ...} of the block in registers (RT rows x CP columns, RT * CP
// = 64 doubles), so a reflector step is one lane-local dot-product pass, one
// reduce-scatter through a conflict-free shared-memory transpose and one
// lane-local update; the live columns shift one register to the left per
// step, so the rolled step loop only ever touches statically indexed
// registers. Row blocks are combined as a tree inside the CTA (warp R
// factors stacked in shared memory and factored again) and, for tall
// sketches, across CTAs through one stacked-R level in global memory.
//
// Reflector convention of this path: H_j = I - g_j u_j u_j^T with u_j stored
// whole (zeros above the diagonal, u_jj = alpha - beta on it, the column
// tail below), g_j = 2 / (u_j^T u_j) computed from the stored u_j.
//
// The small SVD: R^T = Q_1 R_1 (a second register QR), one-sided Jacobi on
// the rows of R_1 without accumulating the rotations: R_1 = J S W^T, and
// the left singular vectors of R (= those of Z up to Q) are the normalised
// rows of the rotated matrix, W = (J^T R_1)^T S^-1.
// ===========================================================================
constexpr int kTreeMaxLevels = 12;

// development: per-segment clocks of the QR step (tools/microbench/wqr.cu)
#ifdef SRTT_WQR_PROF
__device__ long long g_wqr_clk[8];
#define WQR_CLK_DECL long long wq_t[6], wq_acc[6] = {0, 0, 0, 0, 0, 0}
#define WQR_CLK(i)                                        \
  do {                                                    \
    wq_t[i] = clock64();                                  \
    if (i > 0) wq_acc[i] += wq_t[i] - wq_t[i - 1];        \
  } while (0)
#define WQR_CLK_OUT                                                   \
  do {                                                                \
    if (threadIdx.x == 0 && blockIdx.x == 0)                          \
      for (int i = 0; i < 6; ++i) g_wqr_clk[i] = wq_acc[i];           \
  } while (0)
#else
#define WQR_CLK_DECL
#define WQR_CLK(i)
#define WQR_CLK_OUT
#endif

struct WTree {
  int L;                           // QR levels; the final R is S[L]
  int rows[kTreeMaxLevels + 1];    // rows entering level l
  int nblk[kTreeMaxLevels];
  int soff[kTreeMaxLevels + 1];    // S_l, l >= 1: stacked R entering level l (then V_l in place), ld = rows | 1
  int goff[kTreeMaxLevels];        // g_l: nblk x c
  int yoff[kTreeMaxLevels + 1];    // Y_l, l >= 1 (back-application), ld = rows | 1
  int persist;                     // doubles of the S + g part (kept for the apply kernel)
  int total;
};

__host__ __device__ inline WTree wtree_plan(int n0, int c, int chunk) {
  WTree t;
  int rows = n0, l = 0;
  t.rows[0] = n0;
  for (;;) {
    const int nb = (rows + chunk - 1) / chunk;
    const int rem = rows - (nb - 1) * chunk;
    t.nblk[l] = nb;
    rows = (nb - 1) * c + (rem < c ? rem : c);
    ++l;
    t.rows[l] = rows;
    if (nb == 1 || l >= kTreeMaxLevels) break;
  }
  t.L = l;
  int off = 0;
  for (int i = 1; i <= l; ++i) { t.soff[i] = off; off += (t.rows[i] | 1) * c; }
  for (int i = 0; i < l; ++i) { t.goff[i] = off; off += t.nblk[i] * c; }
  t.persist = off;
  for (int i = 1; i <= l; ++i) { t.yoff[i] = off; off += (t.rows[i] | 1) * c; }
  t.total = off;
  return t;
}

template <int CP> struct WTile {
  static constexpr int RT = 64 / CP;      // rows per lane
  static constexpr int CHUNK = 32 * RT;   // rows per warp block
  static constexpr int LPC = 32 / CP;     // lanes sharing a column after the reduce-scatter
  static constexpr int PADG = LPC == 1 ? 0 : 16 / LPC;  // pad between the source-lane groups (bank spread)
  static constexpr int RED = 32 * (CP + 2) + (LPC - 1) * PADG;  // reduce-scatter transpose area
  static constexpr int WSCR = RED + 3 * CP;  // per-warp scratch doubles (+ pivot row, coefficients, dump row)
};

// Sum D[p] over the 32 lanes; afterwards the lanes [col * 32 / CP, ...)
// hold the total of column col (fixed summation order). The scratch rows
// are CP + 2 doubles apart: 16-byte vector stores, and both the stores and
// the column reads are bank-conflict free. The caller must pass a warp
// barrier before the next call (every user below does: the coefficient
// broadcast follows each reduction).
template <int CP>
__device__ __forceinline__ double reduce_scatter_sm(const double (&D)[CP], double* red, int lane) {
  constexpr int LPC = 32 / CP, SPL = 32 / LPC, LD = CP + 2, PADG = WTile<CP>::PADG;
  double2* row = reinterpret_cast<double2*>(red + lane * LD + (lane / SPL) * PADG);
#pragma unroll
  for (int p = 0; p < CP; p += 2) row[p / 2] = make_double2(D[p], D[p + 1]);
  __syncwarp();
  const int col = lane / LPC, part = lane % LPC;
  const double* q = red + (size_t)(part * SPL) * LD + part * PADG + col;
  double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
#pragma unroll
  for (int i = 0; i < SPL; i += 4) {
    s0 += q[(i + 0) * LD];
    s1 += q[(i + 1) * LD];
    s2 += q[(i + 2) * LD];
    s3 += q[(i + 3) * LD];
  }
  double s = (s0 + s1) + (s2 + s3);
#pragma unroll
  for (int o = 1; o < LPC; o <<= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  return s;
}

// Shared-memory accesses by 32-bit shared-window address: the reflector,
// g and R destinations of the step loops are always shared memory, and a
// generic store there costs a few hundred cycles at the next warp barrier.
__device__ __forceinline__ uint32_t smem_addr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void sts_f64(uint32_t addr, double v) {
  asm volatile("st.shared.f64 [%0], %1;" ::"r"(addr), "d"(v) : "memory");
}
__device__ __forceinline__ double lds_f64(uint32_t addr) {
  double v;
  asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(addr) : "memory");
  return v;
}

// Householder QR of the warp's register block a (nr rows, c columns; rows
// beyond nr and columns beyond c are zero). Reflector j goes to
// vout[row + j * ldv] (STOREV), g_j to gout[j], row j of R to
// rout[j * rs + col * cs] (entries on and right of the diagonal only).
// RTL: row groups that can hold rows (compile time; the second QR of the small
// SVD has at most 32 rows: one group, a quarter of the FMA work)
template <int CP, bool STOREV, int RTL = WTile<CP>::RT>
__device__ void wqr_factor(double (&a)[WTile<CP>::RT][CP], int nr, int c, double* vout, int ldv, double* gout,
                           double* rout, int rs, int cs, double* wsm) {
  constexpr int RT = WTile<CP>::RT, LPC = 32 / CP;
  const int lane = threadIdx.x & 31;
  const int mycol = lane / LPC;
  double* red = wsm;
  double* prow = wsm + WTile<CP>::RED;
  double* csm = prow + CP;
  const int kb = nr < c ? nr : c;
  // all destinations are shared memory (see smem_addr)
  uint32_t va = STOREV ? smem_addr(vout) + 8u * lane : 0u;   // element (lane, j = 0)
  uint32_t ga = STOREV ? smem_addr(gout) : 0u;
  uint32_t ra = smem_addr(rout) + 8u * (uint32_t)(mycol * cs);  // element (j = 0, col = mycol)
  const uint32_t vstep = 8u * (uint32_t)ldv, rstep = 8u * (uint32_t)(rs + cs);
  WQR_CLK_DECL;
  for (int j = 0; j < kb; ++j) {
    const int lj = j & 31, tj = j >> 5;
    WQR_CLK(0);
    {
      // pivot row to shared memory without a divergent branch: the owner
      // lane stores to prow, every other lane to the dump row behind csm
      double2* pdst = reinterpret_cast<double2*>(lane == lj ? prow : csm + CP);
#pragma unroll
      for (int t = 0; t < RT; ++t)
        if (tj == t) {
#pragma unroll
          for (int p = 0; p < CP; p += 2) pdst[p / 2] = make_double2(a[t][p], a[t][p + 1]);
        }
    }
    double xm[RT];
#pragma unroll
    for (int t = 0; t < RT; ++t) xm[t] = (t * 32 + lane > j) ? a[t][0] : 0.0;
    double D[CP];
#pragma unroll
    for (int p = 0; p < CP; ++p) {
      double s = 0.0;
#pragma unroll
      for (int t = 0; t < RTL; ++t) s = fma(xm[t], a[t][p], s);
      D[p] = s;
    }
    WQR_CLK(1);
    const double dtot = reduce_scatter_sm<CP>(D, red, lane);  // (its barrier also publishes prow)
    WQR_CLK(2);
    const double ss = __shfl_sync(0xffffffffu, dtot, 0);
    const double alpha = prow[0];
    double beta = alpha, ujj = 0.0, g = 0.0;
    if (ss != 0.0) {
      // g = 2 / (ss + u_jj^2) = 1 / (nrm |u_jj|), from one reciprocal square
      // root and one reciprocal (the chain is the step's critical path)
      const double n2 = fma(alpha, alpha, ss);
      const double rn = rsqrt(n2);
      const double nrm = n2 * rn;
      beta = -copysign(nrm, alpha);
      ujj = alpha - beta;
      g = rn * __drcp_rn(fabs(ujj));
    }
    const double arow = prow[mycol];
    const double cl = g * fma(ujj, arow, dtot);
    WQR_CLK(3);
    if (lane % LPC == 0) {
      csm[mycol] = cl;
      if (j + mycol < c) sts_f64(ra, mycol == 0 ? beta : arow - cl * ujj);
    }
    ra += rstep;
    if (STOREV) {
#pragma unroll
      for (int t = 0; t < RT; ++t) {
        const int row = t * 32 + lane;
        if (row < nr) sts_f64(va + 256u * t, row > j ? xm[t] : (row == j ? ujj : 0.0));
      }
      if (lane == 0) sts_f64(ga + 8u * j, g);
      va += vstep;
    }
    __syncwarp();
    WQR_CLK(4);
#pragma unroll
    for (int p = 0; p < CP; p += 2) {
      const double2 e = reinterpret_cast<const double2*>(csm)[p / 2];
#pragma unroll
      for (int t = 0; t < RTL; ++t) {
        if (p > 0) a[t][p - 1] = fma(-e.x, xm[t], a[t][p]);
        a[t][p] = fma(-e.y, xm[t], a[t][p + 1 < CP ? p + 1 : p]);
      }
    }
#pragma unroll
    for (int t = 0; t < RTL; ++t) a[t][CP - 1] = 0.0;
    __syncwarp();
    WQR_CLK(5);
  }
  WQR_CLK_OUT;
}

// y <- H_0 ... H_{kb-1} y for the warp's register block y (nr rows).
template <int CP, int RTL = WTile<CP>::RT>
__device__ void wqr_apply(double (&y)[WTile<CP>::RT][CP], int nr, int kb, const double* v, int ldv, const double* g,
                          double* wsm) {
  constexpr int RT = WTile<CP>::RT, LPC = 32 / CP;
  const int lane = threadIdx.x & 31;
  const int mycol = lane / LPC;
  double* red = wsm;
  double* esm = wsm + WTile<CP>::RED;
  // v and g are shared memory (see smem_addr)
  const uint32_t vstep = 8u * (uint32_t)ldv;
  uint32_t va = smem_addr(v) + 8u * lane + vstep * (uint32_t)(kb > 0 ? kb - 1 : 0);
  const uint32_t ga = smem_addr(g);
  double vt[RT];
#pragma unroll
  for (int t = 0; t < RT; ++t) vt[t] = (kb > 0 && t * 32 + lane < nr) ? lds_f64(va + 256u * t) : 0.0;
  for (int j = kb - 1; j >= 0; --j) {
    va -= vstep;
    double vn[RT];
#pragma unroll
    for (int t = 0; t < RT; ++t) vn[t] = (j > 0 && t * 32 + lane < nr) ? lds_f64(va + 256u * t) : 0.0;
    const double gj = lds_f64(ga + 8u * j);
    double D[CP];
#pragma unroll
    for (int p = 0; p < CP; ++p) {
      double s = 0.0;
#pragma unroll
      for (int t = 0; t < RTL; ++t) s = fma(vt[t], y[t][p], s);
      D[p] = s;
    }
    const double dtot = reduce_scatter_sm<CP>(D, red, lane);
    if (lane % LPC == 0) esm[mycol] = gj * dtot;
    __syncwarp();
#pragma unroll
    for (int p = 0; p < CP; p += 2) {
      const double2 e = reinterpret_cast<const double2*>(esm)[p / 2];
#pragma unroll
      for (int t = 0; t < RTL; ++t) {
        y[t][p] = fma(-e.x, vt[t], y[t][p]);
        y[t][p + 1] = fma(-e.y, vt[t], y[t][p + 1]);
      }
    }
    __syncwarp();
#pragma unroll
    for (int t = 0; t < RT; ++t) vt[t] = vn[t];
  }
}

// One-sided Jacobi on the rows of B (k x k, row-major, ld ldb) by one warp,
// rows resident in registers (circle method as jacobi_rows_reg), rotations
// not accumulated. A sweep in which every rotated pair had
// |cos(angle between the rows)| <= 3e-7 AND a rotation angle below 1e-6 is
// the last one (the couplings left behind are products of two such small
// numbers; pairs inside a cluster of equal singular values rotate by large
// angles whatever their coupling, so they keep the sweeps going until no
// pair exceeds the 2 eps threshold).
template <int G, int E>
__device__ int jacobi_rows_nov(double* B, int ldb, int k) {
  const int lane = threadIdx.x & 31;
  const int g = lane / G, gl = lane % G;
  const int kk = (k + 1) & ~1;
  const int np = kk / 2;
  const bool live = g < np;
  const double tol2 = 4.0 * DBL_EPSILON * DBL_EPSILON;
  int tp = g, bp = kk - 1 - g;
  double tb[E], bb[E];
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const int j = gl + G * e;
    tb[e] = (live && tp < k && j < k) ? B[(size_t)tp * ldb + j] : 0.0;
    bb[e] = (live && bp < k && j < k) ? B[(size_t)bp * ldb + j] : 0.0;
  }
  const int src_prev = (lane - G) & 31, src_next = (lane + G) & 31;
  int sweep = 0;
  if (k >= 2) {
    for (; sweep < 80; ++sweep) {
      int rotated = 0, big = 0;
      for (int rd = 0; rd < kk - 1; ++rd) {
        double app = 0.0, aqq = 0.0, apq = 0.0;
#pragma unroll
        for (int e = 0; e < E; ++e) {
          app = fma(tb[e], tb[e], app);
          aqq = fma(bb[e], bb[e], aqq);
          apq = fma(tb[e], bb[e], apq);
        }
#pragma unroll
        for (int o = 1; o < G; o <<= 1) {
          app += __shfl_xor_sync(0xffffffffu, app, o);
          aqq += __shfl_xor_sync(0xffffffffu, aqq, o);
          apq += __shfl_xor_sync(0xffffffffu, apq, o);
        }
        const double a2 = apq * apq, pq = app * aqq;
        if (live && apq != 0.0 && a2 > tol2 * pq) {
          double cs, sn;
          jacobi_rotation(app, aqq, apq, &cs, &sn);
#pragma unroll
          for (int e = 0; e < E; ++e) {
            const double x = tb[e], y = bb[e];
            tb[e] = cs * x - sn * y;
            bb[e] = sn * x + cs * y;
          }
          rotated = 1;
          if (a2 > 1e-13 * pq || fabs(sn) > 1e-6) big = 1;
        }
        if (np > 1) {
          // advance: top[0] stays, top[1] <- bot[0], top[g] <- top[g-1],
          // bot[g] <- bot[g+1], bot[np-1] <- top[np-1]
#pragma unroll
          for (int e = 0; e < E; ++e) {
            const double send = g == 0 ? bb[e] : tb[e];
            const double fp = __shfl_sync(0xffffffffu, send, src_prev);
            const double fn = __shfl_sync(0xffffffffu, bb[e], src_next);
            const double otb = tb[e];
            if (g >= 1) tb[e] = fp;
            bb[e] = g == np - 1 ? otb : fn;
          }
          const int sendp = g == 0 ? bp : tp;
          const int fpp = __shfl_sync(0xffffffffu, sendp, src_prev);
          const int fnp = __shfl_sync(0xffffffffu, bp, src_next);
          const int otp = tp;
          if (g >= 1) tp = fpp;
          bp = g == np - 1 ? otp : fnp;
        }
      }
      if (!__any_sync(0xffffffffu, rotated)) break;
      if (!__any_sync(0xffffffffu, big)) { ++sweep; break; }
    }
  }
  __syncwarp();
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const int j = gl + G * e;
    if (live && tp < k && j < k) B[(size_t)tp * ldb + j] = tb[e];
    if (live && bp < k && j < k) B[(size_t)bp * ldb + j] = bb[e];
  }
  __syncwarp();
  return sweep;
}

// ---- row-split teams ---------------------------------------------------------
// A block taller than one warp's 32 RT rows is factored by several warps
// TOGETHER instead of warp by warp plus another tree level: warp w holds rows
// [w rpw, (w + 1) rpw) of the block (rpw a multiple of 32, all columns), the
// per-warp column totals of a step meet in shared memory (double-buffered,
// ONE named barrier per step), every warp derives the same reflector scalars
// and updates its own rows. The pivot rows 0..c-1 all live in warp 0
// (c <= 32 <= rpw). One level of c steps replaces two.
template <int CP> struct TeamRows {
  static constexpr int SCR = 2 * 8 * CP + 2 * 2 * CP;  // CTA-shared doubles: warp totals + pivot row (+ dump), x2
};

__device__ __forceinline__ void team_bar(int nthreads) {
  asm volatile("bar.sync 1, %0;" ::"r"(nthreads) : "memory");
}

// rows per warp and active warps for a block of nr rows on nw warps: one
// warp when the block fits its registers, else an even split
__device__ __forceinline__ void team_split(int nr, int nw, int chunk, int* nwa, int* rpw) {
  if (nr <= chunk) {
    *nwa = 1;
    *rpw = chunk;
    return;
  }
  const int a = min(nw, (nr + chunk - 1) / chunk);
  int r = ((nr + a - 1) / a + 31) & ~31;
  if (r > chunk) r = chunk;
  *rpw = r;
  *nwa = (nr + r - 1) / r;
}

template <int CP>
__device__ void trows_factor(double (&a)[WTile<CP>::RT][CP], int w, int nwa, int rpw, int nr, int c, double* vout, int ldv,
                             double* gout, double* rout, int rs, int cs, double* wsm, double* tscr) {
  constexpr int RT = WTile<CP>::RT, LPC = 32 / CP;
  const int lane = threadIdx.x & 31;
  const int mycol = lane / LPC;
  double* red = wsm;
  double* csm = wsm + WTile<CP>::RED + CP;
  const int row0 = w * rpw;
  const int kb = nr < c ? nr : c;
  uint32_t va = smem_addr(vout) + 8u * (uint32_t)(row0 + lane);
  const uint32_t ga = smem_addr(gout);
  uint32_t ra = smem_addr(rout) + 8u * (uint32_t)(mycol * cs);
  const uint32_t vstep = 8u * (uint32_t)ldv, rstep = 8u * (uint32_t)(rs + cs);
  for (int j = 0; j < kb; ++j) {
    double* xsb = tscr + (j & 1) * 8 * CP;
    double* prb = tscr + 2 * 8 * CP + (j & 1) * 2 * CP;
    if (w == 0) {
      double2* pdst = reinterpret_cast<double2*>(lane == j ? prb : prb + CP);
#pragma unroll
      for (int p = 0; p < CP; p += 2) pdst[p / 2] = make_double2(a[0][p], a[0][p + 1]);
    }
    double xm[RT];
#pragma unroll
    for (int t = 0; t < RT; ++t) xm[t] = (row0 + t * 32 + lane > j) ? a[t][0] : 0.0;
    double D[CP];
#pragma unroll
    for (int p = 0; p < CP; ++p) {
      double s = 0.0;
#pragma unroll
      for (int t = 0; t < RT; ++t) s = fma(xm[t], a[t][p], s);
      D[p] = s;
    }
    const double dw = reduce_scatter_sm<CP>(D, red, lane);
    if (lane % LPC == 0) xsb[w * CP + mycol] = dw;
    team_bar(nwa * 32);
    // all 8 warp slots, fixed order (the slots of inactive warps are zero)
    double d0 = 0.0, d1 = 0.0, s0 = 0.0, s1 = 0.0;
#pragma unroll
    for (int v = 0; v < 8; v += 2) {
      d0 += xsb[v * CP + mycol];
      d1 += xsb[(v + 1) * CP + mycol];
      s0 += xsb[v * CP];
      s1 += xsb[(v + 1) * CP];
    }
    const double dtot = d0 + d1, ss = s0 + s1;
    const double alpha = prb[0];
    double beta = alpha, ujj = 0.0, g = 0.0;
    if (ss != 0.0) {
      const double n2 = fma(alpha, alpha, ss);
      const double rn = rsqrt(n2);
      const double nrm = n2 * rn;
      beta = -copysign(nrm, alpha);
      ujj = alpha - beta;
      g = rn * __drcp_rn(fabs(ujj));
    }
    const double arow = prb[mycol];
    const double cl = g * fma(ujj, arow, dtot);
    if (lane % LPC == 0) {
      csm[mycol] = cl;
      if (w == 0 && j + mycol < c) sts_f64(ra, mycol == 0 ? beta : arow - cl * ujj);
    }
    ra += rstep;
#pragma unroll
    for (int t = 0; t < RT; ++t) {
      const int row = row0 + t * 32 + lane;
      if (t * 32 < rpw && row < nr) sts_f64(va + 256u * t, row > j ? xm[t] : (row == j ? ujj : 0.0));
    }
    if (w == 0 && lane == 0) sts_f64(ga + 8u * j, g);
    va += vstep;
    __syncwarp();
#pragma unroll
    for (int p = 0; p < CP; p += 2) {
      const double2 e = reinterpret_cast<const double2*>(csm)[p / 2];
#pragma unroll
      for (int t = 0; t < RT; ++t) {
        if (p > 0) a[t][p - 1] = fma(-e.x, xm[t], a[t][p]);
        a[t][p] = fma(-e.y, xm[t], a[t][p + 1 < CP ? p + 1 : p]);
      }
    }
#pragma unroll
    for (int t = 0; t < RT; ++t) a[t][CP - 1] = 0.0;
    __syncwarp();
  }
}

template <int CP>
__device__ void trows_apply(double (&y)[WTile<CP>::RT][CP], int w, int nwa, int rpw, int nr, int kb, const double* v, int ldv,
                            const double* g, double* wsm, double* tscr) {
  constexpr int RT = WTile<CP>::RT, LPC = 32 / CP;
  const int lane = threadIdx.x & 31;
  const int mycol = lane / LPC;
  double* red = wsm;
  double* esm = wsm + WTile<CP>::RED;
  const int row0 = w * rpw;
  const uint32_t vstep = 8u * (uint32_t)ldv;
  uint32_t va = smem_addr(v) + 8u * (uint32_t)(row0 + lane) + vstep * (uint32_t)(kb > 0 ? kb - 1 : 0);
  const uint32_t ga = smem_addr(g);
  double vt[RT];
#pragma unroll
  for (int t = 0; t < RT; ++t)
    vt[t] = (kb > 0 && t * 32 < rpw && row0 + t * 32 + lane < nr) ? lds_f64(va + 256u * t) : 0.0;
  for (int j = kb - 1; j >= 0; --j) {
    double* xsb = tscr + (j & 1) * 8 * CP;
    va -= vstep;
    double vn[RT];
#pragma unroll
    for (int t = 0; t < RT; ++t)
      vn[t] = (j > 0 && t * 32 < rpw && row0 + t * 32 + lane < nr) ? lds_f64(va + 256u * t) : 0.0;
    const double gj = lds_f64(ga + 8u * j);
    double D[CP];
#pragma unroll
    for (int p = 0; p < CP; ++p) {
      double s = 0.0;
#pragma unroll
      for (int t = 0; t < RT; ++t) s = fma(vt[t], y[t][p], s);
      D[p] = s;
    }
    const double dw = reduce_scatter_sm<CP>(D, red, lane);
    if (lane % LPC == 0) xsb[w * CP + mycol] = dw;
    team_bar(nwa * 32);
    double d0 = 0.0, d1 = 0.0;
#pragma unroll
    for (int u = 0; u < 8; u += 2) {
      d0 += xsb[u * CP + mycol];
      d1 += xsb[(u + 1) * CP + mycol];
    }
    const double dtot = d0 + d1;
    if (lane % LPC == 0) esm[mycol] = gj * dtot;
    __syncwarp();
#pragma unroll
    for (int p = 0; p < CP; p += 2) {
      const double2 e = reinterpret_cast<const double2*>(esm)[p / 2];
#pragma unroll
      for (int t = 0; t < RT; ++t) {
        y[t][p] = fma(-e.x, vt[t], y[t][p]);
        y[t][p + 1] = fma(-e.y, vt[t], y[t][p + 1]);
      }
    }
    __syncwarp();
#pragma unroll
    for (int t = 0; t < RT; ++t) vt[t] = vn[t];
  }
}

// Factor the levels of a CTA's tree: every level cuts its rows into team
// blocks of (warps x 32 RT) rows taken one after the other by the whole CTA
// (normally there is exactly one). Level 0 reads in0 (ld ld0) and writes its
// reflectors to v0 (ld ldv0; may alias in0); with stage0 set (v0 is global
// memory) a block's reflectors are staged in shared memory during the step
// loop -- a global store there would make every barrier of the step wait for
// its acknowledgement -- and copied out afterwards. Upper levels live in the
// arena.
// RTLM = 0: blocks taller than one warp's run as row teams; RTLM = r > 0: the
// target has at most 32 r rows (one warp block), the team code is left out
// and the FMA loops touch r row groups only (compile time).
template <int CP, int RTLM = 0>
__device__ void wtree_factor(const WTree& tr, int c, const double* in0, int64_t ld0, double* v0, int64_t ldv0,
                             double* arena, double* wscr_all, double* tscr, double* stage0 = nullptr) {
  constexpr int RT = WTile<CP>::RT, CHUNK = WTile<CP>::CHUNK;
  constexpr bool TEAM = RTLM == 0;
  constexpr int RTL = TEAM ? RT : RTLM;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int TB = nw * CHUNK;
  double* wsm = wscr_all + (size_t)warp * WTile<CP>::WSCR;
  for (int l = 0; l < tr.L; ++l) {
    const int rows = tr.rows[l];
    const double* src = l == 0 ? in0 : arena + tr.soff[l];
    const int64_t lds = l == 0 ? ld0 : (rows | 1);
    double* vdst = l == 0 ? v0 : arena + tr.soff[l];
    const int64_t ldv = l == 0 ? ldv0 : (rows | 1);
    double* rnext = arena + tr.soff[l + 1];
    const int ldr = tr.rows[l + 1] | 1;
    for (int b = 0; b < tr.nblk[l]; ++b) {
      const int r0 = b * TB;
      const int nr = min(TB, rows - r0);
      int nwa, rpw;
      team_split(nr, nw, CHUNK, &nwa, &rpw);
      const bool staged = l == 0 && stage0 != nullptr;
      double* vb = staged ? stage0 : vdst + r0;
      const int ldvb = staged ? TB + 1 : (int)ldv;
      if (TEAM && nwa > 1) {  // warp-total slots of the inactive warps must read zero
        for (int i = threadIdx.x; i < 2 * 8 * CP; i += blockDim.x) tscr[i] = 0.0;
        __syncthreads();
      }
      if (warp < nwa) {
        double a[RT][CP];
#pragma unroll
        for (int t = 0; t < RT; ++t) {
          const int row = warp * rpw + t * 32 + lane;
#pragma unroll
          for (int p = 0; p < CP; ++p)
            a[t][p] = (t * 32 < rpw && row < nr && p < c) ? src[r0 + row + (int64_t)p * lds] : 0.0;
        }
        __syncwarp();
        if (!TEAM || nwa == 1)
          wqr_factor<CP, true, RTL>(a, nr, c, vb, ldvb, arena + tr.goff[l] + b * c, rnext + b * c, 1, ldr, wsm);
        else
          trows_factor<CP>(a, warp, nwa, rpw, nr, c, vb, ldvb, arena + tr.goff[l] + b * c, rnext + b * c, 1, ldr, wsm,
                           tscr);
      }
      __syncthreads();
      if (staged) {
        const int kb = min(nr, c);
        for (int idx = threadIdx.x; idx < nr * kb; idx += blockDim.x) {
          const int i = idx % nr, j = idx / nr;
          vdst[r0 + i + (int64_t)j * ldv] = stage0[i + j * (TB + 1)];
        }
        __syncthreads();
      }
    }
  }
}

// Back-application through levels L-1..0: Y_L (arena) holds the kb_top x q
// input; the level-0 result goes to out0 (ld ldo). With stage0 set the
// level-0 reflectors (global memory) are copied to shared memory first.
template <int CP, int RTLM = 0>
__device__ void wtree_apply(const WTree& tr, int c, int q, const double* v0, int64_t ldv0, double* arena,
                            double* wscr_all, double* tscr, double* out0, int64_t ldo, double* stage0) {
  constexpr int RT = WTile<CP>::RT, CHUNK = WTile<CP>::CHUNK;
  constexpr bool TEAM = RTLM == 0;
  constexpr int RTL = TEAM ? RT : RTLM;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int TB = nw * CHUNK;
  double* wsm = wscr_all + (size_t)warp * WTile<CP>::WSCR;
  auto stage_block = [&](int b) {  // cooperative, coalesced; ends with a CTA barrier
    const int r0 = b * TB;
    const int nr = min(TB, tr.rows[0] - r0);
    const int kb = min(nr, c);
    // batches of 16 independent loads per thread: the block comes from L2 /
    // HBM, and a load-store-load-store loop would pay the latency per element
    const int tot = nr * kb, nth = blockDim.x;
    for (int i0 = threadIdx.x; i0 < tot; i0 += nth * 16) {
      double tmp[16];
#pragma unroll
      for (int u = 0; u < 16; ++u) {
        const int idx = i0 + u * nth;
        tmp[u] = idx < tot ? v0[r0 + idx % nr + (int64_t)(idx / nr) * ldv0] : 0.0;
      }
#pragma unroll
      for (int u = 0; u < 16; ++u) {
        const int idx = i0 + u * nth;
        if (idx < tot) stage0[idx % nr + (idx / nr) * (TB + 1)] = tmp[u];
      }
    }
    __syncthreads();
  };
  const bool prestaged = stage0 != nullptr && tr.nblk[0] == 1;
  if (prestaged) stage_block(0);
  for (int l = tr.L - 1; l >= 0; --l) {
    const int rows = tr.rows[l];
    const double* vsrc = l == 0 ? v0 : arena + tr.soff[l];
    const int64_t ldv = l == 0 ? ldv0 : (rows | 1);
    const double* yin = arena + tr.yoff[l + 1];
    const int64_t ldyi = tr.rows[l + 1] | 1;
    double* yout = l == 0 ? out0 : arena + tr.yoff[l];
    const int64_t ldyo = l == 0 ? ldo : (rows | 1);
    for (int b = 0; b < tr.nblk[l]; ++b) {
      const int r0 = b * TB;
      const int nr = min(TB, rows - r0);
      const int kb = min(nr, c);
      int nwa, rpw;
      team_split(nr, nw, CHUNK, &nwa, &rpw);
      const bool staged = l == 0 && stage0 != nullptr;
      if (staged && !prestaged) stage_block(b);
      const double* vb = staged ? stage0 : vsrc + r0;
      const int ldvb = staged ? TB + 1 : (int)ldv;
      if (TEAM && nwa > 1) {
        for (int i = threadIdx.x; i < 2 * 8 * CP; i += blockDim.x) tscr[i] = 0.0;
        __syncthreads();
      }
      if (warp < nwa) {
        double y[RT][CP];
#pragma unroll
        for (int t = 0; t < RT; ++t) {
          const int row = warp * rpw + t * 32 + lane;
#pragma unroll
          for (int p = 0; p < CP; ++p)
            y[t][p] = (t * 32 < rpw && row < kb && p < q) ? yin[b * c + row + (int64_t)p * ldyi] : 0.0;
        }
        if (!TEAM || nwa == 1)
          wqr_apply<CP, RTL>(y, nr, kb, vb, ldvb, arena + tr.goff[l] + b * c, wsm);
        else
          trows_apply<CP>(y, warp, nwa, rpw, nr, kb, vb, ldvb, arena + tr.goff[l] + b * c, wsm, tscr);
#pragma unroll
        for (int t = 0; t < RT; ++t) {
          const int row = warp * rpw + t * 32 + lane;
#pragma unroll
          for (int p = 0; p < CP; ++p)
            if (t * 32 < rpw && row < nr && p < q) yout[r0 + row + (int64_t)p * ldyo] = y[t][p];
        }
      }
      __syncthreads();
    }
  }
}

struct WTopSmem {
  double* v0;     // (n0 | 1) x c level-0 reflectors
  double* arena;  // tree arena
  double* wscr;   // per-warp scratch
  double* tscr;   // row-team scratch
  double* B;      // CP x (CP + 1) Jacobi rows
  double* sig;
  double* dots;
  double* red;
  double* vpad;   // n0 (padding scratch, single-CTA targets)
  int* perm;
};

__host__ __device__ inline size_t wtop_doubles(int n0, int c, int CP, int nwarps, int chunk, bool pad) {
  const WTree tr = wtree_plan(n0, c, chunk);
  return (size_t)(n0 | 1) * c + tr.total + 4 + (size_t)nwarps * (CP == 16 ? WTile<16>::WSCR : WTile<32>::WSCR) + 20 * CP +
         (size_t)CP * (CP + 1) + CP + CP +
         64 + (pad ? n0 : 0) + CP / 2 + 2;
}

// Whole basis of a single-CTA target (nlevels == 0), or the top of a tall
// one (nlevels == 1: input = the stacked R of the factor kernel, output =
// the stacked Y for the apply kernel).
// RTLM > 0: targets of at most one warp block with 32 RTLM rows (every block of
// the tree is a single warp's): the row-team code is left out of the kernel,
// whose once-executed straight-line parts are instruction-fetch bound, and
// the FMA loops cover RTLM row groups. RTLM = 0: row teams, all row groups.
template <int CP, int RTLM>
__global__ void __launch_bounds__(kThreads) basis_wtree_kernel(const BasisTarget* __restrict__ targets,
                                                              const int* __restrict__ list) {
  constexpr int RT = WTile<CP>::RT, CHUNK = WTile<CP>::CHUNK;
  constexpr int LDB = CP + 1;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ BasisTarget T;
  stage_target(&T, &targets[list[blockIdx.x]]);
  __syncthreads();
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const bool tall = T.nlevels > 0;
  const QrLevel L = T.lv[T.nlevels];
  const int n0 = (int)L.n, c = T.c, r = T.r;
  const WTree tr = wtree_plan(n0, c, kWarps * CHUNK);
  WTopSmem s;
  {
    double* p = reinterpret_cast<double*>(smem_raw);
    s.v0 = p; p += ((size_t)(n0 | 1) * c + 1) & ~(size_t)1;
    s.arena = p; p += (tr.total + 1) & ~1;
    s.wscr = p; p += (size_t)kWarps * WTile<CP>::WSCR;  // 16-byte aligned (vector accesses)
    s.tscr = p; p += TeamRows<CP>::SCR;
    s.B = p; p += CP * LDB;
    s.sig = p; p += CP;
    s.dots = p; p += CP;
    s.red = p; p += 64;
    s.vpad = p; p += tall ? 0 : n0;
    s.perm = reinterpret_cast<int*>(p);
  }
  PROF_MARK_CTA(0);
  for (int i = tid; i < tr.persist; i += blockDim.x) s.arena[i] = 0.0;
  for (int i = tid; i < CP * LDB; i += blockDim.x) s.B[i] = 0.0;
  __syncthreads();
  wtree_factor<CP, RTLM>(tr, c, L.a, L.n, s.v0, n0 | 1, s.arena, s.wscr, s.tscr);
  PROF_MARK_CTA(1);
  // R^T = Q_1 R_1, then Jacobi on the rows of R_1 (warp 0)
  const int k = tr.rows[tr.L];
  int sweeps = 0;
  if (warp == 0) {
    const double* Rf = s.arena + tr.soff[tr.L];
    const int ldr = k | 1;
    double a[RT][CP];
#pragma unroll
    for (int t = 0; t < RT; ++t) {
      const int row = t * 32 + lane;  // column index of R
#pragma unroll
      for (int p = 0; p < CP; ++p) a[t][p] = (row < c && p < k) ? Rf[p + (size_t)row * ldr] : 0.0;
    }
    wqr_factor<CP, false, 1>(a, c, k, nullptr, 0, nullptr, s.B, LDB, 1, s.wscr);  // c <= 32 rows: one row group
    __syncwarp();
    PROF_MARK(2);
    if (CP == 16) sweeps = k <= 12 ? jacobi_rows_nov<4, 3>(s.B, LDB, k) : jacobi_rows_nov<4, 4>(s.B, LDB, k);
    else sweeps = k <= 20 ? jacobi_rows_nov<2, 10>(s.B, LDB, k)
                          : (k <= 24 ? jacobi_rows_nov<2, 12>(s.B, LDB, k) : jacobi_rows_nov<2, 16>(s.B, LDB, k));
  }
  __syncthreads();
  PROF_MARK_CTA(3);
  for (int i = tid; i < k; i += blockDim.x) {
    const double* bi = s.B + (size_t)i * LDB;
    s.sig[i] = sqrt(dot4(bi, bi, 0, k));
  }
  __syncthreads();
  for (int i = tid; i < k; i += blockDim.x) {
    int rank = 0;
    for (int j = 0; j < k; ++j) rank += (s.sig[j] > s.sig[i]) || (s.sig[j] == s.sig[i] && j < i);
    s.perm[rank] = i;
  }
  __syncthreads();
  const double smax = k > 0 ? s.sig[s.perm[0]] : 0.0;
  const double tol_rank = (double)srtt_dev::max64(T.n, (int64_t)c) * DBL_EPSILON * smax;
  int nrank = 0;
  for (int i = 0; i < k; ++i) nrank += s.sig[i] > tol_rank;
  const int q = min(nrank, r);
  if (tid == 0) {
    T.info[0] = q;
    T.info[1] = nrank;
    T.info[2] = sweeps;
  }
  if (T.sv)
    for (int i = tid; i < k; i += blockDim.x) T.sv[i] = s.sig[s.perm[i]];
  // Y_L = W(:, perm[:q]): normalised rows of the rotated R_1
  {
    double* yt = s.arena + tr.yoff[tr.L];
    const int ldy = k | 1;
    for (int idx = tid; idx < k * q; idx += blockDim.x) {
      const int i = idx % k, col = idx / k;
      const int src = s.perm[col];
      yt[i + (size_t)col * ldy] = s.B[(size_t)src * LDB + i] / s.sig[src];
    }
  }
  __syncthreads();
  PROF_MARK_CTA(4);
  wtree_apply<CP, RTLM>(tr, c, q, s.v0, n0 | 1, s.arena, s.wscr, s.tscr, tall ? L.y : T.u, tall ? L.n : T.n, nullptr);
  PROF_MARK_CTA(5);
  if (!tall && q < r)
    pad_columns(T.u, n0, n0, q, r, T.state0, T.draw_offset, (uint64_t)T.normal_base, s.vpad, s.dots, s.red);
  PROF_MARK_CTA(6);
  PROF_MARK_CTA(7);
}

// ===========================================================================
// Wide sketches (32 < c <= 64): a TEAM of 8 warps (one CTA) owns a row block
// of 256 rows. Lane l of every warp holds rows {l, l + 32, ...} (8 rows);
// the columns are dealt cyclically over the warps (warp w holds columns
// w, w + 8, ...: 8 local columns, 64 doubles per lane). In step j the owner
// warp of column j reduces its norm, publishes the masked column and
// (ss, alpha) through shared memory (double-buffered: one CTA barrier per
// step); then every warp forms its own dot products, reduce-scatters them
// inside the warp and updates its own columns; only the owner shifts its
// live columns one register to the left. The back-application needs no
// team communication at all: warp w applies all reflectors to its own 8
// columns of Y (wqr_apply<8>).
// ===========================================================================
constexpr int kTeamWarps = 8, kTeamCP = 8, kTeamRT = 8, kTeamRows = 256;

struct TeamScratch {
  double* xs;    // 2 x 256 masked pivot column
  double* hdr;   // 2 x 2 (ss, alpha)
  double* wscr;  // kTeamWarps x WTile<8>::WSCR
};
constexpr int kTeamScratchDoubles = 2 * kTeamRows + 4 + kTeamWarps * WTile<kTeamCP>::WSCR;

__device__ __forceinline__ TeamScratch team_scratch(double* p) {
  TeamScratch t;
  t.xs = p;
  t.hdr = p + 2 * kTeamRows;
  t.wscr = t.hdr + 4;
  return t;
}

// Team Householder QR of the block in registers (nr rows, c columns; warp w
// local column p = global column 8 p + w). All destinations are shared
// memory: reflector j to vout[row + j * ldv] (STOREV), g_j to gout[j], row j
// of R to rout[j * rs + col * cs].
template <bool STOREV>
__device__ void tqr_factor(double (&a)[kTeamRT][kTeamCP], int nr, int c, double* vout, int ldv, double* gout,
                           double* rout, int rs, int cs, const TeamScratch& ts) {
  constexpr int RT = kTeamRT, CP = kTeamCP, NW = kTeamWarps, LPC = 32 / CP;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int mycol = lane / LPC;
  double* wsm = ts.wscr + (size_t)warp * WTile<CP>::WSCR;
  double* red = wsm;
  double* prow = wsm + WTile<CP>::RED;
  double* csm = prow + CP;
  const int kb = nr < c ? nr : c;
  const uint32_t ra0 = smem_addr(rout);
  const uint32_t va0 = STOREV ? smem_addr(vout) + 8u * lane : 0u;
  const uint32_t ga0 = STOREV ? smem_addr(gout) : 0u;
  int sh = 0;  // live columns of this warp start at global column NW * sh + warp
  for (int j = 0; j < kb; ++j) {
    const int wj = j % NW, lj = j & 31, tj = j >> 5;
    double* xsb = ts.xs + (j & 1) * kTeamRows;
    double* hb = ts.hdr + (j & 1) * 2;
    double xm[RT];
    if (warp == wj) {
      double part = 0.0, al = 0.0;
#pragma unroll
      for (int t = 0; t < RT; ++t) {
        xm[t] = (t * 32 + lane > j) ? a[t][0] : 0.0;
        part = fma(xm[t], xm[t], part);
        if (tj == t) al = a[t][0];
        xsb[t * 32 + lane] = xm[t];
      }
      part = warp_sum(part);
      al = __shfl_sync(0xffffffffu, al, lj);
      if (lane == 0) {
        hb[0] = part;
        hb[1] = al;
      }
    }
    __syncthreads();
    if (warp != wj) {
#pragma unroll
      for (int t = 0; t < RT; ++t) xm[t] = xsb[t * 32 + lane];
    }
    const double ss = hb[0], alpha = hb[1];
    {
      double2* pdst = reinterpret_cast<double2*>(lane == lj ? prow : csm + CP);
#pragma unroll
      for (int t = 0; t < 2; ++t)  // j < 64: the pivot row is one of the first 64
        if (tj == t) {
#pragma unroll
          for (int p = 0; p < CP; p += 2) pdst[p / 2] = make_double2(a[t][p], a[t][p + 1]);
        }
    }
    double D[CP];
#pragma unroll
    for (int p = 0; p < CP; ++p) {
      double s0 = 0.0, s1 = 0.0;
#pragma unroll
      for (int t = 0; t < RT; t += 2) {
        s0 = fma(xm[t], a[t][p], s0);
        s1 = fma(xm[t + 1], a[t + 1][p], s1);
      }
      D[p] = s0 + s1;
    }
    const double dtot = reduce_scatter_sm<CP>(D, red, lane);
    double beta = alpha, ujj = 0.0, g = 0.0;
    if (ss != 0.0) {
      const double n2 = fma(alpha, alpha, ss);
      const double rn = rsqrt(n2);
      const double nrm = n2 * rn;
      beta = -copysign(nrm, alpha);
      ujj = alpha - beta;
      g = rn * __drcp_rn(fabs(ujj));
    }
    const double arow = prow[mycol];
    const double cl = g * fma(ujj, arow, dtot);
    if (lane % LPC == 0) {
      csm[mycol] = cl;
      const int col = NW * (mycol + sh) + warp;
      if (col < c) sts_f64(ra0 + 8u * (uint32_t)(j * rs + col * cs), col == j ? beta : arow - cl * ujj);
    }
    if (STOREV && warp == wj) {
#pragma unroll
      for (int t = 0; t < RT; ++t) {
        const int row = t * 32 + lane;
        if (row < nr) sts_f64(va0 + 8u * (uint32_t)(j * ldv) + 256u * t, row > j ? xm[t] : (row == j ? ujj : 0.0));
      }
      if (lane == 0) sts_f64(ga0 + 8u * j, g);
    }
    __syncwarp();
    if (warp == wj) {
#pragma unroll
      for (int p = 0; p < CP; p += 2) {
        const double2 e = reinterpret_cast<const double2*>(csm)[p / 2];
#pragma unroll
        for (int t = 0; t < RT; ++t) {
          if (p > 0) a[t][p - 1] = fma(-e.x, xm[t], a[t][p]);
          a[t][p] = fma(-e.y, xm[t], a[t][p + 1]);
        }
      }
#pragma unroll
      for (int t = 0; t < RT; ++t) a[t][CP - 1] = 0.0;
      ++sh;
    } else {
#pragma unroll
      for (int p = 0; p < CP; p += 2) {
        const double2 e = reinterpret_cast<const double2*>(csm)[p / 2];
#pragma unroll
        for (int t = 0; t < RT; ++t) {
          a[t][p] = fma(-e.x, xm[t], a[t][p]);
          a[t][p + 1] = fma(-e.y, xm[t], a[t][p + 1]);
        }
      }
    }
    __syncwarp();
  }
  __syncthreads();
}

// Register block of the team: element (row, global column NW p + w) from
// src[row * rstride + col * cstride].
__device__ __forceinline__ void team_load(double (&a)[kTeamRT][kTeamCP], const double* src, int64_t rstride,
                                          int64_t cstride, int nr, int c) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int t = 0; t < kTeamRT; ++t) {
    const int row = t * 32 + lane;
#pragma unroll
    for (int p = 0; p < kTeamCP; ++p) {
      const int col = kTeamWarps * p + warp;
      a[t][p] = (row < nr && col < c) ? src[row * rstride + col * cstride] : 0.0;
    }
  }
}

// Back-application of one team block: warp w applies the kb reflectors (vst,
// ld ldv, shared memory) to columns [8 w, 8 w + 8) of Y. Input: the kb x q
// matrix yin (ld ldyi), zero below; output rows to yout (ld ldyo).
__device__ void team_apply(int nr, int kb, int q, const double* vst, int ldv, const double* gst, const double* yin,
                           int64_t ldyi, double* yout, int64_t ldyo, const TeamScratch& ts) {
  constexpr int RT = kTeamRT, CP = kTeamCP;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int c0 = warp * CP;
  if (c0 < q) {
    double y[RT][CP];
#pragma unroll
    for (int t = 0; t < RT; ++t) {
      const int row = t * 32 + lane;
#pragma unroll
      for (int p = 0; p < CP; ++p) y[t][p] = (row < kb && c0 + p < q) ? yin[row + (int64_t)(c0 + p) * ldyi] : 0.0;
    }
    wqr_apply<CP>(y, nr, kb, vst, ldv, gst, ts.wscr + (size_t)warp * WTile<CP>::WSCR);
#pragma unroll
    for (int t = 0; t < RT; ++t) {
      const int row = t * 32 + lane;
#pragma unroll
      for (int p = 0; p < CP; ++p)
        if (row < nr && c0 + p < q) yout[row + (int64_t)(c0 + p) * ldyo] = y[t][p];
    }
  }
}

// One-sided Jacobi on the rows of B (k x k, row-major, ld ldb, shared
// memory), rotations not accumulated, all warps of the CTA: 4-lane groups
// take the round-robin pairs of a round, one CTA barrier per round.
template <int E>
__device__ int jacobi_rows_cta(double* B, int ldb, int k, const unsigned short* pairs) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int gid = warp * 8 + (lane >> 2), gl = lane & 3;
  const int kk = (k + 1) & ~1;
  const int npairs = kk / 2;
  const double tol2 = 4.0 * DBL_EPSILON * DBL_EPSILON;
  if (k < 2) return 0;
  int sweep = 0;
  for (; sweep < 80; ++sweep) {
    int rotated = 0, big = 0;
    for (int rd = 0; rd < kk - 1; ++rd) {
      int p = 0, q = 0;
      bool valid = gid < npairs;
      if (valid) {
        const unsigned short e = pairs[rd * npairs + gid];
        p = e & 0xff;
        q = e >> 8;
        valid = q < k;
      }
      double* bp = B + (size_t)p * ldb;
      double* bq = B + (size_t)q * ldb;
      double x[E], y[E];
      double app = 0.0, aqq = 0.0, apq = 0.0;
#pragma unroll
      for (int e = 0; e < E; ++e) {
        const int j = gl + 4 * e;
        const bool in = valid && j < k;
        x[e] = in ? bp[j] : 0.0;
        y[e] = in ? bq[j] : 0.0;
        app = fma(x[e], x[e], app);
        aqq = fma(y[e], y[e], aqq);
        apq = fma(x[e], y[e], apq);
      }
      app += __shfl_xor_sync(0xffffffffu, app, 1);
      aqq += __shfl_xor_sync(0xffffffffu, aqq, 1);
      apq += __shfl_xor_sync(0xffffffffu, apq, 1);
      app += __shfl_xor_sync(0xffffffffu, app, 2);
      aqq += __shfl_xor_sync(0xffffffffu, aqq, 2);
      apq += __shfl_xor_sync(0xffffffffu, apq, 2);
      const double a2 = apq * apq, pq = app * aqq;
      if (valid && apq != 0.0 && a2 > tol2 * pq) {
        double cs, sn;
        jacobi_rotation(app, aqq, apq, &cs, &sn);
#pragma unroll
        for (int e = 0; e < E; ++e) {
          const int j = gl + 4 * e;
          if (j < k) {
            bp[j] = cs * x[e] - sn * y[e];
            bq[j] = sn * x[e] + cs * y[e];
          }
        }
        rotated = 1;
        if (a2 > 1e-13 * pq || fabs(sn) > 1e-6) big = 1;
      }
      __syncthreads();
    }
    const int any = __syncthreads_or(rotated);
    if (!any) break;
    if (!__syncthreads_or(big)) { ++sweep; break; }
  }
  __syncthreads();
  return sweep;
}

struct WideTopSmem {
  double* v;      // (m | 1) x c reflectors of the top block
  double* g;      // c
  double* rb;     // c x (c | 1): R (column-major), then R_1 / the Jacobi rows (row-major)
  double* ytop;   // (c | 1) x r
  double* scr;    // team scratch
  double* sig;
  double* dots;
  double* red;
  double* vpad;   // m (padding scratch, single-block targets)
  int* perm;
};

__host__ __device__ inline size_t wide_top_doubles(int m, int c, int r, bool pad) {
  return (size_t)(m | 1) * c + 1 + (c + 2) + (size_t)c * (c | 1) + 1 + (size_t)(c | 1) * r + 1 + kTeamScratchDoubles + c + c +
         64 + (pad ? m : 0) + c / 2 + 4;
}

// Top of a wide target (or all of a single-block one): team QR of the top
// block, R^T = Q_1 R_1, CTA Jacobi on the rows of R_1, rank decision,
// back-application through the top block.
__global__ void __launch_bounds__(kThreads) basis_wide_top_kernel(const BasisTarget* __restrict__ targets,
                                                                 const int* __restrict__ list) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ BasisTarget T;
  __shared__ unsigned short pairs[64 * 32];
  stage_target(&T, &targets[list[blockIdx.x]]);
  __syncthreads();
  const int tid = threadIdx.x;
  const int top = T.nlevels;
  const QrLevel L = T.lv[top];
  const int m = (int)L.n, c = T.c, r = T.r;
  const int k = min(m, c);
  const int ldv = m | 1, ldr = c | 1;
  WideTopSmem s;
  {
    double* p = reinterpret_cast<double*>(smem_raw);
    s.v = p; p += ((size_t)ldv * c + 1) & ~(size_t)1;
    s.g = p; p += (c + 2) & ~1;
    s.rb = p; p += ((size_t)c * ldr + 1) & ~(size_t)1;
    s.ytop = p; p += ((size_t)ldr * r + 1) & ~(size_t)1;
    s.scr = p; p += kTeamScratchDoubles;
    s.sig = p; p += c;
    s.dots = p; p += c;
    s.red = p; p += 64;
    s.vpad = p; p += top == 0 ? m : 0;
    s.perm = reinterpret_cast<int*>(p);
  }
  const TeamScratch ts = team_scratch(s.scr);
  PROF_MARK_CTA(8);
  for (int i = tid; i < c * ldr; i += blockDim.x) s.rb[i] = 0.0;
  build_pairs(pairs, (k + 1) & ~1);
  __syncthreads();
  {
    double a[kTeamRT][kTeamCP];
    team_load(a, L.a, 1, L.n, m, c);
    tqr_factor<true>(a, m, c, s.v, ldv, s.g, s.rb, 1, ldr, ts);  // R(j, col) at rb[j + col * ldr]
  }
  PROF_MARK_CTA(9);
  {
    // second QR on R^T (c x k): element (row, col) = R(col, row); R_1 (k x k) row-major over the same storage
    double a[kTeamRT][kTeamCP];
    team_load(a, s.rb, ldr, 1, c, k);
    __syncthreads();
    for (int i = tid; i < c * ldr; i += blockDim.x) s.rb[i] = 0.0;
    __syncthreads();
    tqr_factor<false>(a, c, k, nullptr, 0, nullptr, s.rb, ldr, 1, ts);  // R_1(j, col) at rb[j * ldr + col]
  }
  const int sweeps = k <= 32 ? jacobi_rows_cta<8>(s.rb, ldr, k, pairs)
                     : (k <= 48 ? jacobi_rows_cta<12>(s.rb, ldr, k, pairs) : jacobi_rows_cta<16>(s.rb, ldr, k, pairs));
  PROF_MARK_CTA(10);
  const int lane = tid & 31, warp = tid >> 5;
  for (int i = warp; i < k; i += kWarps) {
    double ss = 0.0;
    for (int j = lane; j < k; j += 32) ss += s.rb[(size_t)i * ldr + j] * s.rb[(size_t)i * ldr + j];
    ss = warp_sum(ss);
    if (lane == 0) s.sig[i] = sqrt(ss);
  }
  __syncthreads();
  for (int i = tid; i < k; i += blockDim.x) {
    int rank = 0;
    for (int j = 0; j < k; ++j) rank += (s.sig[j] > s.sig[i]) || (s.sig[j] == s.sig[i] && j < i);
    s.perm[rank] = i;
  }
  __syncthreads();
  const double smax = k > 0 ? s.sig[s.perm[0]] : 0.0;
  const double tol = (double)srtt_dev::max64(T.n, (int64_t)c) * DBL_EPSILON * smax;
  int nrank = 0;
  for (int i = 0; i < k; ++i) nrank += s.sig[i] > tol;
  const int q = min(nrank, r);
  if (tid == 0) {
    T.info[0] = q;
    T.info[1] = nrank;
    T.info[2] = sweeps;
  }
  if (T.sv)
    for (int i = tid; i < k; i += blockDim.x) T.sv[i] = s.sig[s.perm[i]];
  for (int idx = tid; idx < k * q; idx += blockDim.x) {
    const int i = idx % k, col = idx / k;
    const int src = s.perm[col];
    s.ytop[i + (size_t)col * ldr] = s.rb[(size_t)src * ldr + i] / s.sig[src];
  }
  __syncthreads();
  PROF_MARK_CTA(11);
  team_apply(m, k, q, s.v, ldv, s.g, s.ytop, ldr, top == 0 ? T.u : L.y, top == 0 ? T.n : L.n, ts);
  __syncthreads();
  PROF_MARK_CTA(12);
  if (top == 0 && q < r)
    pad_columns(T.u, m, m, q, r, T.state0, T.draw_offset, (uint64_t)T.normal_base, s.vpad, s.dots, s.red);
  PROF_MARK_CTA(13);
}

__host__ __device__ inline size_t wide_level_doubles(int mb, int c) {
  return (size_t)(mb | 1) * c + 1 + (c + 2) + (size_t)c * (c | 1) + 1 + kTeamScratchDoubles + 4;
}

// One level below the top of a wide target: CTA (target, b) factors row
// block b in place (reflectors u_j whole, g in L.tau) and stacks its R.
__global__ void __launch_bounds__(kThreads) basis_wide_factor_kernel(const BasisTarget* __restrict__ targets,
                                                                    const int2* __restrict__ map, int level) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ BasisTarget T;
  const int2 tb = map[blockIdx.x];
  stage_target(&T, &targets[tb.x]);
  __syncthreads();
  const QrLevel L = T.lv[level];
  const QrLevel P = T.lv[level + 1];
  const int b = tb.y, c = T.c;
  const int64_t r0 = (int64_t)b * L.blk_rows;
  const int mb = (int)srtt_dev::min64(L.blk_rows, L.n - r0);
  const int kb = min(mb, c);
  const int ldv = mb | 1, ldr = c | 1;
  double* p = reinterpret_cast<double*>(smem_raw);
  double* vst = p; p += ((size_t)ldv * c + 1) & ~(size_t)1;
  double* gst = p; p += (c + 2) & ~1;
  double* rst = p; p += ((size_t)c * ldr + 1) & ~(size_t)1;
  const TeamScratch ts = team_scratch(p);
  for (int i = threadIdx.x; i < c * ldr; i += blockDim.x) rst[i] = 0.0;
  for (int i = threadIdx.x; i < c; i += blockDim.x) gst[i] = 0.0;
  __syncthreads();
  {
    double a[kTeamRT][kTeamCP];
    team_load(a, L.a + r0, 1, L.n, mb, c);
    tqr_factor<true>(a, mb, c, vst, ldv, gst, rst, 1, ldr, ts);
  }
  for (int idx = threadIdx.x; idx < mb * kb; idx += blockDim.x) {
    const int i = idx % mb, j = idx / mb;
    L.a[(int64_t)j * L.n + r0 + i] = vst[i + (size_t)j * ldv];
  }
  for (int j = threadIdx.x; j < c; j += blockDim.x) L.tau[(int64_t)b * c + j] = gst[j];
  for (int idx = threadIdx.x; idx < c * c; idx += blockDim.x) {
    const int i = idx % c, j = idx / c;
    P.a[(int64_t)j * P.n + (int64_t)b * c + i] = i < kb ? rst[i + (size_t)j * ldr] : 0.0;
  }
}

__global__ void __launch_bounds__(kThreads) basis_wide_apply_kernel(const BasisTarget* __restrict__ targets,
                                                                   const int2* __restrict__ map, int level) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ BasisTarget T;
  const int2 tb = map[blockIdx.x];
  stage_target(&T, &targets[tb.x]);
  __syncthreads();
  const QrLevel L = T.lv[level];
  const QrLevel P = T.lv[level + 1];
  const int b = tb.y, c = T.c;
  const int q = T.info[0];
  const int64_t r0 = (int64_t)b * L.blk_rows;
  const int mb = (int)srtt_dev::min64(L.blk_rows, L.n - r0);
  const int kb = min(mb, c);
  const int ldv = mb | 1;
  double* p = reinterpret_cast<double*>(smem_raw);
  double* vst = p; p += ((size_t)ldv * c + 1) & ~(size_t)1;
  double* gst = p; p += (c + 2) & ~1;
  p += ((size_t)c * (c | 1) + 1) & ~(size_t)1;
  const TeamScratch ts = team_scratch(p);
  {  // 8 independent loads per thread and pass (the block comes from L2 / HBM)
    const int tot = mb * kb, nth = blockDim.x;
    for (int i0 = threadIdx.x; i0 < tot; i0 += nth * 8) {
      double tmp[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int idx = i0 + u * nth;
        tmp[u] = idx < tot ? L.a[(int64_t)(idx / mb) * L.n + r0 + idx % mb] : 0.0;
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int idx = i0 + u * nth;
        if (idx < tot) vst[idx % mb + (size_t)(idx / mb) * ldv] = tmp[u];
      }
    }
  }
  for (int j = threadIdx.x; j < c; j += blockDim.x) gst[j] = L.tau[(int64_t)b * c + j];
  __syncthreads();
  team_apply(mb, kb, q, vst, ldv, gst, P.y + (int64_t)b * c, P.n, L.y + r0, L.n, ts);
}

// ===========================================================================
// Generic basis kernel (c > 64, up to SRTT_MAX_SKETCH_COLS): the reference
// bounds ranks only by the extents (tucker.hpp:184-197), so sketches wider
// than the register kernels cover still get a basis: one CTA per target,
// everything in global memory (Z factored in place; R rows, the rotation
// accumulator and tau in T.vup), the shared-memory algorithms of the top
// kernel (QRCP Householder, 4-lane Jacobi with accumulated rotations, warp
// back-application). Slow (no TSQR, no registers) but exact to the same
// tolerances; it exists for contract parity, not for the BASELINE configs.
// ===========================================================================
__global__ void __launch_bounds__(kThreads) basis_generic_kernel(const BasisTarget* __restrict__ targets,
                                                                const int* __restrict__ list) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ BasisTarget T;
  stage_target(&T, &targets[list[blockIdx.x]]);
  __syncthreads();
  const int64_t n = T.n;
  const int m = (int)n, c = T.c, r = T.r;
  const int k = min(m, c);
  const int kk = (k + 1) & ~1;
  double* vn = reinterpret_cast<double*>(smem_raw);
  double* sig = vn + c;
  double* dots = sig + c;
  double* red = dots + c;
  double* scal_beta = red + 64;
  int* perm = reinterpret_cast<int*>(scal_beta + 2);
  unsigned short* pairs = reinterpret_cast<unsigned short*>(perm + c + (c & 1));
  double* A = T.lv[0].a;
  double* B = T.vup;
  double* V = B + (size_t)k * c;
  double* tau = V + (size_t)k * k;
  double* vpad = tau + c;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  householder_qr(A, m, c, m, tau, scal_beta, vn);
  __syncthreads();
  for (int idx = threadIdx.x; idx < k * c; idx += blockDim.x) {
    const int i = idx / c, j = idx % c;
    B[idx] = (j >= i) ? A[(size_t)j * n + i] : 0.0;
  }
  for (int idx = threadIdx.x; idx < k * k; idx += blockDim.x) V[idx] = (idx % k == idx / k) ? 1.0 : 0.0;
  build_pairs(pairs, kk);
  __syncthreads();
  const int sweeps = jacobi_rows_g4(B, c, k, c, V, k, pairs);
  for (int i = warp; i < k; i += kWarps) {
    double ss = 0.0;
    for (int j = lane; j < c; j += 32) ss += B[(size_t)i * c + j] * B[(size_t)i * c + j];
    ss = warp_sum(ss);
    if (lane == 0) sig[i] = sqrt(ss);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < k; i += blockDim.x) {
    int rank = 0;
    for (int j = 0; j < k; ++j) rank += (sig[j] > sig[i]) || (sig[j] == sig[i] && j < i);
    perm[rank] = i;
  }
  __syncthreads();
  const double smax = k > 0 ? sig[perm[0]] : 0.0;
  const double tol = (double)srtt_dev::max64(n, (int64_t)c) * DBL_EPSILON * smax;
  int nrank = 0;
  for (int i = 0; i < k; ++i) nrank += sig[i] > tol;
  const int q = min(nrank, r);
  if (threadIdx.x == 0) {
    T.info[0] = q;
    T.info[1] = nrank;
    T.info[2] = sweeps;
  }
  if (T.sv)
    for (int i = threadIdx.x; i < k; i += blockDim.x) T.sv[i] = sig[perm[i]];
  for (int64_t idx = threadIdx.x; idx < n * q; idx += blockDim.x) {
    const int64_t i = idx % n, col = idx / n;
    T.u[idx] = (i < k) ? V[(size_t)perm[col] * k + i] : 0.0;
  }
  __syncthreads();
  for (int col = warp; col < q; col += kWarps) apply_q_warp(A, m, k, m, tau, T.u + (size_t)col * n);
  __syncthreads();
  if (q < r) pad_columns(T.u, n, n, q, r, T.state0, T.draw_offset, (uint64_t)T.normal_base, vpad, dots, red);
}

constexpr int kWfThreads = 128;  // factor / apply CTAs of tall targets: one warp per SM sub-partition

// Tall targets, level 0: CTA (target, i) factors rows [i * rpc, ...) of Z in
// place, keeps its upper tree levels in T.vup and stacks its R.
template <int CP>
__global__ void __launch_bounds__(kWfThreads) basis_wfactor_kernel(const BasisTarget* __restrict__ targets,
                                                                  const int2* __restrict__ map) {
  constexpr int CHUNK = WTile<CP>::CHUNK;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ BasisTarget T;
  const int2 tb = map[blockIdx.x];
  stage_target(&T, &targets[tb.x]);
  __syncthreads();
  const QrLevel L = T.lv[0];
  const QrLevel P = T.lv[1];
  const int c = T.c;
  const int64_t r0 = (int64_t)tb.y * L.blk_rows;
  const int nrows = (int)srtt_dev::min64(L.blk_rows, L.n - r0);
  const WTree tr = wtree_plan(nrows, c, (kWfThreads / 32) * CHUNK);
  double* arena = reinterpret_cast<double*>(smem_raw);
  double* wscr = arena + ((tr.persist + 1) & ~1);
  double* tscr = wscr + (size_t)(kWfThreads / 32) * WTile<CP>::WSCR;
  double* stage = tscr + TeamRows<CP>::SCR;
  for (int i = threadIdx.x; i < tr.persist; i += blockDim.x) arena[i] = 0.0;
  __syncthreads();
  wtree_factor<CP>(tr, c, L.a + r0, L.n, L.a + r0, L.n, arena, wscr, tscr, stage);
  const int k = tr.rows[tr.L];
  const double* Rf = arena + tr.soff[tr.L];
  for (int idx = threadIdx.x; idx < k * c; idx += blockDim.x) {
    const int i = idx % k, j = idx / k;
    P.a[(int64_t)j * P.n + (int64_t)tb.y * c + i] = Rf[i + (size_t)j * (k | 1)];
  }
  double* up = T.vup + (int64_t)tb.y * T.vup_stride;
  for (int i = threadIdx.x; i < tr.persist; i += blockDim.x) up[i] = arena[i];
}

template <int CP>
__global__ void __launch_bounds__(kWfThreads) basis_wapply_kernel(const BasisTarget* __restrict__ targets,
                                                                 const int2* __restrict__ map) {
  constexpr int CHUNK = WTile<CP>::CHUNK;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ BasisTarget T;
  const int2 tb = map[blockIdx.x];
  stage_target(&T, &targets[tb.x]);
  __syncthreads();
  const QrLevel L = T.lv[0];
  const QrLevel P = T.lv[1];
  const int c = T.c;
  const int q = T.info[0];
  const int64_t r0 = (int64_t)tb.y * L.blk_rows;
  const int nrows = (int)srtt_dev::min64(L.blk_rows, L.n - r0);
  const WTree tr = wtree_plan(nrows, c, (kWfThreads / 32) * CHUNK);
  double* arena = reinterpret_cast<double*>(smem_raw);
  double* wscr = arena + ((tr.total + 1) & ~1);
  double* tscr = wscr + (size_t)(kWfThreads / 32) * WTile<CP>::WSCR;
  double* stage = tscr + TeamRows<CP>::SCR;
  const double* up = T.vup + (int64_t)tb.y * T.vup_stride;
  for (int i0 = threadIdx.x; i0 < tr.persist; i0 += blockDim.x * 8) {  // 8 loads in flight per thread
    double tmp[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) tmp[u] = i0 + u * (int)blockDim.x < tr.persist ? up[i0 + u * blockDim.x] : 0.0;
#pragma unroll
    for (int u = 0; u < 8; ++u)
      if (i0 + u * (int)blockDim.x < tr.persist) arena[i0 + u * blockDim.x] = tmp[u];
  }
  const int k = tr.rows[tr.L];
  double* yt = arena + tr.yoff[tr.L];
  for (int idx = threadIdx.x; idx < k * q; idx += blockDim.x) {
    const int i = idx % k, col = idx / k;
    yt[i + (size_t)col * (k | 1)] = P.y[(int64_t)col * P.n + (int64_t)tb.y * c + i];
  }
  __syncthreads();
  wtree_apply<CP>(tr, c, q, L.a + r0, L.n, arena, wscr, tscr, L.y + r0, L.n, stage);
}

}  // namespace

size_t srtt_basis_top_smem(int m, int c, int r) {
  const int k = m < c ? m : c;
  size_t doubles = (size_t)kWarps * 32 + 32 + (size_t)c + (size_t)(m | 1) * c + (size_t)k * c + (size_t)k * k + (size_t)m * r + c + k + r + 32 + m + 2;
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

// Variant of a small target (see basis_small_kernel).
int srtt_basis_small_variant(int m, int c) {
  const int k = m < c ? m : c;
  if (c <= 12) return 4;              // CTA kernel, Jacobi <4, 3> (C2: c = 11)
  if (c <= 16) return 0;              // CTA kernel, Jacobi <4, 4>
  if (k <= 24 && c <= 24) return 3;   // CTA kernel, Jacobi <2, 12> (C3: c = 20)
  if (k <= 32 && c <= 32) return 1;   // CTA kernel, Jacobi <2, 16>
  return 2;                           // <0, 0, 0>
}

cudaError_t srtt_launch_basis_small(int variant, const BasisTarget* d_targets, const int* d_list, int n, size_t smem,
                                    cudaStream_t stream) {
  if (n <= 0) return cudaSuccess;
  switch (variant) {
    case 0:
      SRTT_ENSURE_SMEM((basis_cta_kernel<4, 4>), smem);
      basis_cta_kernel<4, 4><<<n, kThreads, smem, stream>>>(d_targets, d_list);
      break;
    case 1:
      SRTT_ENSURE_SMEM((basis_cta_kernel<2, 16>), smem);
      basis_cta_kernel<2, 16><<<n, kThreads, smem, stream>>>(d_targets, d_list);
      break;
    case 4:
      SRTT_ENSURE_SMEM((basis_cta_kernel<4, 3>), smem);
      basis_cta_kernel<4, 3><<<n, kThreads, smem, stream>>>(d_targets, d_list);
      break;
    case 3:
      SRTT_ENSURE_SMEM((basis_cta_kernel<2, 12>), smem);
      basis_cta_kernel<2, 12><<<n, kThreads, smem, stream>>>(d_targets, d_list);
      break;
    default:
      SRTT_ENSURE_SMEM(basis_small_kernel, smem);
      basis_small_kernel<<<n, 32, smem, stream>>>(d_targets, d_list);
      break;
  }
  return cudaGetLastError();
}

int srtt_basis_top_variant(int c) { return c <= 16 ? 0 : (c <= 32 ? 1 : 2); }

cudaError_t srtt_launch_basis_top(int variant, const BasisTarget* d_targets, const int* d_list, int ntargets,
                                  size_t smem, cudaStream_t stream) {
  if (ntargets <= 0) return cudaSuccess;
  switch (variant) {
    case 0:
      SRTT_ENSURE_SMEM((basis_top_kernel<4, 4>), smem);
      basis_top_kernel<4, 4><<<ntargets, kThreads, smem, stream>>>(d_targets, d_list);
      break;
    case 1:
      SRTT_ENSURE_SMEM((basis_top_kernel<2, 16>), smem);
      basis_top_kernel<2, 16><<<ntargets, kThreads, smem, stream>>>(d_targets, d_list);
      break;
    default:
      SRTT_ENSURE_SMEM((basis_top_kernel<0, 0>), smem);
      basis_top_kernel<0, 0><<<ntargets, kThreads, smem, stream>>>(d_targets, d_list);
      break;
  }
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


// ---- register-tree path (c <= 32): planning helpers and launchers ----------
int srtt_wtree_cp(int c) { return c <= 16 ? 16 : (c <= 32 ? 32 : 0); }
int srtt_wtree_chunk(int cp) { return cp == 16 ? WTile<16>::CHUNK : WTile<32>::CHUNK; }
int srtt_wtree_factor_threads() { return kWfThreads; }

size_t srtt_wtree_top_smem(int n0, int c, bool pad) {
  const int cp = srtt_wtree_cp(c);
  return wtop_doubles(n0, c, cp, kWarps, kWarps * srtt_wtree_chunk(cp), pad) * sizeof(double) + 64;
}

int64_t srtt_wtree_persist_doubles(int rows, int c) {
  const int cp = srtt_wtree_cp(c);
  return wtree_plan(rows, c, (kWfThreads / 32) * srtt_wtree_chunk(cp)).persist;
}

size_t srtt_wtree_factor_smem(int rows, int c) {
  const int cp = srtt_wtree_cp(c);
  const int tb = (kWfThreads / 32) * srtt_wtree_chunk(cp);
  const WTree tr = wtree_plan(rows, c, tb);
  return ((size_t)tr.persist + 2 + (size_t)(kWfThreads / 32) * (cp == 16 ? WTile<16>::WSCR : WTile<32>::WSCR) + 20 * cp +
          (size_t)(tb + 1) * c) * sizeof(double);
}

size_t srtt_wtree_apply_smem(int rows, int c) {
  const int cp = srtt_wtree_cp(c);
  const int chunk = srtt_wtree_chunk(cp);
  const int tb = (kWfThreads / 32) * chunk;
  const WTree tr = wtree_plan(rows, c, tb);
  return ((size_t)tr.total + 2 + (size_t)(kWfThreads / 32) * (cp == 16 ? WTile<16>::WSCR : WTile<32>::WSCR) + 20 * cp +
          (size_t)(tb + 1) * c) * sizeof(double);
}

// mode 0: row teams (blocks taller than one warp's); r > 0: a single-warp-block
// target of at most 32 r rows (r = 1, 2, 4 for c <= 16; 1, 2 for c <= 32)
cudaError_t srtt_launch_wtree_top(int cp, int mode, const BasisTarget* d_targets, const int* d_list, int n, size_t smem,
                                  cudaStream_t stream) {
  if (n <= 0) return cudaSuccess;
#define SRTT_WTOP(CPV, MV)                                                                   \
  do {                                                                                       \
    SRTT_ENSURE_SMEM((basis_wtree_kernel<CPV, MV>), smem);                                   \
    basis_wtree_kernel<CPV, MV><<<n, kThreads, smem, stream>>>(d_targets, d_list);           \
  } while (0)
  if (cp == 16) {
    switch (mode) {
      case 0: SRTT_WTOP(16, 0); break;
      case 1: SRTT_WTOP(16, 1); break;
      case 2: SRTT_WTOP(16, 2); break;
      default: SRTT_WTOP(16, 4); break;
    }
  } else {
    switch (mode) {
      case 0: SRTT_WTOP(32, 0); break;
      case 1: SRTT_WTOP(32, 1); break;
      default: SRTT_WTOP(32, 2); break;
    }
  }
#undef SRTT_WTOP
  return cudaGetLastError();
}

cudaError_t srtt_launch_wtree_factor(int cp, const BasisTarget* d_targets, const int2* d_map, int nctas, size_t smem,
                                     cudaStream_t stream) {
  if (nctas <= 0) return cudaSuccess;
  if (cp == 16) {
    SRTT_ENSURE_SMEM((basis_wfactor_kernel<16>), smem);
    basis_wfactor_kernel<16><<<nctas, kWfThreads, smem, stream>>>(d_targets, d_map);
  } else {
    SRTT_ENSURE_SMEM((basis_wfactor_kernel<32>), smem);
    basis_wfactor_kernel<32><<<nctas, kWfThreads, smem, stream>>>(d_targets, d_map);
  }
  return cudaGetLastError();
}

cudaError_t srtt_launch_wtree_apply(int cp, const BasisTarget* d_targets, const int2* d_map, int nctas, size_t smem,
                                    cudaStream_t stream) {
  if (nctas <= 0) return cudaSuccess;
  if (cp == 16) {
    SRTT_ENSURE_SMEM((basis_wapply_kernel<16>), smem);
    basis_wapply_kernel<16><<<nctas, kWfThreads, smem, stream>>>(d_targets, d_map);
  } else {
    SRTT_ENSURE_SMEM((basis_wapply_kernel<32>), smem);
    basis_wapply_kernel<32><<<nctas, kWfThreads, smem, stream>>>(d_targets, d_map);
  }
  return cudaGetLastError();
}


// ---- generic kernel (c > 64) ----------------------------------------------------
size_t srtt_basis_generic_smem(int c, int r) {
  (void)r;
  const int kk = (c + 1) & ~1;
  return (size_t)(3 * c + 64 + 2) * sizeof(double) + (size_t)(c + 2) * sizeof(int) +
         (size_t)(kk - 1) * (kk / 2) * sizeof(unsigned short) + 64;
}

int64_t srtt_basis_generic_doubles(int64_t n, int c) {
  const int64_t k = n < c ? n : c;
  return k * c + k * k + c + n + 8;
}

cudaError_t srtt_launch_basis_generic(const BasisTarget* d_targets, const int* d_list, int n, size_t smem,
                                      cudaStream_t stream) {
  if (n <= 0) return cudaSuccess;
  SRTT_ENSURE_SMEM(basis_generic_kernel, smem);
  basis_generic_kernel<<<n, kThreads, smem, stream>>>(d_targets, d_list);
  return cudaGetLastError();
}

// ---- wide register path (32 < c <= 64) ---------------------------------------
int srtt_wide_block_rows() { return kTeamRows; }
size_t srtt_wide_top_smem(int m, int c, int r, bool pad) { return wide_top_doubles(m, c, r, pad) * sizeof(double) + 64; }
size_t srtt_wide_level_smem(int mb, int c) { return wide_level_doubles(mb, c) * sizeof(double) + 64; }

cudaError_t srtt_launch_wide_top(const BasisTarget* d_targets, const int* d_list, int n, size_t smem,
                                 cudaStream_t stream) {
  if (n <= 0) return cudaSuccess;
  SRTT_ENSURE_SMEM(basis_wide_top_kernel, smem);
  basis_wide_top_kernel<<<n, kThreads, smem, stream>>>(d_targets, d_list);
  return cudaGetLastError();
}

cudaError_t srtt_launch_wide_factor(const BasisTarget* d_targets, const int2* d_map, int level, int nctas, size_t smem,
                                    cudaStream_t stream) {
  if (nctas <= 0) return cudaSuccess;
  SRTT_ENSURE_SMEM(basis_wide_factor_kernel, smem);
  basis_wide_factor_kernel<<<nctas, kThreads, smem, stream>>>(d_targets, d_map, level);
  return cudaGetLastError();
}

cudaError_t srtt_launch_wide_apply(const BasisTarget* d_targets, const int2* d_map, int level, int nctas, size_t smem,
                                   cudaStream_t stream) {
  if (nctas <= 0) return cudaSuccess;
  SRTT_ENSURE_SMEM(basis_wide_apply_kernel, smem);
  basis_wide_apply_kernel<<<nctas, kThreads, smem, stream>>>(d_targets, d_map, level);
  return cudaGetLastError();
}

#ifdef SRTT_PROF
extern "C" int srtt_debug_basis_clocks(long long* out) {
  return (int)cudaMemcpyFromSymbol(out, g_basis_clk, sizeof(long long) * 16);
}
#endif
