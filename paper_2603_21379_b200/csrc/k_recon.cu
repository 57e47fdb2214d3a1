// Streaming reconstruction error: ||X - A C^T||_F and
// ||X||_F without materialising X-hat, where X is viewed as the n_A x n_B
// matrix of its leading / trailing modes (first index fastest) and the
// low-rank factors are given K-fastest (At: K x n_A, Ct: K x n_B col-major).
//
//   Tucker  (tucker.hpp:18-28):    At = (U_{m-1} (x) ... (x) U_0)^T,
//                                  Ct = G x_m U_m ... x_{d-1} U_{d-1}
//   H-Tucker (htucker.hpp:346-378): At = U_left^T, Ct = B_0 U_right^T
//
// The same kernel writes X-hat tile by tile when `out` is set (the
// reference's reconstruct / ht_reconstruct) and then skips the norms.
//
// residual_kernel: one persistent CTA per SM (static work split ->
// deterministic sums), 128 x 32 (or 64 x 64 for short leading extents)
// output tiles computed with DMMA m8n8k4 (FP64 tensor cores) from an At
// block kept resident in shared memory and Ct tiles; X tiles arrive by TMA
// into an up-to-6-deep ring, so X streams from HBM exactly once while the
// tensor cores run.
#include <cuda.h>

#include <cstdint>

#include "srtt_device.cuh"
#include "srtt_params.h"

using namespace srtt_dev;

namespace {

constexpr int kThreads = 256;

// 8-byte cp.async; src_bytes = 0 zero-fills the destination.
__device__ __forceinline__ void cp_async8(void* smem, const double* g, uint32_t src_bytes = 8) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(smem_u32(smem)), "l"(g), "r"(src_bytes)
               : "memory");
}
// The mbarrier receives this thread's arrival once all its prior cp.async
// copies have landed.
__device__ __forceinline__ void cp_async_arrive(uint64_t* bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}

// 16-byte cp.async through L2 only (no L1 allocation); src_bytes = 0
// zero-fills.
__device__ __forceinline__ void cp_async16(void* smem, const double* g, uint32_t src_bytes = 16) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(smem_u32(smem)), "l"(g), "r"(src_bytes)
               : "memory");
}

// CTA tile TM = 32*WMW rows x TN = 16*WNW columns; WMW x WNW warps, each
// warp a 32 x 16 block = 4 x 2 DMMA m8n8k4 tiles (16 f64
// accumulators per lane). Operand layouts in shared memory are padded so
// the fragment loads are conflict-free: At resident as [k][TM+4] (A frag:
// lane -> (k = lane%4, i = lane/4)), Ct per stage as [TN][K+4] (B frag:
// lane -> (k = lane%4, j = lane/4)).
template <int WMW, int WNW>
struct ResidualCfg {
  static constexpr int TM = 32 * WMW, TN = 16 * WNW;
  __host__ __device__ static size_t at_bytes(int K) { return sizeof(double) * (size_t)K * (TM + 4); }
  __host__ __device__ static size_t x_bytes() { return sizeof(double) * (size_t)TM * TN; }
  __host__ __device__ static size_t c_bytes(int K) { return sizeof(double) * (size_t)TN * (K + 4); }
  __host__ __device__ static size_t stage_bytes(int K) { return x_bytes() + (c_bytes(K) + 127) / 128 * 128; }
  static int stages(int K, size_t budget) {
    const size_t fixed = at_bytes(K) + 1024;
    if (budget < fixed + 2 * stage_bytes(K)) return 0;
    const long ns = (long)((budget - fixed) / stage_bytes(K));
    return ns > 6 ? 6 : (int)ns;
  }
  static size_t smem(int K, int ns) { return at_bytes(K) + ns * stage_bytes(K) + 1024; }
};

template <int WMW, int WNW>
__global__ void __launch_bounds__(32 * WMW * WNW, 1)
    residual_kernel(const __grid_constant__ CUtensorMap tmx, const __grid_constant__ ResidualParams P) {
  using Cfg = ResidualCfg<WMW, WNW>;
  constexpr int TM = Cfg::TM, TN = Cfg::TN;
  constexpr int kThreads = 32 * WMW * WNW, kWarps = WMW * WNW;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int K = P.K, NS = P.stages, KP = P.K + 4;
  unsigned char* base = smem_raw + ((128 - (smem_u32(smem_raw) & 127)) & 127);
  const size_t stage_bytes = Cfg::stage_bytes(K);
  double* at_s = reinterpret_cast<double*>(base + NS * stage_bytes);         // [K][TM+4]
  uint64_t* full = reinterpret_cast<uint64_t*>(at_s + (size_t)K * (TM + 4));  // [NS]
  double* red = reinterpret_cast<double*>(full + 8);                         // [2][kWarps]

  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int wm = warp % WMW, wn = warp / WMW;
  const int lr = lane >> 2, lc = lane & 3;
  const bool norms = P.out == nullptr;
  const bool x_tma = norms && P.x_tma;
  const int64_t tiles_a = (P.nA + TM - 1) / TM, tiles_b = (P.nB + TN - 1) / TN;
  // Work = a contiguous range [f_lo, f_lo + my_tiles) of the row-tile-major
  // tile order (f = rt * tiles_b + ct). With few row tiles, CTA groups of
  // tiles_a CTAs split the columns: the members of a group walk the same
  // column tiles at the same time (Ct from L2). With more row tiles than
  // CTAs the flat order is split evenly (Ct is small then).
  int64_t f_lo, my_tiles;
  if (tiles_a <= gridDim.x && gridDim.x % tiles_a <= gridDim.x / 8) {
    const int64_t groups = gridDim.x / tiles_a;
    const int64_t g = blockIdx.x / tiles_a;
    const int64_t c_lo = g < groups ? g * tiles_b / groups : 0;
    const int64_t c_hi = g < groups ? (g + 1) * tiles_b / groups : 0;
    f_lo = (blockIdx.x % tiles_a) * tiles_b + c_lo;
    my_tiles = c_hi - c_lo;
  } else {
    const int64_t T = tiles_a * tiles_b;
    f_lo = blockIdx.x * T / gridDim.x;
    my_tiles = (blockIdx.x + 1) * T / gridDim.x - f_lo;
  }

  if (threadIdx.x == 0) {
    for (int b = 0; b < NS; ++b) mbar_init(&full[b], kThreads + (x_tma ? 1 : 0));
    fence_mbar_init();
  }
  __syncthreads();

  // tile coordinates advance incrementally (no 64-bit divisions per tile)
  struct Cursor {
    int64_t rt, ct;
  };
  auto advance = [&](Cursor& c) {
    if (++c.ct == tiles_b) {
      c.ct = 0;
      ++c.rt;
    }
  };
  // Ct copy: this thread's first (chunk, column) pair and its per-pass step
  const int kc = K / 2;  // 16-byte chunks per Ct column
  const int q0 = threadIdx.x % kc, jj0 = threadIdx.x / kc;
  const int dq = kThreads % kc, djj = kThreads / kc;
  auto issue = [&](int64_t lt, const Cursor& c) {
    const int stg = (int)(lt % NS);
    double* xs = reinterpret_cast<double*>(base + stg * stage_bytes);
    double* cs = xs + TM * TN;
    const int64_t i0 = c.rt * TM, j0 = c.ct * TN;
    if (x_tma && threadIdx.x == 0) {
      mbar_arrive_expect_tx(&full[stg], (uint32_t)Cfg::x_bytes());
      tma_load_2d(xs, &tmx, &full[stg], (int32_t)i0, (int32_t)j0);
    }
    if (norms && !x_tma) {
      for (int e = threadIdx.x; e < TM * TN; e += kThreads) {
        const int ii = e % TM, jj = e / TM;
        const int64_t i = i0 + ii, j = j0 + jj;
        if (i < P.nA && j < P.nB) cp_async8(xs + jj * TM + ii, P.x + i + P.nA * j);
      }
    }
    int q = q0, jj = jj0;
    while (jj < TN) {
      const int64_t j = j0 + jj;
      const bool ok = j < P.nB;
      cp_async16(cs + jj * KP + 2 * q, ok ? P.ct + (int64_t)K * j + 2 * q : P.ct, ok ? 16u : 0u);
      q += dq;
      jj += djj;
      if (q >= kc) {
        q -= kc;
        ++jj;
      }
    }
    cp_async_arrive(&full[stg]);
  };

  Cursor cur{f_lo / tiles_b, f_lo % tiles_b}, nxt = cur;
  for (int64_t lt = 0; lt < NS && lt < my_tiles; ++lt) {
    issue(lt, nxt);
    advance(nxt);
  }

  double rs[4] = {0.0, 0.0, 0.0, 0.0}, xq[4] = {0.0, 0.0, 0.0, 0.0};
  int64_t cur_rt = -1;
  auto mma = [&](int64_t lt, const Cursor& c, double (&acc)[4][2][2]) {
    if (c.rt != cur_rt) {  // (re)load the resident At block of this row tile
      cur_rt = c.rt;
      __syncthreads();     // every warp is done with the previous block
      const int64_t i0 = c.rt * TM;
      for (int e = threadIdx.x; e < K * TM; e += kThreads) {
        const int kk = e % K, ii = e / K;
        const int64_t i = i0 + ii;
        at_s[kk * (TM + 4) + ii] = i < P.nA ? __ldg(P.at + kk + (int64_t)K * i) : 0.0;
      }
      __syncthreads();
    }
    const int stg = (int)(lt % NS);
    mbar_wait(&full[stg], (uint32_t)((lt / NS) & 1));
    const double* cs = reinterpret_cast<const double*>(base + stg * stage_bytes) + TM * TN;
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int b = 0; b < 2; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
    const double* ap = at_s + lc * (TM + 4) + wm * 32 + lr;
    const double* bp = cs + (wn * 16 + lr) * KP + lc;
    for (int k0 = 0; k0 < K; k0 += 4) {
      double af[4], bf[2];
#pragma unroll
      for (int a = 0; a < 4; ++a) af[a] = ap[k0 * (TM + 4) + 8 * a];
#pragma unroll
      for (int b = 0; b < 2; ++b) bf[b] = bp[8 * b * KP + k0];
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 2; ++b) dmma_8x8x4(acc[a][b][0], acc[a][b][1], af[a], bf[b]);
    }
  };
  // lane holds D[lr][2 lc + e] of each 8 x 8 tile
  auto epi = [&](int64_t lt, const Cursor& c, const double (&acc)[4][2][2]) {
    const int stg = (int)(lt % NS);
    const double* xs = reinterpret_cast<const double*>(base + stg * stage_bytes);
    const int64_t i0 = c.rt * TM, j0 = c.ct * TN;
    const int ib = wm * 32 + lr, jb = wn * 16 + 2 * lc;
    const bool interior = i0 + TM <= P.nA && j0 + TN <= P.nB;
    if (norms && interior) {
      const double* xl = xs + jb * TM + ib;
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 2; ++b)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const double x = xl[(8 * b + e) * TM + 8 * a];
            const double df = x - acc[a][b][e];
            rs[a] = fma(df, df, rs[a]);
            xq[a] = fma(x, x, xq[a]);
          }
    } else {
#pragma unroll
      for (int a = 0; a < 4; ++a) {
        const int ii = ib + 8 * a;
        const int64_t i = i0 + ii;
#pragma unroll
        for (int b = 0; b < 2; ++b)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int jj = jb + 8 * b + e;
            const int64_t j = j0 + jj;
            if (i >= P.nA || j >= P.nB) continue;
            if (!norms) {
              P.out[i + P.nA * j] = acc[a][b][e];
            } else {
              const double x = xs[jj * TM + ii];
              const double df = x - acc[a][b][e];
              rs[a] = fma(df, df, rs[a]);
              xq[a] = fma(x, x, xq[a]);
            }
          }
      }
    }
    __syncthreads();  // stage free for refill
    if (lt + NS < my_tiles) {
      issue(lt + NS, nxt);
      advance(nxt);
    }
  };

  for (int64_t lt = 0; lt < my_tiles; ++lt) {
    double acc[4][2][2];
    mma(lt, cur, acc);
    epi(lt, cur, acc);
    advance(cur);
  }
  double res = (rs[0] + rs[1]) + (rs[2] + rs[3]);
  double xn = (xq[0] + xq[1]) + (xq[2] + xq[3]);
  if (!norms) return;
  res = warp_sum(res);
  xn = warp_sum(xn);
  if (lane == 0) {
    red[warp] = res;
    red[kWarps + warp] = xn;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double r = 0.0, n = 0.0;
    for (int i = 0; i < kWarps; ++i) {
      r += red[i];
      n += red[kWarps + i];
    }
    P.partial[2 * blockIdx.x] = r;
    P.partial[2 * blockIdx.x + 1] = n;
  }
}

// ||x - y||^2 and ||x||^2 of two flat tensors (rel_error, tensor.hpp:241-249);
// static chunking per CTA keeps the sums deterministic.
__global__ void __launch_bounds__(kThreads) diff_norm_kernel(const double* __restrict__ x,
                                                             const double* __restrict__ y, int64_t n,
                                                             double* partial) {
  __shared__ double red[2][kThreads / 32];
  const int64_t chunk = (n + gridDim.x - 1) / gridDim.x;
  const int64_t lo = blockIdx.x * chunk, hi = min64(n, lo + chunk);
  double r0 = 0, r1 = 0, n0 = 0, n1 = 0;
  int64_t i = lo + threadIdx.x;
  for (; i + kThreads < hi; i += 2 * kThreads) {
    const double a = __ldg(x + i), b = __ldg(y + i);
    const double c = __ldg(x + i + kThreads), e = __ldg(y + i + kThreads);
    r0 = fma(a - b, a - b, r0);
    n0 = fma(a, a, n0);
    r1 = fma(c - e, c - e, r1);
    n1 = fma(c, c, n1);
  }
  if (i < hi) {
    const double a = __ldg(x + i), b = __ldg(y + i);
    r0 = fma(a - b, a - b, r0);
    n0 = fma(a, a, n0);
  }
  double res = warp_sum(r0 + r1), xn = warp_sum(n0 + n1);
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) {
    red[0][w] = res;
    red[1][w] = xn;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double r = 0.0, s = 0.0;
    for (int k = 0; k < kThreads / 32; ++k) {
      r += red[0][k];
      s += red[1][k];
    }
    partial[2 * blockIdx.x] = r;
    partial[2 * blockIdx.x + 1] = s;
  }
}

// Fixed-order final sum of the per-CTA partials (one warp, pairwise tree).
__global__ void partial_sum_kernel(const double* partial, int nparts, double* out) {
  double r = 0.0, s = 0.0;
  for (int i = threadIdx.x; i < nparts; i += 32) {
    r += partial[2 * i];
    s += partial[2 * i + 1];
  }
  r = warp_sum(r);
  s = warp_sum(s);
  if (threadIdx.x == 0) {
    out[0] = r;
    out[1] = s;
  }
}

// At (K x n_A) of the Kronecker product U_{m-1} (x) ... (x) U_0 (first
// factor fastest, matching the flat index of the leading m modes).
__global__ void kron_rows_kernel(const KronParams P) {
  const int64_t total = P.K * P.nA;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    int64_t t = e % P.K, i = e / P.K;
    double v = 1.0;
    for (int k = 0; k < P.m; ++k) {
      const int64_t tk = t % P.r[k], ik = i % P.n[k];
      t /= P.r[k];
      i /= P.n[k];
      v *= P.u[k][ik + P.n[k] * tk];
    }
    P.at[e] = v;
  }
}

// K x n (ld K) -> Kp x n (ld Kp), zero rows K..Kp-1.
__global__ void pad_rows_kernel(const double* __restrict__ in, int64_t K, int64_t n, int64_t Kp, double* out) {
  const int64_t total = Kp * n;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t t = e % Kp, j = e / Kp;
    out[e] = t < K ? in[t + K * j] : 0.0;
  }
}

__global__ void transpose_kernel(const double* __restrict__ in, int64_t rows, int64_t cols, double* out) {
  const int64_t total = rows * cols;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e % rows, j = e / rows;
    out[j + cols * i] = in[e];
  }
}

}  // namespace



namespace {
template <int WMW, int WNW>
cudaError_t launch_residual_t(const CUtensorMap* tmx, ResidualParams P, int grid, cudaStream_t s) {
  using Cfg = ResidualCfg<WMW, WNW>;
  P.stages = Cfg::stages(P.K, 232448 - 1024);
  if (P.stages < 2) return cudaErrorInvalidValue;
  const size_t smem = Cfg::smem(P.K, P.stages);
  auto* k = residual_kernel<WMW, WNW>;
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  k<<<grid, 32 * WMW * WNW, smem, s>>>(*tmx, P);
  return cudaGetLastError();
}
}  // namespace

// One CTA per SM. 16 warps (128 x 64 tiles, or 64 x 128 for a short leading
// extent) while the 2-deep ring fits next to the resident At block (K <= 32),
// else 8 warps (128 x 32) with a deeper ring.
int srtt_residual_grid(int sms, int64_t, int) { return sms; }
int srtt_residual_tile_rows(int64_t nA) { return nA <= 64 ? 64 : 128; }
int srtt_residual_tile_cols(int64_t nA, int K) {
  if (nA <= 64) return 128;
  return ResidualCfg<4, 4>::stages(K, 232448 - 1024) >= 2 ? 64 : 32;
}

// P.K must be a multiple of 8 (At / Ct zero-padded), <= 64.
cudaError_t srtt_launch_residual(const CUtensorMap* tmx, const ResidualParams& P, int grid, double* sums,
                                 cudaStream_t s) {
  if (P.K % 8 != 0 || P.K > 64) return cudaErrorInvalidValue;
  cudaError_t e;
  if (srtt_residual_tile_rows(P.nA) == 64)
    e = launch_residual_t<2, 8>(tmx, P, grid, s);
  else if (srtt_residual_tile_cols(P.nA, P.K) == 64)
    e = launch_residual_t<4, 4>(tmx, P, grid, s);
  else
    e = launch_residual_t<4, 2>(tmx, P, grid, s);
  if (e != cudaSuccess) return e;
  if (!P.out) partial_sum_kernel<<<1, 32, 0, s>>>(P.partial, grid, sums);
  return cudaGetLastError();
}

cudaError_t srtt_launch_diff_norm(const double* x, const double* y, int64_t n, int grid, double* partial,
                                  double* sums, cudaStream_t s) {
  diff_norm_kernel<<<grid, kThreads, 0, s>>>(x, y, n, partial);
  partial_sum_kernel<<<1, 32, 0, s>>>(partial, grid, sums);
  return cudaGetLastError();
}

cudaError_t srtt_launch_kron_rows(const KronParams& P, cudaStream_t s) {
  const int64_t total = P.K * P.nA;
  kron_rows_kernel<<<(int)min64(148 * 8, (total + 255) / 256), 256, 0, s>>>(P);
  return cudaGetLastError();
}

cudaError_t srtt_launch_pad_rows(const double* in, int64_t K, int64_t n, int64_t Kp, double* out, cudaStream_t s) {
  const int64_t total = Kp * n;
  pad_rows_kernel<<<(int)min64(148 * 8, (total + 255) / 256), 256, 0, s>>>(in, K, n, Kp, out);
  return cudaGetLastError();
}

cudaError_t srtt_launch_mat_transpose(const double* in, int64_t rows, int64_t cols, double* out, cudaStream_t s) {
  const int64_t total = rows * cols;
  transpose_kernel<<<(int)min64(148 * 8, (total + 255) / 256), 256, 0, s>>>(in, rows, cols, out);
  return cudaGetLastError();
}
