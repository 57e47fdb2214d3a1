// K3 / K5 — fused multi-TTM streaming engine (sm_100a).
//
// Replaces the single full-tensor pass of the reference:
//   core_from_factors -> ttm x d            tucker.hpp:43-50, tensor.hpp:255-306
//   sliced_core (slab reduction + tail TTM)  parallel.hpp:355-445
//   root_transfer  (U_l^T M U_r)             htucker.hpp:67-85
//
// X is viewed as M = n0 x Q (column-major; mode 0 is the only stride-1
// mode, its fibres are M's columns). Work items are (row block, level-m
// group, split) triples; each persistent CTA streams its items' boxes of
// 16 rows x W columns through an 8-stage TMA ring (cp.async.bulk.tensor,
// 128-byte swizzle, mbarrier complete_tx) fed by one producer warp.
// Stage 1 (t1 = U0^T X_box, the only FLOP-heavy step: 2 r0 flop/entry) runs
// on the FP64 tensor cores: each compute warp owns 8-column M-tiles (even /
// odd column interleave so the swizzled A-fragment loads are conflict free)
// and issues mma.sync.m8n8k4.f64 against U0 B-fragments resident in shared
// memory. The t1 tile then folds into nested shared-memory accumulators
// acc_l (modes 1..m-1) with flush-on-index-change, which is linear and
// therefore correct for any item boundary. X is read from HBM exactly once.
// Item results are written to fixed slots and reduced in a fixed order by
// the tail, so the core is bitwise reproducible run to run.
#include <cuda.h>

#include "srtt_device.cuh"
#include "srtt_params.h"

namespace {

using namespace srtt_dev;

constexpr int kComputeWarps = 8;
constexpr int kComputeThreads = kComputeWarps * 32;
constexpr int kThreads = kComputeThreads + 32;  // + producer warp
constexpr int kStages = 8;
constexpr int kFoldScratch = 1024;  // doubles

struct Item {
  int rho;
  int sigma;
  int64_t p;
  int64_t c_lo, c_hi;
};

__device__ __forceinline__ Item decode_item(const CoreParams& P, int64_t it) {
  Item I;
  I.rho = (int)(it % P.nrb);
  const int64_t rest = it / P.nrb;
  I.sigma = (int)(rest % P.S);
  I.p = rest / P.S;
  I.c_lo = I.p * P.GS + (int64_t)I.sigma * P.SL;
  I.c_hi = min(I.c_lo + P.SL, (I.p + 1) * P.GS);
  return I;
}

__device__ __forceinline__ int boxes_of(const CoreParams& P, int rho) {
  const int64_t rows = srtt_dev::min64(P.RB, P.n0 - (int64_t)rho * P.RB);
  return (int)((rows + 15) / 16);
}

// Level-l fold: acc2[a0 + r0*a1] += sum_{j in run} T1[a0][j] * U1[i1(j)][a1].
__device__ void fold_level2(const CoreParams& P, const double* T1, int W, int j0, int len, int64_t i1_0,
                            double* acc2, double* scratch) {
  const int tid = threadIdx.x;
  const int r0 = P.r0, r1 = P.frank[0];
  const double* __restrict__ U1 = P.fu[0];
  const int nb = (r1 + 3) / 4;
  const int units = r0 * nb;
  const int JG = units >= kComputeThreads ? 1 : min(kComputeThreads / units, max(len, 1));
  if (JG == 1) {
    // every (a0, a1) pair has a single owner: accumulate in place
    for (int unit = tid; unit < units; unit += kComputeThreads) {
      const int a0 = unit % r0, a1b = (unit / r0) * 4;
      double s[4] = {0, 0, 0, 0};
      for (int jj = 0; jj < len; ++jj) {
        const double t = T1[a0 * W + j0 + jj];
        const double* ur = U1 + (i1_0 + jj) * r1 + a1b;
#pragma unroll
        for (int e = 0; e < 4; ++e)
          if (a1b + e < r1) s[e] += t * ur[e];
      }
#pragma unroll
      for (int e = 0; e < 4; ++e)
        if (a1b + e < r1) acc2[a0 + r0 * (a1b + e)] += s[e];
    }
    named_sync(1, kComputeThreads);
    return;
  }
  // partial sums into scratch[(jg*units + unit)*4 + e]  (JG*units <= 256)
  for (int u = tid; u < units * JG; u += kComputeThreads) {
    const int unit = u % units, jg = u / units;
    const int a0 = unit % r0, a1b = (unit / r0) * 4;
    double s0 = 0, s1 = 0, s2 = 0, s3 = 0;
    for (int jj = jg; jj < len; jj += JG) {
      const double t = T1[a0 * W + j0 + jj];
      const double* ur = U1 + (i1_0 + jj) * r1 + a1b;
      s0 += t * ur[0];
      if (a1b + 1 < r1) s1 += t * ur[1];
      if (a1b + 2 < r1) s2 += t * ur[2];
      if (a1b + 3 < r1) s3 += t * ur[3];
    }
    double* o = scratch + ((size_t)jg * units + unit) * 4;
    o[0] = s0; o[1] = s1; o[2] = s2; o[3] = s3;
  }
  named_sync(1, kComputeThreads);
  for (int idx = tid; idx < r0 * r1; idx += kComputeThreads) {
    const int a0 = idx % r0, a1 = idx / r0;
    const int unit = a0 + r0 * (a1 / 4), e = a1 % 4;
    double s = 0.0;
    for (int jg = 0; jg < JG; ++jg) s += scratch[((size_t)jg * units + unit) * 4 + e];
    acc2[idx] += s;
  }
  named_sync(1, kComputeThreads);
}

// acc_{l+1}[a + A_l * b] += acc_l[a] * U_l[i][b]; acc_l = 0.
__device__ void flush_level(const CoreParams& P, double* accs, int l, int64_t i) {
  const int tid = threadIdx.x;
  double* src = accs + P.acc_off[l];
  double* dst = accs + P.acc_off[l + 1];
  int Al = P.r0;
  for (int k = 0; k < l - 1; ++k) Al *= P.frank[k];
  const int rl = P.frank[l - 1];
  const double* __restrict__ Ul = P.fu[l - 1] + i * rl;
  for (int idx = tid; idx < Al * rl; idx += kComputeThreads) {
    const int a = idx % Al, b = idx / Al;
    dst[idx] += src[a] * Ul[b];
  }
  named_sync(1, kComputeThreads);
  for (int idx = tid; idx < Al; idx += kComputeThreads) src[idx] = 0.0;
  named_sync(1, kComputeThreads);
}

__device__ void fold_chunk(const CoreParams& P, const double* T1, int W, int64_t q0, int nvalid,
                           bool last_chunk_of_item, double* accs, double* scratch) {
  const int64_t n1 = P.fdim[0];
  int j = 0;
  while (j < nvalid) {
    const int64_t q = q0 + j;
    const int64_t i1 = q % n1;
    const int len = (int)srtt_dev::min64(n1 - i1, nvalid - j);
    fold_level2(P, T1, W, j, len, i1, accs + P.acc_off[2], scratch);
    j += len;
    const int64_t qlast = q + len - 1;
    const bool item_end = last_chunk_of_item && j == nvalid;
    // cascade flushes: level l (2..m-1) completes when digits 1..l-1 of
    // qlast are at their maxima, or at the end of the item.
    int64_t rem = qlast;
    bool complete = (rem % n1 == n1 - 1) || item_end;
    rem /= n1;
    for (int l = 2; l < P.m && complete; ++l) {
      const int64_t nl = P.fdim[l - 1];
      const int64_t il = rem % nl;
      flush_level(P, accs, l, il);
      complete = (il == nl - 1) || item_end;
      rem /= nl;
    }
  }
}

template <int NT, int MT>
__global__ void __launch_bounds__(kThreads, 1)
    core_kernel(const __grid_constant__ CUtensorMap tmap, const __grid_constant__ CoreParams P) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  const int W = P.W;
  const int stage_doubles = 16 * W;
  // carve (stage buffers first: 1024-byte aligned for the 128B swizzle)
  uintptr_t base = (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023);
  double* stages = reinterpret_cast<double*>(base);
  double* ufrag = stages + (size_t)kStages * stage_doubles;
  double* T1 = ufrag + (size_t)P.RB * NT * 8;
  double* accs = T1 + (size_t)P.r0 * W;
  double* scratch = accs + P.acc_total;
  uint64_t* full = reinterpret_cast<uint64_t*>(scratch + kFoldScratch);
  uint64_t* empty = full + kStages;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], P.use_tma ? 1 : 32);
      mbar_init(&empty[s], kComputeWarps);
    }
    fence_mbar_init();
  }
  __syncthreads();

  if (warp == kComputeWarps) {
    // ------------------------- producer warp -------------------------
    if (P.use_tma && lane == 0) prefetch_tmap(&tmap);
    uint32_t it = 0;
    for (int64_t item = blockIdx.x; item < P.nitems; item += gridDim.x) {
      const Item I = decode_item(P, item);
      const int nbox = boxes_of(P, I.rho);
      for (int64_t c0 = I.c_lo; c0 < I.c_hi; c0 += W) {
        for (int b = 0; b < nbox; ++b, ++it) {
          const int s = it % kStages;
          const uint32_t ph = (it / kStages) & 1;
          mbar_wait(&empty[s], ph ^ 1);
          double* dst = stages + (size_t)s * stage_doubles;
          const int64_t row0 = (int64_t)I.rho * P.RB + 16 * b;
          if (P.use_tma) {
            if (lane == 0) {
              mbar_arrive_expect_tx(&full[s], (uint32_t)(stage_doubles * sizeof(double)));
              tma_load_2d(dst, &tmap, &full[s], (int32_t)row0, (int32_t)c0);
            }
          } else {
            // warp copy into the same 128B-swizzled layout (odd n0)
            for (int e = lane; e < stage_doubles; e += 32) {
              const int jj = e >> 4, ii = e & 15;
              const int64_t row = row0 + ii, col = c0 + jj;
              const double v = (row < P.n0 && col < P.Q) ? P.x[col * P.n0 + row] : 0.0;
              dst[jj * 16 + ((((ii >> 1) ^ (jj & 7)) << 1) | (ii & 1))] = v;
            }
            mbar_arrive(&full[s]);
          }
        }
      }
    }
    return;
  }

  // --------------------------- compute warps ---------------------------
  const int tid = threadIdx.x;  // 0..kComputeThreads-1
  const int g = lane >> 2, tq = lane & 3;
  uint32_t it = 0;
  int cur_rho = -1;
  for (int64_t item = blockIdx.x; item < P.nitems; item += gridDim.x) {
    const Item I = decode_item(P, item);
    const int nbox = boxes_of(P, I.rho);
    if (I.rho != cur_rho) {
      named_sync(1, kComputeThreads);
      const double* src = P.ufrag + (size_t)I.rho * P.RB * NT * 8;
      for (int e = tid; e < P.RB * NT * 8; e += kComputeThreads) ufrag[e] = src[e];
      cur_rho = I.rho;
    }
    for (int e = tid; e < P.acc_total; e += kComputeThreads) accs[e] = 0.0;
    named_sync(1, kComputeThreads);

    for (int64_t c0 = I.c_lo; c0 < I.c_hi; c0 += W) {
      double d[MT][NT][2];
#pragma unroll
      for (int mt = 0; mt < MT; ++mt)
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) d[mt][nt][0] = d[mt][nt][1] = 0.0;
      int colg[MT];
#pragma unroll
      for (int mt = 0; mt < MT; ++mt) {
        const int tau = warp * MT + mt;
        colg[mt] = 16 * (tau >> 1) + 2 * g + (tau & 1);
      }
      for (int b = 0; b < nbox; ++b, ++it) {
        const int s = it % kStages;
        const uint32_t ph = (it / kStages) & 1;
        mbar_wait(&full[s], ph);
        const double* st = stages + (size_t)s * stage_doubles;
        const double* uf = ufrag + (size_t)b * 4 * NT * 32;
#pragma unroll
        for (int ks = 0; ks < 4; ++ks) {
          const int ii = 4 * ks + tq;
          double a[MT];
#pragma unroll
          for (int mt = 0; mt < MT; ++mt) {
            const int jj = colg[mt];
            a[mt] = st[jj * 16 + ((((ii >> 1) ^ (jj & 7)) << 1) | (ii & 1))];
          }
#pragma unroll
          for (int nt = 0; nt < NT; ++nt) {
            const double bf = uf[(ks * NT + nt) * 32 + lane];
#pragma unroll
            for (int mt = 0; mt < MT; ++mt) dmma_8x8x4(d[mt][nt][0], d[mt][nt][1], a[mt], bf);
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);
      }
      // t1 tile -> shared memory T1[a][col]
#pragma unroll
      for (int mt = 0; mt < MT; ++mt)
#pragma unroll
        for (int nt = 0; nt < NT; ++nt)
#pragma unroll
          for (int v = 0; v < 2; ++v) {
            const int a = 8 * nt + 2 * tq + v;
            if (a < P.r0) T1[a * W + colg[mt]] = d[mt][nt][v];
          }
      named_sync(1, kComputeThreads);
      const int nvalid = (int)srtt_dev::min64(W, I.c_hi - c0);
      fold_chunk(P, T1, W, c0, nvalid, c0 + W >= I.c_hi, accs, scratch);
    }
    // item result -> fixed slot
    double* out = P.part + (((int64_t)I.rho * P.S + I.sigma) * P.G + I.p) * P.A;
    const double* accm = accs + P.acc_off[P.m];
    for (int e = tid; e < P.A; e += kComputeThreads) out[e] = accm[e];
    named_sync(1, kComputeThreads);
  }
}

// U0 -> B-fragment order; fold factors -> row-major.
__global__ void prep_kernel(const double* __restrict__ u0, int64_t n0, int r0, int RB, int NT, int nrb,
                            double* __restrict__ ufrag) {
  const int64_t total = (int64_t)nrb * RB * NT * 8;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int lane = (int)(e % 32);
    int64_t rest = e / 32;
    const int nt = (int)(rest % NT);
    rest /= NT;
    const int64_t kstep = rest % (RB / 4);
    const int64_t rho = rest / (RB / 4);
    const int64_t row = rho * RB + 4 * kstep + (lane & 3);
    const int col = 8 * nt + (lane >> 2);
    ufrag[e] = (row < n0 && col < r0) ? u0[row + n0 * col] : 0.0;
  }
}

__global__ void transpose_kernel(const double* __restrict__ u, int64_t n, int r, double* __restrict__ ut) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n * r;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e / r;
    const int a = (int)(e % r);
    ut[e] = u[i + n * a];
  }
}

// out(gi, b, pi) = sum_i in(gi, i, pi) * coef(i, b), summed over nparts
// partial inputs in a fixed order.
__global__ void ttm_kernel(const TtmParams T) {
  const int64_t total = T.g * T.rr * T.post;
  for (int64_t o = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; o < total;
       o += (int64_t)gridDim.x * blockDim.x) {
    const int64_t gi = o % T.g;
    const int64_t rest = o / T.g;
    const int64_t b = rest % T.rr;
    const int64_t pi = rest / T.rr;
    double s = 0.0;
    for (int64_t i = 0; i < T.n; ++i) {
      const int64_t idx = gi + T.g * (i + T.n * pi);
      double v = T.in[idx];
      for (int pp = 1; pp < T.nparts; ++pp) v += T.in[idx + pp * T.part_stride];
      const double cf = T.transpose ? T.u[i + T.n * b] : T.u[b + T.rr * i];
      s += v * cf;
    }
    T.out[o] = s;
  }
}

}  // namespace

int srtt_core_threads() { return kThreads; }

size_t srtt_core_smem_bytes(const CoreParams& P) {
  const size_t doubles = (size_t)kStages * 16 * P.W + (size_t)P.RB * P.NT * 8 + (size_t)P.r0 * P.W +
                         P.acc_total + kFoldScratch;
  return 1024 + doubles * sizeof(double) + 2 * kStages * sizeof(uint64_t);
}

template <int NT, int MT>
static cudaError_t launch_core_t(const CUtensorMap* tmap, const CoreParams& P, int grid, cudaStream_t s) {
  const size_t smem = srtt_core_smem_bytes(P);
  cudaError_t e = cudaFuncSetAttribute(core_kernel<NT, MT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem);
  if (e != cudaSuccess) return e;
  core_kernel<NT, MT><<<grid, kThreads, smem, s>>>(*tmap, P);
  return cudaGetLastError();
}

int srtt_core_occupancy(const CoreParams& P) {
  const size_t smem = srtt_core_smem_bytes(P);
  int nb = 0;
#define OCC(NTV)                                                                                    \
  case NTV:                                                                                         \
    cudaFuncSetAttribute(core_kernel<NTV, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); \
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, core_kernel<NTV, 1>, kThreads, smem);        \
    break;
  switch (P.NT) {
    OCC(1) OCC(2) OCC(3) OCC(4) OCC(5) OCC(6) OCC(7) OCC(8)
    default: break;
  }
#undef OCC
  return nb;
}

cudaError_t srtt_launch_core(const CUtensorMap* tmap, const CoreParams& P, int grid, cudaStream_t s) {
  const int MT = P.W / (8 * kComputeWarps);
  if (MT == 1) {
    switch (P.NT) {
      case 1: return launch_core_t<1, 1>(tmap, P, grid, s);
      case 2: return launch_core_t<2, 1>(tmap, P, grid, s);
      case 3: return launch_core_t<3, 1>(tmap, P, grid, s);
      case 4: return launch_core_t<4, 1>(tmap, P, grid, s);
      case 5: return launch_core_t<5, 1>(tmap, P, grid, s);
      case 6: return launch_core_t<6, 1>(tmap, P, grid, s);
      case 7: return launch_core_t<7, 1>(tmap, P, grid, s);
      case 8: return launch_core_t<8, 1>(tmap, P, grid, s);
    }
  } else if (MT == 2) {
    switch (P.NT) {
      case 1: return launch_core_t<1, 2>(tmap, P, grid, s);
      case 2: return launch_core_t<2, 2>(tmap, P, grid, s);
      case 3: return launch_core_t<3, 2>(tmap, P, grid, s);
      case 4: return launch_core_t<4, 2>(tmap, P, grid, s);
    }
  }
  return cudaErrorInvalidValue;
}

cudaError_t srtt_launch_prep(const double* u0, int64_t n0, int r0, int RB, int NT, int nrb, double* ufrag,
                             cudaStream_t s) {
  prep_kernel<<<64, 256, 0, s>>>(u0, n0, r0, RB, NT, nrb, ufrag);
  return cudaGetLastError();
}

cudaError_t srtt_launch_transpose(const double* u, int64_t n, int r, double* ut, cudaStream_t s) {
  const int64_t total = n * r;
  const int blocks = (int)srtt_dev::min64(1024, (total + 255) / 256);
  transpose_kernel<<<blocks > 0 ? blocks : 1, 256, 0, s>>>(u, n, r, ut);
  return cudaGetLastError();
}

cudaError_t srtt_launch_ttm(const TtmParams& T, cudaStream_t s) {
  const int64_t total = T.g * T.rr * T.post;
  const int blocks = (int)srtt_dev::min64(148 * 16, (total + 255) / 256);
  ttm_kernel<<<blocks > 0 ? blocks : 1, 256, 0, s>>>(T);
  return cudaGetLastError();
}
