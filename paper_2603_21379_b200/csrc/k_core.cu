// K3 / K5 — fused multi-TTM streaming engine (sm_100a).
//
// Replaces the single full-tensor pass of the reference:
//   core_from_factors -> ttm x d            tucker.hpp:43-50, tensor.hpp:255-306
//   sliced_core (slab reduction + tail TTM)  parallel.hpp:355-445
//   root_transfer  (U_l^T M U_r)             htucker.hpp:67-85
//
// X is viewed as M = n0 x Q (column-major; mode 0 is the only stride-1 mode
// and its fibres are M's columns). A work item is one contiguous column
// range of one row block inside one level-m group (m = 2 or 3); the CTA's
// 8 warps split the item into contiguous runs of 16-column "tile pairs".
//
// Each warp is its own producer and consumer: lane 0 keeps a private ring
// of NS TMA boxes (16 rows x 16 columns, 128-byte swizzle,
// cp.async.bulk.tensor + mbarrier complete_tx) NS boxes ahead of the
// consumer, across item boundaries. Per box, stage 1 computes
//   T(ranks0 x 16 cols) += U0^T(ranks0 x 16 rows) X(16 rows x 16 cols)
// on the FP64 tensor cores (mma.sync.m8n8k4.f64 = DMMA.8x8x4): A = U0
// fragments resident in shared memory, B = X fragments read conflict-free
// from the swizzled box (even/odd column interleave). When a tile pair's
// rows are done, stage 2 folds mode 1 with a second DMMA,
//   R2(ranks0 x ranks1) += T(ranks0 x 16 cols) U1[i1(col), :],
// whose A operand is the stage-1 accumulator itself: the column <-> k-slot
// map is chosen so each thread already holds its A values (no shuffles).
// Columns of other level-2 groups or beyond the item are masked through the
// B operand. For m = 3 a finished level-2 group is flushed into a
// warp-private acc3 (r0 r1 r2) with U2[i2, :]. At the end of an item the
// 8 warp partials are summed in a fixed order into the item's output slot,
// so the core is bitwise reproducible run to run. X is read exactly once.
//
// core_flat_kernel (one row block, n0 <= 256) drops the items: every warp
// streams an equal contiguous range of column tiles and its group records
// are reduced in-kernel by the warp that completes each group (see below);
// for short columns one unswizzled TMA box holds whole columns.
#include <cuda.h>

#include <algorithm>

#include "srtt_device.cuh"
#include "srtt_params.h"

namespace {

using namespace srtt_dev;


__device__ __forceinline__ int boxes_of(const CoreParams& P, int rho) {
  const int64_t rows = min64(P.RB, P.n0 - (int64_t)rho * P.RB);
  return (int)((rows + 15) / 16);
}

template <int WARPS>
__device__ __forceinline__ void warp_range(int len, int bc, int warp, int* lo, int* hi) {
  const int ntg = (len + bc - 1) / bc;
  *lo = (ntg * warp) / WARPS;
  *hi = (ntg * (warp + 1)) / WARPS;
}

// Producer-side walk over this warp's (item, tile group, box) sequence.
template <int WARPS>
struct WarpIter {
  int64_t item;
  int tg, tg_end, b, nbox, rho;
  int64_t c_lo;
  bool valid;

  __device__ void seek(const CoreParams& P, int bc, int warp) {
    while (item < P.nitems) {
      const CoreItem I = P.items[item];
      int lo, hi;
      warp_range<WARPS>(I.len, bc, warp, &lo, &hi);
      if (lo < hi) {
        tg = lo;
        tg_end = hi;
        b = 0;
        nbox = boxes_of(P, I.rho);
        rho = I.rho;
        c_lo = I.c_lo;
        valid = true;
        return;
      }
      item += gridDim.x;
    }
    valid = false;
  }
  __device__ __forceinline__ void next(const CoreParams& P, int bc, int warp) {
    if (++b < nbox) return;
    b = 0;
    if (++tg < tg_end) return;
    item += gridDim.x;
    seek(P, bc, warp);
  }
};

// MT: 8-rank tiles of mode 0; NT1: of mode 1; M3: fold depth 3;
// TPB: 16-column tile pairs per TMA box (box = 16 rows x 16*TPB columns);
// WARPS: warps per CTA (each its own producer/consumer).
template <int MT, int NT1, bool M3, int TPB, int WARPS>
__global__ void __launch_bounds__(WARPS * 32, 1)
    core_kernel(const __grid_constant__ CUtensorMap tmap, const __grid_constant__ CoreParams P) {
  constexpr int BC = 16 * TPB;
  constexpr int BOX = 16 * BC;
  constexpr int KP = MT == 1 ? 2 : 1;  // split-K accumulators for DMMA ILP
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  const int NS = P.nstages;
  // 1024-byte alignment for the 128B swizzle, computed on the shared-window
  // address so every pointer below stays in the shared state space (LDS/STS,
  // not generic LD/ST).
  const uint32_t pad = (1024u - (smem_u32(smem_raw) & 1023u)) & 1023u;
  double* rings = reinterpret_cast<double*>(smem_raw + pad);
  double* ufrag = rings + (size_t)WARPS * NS * BOX;
  // m = 2 with a large r0 r1 (C5: 1024) reduces the warp partials in
  // chunks of P.slot_ch entries, so 512-row blocks fit next to U0
  const int SLOT = (!M3 && P.slot_ch) ? P.slot_ch : P.A;
  double* slots = ufrag + (size_t)(P.RB / 4) * MT * 32;
  uint64_t* bars = reinterpret_cast<uint64_t*>(slots + (size_t)WARPS * SLOT);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, tq = lane & 3;
  double* ring = rings + (size_t)warp * NS * BOX;
  uint64_t* bar = bars + warp * NS;
  double* slot = slots + (size_t)warp * SLOT;

  const int r0 = P.r0, r1 = P.frank[0];
  const int n1 = (int)P.fdim[0];
  const double* __restrict__ U1 = P.fu[0];

  // per-lane swizzled offsets of the B fragments: column 2g+par, row 4ks+tq
  int boff[2][4];
#pragma unroll
  for (int par = 0; par < 2; ++par)
#pragma unroll
    for (int ks = 0; ks < 4; ++ks) {
      const int col = 2 * g + par, row = 4 * ks + tq;
      boff[par][ks] = col * 16 + ((((row >> 1) ^ (col & 7)) << 1) | (row & 1));
    }

  if (lane == 0) {
    for (int s = 0; s < NS; ++s) mbar_init(&bar[s], 1);
    fence_mbar_init();
  }
  __syncthreads();

  WarpIter<WARPS> pit;
  pit.item = blockIdx.x;
  pit.seek(P, BC, warp);
  if (P.use_tma && lane == 0) {
    prefetch_tmap(&tmap);
    for (int s = 0; s < NS && pit.valid; ++s) {
      mbar_arrive_expect_tx(&bar[s], BOX * sizeof(double));
      tma_load_2d(ring + s * BOX, &tmap, &bar[s], pit.rho * P.RB + 16 * pit.b, (int32_t)(pit.c_lo + BC * pit.tg));
      pit.next(P, BC, warp);
    }
  }

  int stage = 0;
  uint32_t phase = 0;
  int cur_rho = -1;
  for (int64_t item = blockIdx.x; item < P.nitems; item += gridDim.x) {
    const CoreItem I = P.items[item];
    if (I.rho != cur_rho) {
      __syncthreads();
      const double* src = P.ufrag + (size_t)I.rho * (P.RB / 4) * MT * 32;
      for (int e = threadIdx.x; e < (P.RB / 4) * MT * 32; e += WARPS * 32) ufrag[e] = src[e];
      cur_rho = I.rho;
      __syncthreads();
    }
    const int nbox = boxes_of(P, I.rho);
    const int len = I.len;
    if (M3)
      for (int e = lane; e < P.A; e += 32) slot[e] = 0.0;
    __syncwarp();
    double r2[MT][NT1][2];
#pragma unroll
    for (int mt = 0; mt < MT; ++mt)
#pragma unroll
      for (int nt = 0; nt < NT1; ++nt) r2[mt][nt][0] = r2[mt][nt][1] = 0.0;
    int64_t cur_g2 = -1;  // level-2 group held in r2 (M3 only)

    auto flush = [&](int64_t grp) {
      const int r2n = P.frank[1];
      const int64_t i2 = grp % P.fdim[1];
      const double* __restrict__ U2 = P.fu[1] + i2 * r2n;
#pragma unroll
      for (int mt = 0; mt < MT; ++mt)
#pragma unroll
        for (int nt = 0; nt < NT1; ++nt)
#pragma unroll
          for (int v = 0; v < 2; ++v) {
            const int a0 = g + 8 * mt, a1 = 2 * tq + v + 8 * nt;
            if (a0 < r0 && a1 < r1) {
              const double val = r2[mt][nt][v];
              double* dst = slot + a0 + r0 * a1;
              for (int a2 = 0; a2 < r2n; ++a2) dst[(size_t)r0 * r1 * a2] += val * __ldg(U2 + a2);
            }
            r2[mt][nt][v] = 0.0;
          }
      __syncwarp();
    };

    int tg_lo, tg_hi;
    warp_range<WARPS>(len, BC, warp, &tg_lo, &tg_hi);
    // level-2 group tracking of this warp's first column (32-bit)
    int64_t grp = I.grp0;
    int off = I.off0 + BC * tg_lo;
    if (off >= n1) {
      grp += off / n1;
      off %= n1;
    }
    for (int tg = tg_lo; tg < tg_hi; ++tg) {
      const int64_t c0 = I.c_lo + (int64_t)BC * tg;
      double t[TPB][2][MT][KP][2];
#pragma unroll
      for (int h = 0; h < TPB; ++h)
#pragma unroll
        for (int par = 0; par < 2; ++par)
#pragma unroll
          for (int mt = 0; mt < MT; ++mt)
#pragma unroll
            for (int kp = 0; kp < KP; ++kp) t[h][par][mt][kp][0] = t[h][par][mt][kp][1] = 0.0;
      const double* uf = ufrag + lane;
      for (int b = 0; b < nbox; ++b, uf += 4 * MT * 32) {
        double* st = ring + stage * BOX;
        if (P.use_tma) {
          mbar_wait(&bar[stage], phase);
        } else {
          const int64_t row0 = (int64_t)I.rho * P.RB + 16 * b;
          for (int e = lane; e < BOX; e += 32) {
            const int jj = e >> 4, ii = e & 15;
            const int64_t row = row0 + ii, col = c0 + jj;
            const double v = (row < P.n0 && col < P.Q) ? P.x[col * P.n0 + row] : 0.0;
            st[jj * 16 + ((((ii >> 1) ^ (jj & 7)) << 1) | (ii & 1))] = v;
          }
          __syncwarp();
        }
#pragma unroll
        for (int ks = 0; ks < 4; ++ks) {
          double a[MT];
#pragma unroll
          for (int mt = 0; mt < MT; ++mt) a[mt] = uf[(ks * MT + mt) * 32];
#pragma unroll
          for (int h = 0; h < TPB; ++h) {
            const double x0 = st[h * 256 + boff[0][ks]];
            const double x1 = st[h * 256 + boff[1][ks]];
#pragma unroll
            for (int mt = 0; mt < MT; ++mt) {
              double* d0 = t[h][0][mt][ks % KP];
              double* d1 = t[h][1][mt][ks % KP];
              dmma_8x8x4(d0[0], d0[1], a[mt], x0);
              dmma_8x8x4(d1[0], d1[1], a[mt], x1);
            }
          }
        }
        __syncwarp();
        if (P.use_tma && lane == 0 && pit.valid) {
          mbar_arrive_expect_tx(&bar[stage], BOX * sizeof(double));
          tma_load_2d(st, &tmap, &bar[stage], pit.rho * P.RB + 16 * pit.b, (int32_t)(pit.c_lo + BC * pit.tg));
          pit.next(P, BC, warp);
        }
        if (++stage == NS) {
          stage = 0;
          phase ^= 1;
        }
      }
      if (KP == 2) {
#pragma unroll
        for (int h = 0; h < TPB; ++h)
#pragma unroll
          for (int par = 0; par < 2; ++par)
#pragma unroll
            for (int mt = 0; mt < MT; ++mt) {
              t[h][par][mt][0][0] += t[h][par][mt][KP - 1][0];
              t[h][par][mt][0][1] += t[h][par][mt][KP - 1][1];
            }
      }
      // ---- stage 2: fold mode 1; thread holds T[g+8mt][col], col = c0h + 4tq + 2s + par
#pragma unroll
      for (int h = 0; h < TPB; ++h) {
        const int rel = BC * tg + 16 * h;  // column offset inside the item
        if (rel >= len) break;
        if (off + 16 <= n1 && rel + 16 <= len) {
          if (M3) {
            if (cur_g2 >= 0 && grp != cur_g2) flush(cur_g2);
            cur_g2 = grp;
          }
          const double* urow = U1 + (off + 4 * tq) * r1 + g;
#pragma unroll
          for (int par = 0; par < 2; ++par)
#pragma unroll
            for (int s2 = 0; s2 < 2; ++s2) {
              double bv[NT1];
#pragma unroll
              for (int nt = 0; nt < NT1; ++nt)
                bv[nt] = (g + 8 * nt < r1) ? __ldg(urow + (2 * s2 + par) * r1 + 8 * nt) : 0.0;
#pragma unroll
              for (int mt = 0; mt < MT; ++mt)
#pragma unroll
                for (int nt = 0; nt < NT1; ++nt)
                  dmma_8x8x4(r2[mt][nt][0], r2[mt][nt][1], t[h][par][mt][0][s2], bv[nt]);
            }
        } else {
          // straddles a level-2 group boundary or the item end: per group
          // segment [lo, hi) of the 16 columns, mask the others in B
          int64_t gg = grp;
          int oo = off;
          const int lim = min(16, len - rel);
          for (int lo = 0; lo < lim;) {
            const int hi = min(lim, lo + n1 - oo);
            if (M3) {
              if (cur_g2 >= 0 && gg != cur_g2) flush(cur_g2);
              cur_g2 = gg;
            }
            const double* ubase = U1 + (oo - lo) * r1 + g;
#pragma unroll
            for (int par = 0; par < 2; ++par)
#pragma unroll
              for (int s2 = 0; s2 < 2; ++s2) {
                const int j = 4 * tq + 2 * s2 + par;
                const bool ok = j >= lo && j < hi;
                double bv[NT1];
#pragma unroll
                for (int nt = 0; nt < NT1; ++nt)
                  bv[nt] = (ok && g + 8 * nt < r1) ? __ldg(ubase + j * r1 + 8 * nt) : 0.0;
#pragma unroll
                for (int mt = 0; mt < MT; ++mt)
#pragma unroll
                  for (int nt = 0; nt < NT1; ++nt)
                    dmma_8x8x4(r2[mt][nt][0], r2[mt][nt][1], t[h][par][mt][0][s2], bv[nt]);
              }
            oo += hi - lo;
            lo = hi;
            if (oo >= n1) {
              oo -= n1;
              ++gg;
            }
          }
        }
        off += 16;
        while (off >= n1) {
          off -= n1;
          ++grp;
        }
      }
    }
    // ---- item end: warp partial -> slot, fixed-order CTA reduction
    // (chunks of SLOT entries; one chunk unless P.slot_ch is set)
    double* out = P.part + I.out_off;
    if (M3 && cur_g2 >= 0) flush(cur_g2);
    for (int c0 = 0; c0 < P.A; c0 += SLOT) {
      if (!M3) {
#pragma unroll
        for (int mt = 0; mt < MT; ++mt)
#pragma unroll
          for (int nt = 0; nt < NT1; ++nt)
#pragma unroll
            for (int v = 0; v < 2; ++v) {
              const int a0 = g + 8 * mt, a1 = 2 * tq + v + 8 * nt;
              const int e = a0 + r0 * a1 - c0;
              if (a0 < r0 && a1 < r1 && e >= 0 && e < SLOT) slot[e] = r2[mt][nt][v];
            }
      }
      __syncthreads();
      const int ce = min(SLOT, P.A - c0);
      for (int e = threadIdx.x; e < ce; e += WARPS * 32) {
        double sum = 0.0;
#pragma unroll
        for (int w = 0; w < WARPS; ++w) sum += slots[(size_t)w * SLOT + e];
        out[c0 + e] = sum;
      }
      __syncthreads();
    }
  }
}

// ---- flat mode (single row block, n0 <= 256) --------------------------------
// Global warp gw owns tiles [T*gw/NW, T*(gw+1)/NW) of BC columns: every warp
// streams the same number of tiles (+-1), with no CTA barrier after the
// start, so an item's slowest warp no longer sets the pace. A warp folds its
// columns exactly as core_kernel does and emits one record per level-m group
// its range touches; the warp whose record completes a group sums the
// group's records in warp order (deterministic) into the compact R_m.
__device__ __forceinline__ int64_t flat_tile_lo(int64_t T, int64_t gw, int64_t nw) { return T * gw / nw; }
// the (non-empty) warp whose tile range contains tile t
__device__ __forceinline__ int64_t flat_warp_of(int64_t T, int64_t t, int64_t nw) {
  return ((t + 1) * nw + T - 1) / T - 1;
}

template <int WARPS>
__device__ __forceinline__ void flat_emit(const CoreParams& P, int64_t gw, int64_t p, int lane, int BC) {
  // record of (gw, p) is in global memory (written by all lanes); publish it
  __threadfence();
  __syncwarp();
  uint32_t last = 0;
  const int64_t c_first = p * P.GS, c_last = min64((p + 1) * P.GS, P.Q) - 1;
  const int64_t w_lo = flat_warp_of(P.ntiles, c_first / BC, P.nw);
  const int64_t w_hi = flat_warp_of(P.ntiles, c_last / BC, P.nw);
  if (lane == 0) {
    const uint32_t old = atomicAdd(P.cnt + p, 1u);
    last = (old == (uint32_t)(w_hi - w_lo)) ? 1u : 0u;
  }
  last = __shfl_sync(0xffffffffu, last, 0);
  if (!last) return;
  __threadfence();
  for (int e = lane; e < P.A; e += 32) {
    double sum = __ldcg(P.rec + (w_lo + p) * P.A + e);
    for (int64_t w = w_lo + 1; w <= w_hi; ++w) sum += __ldcg(P.rec + (w + p) * P.A + e);
    P.part[p * P.A + e] = sum;
  }
  if (lane == 0) P.cnt[p] = 0u;  // ready for the next call (stream order)
}

template <int MT, int NT1, bool M3, int TPB, int WARPS, bool CB>
__global__ void __launch_bounds__(WARPS * 32, 1)
    core_flat_kernel(const __grid_constant__ CUtensorMap tmap, const __grid_constant__ CoreParams P) {
  constexpr int BC = 16 * TPB;
  const int BOX = CB ? P.cb * BC : 16 * BC;  // doubles per TMA box
  constexpr int KP = MT == 1 ? 2 : 1;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  const int NS = P.nstages;
  const uint32_t pad = (1024u - (smem_u32(smem_raw) & 1023u)) & 1023u;
  double* rings = reinterpret_cast<double*>(smem_raw + pad);
  double* ufrag = rings + (size_t)WARPS * NS * BOX;
  double* slots = ufrag + (size_t)(P.RB / 4) * MT * 32;
  uint64_t* bars = reinterpret_cast<uint64_t*>(slots + (size_t)WARPS * P.A);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, tq = lane & 3;
  double* ring = rings + (size_t)warp * NS * BOX;
  uint64_t* bar = bars + warp * NS;
  double* slot = slots + (size_t)warp * P.A;

  const int r0 = P.r0, r1 = P.frank[0];
  const int n1 = (int)P.fdim[0];
  const double* __restrict__ U1 = P.fu[0];
  const int nbox = CB ? 1 : (int)((P.n0 + 15) / 16);
  const int KS = P.RB / 4;  // k-steps of a whole-column box (CB)
  // CB: column (2g + par) of the box, row tq; + 4 ks per k-step, + 16 cb per h
  const int boffc0 = (2 * g) * P.cb + tq, boffc1 = boffc0 + P.cb;

  int boff[2][4];
#pragma unroll
  for (int par = 0; par < 2; ++par)
#pragma unroll
    for (int ks = 0; ks < 4; ++ks) {
      const int col = 2 * g + par, row = 4 * ks + tq;
      boff[par][ks] = col * 16 + ((((row >> 1) ^ (col & 7)) << 1) | (row & 1));
    }

  for (int e = threadIdx.x; e < (P.RB / 4) * MT * 32; e += WARPS * 32) ufrag[e] = P.ufrag[e];
  if (lane == 0) {
    for (int s = 0; s < NS; ++s) mbar_init(&bar[s], 1);
    fence_mbar_init();
  }
  if (M3)
    for (int e = lane; e < P.A; e += 32) slot[e] = 0.0;
  __syncthreads();

  const int64_t gw = (int64_t)blockIdx.x * WARPS + warp;
  const int64_t t_lo = flat_tile_lo(P.ntiles, gw, P.nw), t_hi = flat_tile_lo(P.ntiles, gw + 1, P.nw);
  if (t_lo >= t_hi) return;

  // producer walk over (tile, box)
  int64_t pt = t_lo;
  int pb = 0;
  if (P.use_tma && lane == 0) {
    prefetch_tmap(&tmap);
    for (int s = 0; s < NS && pt < t_hi; ++s) {
      mbar_arrive_expect_tx(&bar[s], BOX * sizeof(double));
      tma_load_2d(ring + s * BOX, &tmap, &bar[s], 16 * pb, (int32_t)(BC * pt));
      if (++pb == nbox) {
        pb = 0;
        ++pt;
      }
    }
  }
  (void)pb;

  int stage = 0;
  uint32_t phase = 0;
  double r2[MT][NT1][2];
#pragma unroll
  for (int mt = 0; mt < MT; ++mt)
#pragma unroll
    for (int nt = 0; nt < NT1; ++nt) r2[mt][nt][0] = r2[mt][nt][1] = 0.0;
  int64_t cur_g2 = -1;  // level-2 group held in r2
  int64_t cur_p = -1;   // level-3 group held in the slot (M3)
  const int64_t n2 = M3 ? P.fdim[1] : 1;

  // r2 (level-2 group g2) -> record (m = 2) or -> slot of its level-3 group
  auto retire = [&](int64_t g2) {
    if (M3) {
      const int64_t p = g2 / n2;
      if (p != cur_p) {
        if (cur_p >= 0) {
          __syncwarp();
          double* dst = P.rec + (gw + cur_p) * P.A;
          for (int e = lane; e < P.A; e += 32) {
            dst[e] = slot[e];
            slot[e] = 0.0;
          }
          flat_emit<WARPS>(P, gw, cur_p, lane, BC);
          __syncwarp();
        }
        cur_p = p;
      }
      const int r2n = P.frank[1];
      const double* __restrict__ U2 = P.fu[1] + (g2 % n2) * r2n;
#pragma unroll
      for (int mt = 0; mt < MT; ++mt)
#pragma unroll
        for (int nt = 0; nt < NT1; ++nt)
#pragma unroll
          for (int v = 0; v < 2; ++v) {
            const int a0 = g + 8 * mt, a1 = 2 * tq + v + 8 * nt;
            if (a0 < r0 && a1 < r1) {
              const double val = r2[mt][nt][v];
              double* dst = slot + a0 + r0 * a1;
              for (int a2 = 0; a2 < r2n; ++a2) dst[(size_t)r0 * r1 * a2] += val * __ldg(U2 + a2);
            }
            r2[mt][nt][v] = 0.0;
          }
      __syncwarp();
    } else {
      double* dst = P.rec + (gw + g2) * P.A;
#pragma unroll
      for (int mt = 0; mt < MT; ++mt)
#pragma unroll
        for (int nt = 0; nt < NT1; ++nt)
#pragma unroll
          for (int v = 0; v < 2; ++v) {
            const int a0 = g + 8 * mt, a1 = 2 * tq + v + 8 * nt;
            if (a0 < r0 && a1 < r1) dst[a0 + r0 * a1] = r2[mt][nt][v];
            r2[mt][nt][v] = 0.0;
          }
      flat_emit<WARPS>(P, gw, g2, lane, BC);
    }
  };

  int64_t grp = (t_lo * BC) / n1;
  int off = (int)(t_lo * BC - grp * n1);
  for (int64_t t = t_lo; t < t_hi; ++t) {
    const int64_t c0 = (int64_t)BC * t;
    double tacc[TPB][2][MT][KP][2];
#pragma unroll
    for (int h = 0; h < TPB; ++h)
#pragma unroll
      for (int par = 0; par < 2; ++par)
#pragma unroll
        for (int mt = 0; mt < MT; ++mt)
#pragma unroll
          for (int kp = 0; kp < KP; ++kp) tacc[h][par][mt][kp][0] = tacc[h][par][mt][kp][1] = 0.0;
    const double* uf = ufrag + lane;
    if constexpr (CB) {
      // one box = BC whole columns (pitch cb), KS k-steps of 4 rows each
      double* st = ring + stage * BOX;
      mbar_wait(&bar[stage], phase);
      auto kstep = [&](int ks, int kp) {
        double a[MT];
#pragma unroll
        for (int mt = 0; mt < MT; ++mt) a[mt] = uf[(ks * MT + mt) * 32];
#pragma unroll
        for (int h = 0; h < TPB; ++h) {
          const double x0 = st[h * 16 * P.cb + boffc0 + 4 * ks];
          const double x1 = st[h * 16 * P.cb + boffc1 + 4 * ks];
#pragma unroll
          for (int mt = 0; mt < MT; ++mt) {
            dmma_8x8x4(tacc[h][0][mt][kp][0], tacc[h][0][mt][kp][1], a[mt], x0);
            dmma_8x8x4(tacc[h][1][mt][kp][0], tacc[h][1][mt][kp][1], a[mt], x1);
          }
        }
      };
      int ks = 0;
      for (; ks + 1 < KS; ks += 2) {
        kstep(ks, 0);
        kstep(ks + 1, KP - 1);
      }
      if (ks < KS) kstep(ks, 0);
      __syncwarp();
      if (lane == 0 && pt < t_hi) {
        mbar_arrive_expect_tx(&bar[stage], BOX * sizeof(double));
        tma_load_2d(st, &tmap, &bar[stage], 0, (int32_t)(BC * pt));
        ++pt;
      }
      if (++stage == NS) {
        stage = 0;
        phase ^= 1;
      }
    }
    for (int b = 0; b < (CB ? 0 : nbox); ++b, uf += 4 * MT * 32) {
      double* st = ring + stage * BOX;
      if (P.use_tma) {
        mbar_wait(&bar[stage], phase);
      } else {
        const int64_t row0 = 16 * b;
        for (int e = lane; e < BOX; e += 32) {
          const int jj = e >> 4, ii = e & 15;
          const int64_t row = row0 + ii, col = c0 + jj;
          const double v = (row < P.n0 && col < P.Q) ? P.x[col * P.n0 + row] : 0.0;
          st[jj * 16 + ((((ii >> 1) ^ (jj & 7)) << 1) | (ii & 1))] = v;
        }
        __syncwarp();
      }
#pragma unroll
      for (int ks = 0; ks < 4; ++ks) {
        double a[MT];
#pragma unroll
        for (int mt = 0; mt < MT; ++mt) a[mt] = uf[(ks * MT + mt) * 32];
#pragma unroll
        for (int h = 0; h < TPB; ++h) {
          const double x0 = st[h * 256 + boff[0][ks]];
          const double x1 = st[h * 256 + boff[1][ks]];
#pragma unroll
          for (int mt = 0; mt < MT; ++mt) {
            double* d0 = tacc[h][0][mt][ks % KP];
            double* d1 = tacc[h][1][mt][ks % KP];
            dmma_8x8x4(d0[0], d0[1], a[mt], x0);
            dmma_8x8x4(d1[0], d1[1], a[mt], x1);
          }
        }
      }
      __syncwarp();
      if (P.use_tma && lane == 0 && pt < t_hi) {
        mbar_arrive_expect_tx(&bar[stage], BOX * sizeof(double));
        tma_load_2d(st, &tmap, &bar[stage], 16 * pb, (int32_t)(BC * pt));
        if (++pb == nbox) {
          pb = 0;
          ++pt;
        }
      }
      if (++stage == NS) {
        stage = 0;
        phase ^= 1;
      }
    }
    if (KP == 2) {
#pragma unroll
      for (int h = 0; h < TPB; ++h)
#pragma unroll
        for (int par = 0; par < 2; ++par)
#pragma unroll
          for (int mt = 0; mt < MT; ++mt) {
            tacc[h][par][mt][0][0] += tacc[h][par][mt][KP - 1][0];
            tacc[h][par][mt][0][1] += tacc[h][par][mt][KP - 1][1];
          }
    }
#pragma unroll
    for (int h = 0; h < TPB; ++h) {
      const int64_t ch = c0 + 16 * h;
      if (ch >= P.Q) break;
      const int lim = (int)min64(16, P.Q - ch);
      if (off + 16 <= n1 && lim == 16) {
        if (grp != cur_g2) {
          if (cur_g2 >= 0) retire(cur_g2);
          cur_g2 = grp;
        }
        const double* urow = U1 + (off + 4 * tq) * r1 + g;
#pragma unroll
        for (int par = 0; par < 2; ++par)
#pragma unroll
          for (int s2 = 0; s2 < 2; ++s2) {
            double bv[NT1];
#pragma unroll
            for (int nt = 0; nt < NT1; ++nt)
              bv[nt] = (g + 8 * nt < r1) ? __ldg(urow + (2 * s2 + par) * r1 + 8 * nt) : 0.0;
#pragma unroll
            for (int mt = 0; mt < MT; ++mt)
#pragma unroll
              for (int nt = 0; nt < NT1; ++nt)
                dmma_8x8x4(r2[mt][nt][0], r2[mt][nt][1], tacc[h][par][mt][0][s2], bv[nt]);
          }
      } else {
        int64_t gg = grp;
        int oo = off;
        for (int lo = 0; lo < lim;) {
          const int hi = min(lim, lo + n1 - oo);
          if (gg != cur_g2) {
            if (cur_g2 >= 0) retire(cur_g2);
            cur_g2 = gg;
          }
          const double* ubase = U1 + (oo - lo) * r1 + g;
#pragma unroll
          for (int par = 0; par < 2; ++par)
#pragma unroll
            for (int s2 = 0; s2 < 2; ++s2) {
              const int j = 4 * tq + 2 * s2 + par;
              const bool ok = j >= lo && j < hi;
              double bv[NT1];
#pragma unroll
              for (int nt = 0; nt < NT1; ++nt)
                bv[nt] = (ok && g + 8 * nt < r1) ? __ldg(ubase + j * r1 + 8 * nt) : 0.0;
#pragma unroll
              for (int mt = 0; mt < MT; ++mt)
#pragma unroll
                for (int nt = 0; nt < NT1; ++nt)
                  dmma_8x8x4(r2[mt][nt][0], r2[mt][nt][1], tacc[h][par][mt][0][s2], bv[nt]);
            }
          oo += hi - lo;
          lo = hi;
          if (oo >= n1) {
            oo -= n1;
            ++gg;
          }
        }
      }
      off += 16;
      while (off >= n1) {
        off -= n1;
        ++grp;
      }
    }
  }
  // range end: retire the open level-2 group, then (M3) the open slot
  if (cur_g2 >= 0) retire(cur_g2);
  if (M3 && cur_p >= 0) {
    __syncwarp();
    double* dst = P.rec + (gw + cur_p) * P.A;
    for (int e = lane; e < P.A; e += 32) dst[e] = slot[e];
    flat_emit<WARPS>(P, gw, cur_p, lane, BC);
  }
}

// U0 -> fragment order [rho][kstep][mt][lane] = U0[rho*RB + 4 kstep + lane%4][8 mt + lane/4].
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
// partial inputs in a fixed order. Four independent accumulators keep
// several loads in flight per thread (the tail is latency-, not
// bandwidth-bound).
__global__ void ttm_kernel(const TtmParams T) {
  const int64_t total = T.g * T.rr * T.post;
  for (int64_t o = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; o < total;
       o += (int64_t)gridDim.x * blockDim.x) {
    const int64_t gi = o % T.g;
    const int64_t rest = o / T.g;
    const int64_t b = rest % T.rr;
    const int64_t pi = rest / T.rr;
    const double* in = T.in + gi + T.g * T.n * pi;
    const int64_t cs = T.transpose ? 1 : T.rr;  // coef stride along i
    const double* cf = T.transpose ? T.u + T.n * b : T.u + b;
    double s0 = 0, s1 = 0, s2 = 0, s3 = 0;
    int64_t i = 0;
    if (T.nparts == 1) {
      for (; i + 3 < T.n; i += 4) {
        s0 += in[T.g * i] * cf[cs * i];
        s1 += in[T.g * (i + 1)] * cf[cs * (i + 1)];
        s2 += in[T.g * (i + 2)] * cf[cs * (i + 2)];
        s3 += in[T.g * (i + 3)] * cf[cs * (i + 3)];
      }
      for (; i < T.n; ++i) s0 += in[T.g * i] * cf[cs * i];
    } else {
      for (; i < T.n; ++i) {
        const double* pp = in + T.g * i;
        double v0 = pp[0], v1 = 0, v2 = 0, v3 = 0;
        int q = 1;
        for (; q + 2 < T.nparts; q += 3) {
          v1 += pp[q * T.part_stride];
          v2 += pp[(q + 1) * T.part_stride];
          v3 += pp[(q + 2) * T.part_stride];
        }
        for (; q < T.nparts; ++q) v1 += pp[q * T.part_stride];
        s0 += ((v0 + v1) + (v2 + v3)) * cf[cs * i];
      }
    }
    T.out[o] = (s0 + s1) + (s2 + s3);
  }
}

// Latency-bound variant for small outputs: S lanes share one output, each
// summing every S-th term of the contraction (and of the part sum), then a
// fixed xor-tree combines them -- about one memory round trip per output
// instead of n / 4. Deterministic (fixed order).
template <int S>
__global__ void ttm_split_kernel(const TtmParams T) {
  const int64_t total = T.g * T.rr * T.post;
  const int lane = threadIdx.x & 31, sub = lane % S;
  const int64_t per_warp = 32 / S;
  const int64_t warp_id = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) / 32;
  const int64_t nwarps = (int64_t)gridDim.x * blockDim.x / 32;
  for (int64_t o0 = warp_id * per_warp; o0 < total; o0 += nwarps * per_warp) {
    const int64_t o = o0 + lane / S;
    const bool act = o < total;
    double s0 = 0.0, s1 = 0.0;
    if (act) {
      const int64_t gi = o % T.g;
      const int64_t rest = o / T.g;
      const int64_t b = rest % T.rr;
      const int64_t pi = rest / T.rr;
      const double* in = T.in + gi + T.g * T.n * pi;
      const int64_t cs = T.transpose ? 1 : T.rr;
      const double* cf = T.transpose ? T.u + T.n * b : T.u + b;
      if (T.nparts == 1) {
        int64_t i = sub;
        for (; i + S < T.n; i += 2 * S) {
          s0 = fma(in[T.g * i], cf[cs * i], s0);
          s1 = fma(in[T.g * (i + S)], cf[cs * (i + S)], s1);
        }
        if (i < T.n) s0 = fma(in[T.g * i], cf[cs * i], s0);
      } else {
        // lanes split the flattened (i, part) space: lane sub takes every
        // S-th (i, q) pair in i-major order (fixed order per lane)
        // (four loads in flight, the sum in the same order)
        const int64_t np = T.nparts, total_iq = T.n * np;
        for (int64_t e = sub; e < total_iq; e += 4 * S) {
          double v[4], w[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int64_t ee = e + (int64_t)u * S;
            const bool in_range = ee < total_iq;
            const int64_t i = in_range ? ee / np : 0, q = in_range ? ee - i * np : 0;
            v[u] = in_range ? in[T.g * i + q * T.part_stride] : 0.0;
            w[u] = in_range ? cf[cs * i] : 0.0;
          }
#pragma unroll
          for (int u = 0; u < 4; ++u)
            if (e + (int64_t)u * S < total_iq) s0 = fma(v[u], w[u], s0);
        }
      }
    }
    double s = s0 + s1;
#pragma unroll
    for (int off = S / 2; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
    if (act && sub == 0) T.out[o] = s;
  }
}

// Input-once variant: one thread per (gi, pi) accumulates all rr outputs in
// registers, so every input element (and the part sum) is read exactly once;
// consecutive threads take consecutive gi (coalesced loads and stores).
template <int RR>
__global__ void ttm_all_kernel(const TtmParams T) {
  const int64_t pairs = T.g * T.post;
  for (int64_t o = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; o < pairs;
       o += (int64_t)gridDim.x * blockDim.x) {
    const int64_t gi = o % T.g, pi = o / T.g;
    const double* in = T.in + gi + T.g * T.n * pi;
    double acc[RR];
#pragma unroll
    for (int b = 0; b < RR; ++b) acc[b] = 0.0;
    // coefficient (i, b): U^T (u is n x rr) or U (u is rr x n)
    const int64_t cs = T.transpose ? T.n : 1, ci = T.transpose ? 1 : T.rr;
    constexpr int kB = 8;  // rows per batch: their loads are in flight together
    for (int64_t i0 = 0; i0 < T.n; i0 += kB) {
      double v[kB];
#pragma unroll
      for (int u = 0; u < kB; ++u) {
        const int64_t i = i0 + u;
        v[u] = 0.0;
        if (i < T.n) {
          const double* pp = in + T.g * i;
          double s0 = pp[0];
          for (int q = 1; q < T.nparts; ++q) s0 += pp[q * T.part_stride];
          v[u] = s0;
        }
      }
#pragma unroll
      for (int u = 0; u < kB; ++u) {
        const int64_t i = i0 + u;
        if (i < T.n) {
          const double* cf = T.u + ci * i;
#pragma unroll
          for (int b = 0; b < RR; ++b)
            if (b < T.rr) acc[b] = fma(v[u], __ldg(cf + cs * b), acc[b]);
        }
      }
    }
    double* out = T.out + gi + T.g * T.rr * pi;
#pragma unroll
    for (int b = 0; b < RR; ++b)
      if (b < T.rr) out[T.g * b] = acc[b];
  }
}

// Bandwidth variant for large inputs: CTA (pi, gi-block) with 64 gi x 4
// i-groups; each thread accumulates all rr outputs of its gi over every 4th
// i (coalesced 512-byte rows of the input, U through shared memory), then
// the 4 i-groups are combined in a fixed order (deterministic).
template <int RR>
__global__ void __launch_bounds__(256) ttm_block_kernel(const TtmParams T) {
  __shared__ double red[4][RR][64];
  extern __shared__ double ush[];  // n x rr coefficients, [i][b]
  const int tx = threadIdx.x & 63, ty = threadIdx.x >> 6;
  const int64_t pi = blockIdx.x;
  const int64_t gi = (int64_t)blockIdx.y * 64 + tx;
  const int64_t cs = T.transpose ? T.n : 1, ci = T.transpose ? 1 : T.rr;
  for (int64_t e = threadIdx.x; e < T.n * T.rr; e += 256) {
    const int64_t i = e / T.rr, b = e % T.rr;
    ush[e] = T.u[ci * i + cs * b];
  }
  __syncthreads();
  double acc[RR];
#pragma unroll
  for (int b = 0; b < RR; ++b) acc[b] = 0.0;
  if (gi < T.g) {
    const double* in = T.in + gi + T.g * T.n * pi;
    constexpr int kB = 8;  // loads in flight per thread
    for (int64_t i0 = ty; i0 < T.n; i0 += 4 * kB) {
      double v[kB];
#pragma unroll
      for (int u = 0; u < kB; ++u) {
        const int64_t i = i0 + 4 * u;
        v[u] = 0.0;
        if (i < T.n) {
          const double* pp = in + T.g * i;
          double s0 = pp[0];
          for (int q = 1; q < T.nparts; ++q) s0 += pp[q * T.part_stride];
          v[u] = s0;
        }
      }
#pragma unroll
      for (int u = 0; u < kB; ++u) {
        const int64_t i = i0 + 4 * u;
        if (i < T.n) {
          const double* uc = ush + i * T.rr;
#pragma unroll
          for (int b = 0; b < RR; ++b)
            if (b < T.rr) acc[b] = fma(v[u], uc[b], acc[b]);
        }
      }
    }
  }
#pragma unroll
  for (int b = 0; b < RR; ++b) red[ty][b][tx] = acc[b];
  __syncthreads();
  for (int e = threadIdx.x; e < RR * 64; e += 256) {
    const int b = e / 64, x = e % 64;
    const int64_t go = (int64_t)blockIdx.y * 64 + x;
    if (b < T.rr && go < T.g)
      T.out[go + T.g * (b + T.rr * pi)] = ((red[0][b][x] + red[1][b][x]) + red[2][b][x]) + red[3][b][x];
  }
}

// Few slabs (post < 64), long contraction: split the mode over gridDim.y
// chunks; CTA (gi-block, chunk) writes a partial of its 64 rows x rr
// outputs, and ttm_splitk_reduce_kernel sums the chunks in order
// (deterministic). post is looped inside the CTA.
template <int RR>
__global__ void __launch_bounds__(256) ttm_splitk_kernel(const TtmParams T, int64_t chunk, double* partial) {
  __shared__ double red[2][RR][64];
  // the factor rows of one 64-row tile of the mode (read by every thread);
  // overlays red, which is only used after the accumulation (barrier between)
  double (*us)[RR + 1] = reinterpret_cast<double (*)[RR + 1]>(&red[0][0][0]);
  static_assert(64 * (RR + 1) <= 2 * RR * 64, "tile overlay");
  const int tx = threadIdx.x & 63, ty = threadIdx.x >> 6;
  const int64_t gi = (int64_t)blockIdx.x * 64 + tx;
  const int64_t i_lo = (int64_t)blockIdx.y * chunk, i_hi = min64(T.n, i_lo + chunk);
  const int64_t cs = T.transpose ? T.n : 1, ci = T.transpose ? 1 : T.rr;
  for (int64_t pi = 0; pi < T.post; ++pi) {
    double acc[RR];
#pragma unroll
    for (int b = 0; b < RR; ++b) acc[b] = 0.0;
    const double* in = T.in + gi + T.g * T.n * pi;
    constexpr int kB = 4;
    for (int64_t t0 = i_lo; t0 < i_hi; t0 += 64) {
      __syncthreads();
      for (int e = threadIdx.x; e < 64 * RR; e += 256) {
        const int ii = T.transpose ? e % 64 : e / RR, b = T.transpose ? e / 64 : e % RR;
        const int64_t i = t0 + ii;
        us[ii][b] = (i < i_hi && b < T.rr) ? __ldg(T.u + ci * i + cs * b) : 0.0;
      }
      __syncthreads();
      if (gi < T.g) {
        const int64_t t1 = min64(i_hi, t0 + 64);
        for (int64_t i0 = t0 + ty; i0 < t1; i0 += 4 * kB) {
          double v[kB];
#pragma unroll
          for (int u = 0; u < kB; ++u) {
            const int64_t i = i0 + 4 * u;
            v[u] = 0.0;
            if (i < t1) {
              // the parts four at a time: independent loads, the same left-to-right sum
              const double* pp = in + T.g * i;
              double s0 = 0.0;
              for (int q0 = 0; q0 < T.nparts; q0 += 4) {
                double pv[4];
#pragma unroll
                for (int w = 0; w < 4; ++w) pv[w] = q0 + w < T.nparts ? pp[(int64_t)(q0 + w) * T.part_stride] : 0.0;
#pragma unroll
                for (int w = 0; w < 4; ++w)
                  if (q0 + w < T.nparts) s0 = (q0 + w == 0) ? pv[w] : s0 + pv[w];
              }
              v[u] = s0;
            }
          }
#pragma unroll
          for (int u = 0; u < kB; ++u) {
            const int64_t i = i0 + 4 * u;
            if (i < t1) {
              const double* cf = us[(int)(i - t0)];
#pragma unroll
              for (int b = 0; b < RR; ++b)
                if (b < T.rr) acc[b] = fma(v[u], cf[b], acc[b]);
            }
          }
        }
      }
    }
    // fixed-order combine of the 4 i-groups: (g0 + g2) + (g1 + g3)
    __syncthreads();
    if (ty >= 2)
#pragma unroll
      for (int b = 0; b < RR; ++b) red[ty - 2][b][tx] = acc[b];
    __syncthreads();
    if (ty < 2)
#pragma unroll
      for (int b = 0; b < RR; ++b) acc[b] += red[ty][b][tx];
    __syncthreads();
    if (ty == 1)
#pragma unroll
      for (int b = 0; b < RR; ++b) red[0][b][tx] = acc[b];
    __syncthreads();
    if (ty == 0) {
      const int64_t go = (int64_t)blockIdx.x * 64 + tx;
      if (go < T.g)
#pragma unroll
        for (int b = 0; b < RR; ++b)
          if (b < T.rr)
            partial[(((int64_t)blockIdx.y * T.post + pi) * T.rr + b) * T.g + go] = acc[b] + red[0][b][tx];
    }
  }
}

__global__ void ttm_splitk_reduce_kernel(const TtmParams T, int nchunks, const double* __restrict__ partial) {
  const int64_t total = T.g * T.rr * T.post;  // output order: gi fastest, then b, then pi
  for (int64_t o = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; o < total;
       o += (int64_t)gridDim.x * blockDim.x) {
    const int64_t gi = o % T.g, rest = o / T.g;
    const int64_t b = rest % T.rr, pi = rest / T.rr;
    double sum = 0.0;
    for (int c = 0; c < nchunks; ++c) sum += partial[(((int64_t)c * T.post + pi) * T.rr + b) * T.g + gi];
    T.out[o] = sum;
  }
}

// All factor reformatting of a core pass in one launch: blockIdx.y = 0
// builds U0's fragments, 1..2 transpose U1, U2 to row-major.
struct PrepJobs {
  CoreItem* items;
  int64_t nitems, G, GS, SL, n1;
  int S, A;
  const double* u0;
  double* ufrag;
  int64_t n0;
  int r0, RB, NT, nrb;
  const double* u[2];
  double* ut[2];
  int64_t n[2];
  int r[2];
  int njobs;
  uint32_t* cnt;  // flat mode: group counters to clear
  int64_t ncnt;
};

__global__ void prep_all_kernel(const PrepJobs J) {
  if ((int)blockIdx.y == J.njobs + 1) {
    for (int64_t it = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; it < J.ncnt;
         it += (int64_t)gridDim.x * blockDim.x)
      J.cnt[it] = 0u;
    // item table, rho-major: consecutive items of a CTA share the row block
    for (int64_t it = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; it < J.nitems;
         it += (int64_t)gridDim.x * blockDim.x) {
      const int64_t per_rho = J.G * J.S;
      const int rho = (int)(it / per_rho);
      const int64_t rest = it - (int64_t)rho * per_rho;
      const int64_t p = rest / J.S;
      const int sigma = (int)(rest - p * J.S);
      CoreItem I;
      I.c_lo = p * J.GS + (int64_t)sigma * J.SL;
      const int64_t c_hi = min64(I.c_lo + J.SL, (p + 1) * J.GS);
      I.len = (int)(c_hi - I.c_lo);
      I.rho = rho;
      I.out_off = (((int64_t)rho * J.S + sigma) * J.G + p) * J.A;
      I.grp0 = I.c_lo / J.n1;
      I.off0 = (int)(I.c_lo - I.grp0 * J.n1);
      I.pad = 0;
      J.items[it] = I;
    }
  } else if (blockIdx.y == 0) {
    const int64_t total = (int64_t)J.nrb * J.RB * J.NT * 8;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
         e += (int64_t)gridDim.x * blockDim.x) {
      const int lane = (int)(e % 32);
      int64_t rest = e / 32;
      const int nt = (int)(rest % J.NT);
      rest /= J.NT;
      const int64_t kstep = rest % (J.RB / 4);
      const int64_t rho = rest / (J.RB / 4);
      const int64_t row = rho * J.RB + 4 * kstep + (lane & 3);
      const int col = 8 * nt + (lane >> 2);
      J.ufrag[e] = (row < J.n0 && col < J.r0) ? J.u0[row + J.n0 * col] : 0.0;
    }
  } else if ((int)blockIdx.y <= J.njobs) {
    const int j = blockIdx.y - 1;
    const int64_t n = J.n[j];
    const int r = J.r[j];
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n * r;
         e += (int64_t)gridDim.x * blockDim.x)
      J.ut[j][e] = J.u[j][(e / r) + n * (e % r)];
  }
}

template <int MT, int NT1, bool M3, int TPB, int WARPS>
cudaError_t launch_w(const CUtensorMap* tmap, const CoreParams& P, int grid, size_t smem, cudaStream_t s) {
  if (P.flat) {
    if constexpr (MT == 1 && TPB == 1) {
      if (P.cb) {
        cudaError_t e = SRTT_ENSURE_SMEM((core_flat_kernel<MT, NT1, M3, TPB, WARPS, true>), smem);
        if (e != cudaSuccess) return e;
        core_flat_kernel<MT, NT1, M3, TPB, WARPS, true><<<grid, WARPS * 32, smem, s>>>(*tmap, P);
        return cudaGetLastError();
      }
    }
    if (P.cb) return cudaErrorInvalidValue;
    cudaError_t e = SRTT_ENSURE_SMEM((core_flat_kernel<MT, NT1, M3, TPB, WARPS, false>), smem);
    if (e != cudaSuccess) return e;
    core_flat_kernel<MT, NT1, M3, TPB, WARPS, false><<<grid, WARPS * 32, smem, s>>>(*tmap, P);
    return cudaGetLastError();
  }
  cudaError_t e = SRTT_ENSURE_SMEM((core_kernel<MT, NT1, M3, TPB, WARPS>), smem);
  if (e != cudaSuccess) return e;
  core_kernel<MT, NT1, M3, TPB, WARPS><<<grid, WARPS * 32, smem, s>>>(*tmap, P);
  return cudaGetLastError();
}

template <int MT, int NT1, bool M3, int TPB>
cudaError_t launch_t(const CUtensorMap* tmap, const CoreParams& P, int grid, size_t smem, cudaStream_t s) {
  if (MT * NT1 <= 4 && P.warps == 16) return launch_w<MT, NT1, M3, TPB, (MT * NT1 <= 4 ? 16 : 8)>(tmap, P, grid, smem, s);
  return launch_w<MT, NT1, M3, TPB, 8>(tmap, P, grid, smem, s);
}

template <int MT, int NT1, bool M3>
cudaError_t launch_b(const CUtensorMap* tmap, const CoreParams& P, int grid, size_t smem, cudaStream_t s) {
  switch (P.tpb) {
    case 1: return launch_t<MT, NT1, M3, 1>(tmap, P, grid, smem, s);
    case 2: return launch_t<MT, NT1, M3, (MT <= 2 && NT1 <= 2 ? 2 : 1)>(tmap, P, grid, smem, s);
  }
  return cudaErrorInvalidValue;
}

template <int MT, int NT1>
cudaError_t launch_m(const CUtensorMap* tmap, const CoreParams& P, int grid, size_t smem, cudaStream_t s) {
  return P.m == 3 ? launch_b<MT, NT1, true>(tmap, P, grid, smem, s)
                  : launch_b<MT, NT1, false>(tmap, P, grid, smem, s);
}

template <int MT>
cudaError_t launch_n(const CUtensorMap* tmap, const CoreParams& P, int grid, size_t smem, cudaStream_t s) {
  switch (P.NT1) {
    case 1: return launch_m<MT, 1>(tmap, P, grid, smem, s);
    case 2: return launch_m<MT, 2>(tmap, P, grid, smem, s);
    case 4: return launch_m<MT, 4>(tmap, P, grid, smem, s);
  }
  return cudaErrorInvalidValue;
}

}  // namespace

int srtt_core_threads() { return 256; }

// Shared memory of the core kernel for a given stage count.
size_t srtt_core_smem_bytes(const CoreParams& P) {
  const size_t w = P.warps;
  const size_t box = P.cb ? (size_t)P.cb * 16 * P.tpb : (size_t)256 * P.tpb;
  const size_t slot = (P.m == 2 && P.slot_ch && !P.flat) ? (size_t)P.slot_ch : (size_t)P.A;
  const size_t doubles = w * P.nstages * box + (size_t)(P.RB / 4) * P.NT * 32 + w * slot;
  return 1024 + doubles * sizeof(double) + w * P.nstages * sizeof(uint64_t);
}

int srtt_core_max_stages(const CoreParams& P, size_t budget) {
  CoreParams Q = P;
  int best = 0;
  for (int ns = 2; ns <= 16; ++ns) {
    Q.nstages = ns;
    if (srtt_core_smem_bytes(Q) <= budget) best = ns;
  }
  return best;
}

int srtt_core_occupancy(const CoreParams&) { return 1; }

cudaError_t srtt_launch_core(const CUtensorMap* tmap, const CoreParams& P, int grid, cudaStream_t s) {
  const size_t smem = srtt_core_smem_bytes(P);
  switch (P.NT) {
    case 1: return launch_n<1>(tmap, P, grid, smem, s);
    case 2: return launch_n<2>(tmap, P, grid, smem, s);
    case 4: return launch_n<4>(tmap, P, grid, smem, s);
  }
  return cudaErrorInvalidValue;
}

cudaError_t srtt_launch_prep(const double* u0, int64_t n0, int r0, int RB, int NT, int nrb, double* ufrag,
                             cudaStream_t s) {
  prep_kernel<<<64, 256, 0, s>>>(u0, n0, r0, RB, NT, nrb, ufrag);
  return cudaGetLastError();
}

cudaError_t srtt_launch_prep_all(const CoreParams& P, CoreItem* items, const double* u0, int64_t n0, int r0,
                                 int RB, int NT, int nrb, double* ufrag, int njobs, const double* const* u,
                                 double* const* ut, const int64_t* n, const int* r, cudaStream_t s) {
  PrepJobs J{};
  J.items = items;
  J.nitems = P.nitems;
  J.G = P.G;
  J.GS = P.GS;
  J.SL = P.SL;
  J.n1 = P.fdim[0];
  J.S = P.S;
  J.A = P.A;
  J.u0 = u0;
  J.ufrag = ufrag;
  J.n0 = n0;
  J.r0 = r0;
  J.RB = RB;
  J.NT = NT;
  J.nrb = nrb;
  J.njobs = njobs;
  J.cnt = P.flat ? P.cnt : nullptr;
  J.ncnt = P.flat ? P.G : 0;
  for (int j = 0; j < njobs; ++j) {
    J.u[j] = u[j];
    J.ut[j] = ut[j];
    J.n[j] = n[j];
    J.r[j] = r[j];
  }
  const int64_t total = (int64_t)nrb * RB * NT * 8;
  const int bx = (int)min64(256, (total + 255) / 256);
  prep_all_kernel<<<dim3(bx > 0 ? bx : 1, 2 + njobs), 256, 0, s>>>(J);
  return cudaGetLastError();
}

cudaError_t srtt_launch_transpose(const double* u, int64_t n, int r, double* ut, cudaStream_t s) {
  const int64_t total = n * r;
  const int blocks = (int)min64(1024, (total + 255) / 256);
  transpose_kernel<<<blocks > 0 ? blocks : 1, 256, 0, s>>>(u, n, r, ut);
  return cudaGetLastError();
}

cudaError_t srtt_launch_ttm(const TtmParams& T, cudaStream_t s) {
  const int64_t total = T.g * T.rr * T.post;
  const int64_t pairs = T.g * T.post;
  const double in_bytes = 8.0 * (double)T.g * T.n * T.post * T.nparts;
  if (T.rr <= 16 && T.post >= 64 && T.post < 65536 && in_bytes * T.rr > 64e6 && T.n * T.rr * 8 <= 48 * 1024) {
    // large input, many slabs: CTA per (slab, 64 rows), i split over 4 groups
    const dim3 grid((unsigned)T.post, (unsigned)((T.g + 63) / 64));
    const size_t sm = (size_t)T.n * T.rr * sizeof(double);
    cudaError_t e = T.rr <= 8 ? SRTT_ENSURE_SMEM(ttm_block_kernel<8>, sm) : SRTT_ENSURE_SMEM(ttm_block_kernel<16>, sm);
    if (e != cudaSuccess) return e;
    if (T.rr <= 8) ttm_block_kernel<8><<<grid, 256, sm, s>>>(T);
    else ttm_block_kernel<16><<<grid, 256, sm, s>>>(T);
    return cudaGetLastError();
  }
  if (T.rr <= 32 && T.post < 64 && T.scratch && in_bytes > 16e6) {
    // few slabs, long contraction (C5 tail: 1024 x 2048 x 4 parts): split-K
    const int64_t gblk = (T.g + 63) / 64;
    int64_t nch = std::max<int64_t>(1, std::min<int64_t>((148 * 4 + gblk - 1) / gblk, (T.n + 63) / 64));
    nch = std::min<int64_t>(nch, T.scratch_doubles / std::max<int64_t>(1, T.g * T.rr * T.post));
    if (nch >= 2) {
      const int64_t chunk = (T.n + nch - 1) / nch;
      nch = (T.n + chunk - 1) / chunk;
      const dim3 grid((unsigned)gblk, (unsigned)nch);
      if (T.rr <= 8) ttm_splitk_kernel<8><<<grid, 256, 0, s>>>(T, chunk, T.scratch);
      else if (T.rr <= 16) ttm_splitk_kernel<16><<<grid, 256, 0, s>>>(T, chunk, T.scratch);
      else ttm_splitk_kernel<32><<<grid, 256, 0, s>>>(T, chunk, T.scratch);
      cudaError_t e = cudaGetLastError();
      if (e != cudaSuccess) return e;
      const int64_t total = T.g * T.rr * T.post;
      ttm_splitk_reduce_kernel<<<(unsigned)min64(148 * 8, (total + 255) / 256), 256, 0, s>>>(T, (int)nch,
                                                                                            T.scratch);
      return cudaGetLastError();
    }
  }
  if (T.rr <= 32 && pairs >= 148 * 128 && in_bytes * T.rr > 64e6) {
    // large input re-read rr times by the per-output kernels: read it once
    const int blocks = (int)min64(148 * 8, (pairs + 127) / 128);
    if (T.rr <= 8) ttm_all_kernel<8><<<blocks, 128, 0, s>>>(T);
    else if (T.rr <= 16) ttm_all_kernel<16><<<blocks, 128, 0, s>>>(T);
    else ttm_all_kernel<32><<<blocks, 128, 0, s>>>(T);
    return cudaGetLastError();
  }
  if (total <= 148 * 256 * 2 && T.n * T.nparts >= 8) {
    // few outputs: spread each contraction (and part sum) over 8 lanes
    const int64_t threads = total * 8;
    const int blocks = (int)min64(148 * 8, (threads + 255) / 256);
    ttm_split_kernel<8><<<blocks > 0 ? blocks : 1, 256, 0, s>>>(T);
    return cudaGetLastError();
  }
  const int blocks = (int)min64(148 * 16, (total + 255) / 256);
  ttm_kernel<<<blocks > 0 ? blocks : 1, 256, 0, s>>>(T);
  return cudaGetLastError();
}
