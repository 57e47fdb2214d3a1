// K1 — fused fibre-sampling gather + Gaussian sketch (sm_100a).
//
// Replaces, per target (Tucker mode or H-Tucker node):
//   extract_fibers / extract_group_fibers   unfolding.hpp:32-111
//   gaussian_matrix (after the sampling draws) sampling.hpp:69-77
//   sketch = y * omega                       tucker.hpp:159-161, htucker.hpp:279-281
// with ONE grouped launch over all targets. Each thread owns one row i of the
// target's unfolding; it walks the sampled fibres j, loads X[base_j + off(i)]
// straight into a register (consecutive rows of a contiguous fibre are
// consecutive addresses, so warps issue coalesced loads) and accumulates
// Z(i, :) += x * Omega(j, :). Omega rows are generated in shared memory from
// the reference's counter-derived stream, chunk by chunk. The sampled fibres
// are never written anywhere. Partial sums over fibre groups are reduced in a
// fixed order, so Z is bitwise reproducible run to run.
#include "srtt_device.cuh"
#include "srtt_params.h"

namespace {

constexpr int kThreads = 256;
constexpr int kChunk = 128;  // fibres per Omega chunk held in shared memory

// Gather load with the smallest L2 fetch size: a strided target uses 8 bytes
// of every line it touches, so anything the L2 fetches beyond the sector is
// wasted DRAM traffic (ncu: 128 bytes per element with the default policy).
__device__ __forceinline__ double ldg_gather(const double* p) {
  double v;
  asm volatile("ld.global.nc.L2::64B.f64 %0, [%1];" : "=d"(v) : "l"(p));
  return v;
}

template <int CMAX>
__global__ void __launch_bounds__(kThreads) sketch_kernel(const SketchTarget* __restrict__ targets,
                                                          int ntargets) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ SketchTarget T;
  __shared__ int tsel;
  const int tid = threadIdx.x;
  if (tid == 0) {
    int lo = 0, hi = ntargets - 1;
    while (lo < hi) {  // last target with cta_begin <= blockIdx.x
      const int mid = (lo + hi + 1) >> 1;
      if (targets[mid].cta_begin <= (int64_t)blockIdx.x) lo = mid; else hi = mid - 1;
    }
    tsel = lo;
  }
  __syncthreads();
  {
    const int* src = reinterpret_cast<const int*>(&targets[tsel]);
    int* dst = reinterpret_cast<int*>(&T);
    for (int k = tid; k < (int)(sizeof(SketchTarget) / sizeof(int)); k += kThreads) dst[k] = src[k];
  }
  __syncthreads();

  const int ctot = T.c;
  const int cw = ctot < CMAX ? ctot : CMAX;  // columns per pass (more than CMAX columns: several passes)
  const int RT = T.row_tile;
  const int JS = kThreads / RT;
  const int il = tid % RT;
  const int js = tid / RT;
  // CTA -> (row tile, fibre chunk)
  const int64_t local = (int64_t)blockIdx.x - T.cta_begin;
  const int64_t row_ctas = (T.rows + RT - 1) / RT;
  const int64_t rt = local % row_ctas;
  const int fchunk = (int)(local / row_ctas);
  const int64_t flen = (T.w + T.fsplit - 1) / T.fsplit;
  const int64_t jbeg = (int64_t)fchunk * flen;
  const int64_t jend = srtt_dev::min64(T.w, jbeg + flen);
  const int64_t i = rt * RT + il;
  const bool active = (js < JS) && (i < T.rows);

  double* om = reinterpret_cast<double*>(smem_raw);         // kChunk x cw
  int64_t* base = reinterpret_cast<int64_t*>(om + kChunk * cw);  // kChunk
  double* red = reinterpret_cast<double*>(base + kChunk);    // kThreads x cw

  // Row offset of row i in the flat tensor: mixed-radix decode over S's
  // modes, first mode fastest (unfolding.hpp:81-108 row odometer).
  int64_t roff = 0;
  if (active) {
    int64_t rem = i;
    for (int mm = 0; mm < T.nrow_modes; ++mm) {
      const int64_t dm = T.row_dim[mm];
      roff += (rem % dm) * T.row_stride[mm];
      rem /= dm;
    }
  }

  const double* __restrict__ x = T.x;
  // flat-range sharding: only [flo, fhi) of the global flat index is local
  const int64_t flo = T.flat_lo, fhi = T.flat_hi;
  const bool ranged = fhi > 0;
  // Sketches wider than CMAX columns (r + p > 64) take one pass over the
  // sampled fibres per window of CMAX columns [c0, c0 + c).
  for (int c0 = 0; c0 < ctot; c0 += CMAX) {
  const int c = ctot - c0 < CMAX ? ctot - c0 : CMAX;
  double acc[CMAX];
#pragma unroll
  for (int cc = 0; cc < CMAX; ++cc) acc[cc] = 0.0;
  for (int64_t j0 = jbeg; j0 < jend; j0 += kChunk) {
    const int jn = (int)srtt_dev::min64(kChunk, jend - j0);
    __syncthreads();
    // Omega(j, cc) is normal number t = j + cc * w of the stream
    // (column-major gaussian_matrix fill, sampling.hpp:74-75).
    for (int idx = tid; idx < jn * c; idx += kThreads) {
      const int jl = idx / c, cc = idx - jl * c;
      const uint64_t t = (uint64_t)(j0 + jl) + (uint64_t)(cc + c0) * (uint64_t)T.w;
      om[jl * c + cc] = T.omega ? T.omega[t] : srtt_dev::normal_at(T.state0, T.draw_offset, t, T.flags);
    }
    // Fibre base offsets: decode the sampled column over the complement
    // modes, ascending, first fastest (unfolding.hpp:36-41, 71-75).
    for (int jl = tid; jl < jn; jl += kThreads) {
      int64_t col = T.cols[j0 + jl], b = 0;
      for (int mm = 0; mm < T.ncol_modes; ++mm) {
        const int64_t dm = T.col_dim[mm];
        int64_t dig = col % dm;
        if (mm == T.slab_digit) {
          if (dig < T.slab_lo || dig >= T.slab_hi) b = INT64_MIN / 2;  // not in this slab
          dig -= T.slab_lo;
        }
        b += dig * T.col_stride[mm];
        col /= dm;
      }
      base[jl] = b < 0 ? -1 : b;
    }
    __syncthreads();
    if (active && ranged) {
      for (int jl = js; jl < jn; jl += JS) {
        const int64_t o = base[jl] + roff;
        const double v = (o >= flo && o < fhi) ? __ldg(x + (o - flo)) : 0.0;
        const double* om_j = om + jl * c;
#pragma unroll
        for (int cc = 0; cc < CMAX; ++cc)
          if (cc < c) acc[cc] += v * om_j[cc];
      }
    } else if (active) {
      int jl = js;
      // 8, then 4, independent loads in flight per thread before the FMAs
      // (strided targets pay one DRAM burst per element: latency-bound).
      for (; jl + 7 * JS < jn; jl += 8 * JS) {
        double v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int64_t bu = base[jl + u * JS];
          v[u] = bu >= 0 ? ldg_gather(x + bu + roff) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const double* ou = om + (jl + u * JS) * c;
#pragma unroll
          for (int cc = 0; cc < CMAX; ++cc)
            if (cc < c) acc[cc] += v[u] * ou[cc];
        }
      }
      for (; jl + 3 * JS < jn; jl += 4 * JS) {
        const int64_t b0 = base[jl], b1 = base[jl + JS], b2 = base[jl + 2 * JS], b3 = base[jl + 3 * JS];
        const double v0 = b0 >= 0 ? ldg_gather(x + b0 + roff) : 0.0;
        const double v1 = b1 >= 0 ? ldg_gather(x + b1 + roff) : 0.0;
        const double v2 = b2 >= 0 ? ldg_gather(x + b2 + roff) : 0.0;
        const double v3 = b3 >= 0 ? ldg_gather(x + b3 + roff) : 0.0;
        const double* o0 = om + jl * c;
        const double* o1 = o0 + JS * c;
        const double* o2 = o1 + JS * c;
        const double* o3 = o2 + JS * c;
#pragma unroll
        for (int cc = 0; cc < CMAX; ++cc)
          if (cc < c) acc[cc] += v0 * o0[cc] + v1 * o1[cc] + v2 * o2[cc] + v3 * o3[cc];
      }
      for (; jl < jn; jl += JS) {
        const int64_t bj = base[jl];
        const double v = bj >= 0 ? ldg_gather(x + bj + roff) : 0.0;
        const double* o = om + jl * c;
#pragma unroll
        for (int cc = 0; cc < CMAX; ++cc)
          if (cc < c) acc[cc] += v * o[cc];
      }
    }
  }
  // Fixed-order reduction over the fibre groups js = 0..JS-1.
  __syncthreads();
  if (js < JS) {
#pragma unroll
    for (int cc = 0; cc < CMAX; ++cc)
      if (cc < c) red[(js * RT + il) * c + cc] = acc[cc];
  }
  __syncthreads();
  const int64_t ldz = T.ldz > 0 ? T.ldz : T.rows;
  for (int idx = tid; idx < RT * c; idx += kThreads) {
    const int rl = idx % RT, cc = idx / RT;
    const int64_t row = rt * RT + rl;
    if (row >= T.rows) continue;
    double s = 0.0;
    for (int g = 0; g < JS; ++g) s += red[(g * RT + rl) * c + cc];
    if (T.fsplit > 1)
      T.zpart[((int64_t)fchunk * ctot + cc + c0) * T.rows + row] = s;
    else
      T.z[row + (int64_t)(cc + c0) * ldz] = s;
  }
  }  // column windows
}

// ---------------------------------------------------------------------------
// Staged DMMA sketch for contiguous fibres with many fibres (K1c).
// Z(i, :) = sum_j X[cols[j] * rows + i] Omega(j, :): a GEMM whose A operand
// (rows x fibres) is gathered column by column. A CTA owns 64 rows and one
// fibre chunk; each stage brings 32 fibre segments (64 rows, coalesced
// 8-byte cp.async, any alignment; rows / fibres beyond the ends zero-fill)
// and the matching 32 rows of Omega into shared memory, kCStages deep, and
// the 8 warps (8 rows each) accumulate Z tiles with DMMA m8n8k4 (A = the
// fibre values, B = Omega, c padded to multiples of 8). Fixed k order:
// deterministic. Partials per fibre chunk as in sketch_kernel.
// ---------------------------------------------------------------------------
constexpr int kCRows = 128, kCFib = 28, kCStages = 3;  // ~101 KB: two CTAs per SM
constexpr int kCMW = kCRows / (8 * (kThreads / 32));  // 8-row tiles per warp (2: 16 rows)
constexpr int kCYld = kCRows + 4;  // = 4 (mod 16): conflict-free A fragment reads
constexpr int kCOld = 36;          // Omega stored transposed (column cc, fibre f), pitch = 4 (mod 16)
static_assert(kCFib % 4 == 0 && kCOld >= kCFib && kCOld % 16 == 4, "K1c stage geometry");

__device__ __forceinline__ void cp_async8z(void* smem, const double* g, bool ok) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(srtt_dev::smem_u32(smem)), "l"(g),
               "r"(ok ? 8u : 0u)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void cp_async16z(void* smem, const double* g, bool ok) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(srtt_dev::smem_u32(smem)), "l"(g),
               "r"(ok ? 16u : 0u)
               : "memory");
}
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

constexpr int kTYld = kCFib + 8;  // K1t: Y stored [row][fibre], pitch = 4 (mod 16)
static_assert(kTYld % 16 == 4, "K1t stage geometry");

// CT: 8-column tiles of c. TR = false: K1c (fibres contiguous, Y stored
// [fibre][row]); TR = true: K1t (sorted columns of a trailing-mode target,
// neighbouring fibres are neighbouring addresses; Y stored [row][fibre]).
template <int CT, bool TR>
__global__ void __launch_bounds__(kThreads) sketch_contig_kernel(const SketchTarget* __restrict__ targets,
                                                                 int ntargets) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ SketchTarget T;
  __shared__ int tsel;
  constexpr int CP = 8 * CT;  // Omega columns (c padded to the 8-wide tiles)
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, tq = lane & 3;
  if (tid == 0) {
    int lo = 0, hi = ntargets - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if ((TR ? targets[mid].cta_begin_t : targets[mid].cta_begin_c) <= (int64_t)blockIdx.x) lo = mid;
      else hi = mid - 1;
    }
    tsel = lo;
  }
  __syncthreads();
  {
    const int* src = reinterpret_cast<const int*>(&targets[tsel]);
    int* dst = reinterpret_cast<int*>(&T);
    for (int k = tid; k < (int)(sizeof(SketchTarget) / sizeof(int)); k += kThreads) dst[k] = src[k];
  }
  __syncthreads();
  const int c = T.c;
  const int64_t rows = T.rows;
  const int64_t local = (int64_t)blockIdx.x - (TR ? T.cta_begin_t : T.cta_begin_c);
  const int64_t row_ctas = (rows + kCRows - 1) / kCRows;
  const int64_t rt = local % row_ctas;
  const int fchunk = (int)(local / row_ctas);
  const int64_t flen = (T.w + T.fsplit - 1) / T.fsplit;
  const int64_t jbeg = (int64_t)fchunk * flen;
  const int64_t jend = srtt_dev::min64(T.w, jbeg + flen);
  const int64_t row0 = rt * kCRows;
  constexpr int kYst = TR ? kCRows * kTYld : kCFib * kCYld;  // Y doubles per stage
  double* Ys = reinterpret_cast<double*>(smem_raw);     // kCStages x (K1c: kCFib x kCYld, K1t: kCRows x kTYld)
  double* Os = Ys + kCStages * kYst;                    // kCStages x CP x kCOld (transposed)
  const double* __restrict__ x = T.x;
  const double* __restrict__ om = T.omega;

  // Fibre start offsets (cols[j] * rows) live in a small per-stage table in
  // shared memory, written by warp 0 one iteration ahead of the copies that
  // use them (its cols[] loads are issued another iteration earlier), so no
  // copy waits on a cols[] load and the 64-bit products are formed once.
  // Even `rows` (fibre starts 16-byte aligned): 2 rows per 16-byte
  // cp.async, else 1 row per 8-byte cp.async.
  __shared__ int64_t sbase[kCStages][kCFib];
  const bool pairs = (rows & 1) == 0;
  const int rpt = pairs ? 2 : 1;            // rows per copy
  const int tpf = kCRows / rpt;             // threads per fibre segment
  const int fstep = kThreads / tpf;         // fibres per pass
  const int npass = kCFib / fstep;
  const int r_me = (tid % tpf) * rpt, f_me = tid / tpf;
  const int64_t* __restrict__ cols = T.cols;
  int64_t creg = -1;                        // warp 0, lane < kCFib: cols[] of the stage after next
  auto fetch_cols = [&](int64_t j0) {
    if (warp == 0 && lane < kCFib) {
      const int64_t j = j0 + lane;
      creg = j < jend ? __ldg(cols + j) : -1;
    }
  };
  auto put_bases = [&](int s) {
    if (warp == 0 && lane < kCFib) sbase[s][lane] = creg >= 0 ? (TR ? creg : creg * rows) : -1;
  };
  // stage s <- fibres [j0, j0 + kCFib) (table sbase[s] already written)
  auto load = [&](int s, int64_t j0) {
    double* ys = Ys + s * kYst;
    double* os = Os + s * CP * kCOld;
    if constexpr (TR) {  // element (row i, fibre f) = X[cols_sorted[f] + ncols * i]: lanes = fibres
      if (lane < kCFib) {
        const int64_t b = sbase[s][lane];
        for (int i = warp; i < kCRows; i += kThreads / 32) {
          const int64_t row = row0 + i;
          const bool ok = b >= 0 && row < rows;
          cp_async8z(ys + i * kTYld + lane, ok ? x + b + T.ncols * row : x, ok);
        }
      }
    } else {
    const int64_t row = row0 + r_me;
    for (int i = 0; i < npass; ++i) {
      const int f = f_me + fstep * i;
      const int64_t b = sbase[s][f];
      const bool ok = b >= 0 && row < rows;  // rows even: row + 1 < rows too
      if (pairs)
        cp_async16z(ys + f * kCYld + r_me, ok ? x + b + row : x, ok);
      else
        cp_async8z(ys + f * kCYld + r_me, ok ? x + b + row : x, ok);
    }
    }
    // Omega(j, cc) column-major (ld w): warp w copies columns w, w + 8, ...
    // with one fibre per lane (coalesced), stored transposed
    if (lane < kCFib) {
      const int64_t j = j0 + lane;
      for (int cc = warp; cc < CP; cc += kThreads / 32) {
        const bool ok = j < jend && cc < c;
        cp_async8z(os + cc * kCOld + lane, ok ? om + j + (int64_t)cc * T.w : om, ok);
      }
    }
  };

  // KS interleaved accumulator sets (k steps kk = s mod KS) keep >= 4
  // independent DMMA chains per warp; summed in a fixed order at the end
  constexpr int KS = kCMW * CT >= 4 ? 1 : 4 / (kCMW * CT);
  double acc[KS][kCMW][CT][2];
#pragma unroll
  for (int ks = 0; ks < KS; ++ks)
#pragma unroll
    for (int m = 0; m < kCMW; ++m)
#pragma unroll
      for (int ct = 0; ct < CT; ++ct) acc[ks][m][ct][0] = acc[ks][m][ct][1] = 0.0;
  const int64_t nst = (jend - jbeg + kCFib - 1) / kCFib;
  // prologue: tables of stages 0 .. NST-1, copies of stages 0 .. NST-2
  for (int s = 0; s < kCStages; ++s) {
    fetch_cols(jbeg + (int64_t)s * kCFib);
    put_bases(s);
  }
  __syncthreads();
#pragma unroll
  for (int s = 0; s < kCStages - 1; ++s) {
    if (s < nst) load(s, jbeg + (int64_t)s * kCFib);
    cp_async_commit();
  }
  fetch_cols(jbeg + (int64_t)kCStages * kCFib);  // table of stage NST, written at iteration 0
  for (int64_t st = 0; st < nst; ++st) {
    cp_async_wait<kCStages - 2>();
    __syncthreads();
    {  // refill the stage freed by the previous iteration (its table was
       // written before the barrier); then the table of the stage after it
      const int64_t nx = st + kCStages - 1;
      if (nx < nst) load((int)(nx % kCStages), jbeg + nx * kCFib);
      cp_async_commit();
      put_bases((int)((nx + 1) % kCStages));
      fetch_cols(jbeg + (nx + 2) * kCFib);
    }
    const int s = (int)(st % kCStages);
    const double* ys = TR ? Ys + s * kYst + (8 * kCMW * warp + g) * kTYld + tq
                          : Ys + s * kYst + 8 * kCMW * warp + g;
    const double* os = Os + s * CP * kCOld + g * kCOld + tq;  // B(k = tq, n = g) = Omega(f, 8 ct + g)
#pragma unroll
    for (int kk = 0; kk < kCFib / 4; ++kk) {
      double a[kCMW];
#pragma unroll
      for (int m = 0; m < kCMW; ++m) a[m] = TR ? ys[8 * m * kTYld + 4 * kk] : ys[(4 * kk + tq) * kCYld + 8 * m];
#pragma unroll
      for (int ct = 0; ct < CT; ++ct) {
        const double b = os[8 * ct * kCOld + 4 * kk];
#pragma unroll
        for (int m = 0; m < kCMW; ++m)
          srtt_dev::dmma_8x8x4(acc[kk % KS][m][ct][0], acc[kk % KS][m][ct][1], a[m], b);
      }
    }
  }
  cp_async_wait<0>();
#pragma unroll
  for (int ks = 1; ks < KS; ++ks)
#pragma unroll
    for (int m = 0; m < kCMW; ++m)
#pragma unroll
      for (int ct = 0; ct < CT; ++ct) {
        acc[0][m][ct][0] += acc[ks][m][ct][0];
        acc[0][m][ct][1] += acc[ks][m][ct][1];
      }
  // D fragment: row 16 warp + 8 m + g, columns 8 ct + 2 tq + {0, 1}
  const int64_t ldz = T.ldz > 0 ? T.ldz : rows;
#pragma unroll
  for (int m = 0; m < kCMW; ++m) {
    const int64_t row = row0 + 8 * kCMW * warp + 8 * m + g;
    if (row >= rows) continue;
#pragma unroll
    for (int ct = 0; ct < CT; ++ct)
#pragma unroll
      for (int v = 0; v < 2; ++v) {
        const int cc = 8 * ct + 2 * tq + v;
        if (cc >= c) continue;
        if (T.fsplit > 1)
          T.zpart[((int64_t)fchunk * c + cc) * rows + row] = acc[0][m][ct][v];
        else
          T.z[row + (int64_t)cc * ldz] = acc[0][m][ct][v];
      }
  }
}

// Omega of the targets with omega_gen set, generated once: normal number
// t = j + cc * w of the target's stream after its sampling draws.
__global__ void __launch_bounds__(256) omega_kernel(const SketchTarget* __restrict__ targets, int ntargets) {
  for (int t = 0; t < ntargets; ++t) {
    const SketchTarget& T = targets[t];
    if (!T.omega_gen) continue;
    const int64_t n = T.w * T.c;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
      // K1t targets: row k of Omega is the sorted column's sampled position
      const int64_t k = e % T.w, cc = e / T.w;
      const int64_t t = T.perm ? T.perm[k] + cc * T.w : e;
      T.omega_gen[e] = srtt_dev::normal_at(T.state0, T.draw_offset, (uint64_t)t, T.flags);
    }
  }
}

// Fixed-order sum of the fibre-chunk partials of the split targets.
__global__ void __launch_bounds__(256) sketch_reduce_kernel(const SketchTarget* __restrict__ targets,
                                                            int ntargets) {
  for (int t = 0; t < ntargets; ++t) {
    const SketchTarget& T = targets[t];
    if (T.fsplit <= 1) continue;
    const int64_t n = T.rows * T.c;
    const int64_t ldz = T.ldz > 0 ? T.ldz : T.rows;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
      const int64_t row = e % T.rows, cc = e / T.rows;
      double s = 0.0;
      for (int f = 0; f < T.fsplit; ++f) s += T.zpart[((int64_t)f * T.c + cc) * T.rows + row];
      T.z[row + cc * ldz] = s;
    }
  }
}

}  // namespace

size_t srtt_sketch_contig_smem(int ct, bool tr) {
  const size_t y = tr ? (size_t)kCRows * kTYld : (size_t)kCFib * kCYld;
  return sizeof(double) * (size_t)kCStages * (y + (size_t)8 * ct * kCOld);
}

cudaError_t srtt_launch_sketch_contig(const SketchTarget* d_targets, int ntargets, int64_t total_ctas, int cmax,
                                      int trans, cudaStream_t stream) {
  if (total_ctas <= 0) return cudaSuccess;
  const int ct = (cmax + 7) / 8;
  const size_t smem = srtt_sketch_contig_smem(ct, trans != 0);
#define SRTT_CONTIG_CASE(N)                                                                                   \
  case N:                                                                                                     \
    if (trans) {                                                                                              \
      SRTT_ENSURE_SMEM((sketch_contig_kernel<N, true>), smem);                                                \
      sketch_contig_kernel<N, true><<<(unsigned)total_ctas, kThreads, smem, stream>>>(d_targets, ntargets);  \
    } else {                                                                                                  \
      SRTT_ENSURE_SMEM((sketch_contig_kernel<N, false>), smem);                                               \
      sketch_contig_kernel<N, false><<<(unsigned)total_ctas, kThreads, smem, stream>>>(d_targets, ntargets); \
    }                                                                                                         \
    break;
  switch (ct) {
    SRTT_CONTIG_CASE(1)
    SRTT_CONTIG_CASE(2)
    SRTT_CONTIG_CASE(3)
    SRTT_CONTIG_CASE(4)
    SRTT_CONTIG_CASE(5)
    SRTT_CONTIG_CASE(6)
    SRTT_CONTIG_CASE(7)
    SRTT_CONTIG_CASE(8)
    default:
      return cudaErrorInvalidValue;
  }
#undef SRTT_CONTIG_CASE
  return cudaGetLastError();
}

cudaError_t srtt_launch_omega(const SketchTarget* d_targets, int ntargets, int64_t max_elems, cudaStream_t stream) {
  const int grid = (int)srtt_dev::min64(4 * 148, (max_elems + 255) / 256);
  omega_kernel<<<grid > 0 ? grid : 1, 256, 0, stream>>>(d_targets, ntargets);
  return cudaGetLastError();
}

cudaError_t srtt_launch_sketch_reduce(const SketchTarget* d_targets, int ntargets, int64_t max_elems,
                                      cudaStream_t stream) {
  const int grid = (int)srtt_dev::min64(4 * 148, (max_elems + 255) / 256);
  sketch_reduce_kernel<<<grid > 0 ? grid : 1, 256, 0, stream>>>(d_targets, ntargets);
  return cudaGetLastError();
}

size_t srtt_sketch_smem_bytes(int cmax) {
  return (size_t)kChunk * cmax * sizeof(double) + kChunk * sizeof(int64_t) +
         (size_t)kThreads * cmax * sizeof(double);
}

int srtt_sketch_threads() { return kThreads; }

cudaError_t srtt_launch_sketch(const SketchTarget* d_targets, int ntargets, int64_t total_ctas,
                               int cmax, cudaStream_t stream) {
  if (total_ctas <= 0) return cudaSuccess;
  const size_t smem = srtt_sketch_smem_bytes(cmax < 64 ? cmax : 64);
  if (cmax <= 16) {
    SRTT_ENSURE_SMEM((sketch_kernel<16>), smem);
    sketch_kernel<16><<<(unsigned)total_ctas, kThreads, smem, stream>>>(d_targets, ntargets);
  } else if (cmax <= 32) {
    SRTT_ENSURE_SMEM((sketch_kernel<32>), smem);
    sketch_kernel<32><<<(unsigned)total_ctas, kThreads, smem, stream>>>(d_targets, ntargets);
  } else {
    SRTT_ENSURE_SMEM((sketch_kernel<64>), smem);
    sketch_kernel<64><<<(unsigned)total_ctas, kThreads, smem, stream>>>(d_targets, ntargets);
  }
  return cudaGetLastError();
}
