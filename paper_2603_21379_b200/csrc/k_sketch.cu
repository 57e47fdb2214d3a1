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

  const int c = T.c;
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

  double* om = reinterpret_cast<double*>(smem_raw);         // kChunk x c
  int64_t* base = reinterpret_cast<int64_t*>(om + kChunk * c);  // kChunk
  double* red = reinterpret_cast<double*>(base + kChunk);    // kThreads x c

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

  double acc[CMAX];
#pragma unroll
  for (int cc = 0; cc < CMAX; ++cc) acc[cc] = 0.0;

  const double* __restrict__ x = T.x;
  // flat-range sharding: only [flo, fhi) of the global flat index is local
  const int64_t flo = T.flat_lo, fhi = T.flat_hi;
  const bool ranged = fhi > 0;
  for (int64_t j0 = jbeg; j0 < jend; j0 += kChunk) {
    const int jn = (int)srtt_dev::min64(kChunk, jend - j0);
    __syncthreads();
    // Omega(j, cc) is normal number t = j + cc * w of the stream
    // (column-major gaussian_matrix fill, sampling.hpp:74-75).
    for (int idx = tid; idx < jn * c; idx += kThreads) {
      const int jl = idx / c, cc = idx - jl * c;
      const uint64_t t = (uint64_t)(j0 + jl) + (uint64_t)cc * (uint64_t)T.w;
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
      // 4 independent loads in flight per thread before the FMAs.
      for (; jl + 3 * JS < jn; jl += 4 * JS) {
        const int64_t b0 = base[jl], b1 = base[jl + JS], b2 = base[jl + 2 * JS], b3 = base[jl + 3 * JS];
        const double v0 = b0 >= 0 ? __ldg(x + b0 + roff) : 0.0;
        const double v1 = b1 >= 0 ? __ldg(x + b1 + roff) : 0.0;
        const double v2 = b2 >= 0 ? __ldg(x + b2 + roff) : 0.0;
        const double v3 = b3 >= 0 ? __ldg(x + b3 + roff) : 0.0;
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
        const double v = bj >= 0 ? __ldg(x + bj + roff) : 0.0;
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
      T.zpart[((int64_t)fchunk * c + cc) * T.rows + row] = s;
    else
      T.z[row + (int64_t)cc * ldz] = s;
  }
}

// Omega of the targets with omega_gen set, generated once: normal number
// t = j + cc * w of the target's stream after its sampling draws.
__global__ void __launch_bounds__(256) omega_kernel(const SketchTarget* __restrict__ targets, int ntargets) {
  for (int t = 0; t < ntargets; ++t) {
    const SketchTarget& T = targets[t];
    if (!T.omega_gen) continue;
    const int64_t n = T.w * T.c;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x)
      T.omega_gen[e] = srtt_dev::normal_at(T.state0, T.draw_offset, (uint64_t)e, T.flags);
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
  const size_t smem = srtt_sketch_smem_bytes(cmax);
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
