// Device-side helpers shared by the sm_100a kernels: the reference's
// counter-derived random stream restated as a random-access generator,
// warp reductions, and the mbarrier / TMA primitives (inline PTX).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace srtt_dev {

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) only when the requested
// size grows (the attribute call costs microseconds on every launch); one
// static watermark per call site / kernel.
template <class K>
inline cudaError_t ensure_smem_at(size_t& current, K kernel, size_t bytes) {
  if (bytes <= current) return cudaSuccess;
  cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  if (e == cudaSuccess) current = bytes;
  return e;
}
#define SRTT_ENSURE_SMEM(kernel, bytes) \
  ([&]() { static size_t wm_ = 0; return ::srtt_dev::ensure_smem_at(wm_, kernel, bytes); }())

__host__ __device__ __forceinline__ int64_t min64(int64_t a, int64_t b) { return a < b ? a : b; }
__host__ __device__ __forceinline__ int64_t max64(int64_t a, int64_t b) { return a > b ? a : b; }

constexpr uint64_t kGolden = 0x9E3779B97F4A7C15ULL;

// splitmix64 finalizer (reference rng.hpp:12-19).
__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z ^= z >> 30;
  z *= 0xBF58476D1CE4E5B9ULL;
  z ^= z >> 27;
  z *= 0x94D049BB133111EBULL;
  z ^= z >> 31;
  return z;
}

// Normal number t (0-based) drawn from a stream after `draw_offset` u64 draws
// were consumed, exactly as RngStream::normal() would produce it
// (rng.hpp:65-78): pair q = t/2 uses draws D+2q+1 (u1) and D+2q+2 (u2);
// even t -> radius*cos, odd t -> the cached radius*sin. The stream is
// counter-derived (draw j = mix64(state0 + j*G)), so any t is random-access.
// The reference retries u1 == 0 (probability 2^-53 per pair), which would
// shift every later draw; that event is flagged in *flags instead.
__device__ __forceinline__ double normal_at(uint64_t state0, uint64_t draw_offset, uint64_t t,
                                            int32_t* flags) {
  const uint64_t q = t >> 1;
  const uint64_t s1 = state0 + (draw_offset + 2 * q + 1) * kGolden;
  const uint64_t b1 = mix64(s1) >> 11;
  const uint64_t b2 = mix64(s1 + kGolden) >> 11;
  if (b1 == 0 && flags) atomicOr(flags, 1);
  const double u1 = static_cast<double>(b1) * 0x1.0p-53;
  const double u2 = static_cast<double>(b2) * 0x1.0p-53;
  const double radius = sqrt(-2.0 * log(u1));
  const double angle = 6.283185307179586 * u2;  // 2.0 * pi * u2, same rounding
  double sn, cs;
  sincos(angle, &sn, &cs);
  return (t & 1) ? radius * sn : radius * cs;
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// ---- mbarrier / TMA (PTX) -------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@P1 bra DONE_%=;\n\t"
      "bra WAIT_%=;\n"
      "DONE_%=:\n\t}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// 2-D tiled TMA load of one box into shared memory, completing on `bar`.
__device__ __forceinline__ void tma_load_2d(void* dst, const void* tmap, uint64_t* bar, int32_t c0,
                                            int32_t c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];\n" ::"r"(smem_u32(dst)),
      "l"(tmap), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}

__device__ __forceinline__ void prefetch_tmap(const void* tmap) {
  asm volatile("prefetch.tensormap [%0];\n" ::"l"(tmap) : "memory");
}

// Named barrier among `nthreads` threads (ids 1..15; 0 is __syncthreads).
__device__ __forceinline__ void named_sync(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(nthreads) : "memory");
}

// D(8x8) += A(8x4) * B(4x8), FP64 tensor-core MMA (SASS: DMMA.8x8x4).
__device__ __forceinline__ void dmma_8x8x4(double& d0, double& d1, double a, double b) {
  asm volatile(
      "mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(d0), "+d"(d1)
      : "d"(a), "d"(b));
}

}  // namespace srtt_dev
