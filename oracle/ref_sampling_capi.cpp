// Test infrastructure (oracle/_ref): a C-callable wrapper around the
// REFERENCE's own srtt::RngStream and srtt::sample_indices[_partitioned]
// (/root/reference/proj/include/srtt/{rng,sampling}.hpp), compiled straight
// from the reference sources with the declaration shim in ref_shim/. Used
// only by tests/ and tests/golden/make_golden.py to pin the oracle's and the
// product's host sampler bit-for-bit. Never linked into the product.
#include "srtt/sampling.hpp"

#include <cstdint>
#include <cstring>
#include <exception>

extern "C" {

// Draws s indices of [0, m) with stream (seed, stream_id) exactly as
// sub_r_hosvd's mode job does (tucker.hpp:145-149; partitions>1 follows
// sampling.hpp:41-66), then n_normals normals from the same stream as
// gaussian_matrix would (sampling.hpp:69-77). Returns 0 on success, 1 on
// std::invalid_argument.
int ref_sample_then_normals(uint64_t seed, uint64_t stream_id, int64_t m, int64_t s,
                            int64_t partitions, int64_t* idx_out, int64_t n_normals,
                            double* normals_out) {
  try {
    srtt::RngStream rng(seed, stream_id);
    std::vector<srtt::Index> idx = partitions > 1
                                       ? srtt::sample_indices_partitioned(m, s, partitions, rng)
                                       : srtt::sample_indices(m, s, rng);
    for (std::size_t i = 0; i < idx.size(); ++i) idx_out[i] = idx[i];
    for (int64_t t = 0; t < n_normals; ++t) normals_out[t] = rng.normal();
    return 0;
  } catch (const std::exception&) {
    return 1;
  }
}

// Raw u64 draws of a stream (rng.hpp:47-50).
void ref_next_u64(uint64_t seed, uint64_t stream_id, int64_t n, uint64_t* out) {
  srtt::RngStream rng(seed, stream_id);
  for (int64_t i = 0; i < n; ++i) out[i] = rng.next_u64();
}

// Child-stream derivation (rng.hpp:43-45): n raw draws of rng(seed,id).child(i).
void ref_child_u64(uint64_t seed, uint64_t stream_id, uint64_t child, int64_t n, uint64_t* out) {
  srtt::RngStream rng = srtt::RngStream(seed, stream_id).child(child);
  for (int64_t i = 0; i < n; ++i) out[i] = rng.next_u64();
}

// uniform01 and bounded draws (rng.hpp:53-62), interleaved as the caller asks:
// kinds[i]==0 -> uniform01, else bounded(kinds[i]) stored as double.
void ref_mixed_draws(uint64_t seed, uint64_t stream_id, int64_t n, const uint64_t* kinds,
                     double* out) {
  srtt::RngStream rng(seed, stream_id);
  for (int64_t i = 0; i < n; ++i)
    out[i] = kinds[i] == 0 ? rng.uniform01() : static_cast<double>(rng.bounded(kinds[i]));
}

}  // extern "C"
