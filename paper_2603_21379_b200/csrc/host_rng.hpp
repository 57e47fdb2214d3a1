// Host-side sampler of the product path: the reference's counter-derived
// stream and Floyd sampling, restated in C++ (rng.hpp:12-78,
// sampling.hpp:14-66). Indices must be bit-exact with the reference; this
// is pinned against the reference's own headers by tests/test_sampler.py.
// It additionally reports how many u64 draws the sampling consumed, which
// is where the device Gaussian generator starts (gaussian_matrix follows
// the sampling on the same stream, tucker.hpp:145-159).
#pragma once
#include <cstdint>
#include <stdexcept>
#include <string>
#include <unordered_set>
#include <vector>

namespace srtt_host {

constexpr uint64_t kGolden = 0x9E3779B97F4A7C15ULL;

inline uint64_t mix64(uint64_t z) {
  z ^= z >> 30;
  z *= 0xBF58476D1CE4E5B9ULL;
  z ^= z >> 27;
  z *= 0x94D049BB133111EBULL;
  z ^= z >> 31;
  return z;
}

inline uint64_t stream_state0(uint64_t seed, uint64_t id) {
  return mix64(mix64(seed + kGolden) ^ mix64(id * kGolden + 1));
}

struct Stream {
  uint64_t seed, id, state, draws = 0;
  Stream(uint64_t s, uint64_t i) : seed(s), id(i), state(stream_state0(s, i)) {}
  Stream child(uint64_t i) const { return Stream(seed, mix64(id ^ kGolden) + i + 1); }
  uint64_t next_u64() {
    state += kGolden;
    ++draws;
    return mix64(state);
  }
  uint64_t bounded(uint64_t n) {
    const uint64_t threshold = (0 - n) % n;
    for (;;) {
      const uint64_t r = next_u64();
      if (r >= threshold) return r % n;
    }
  }
};

// Open-addressing set of sampled indices (membership is all Floyd needs;
// the reference's std::unordered_set gives identical results).
struct IndexSet {
  std::vector<int64_t> keys;
  uint64_t mask = 0;
  void reset(int64_t n) {
    uint64_t cap = 16;
    while (cap < static_cast<uint64_t>(4 * n + 4)) cap <<= 1;
    keys.assign(cap, -1);
    mask = cap - 1;
  }
  bool insert(int64_t k) {  // true if newly inserted
    uint64_t i = mix64(static_cast<uint64_t>(k)) & mask;
    while (keys[i] != -1) {
      if (keys[i] == k) return false;
      i = (i + 1) & mask;
    }
    keys[i] = k;
    return true;
  }
};

// Floyd's algorithm, indices in sampled order (sampling.hpp:14-32).
inline void sample_indices(int64_t m, int64_t s, Stream& rng, std::vector<int64_t>& out) {
  if (s < 1 || s > m)
    throw std::invalid_argument("sample_indices: need 1 <= s <= m, got s=" + std::to_string(s) +
                                " m=" + std::to_string(m));
  out.clear();
  out.reserve(static_cast<size_t>(s));
  thread_local IndexSet chosen;
  chosen.reset(s);
  for (int64_t j = m - s; j < m; ++j) {
    const int64_t t = static_cast<int64_t>(rng.bounded(static_cast<uint64_t>(j) + 1));
    if (chosen.insert(t)) {
      out.push_back(t);
    } else {
      chosen.insert(j);
      out.push_back(j);
    }
  }
}

// sampling.hpp:41-66 (child streams; the parent stream is not advanced).
inline void sample_indices_partitioned(int64_t m, int64_t s, int64_t partitions, Stream& rng,
                                       std::vector<int64_t>& out) {
  if (partitions < 1) throw std::invalid_argument("sample_indices_partitioned: partitions >= 1");
  if (partitions > s)
    throw std::invalid_argument("sample_indices_partitioned: partitions must not exceed s");
  if (s > m) throw std::invalid_argument("sample_indices_partitioned: s must not exceed m");
  if (partitions == 1) {
    sample_indices(m, s, rng, out);
    return;
  }
  const int64_t base_len = m / partitions;
  if (base_len == 0)
    throw std::invalid_argument("sample_indices_partitioned: more partitions than indices");
  const int64_t base_cnt = s / partitions;
  out.clear();
  std::vector<int64_t> part_idx;
  for (int64_t part = 0; part < partitions; ++part) {
    const int64_t lo = part * base_len;
    const int64_t len = (part == partitions - 1) ? (m - lo) : base_len;
    const int64_t cnt = (part == partitions - 1) ? (base_cnt + s % partitions) : base_cnt;
    if (cnt > len)
      throw std::invalid_argument("sample_indices_partitioned: subinterval too small for draw");
    Stream sub = rng.child(static_cast<uint64_t>(part));
    sample_indices(len, cnt, sub, part_idx);
    for (int64_t v : part_idx) out.push_back(lo + v);
  }
}

}  // namespace srtt_host
