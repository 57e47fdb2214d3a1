/*
 * ORACLE (test infrastructure only; never linked into the product).
 *
 * Plain-C restatement of the reference's counter-derived random stream and
 * Floyd fiber sampling:
 *   - mix64 / kGolden              rng.hpp:12-21
 *   - RngStream(seed, id) state     rng.hpp:30-36
 *   - child(i)                     rng.hpp:43-45
 *   - next_u64                     rng.hpp:47-50
 *   - uniform01                    rng.hpp:53
 *   - bounded (rejection)          rng.hpp:56-62
 *   - normal (Box-Muller, cached)  rng.hpp:65-78
 *   - sample_indices (Floyd)       sampling.hpp:14-32
 *   - sample_indices_partitioned   sampling.hpp:41-66
 *   - gaussian_matrix (col-major)  sampling.hpp:69-77
 * Pinned bit-for-bit against the reference's own headers (oracle/_ref) and
 * the Appendix-A known answers in SURVEY.md by tests/test_oracle_rng.py.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define KGOLDEN 0x9E3779B97F4A7C15ULL

static uint64_t mix64(uint64_t z) {
  z ^= z >> 30;
  z *= 0xBF58476D1CE4E5B9ULL;
  z ^= z >> 27;
  z *= 0x94D049BB133111EBULL;
  z ^= z >> 31;
  return z;
}

typedef struct {
  uint64_t seed, id, state;
  double cached;
  int have_cached;
  uint64_t draws; /* number of next_u64 calls so far */
} orc_stream;

void orc_stream_init(orc_stream* s, uint64_t seed, uint64_t id) {
  s->seed = seed;
  s->id = id;
  s->state = mix64(mix64(seed + KGOLDEN) ^ mix64(id * KGOLDEN + 1));
  s->cached = 0.0;
  s->have_cached = 0;
  s->draws = 0;
}

uint64_t orc_stream_state0(uint64_t seed, uint64_t id) {
  return mix64(mix64(seed + KGOLDEN) ^ mix64(id * KGOLDEN + 1));
}

uint64_t orc_child_id(uint64_t id, uint64_t i) { return mix64(id ^ KGOLDEN) + i + 1; }

uint64_t orc_next_u64(orc_stream* s) {
  s->state += KGOLDEN;
  s->draws++;
  return mix64(s->state);
}

double orc_uniform01(orc_stream* s) { return (double)(orc_next_u64(s) >> 11) * 0x1.0p-53; }

uint64_t orc_bounded(orc_stream* s, uint64_t n) {
  const uint64_t threshold = (0 - n) % n;
  for (;;) {
    const uint64_t r = orc_next_u64(s);
    if (r >= threshold) return r % n;
  }
}

double orc_normal(orc_stream* s) {
  if (s->have_cached) {
    s->have_cached = 0;
    return s->cached;
  }
  double u1 = orc_uniform01(s);
  while (u1 == 0.0) u1 = orc_uniform01(s);
  const double u2 = orc_uniform01(s);
  const double radius = sqrt(-2.0 * log(u1));
  const double angle = 2.0 * 3.14159265358979323846 * u2;
  s->cached = radius * sin(angle);
  s->have_cached = 1;
  return radius * cos(angle);
}

/* Open-addressing set of int64 (the reference uses std::unordered_set; only
 * membership matters for the result). */
typedef struct {
  int64_t* keys;
  uint8_t* used;
  uint64_t cap;
} orc_set;

static void set_init(orc_set* h, int64_t n) {
  uint64_t cap = 16;
  while (cap < (uint64_t)(4 * n + 4)) cap <<= 1;
  h->cap = cap;
  h->keys = (int64_t*)malloc(cap * sizeof(int64_t));
  h->used = (uint8_t*)calloc(cap, 1);
}
static void set_free(orc_set* h) {
  free(h->keys);
  free(h->used);
}
/* returns 1 if inserted (was absent) */
static int set_insert(orc_set* h, int64_t k) {
  uint64_t i = mix64((uint64_t)k) & (h->cap - 1);
  while (h->used[i]) {
    if (h->keys[i] == k) return 0;
    i = (i + 1) & (h->cap - 1);
  }
  h->used[i] = 1;
  h->keys[i] = k;
  return 1;
}

/* Floyd's algorithm in sampled order (sampling.hpp:14-32).
 * Returns 0 on success, 1 if s<1 or s>m. */
int orc_sample_indices(int64_t m, int64_t s, orc_stream* rng, int64_t* out) {
  if (s < 1 || s > m) return 1;
  orc_set h;
  set_init(&h, s);
  int64_t n = 0;
  for (int64_t j = m - s; j < m; ++j) {
    const int64_t t = (int64_t)orc_bounded(rng, (uint64_t)j + 1);
    if (set_insert(&h, t)) {
      out[n++] = t;
    } else {
      set_insert(&h, j);
      out[n++] = j;
    }
  }
  set_free(&h);
  return 0;
}

/* sampling.hpp:41-66. Returns 0 ok, 1 invalid argument. The parent stream is
 * not advanced (each part uses child(part)). */
int orc_sample_indices_partitioned(int64_t m, int64_t s, int64_t partitions, orc_stream* rng,
                                   int64_t* out) {
  if (partitions < 1) return 1;
  if (partitions > s) return 1;
  if (s > m) return 1;
  if (partitions == 1) return orc_sample_indices(m, s, rng, out);
  const int64_t base_len = m / partitions;
  if (base_len == 0) return 1;
  const int64_t base_cnt = s / partitions;
  int64_t n = 0;
  for (int64_t part = 0; part < partitions; ++part) {
    const int64_t lo = part * base_len;
    const int64_t len = (part == partitions - 1) ? (m - lo) : base_len;
    const int64_t cnt = (part == partitions - 1) ? (base_cnt + s % partitions) : base_cnt;
    if (cnt > len) return 1;
    orc_stream sub;
    orc_stream_init(&sub, rng->seed, orc_child_id(rng->id, (uint64_t)part));
    if (orc_sample_indices(len, cnt, &sub, out + n)) return 1;
    for (int64_t i = 0; i < cnt; ++i) out[n + i] += lo;
    n += cnt;
  }
  return 0;
}

/* ---- flat C entry points for ctypes ------------------------------------- */

/* Sampling followed by `n_normals` normals from the same stream (the order of
 * subsampled_mode_basis, tucker.hpp:145-159). draws_out receives the number
 * of u64 draws consumed by the sampling step. */
int orc_sample_then_normals(uint64_t seed, uint64_t id, int64_t m, int64_t s, int64_t partitions,
                            int64_t* idx_out, int64_t n_normals, double* normals_out,
                            uint64_t* draws_out) {
  orc_stream rng;
  orc_stream_init(&rng, seed, id);
  int rc = partitions > 1 ? orc_sample_indices_partitioned(m, s, partitions, &rng, idx_out)
                          : orc_sample_indices(m, s, &rng, idx_out);
  if (rc) return rc;
  if (draws_out) *draws_out = rng.draws;
  for (int64_t t = 0; t < n_normals; ++t) normals_out[t] = orc_normal(&rng);
  return 0;
}

/* A resumable stream object for the numpy oracle (padding continues the
 * stream after Omega; sketch.hpp:48-65). */
orc_stream* orc_stream_new(uint64_t seed, uint64_t id) {
  orc_stream* s = (orc_stream*)malloc(sizeof(orc_stream));
  orc_stream_init(s, seed, id);
  return s;
}
void orc_stream_delete(orc_stream* s) { free(s); }
int orc_stream_sample(orc_stream* s, int64_t m, int64_t cnt, int64_t partitions, int64_t* out) {
  return partitions > 1 ? orc_sample_indices_partitioned(m, cnt, partitions, s, out)
                        : orc_sample_indices(m, cnt, s, out);
}
void orc_stream_normals(orc_stream* s, int64_t n, double* out) {
  for (int64_t i = 0; i < n; ++i) out[i] = orc_normal(s);
}
void orc_stream_u64(orc_stream* s, int64_t n, uint64_t* out) {
  for (int64_t i = 0; i < n; ++i) out[i] = orc_next_u64(s);
}
void orc_stream_uniform(orc_stream* s, int64_t n, double* out) {
  for (int64_t i = 0; i < n; ++i) out[i] = orc_uniform01(s);
}
uint64_t orc_stream_draws(const orc_stream* s) { return s->draws; }
