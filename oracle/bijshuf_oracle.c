/*
 * bijshuf_oracle.c -- CPU restatement of the reference bijective shuffle.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker for the
 * sm_100a kernels in paper_2106_06161_b200/csrc.  Only tests/, the
 * __graft_entry__.smoke() check and bench.py's cpu_baseline leg may load
 * it.  The product path (libbsg.so and the Python/C++ host layers) never
 * links, loads or calls anything here, and has no CPU fallback.
 *
 * Every function restates the algorithm of the reference header-only C++
 * library `bijshuf` (/root/reference/proj/include/bijshuf/*.hpp) in plain
 * C99, citing the file:line it follows.  It is deliberately the slow,
 * obvious, sequential form: one counter at a time, full 64-bit arithmetic
 * exactly as the reference writes it, compaction by a running counter.
 *
 * Parity pinning: tests/test_oracle.py checks this restatement against
 *   (1) the reference's own frozen golden value (round keys for seed 42,
 *       proj/tests/unit_bijection.cpp:32-37) and LCG known answers
 *       (unit_bijection.cpp:52-84), the compaction example of
 *       unit_shuffle.cpp:14-37 and the domain-bits table (:39-46);
 *   (2) full-permutation fixtures in tests/golden/ that were produced by
 *       the reference itself (oracle/_ref, compiled from the reference
 *       headers by oracle/Makefile; script tests/golden/make_golden.py).
 */
#include <stddef.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORC_OK 0
#define ORC_EINVAL (-1)  /* std::invalid_argument in the reference */
#define ORC_ERANGE (-2)  /* std::out_of_range in the reference */

enum { ORC_LCG = 0, ORC_PHILOX = 1 }; /* BijectionVariant, shuffle.hpp:20 */

static const uint64_t kGamma = 0x9E3779B97F4A7C15ULL; /* splitmix.hpp:18 */
static const uint64_t kM0 = 0xD2B74407B1CE6E93ULL;    /* bijection.hpp:57 */

/* splitmix.hpp:11-15 */
uint64_t orc_mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

/* splitmix.hpp:22-31: key_i = low32(mix64(seed + (i+1)*gamma)); rounds >= 1. */
int orc_derive_round_keys(uint64_t seed, int rounds, uint32_t* keys) {
  if (rounds < 1) return ORC_EINVAL;
  for (int i = 0; i < rounds; ++i)
    keys[i] = (uint32_t)orc_mix64(seed + ((uint64_t)i + 1) * kGamma);
  return ORC_OK;
}

/* bijection.hpp:25-34 (make_lcg): a forced odd, both reduced mod 2^bits. */
int orc_make_lcg(int bits, uint64_t seed, uint64_t* a, uint64_t* c) {
  if (bits < 1 || bits > 63) return ORC_EINVAL;
  const uint64_t mask = (1ULL << bits) - 1;
  *a = (orc_mix64(seed) | 1ULL) & mask;
  *c = orc_mix64(seed + 1) & mask;
  return ORC_OK;
}

/* bijection.hpp:36-40 (lcg_apply) with LcgParams::domain_mask (:20-22). */
int orc_lcg_apply(int bits, uint64_t a, uint64_t c, uint64_t x, uint64_t* y) {
  const uint64_t mask = bits >= 64 ? ~0ULL : ((1ULL << bits) - 1);
  if (x > mask) return ORC_ERANGE;
  *y = (a * x + c) & mask;
  return ORC_OK;
}

/* bijection.hpp:73-88 (make_philox) parameter checks. */
int orc_philox_check(int bits, int rounds) {
  if (bits < 2 || bits > 63) return ORC_EINVAL;
  if (rounds < 3) return ORC_EINVAL;
  return ORC_OK;
}

/* bijection.hpp:94-111 (philox_apply), without the domain check; the
 * arithmetic is the reference's 64-bit form verbatim. */
uint64_t orc_philox_apply_unchecked(int bits, const uint32_t* keys, int rounds, uint64_t x) {
  const int L = bits / 2, R = bits - L, d = R - L;
  const uint64_t LM = (1ULL << L) - 1, RM = (1ULL << R) - 1;
  uint64_t s0 = x >> R, s1 = x & RM;
  for (int i = 0; i < rounds; ++i) {
    const uint64_t product = kM0 * s0;
    const uint64_t hi = product >> 32;
    uint64_t lo = product & 0xFFFFFFFFULL;
    lo = (lo << d) | (s1 >> L);
    s0 = ((hi ^ keys[i]) ^ s1) & LM;
    s1 = lo & RM;
  }
  return (s0 << R) | s1;
}

/* bijection.hpp:94-111 with the out_of_range check of :96-97. */
int orc_philox_apply(int bits, const uint32_t* keys, int rounds, uint64_t x, uint64_t* y) {
  if (bits < 64 && (x >> bits) != 0) return ORC_ERANGE;
  *y = orc_philox_apply_unchecked(bits, keys, rounds, x);
  return ORC_OK;
}

/* bijection.hpp:61-65 (odd_inverse_pow2_64): Newton iteration mod 2^64. */
uint64_t orc_odd_inverse_pow2_64(uint64_t a) {
  uint64_t x = a;
  for (int i = 0; i < 5; ++i) x *= 2 - a * x;
  return x;
}

/* bijection.hpp:117-143 (philox_invert). */
int orc_philox_invert(int bits, const uint32_t* keys, int rounds, uint64_t y, uint64_t* x) {
  if (bits < 64 && (y >> bits) != 0) return ORC_ERANGE;
  const int L = bits / 2, R = bits - L, d = R - L;
  const uint64_t LM = (1ULL << L) - 1, RM = (1ULL << R) - 1;
  const uint64_t m0_inv = orc_odd_inverse_pow2_64(kM0);
  uint64_t t0 = y >> R, t1 = y & RM;
  (void)RM;
  for (int i = rounds - 1; i >= 0; --i) {
    const uint64_t spare = t1 & ((1ULL << d) - 1);
    const uint64_t lo_mod_left = (t1 >> d) & LM;
    const uint64_t s0 = (m0_inv * lo_mod_left) & LM;
    const uint64_t hi = (kM0 * s0) >> 32;
    const uint64_t s1 = (((hi ^ keys[i]) ^ t0) & LM) | (spare << L);
    t0 = s0;
    t1 = s1;
  }
  *x = (t0 << R) | t1;
  return ORC_OK;
}

/* shuffle.hpp:49-52: max(4, ceil(log2 m)) for m >= 2. */
int orc_domain_bits(uint64_t m) {
  const int needed = m <= 1 ? 0 : 64 - __builtin_clzll(m - 1);
  return needed < 4 ? 4 : needed;
}

/* A resolved bijection: the state run_shuffle_engine builds
 * (shuffle.hpp:151-191) before evaluating counters. */
typedef struct {
  int variant, bits, rounds;
  uint64_t a, c;       /* LCG */
  uint32_t keys[4096]; /* Philox; rounds are capped at 4096 in this oracle */
} orc_bij;

static int orc_bij_init(orc_bij* b, uint64_t m, uint64_t seed, int variant, int rounds) {
  b->bits = orc_domain_bits(m);
  b->variant = variant;
  b->rounds = rounds;
  if (variant == ORC_LCG) return orc_make_lcg(b->bits, seed, &b->a, &b->c); /* shuffle.hpp:157-158 */
  int rc = orc_philox_check(b->bits, rounds);                                 /* shuffle.hpp:171-172 */
  if (rc) return rc;
  if (rounds > 4096) return ORC_EINVAL;
  return orc_derive_round_keys(seed, rounds, b->keys);
}

static inline uint64_t orc_bij_apply(const orc_bij* b, uint64_t x) {
  if (b->variant == ORC_LCG) /* shuffle.hpp:160-162 */
    return (b->a * x + b->c) & ((1ULL << b->bits) - 1);
  return orc_philox_apply_unchecked(b->bits, b->keys, b->rounds, x);
}

/* shuffle.hpp:226-244 (shuffle_indices_core) with the engine
 * (run_shuffle_engine :151-191, chained_compact :107-147, scalar_compact
 * :58-69, IndicesSink :214-224) collapsed to its sequential meaning:
 * evaluate every counter of [0, 2^bits) in order and keep images < m. */
int orc_shuffle_indices(uint64_t m, uint64_t seed, int variant, int rounds, uint64_t* out) {
  if (m == 0) return ORC_OK;
  if (m == 1) { out[0] = 0; return ORC_OK; }
  if (m == 2) { /* :233-240 -- variant and rounds are ignored */
    const uint64_t bit = orc_mix64(seed) & 1;
    out[0] = bit;
    out[1] = bit ^ 1;
    return ORC_OK;
  }
  orc_bij* b = (orc_bij*)malloc(sizeof(orc_bij)); /* key table per call: reentrant */
  if (!b) return ORC_EINVAL;
  int rc = orc_bij_init(b, m, seed, variant, rounds);
  if (rc) { free(b); return rc; }
  const uint64_t n = 1ULL << b->bits;
  uint64_t k = 0;
  for (uint64_t i = 0; i < n; ++i) {
    const uint64_t y = orc_bij_apply(b, i);
    if (y < m) out[k++] = y;
  }
  free(b);
  return ORC_OK;
}

/* Survivors of the counter range [c0, c1) of the same engine, in counter
 * order; returns the count through *count.  This is the per-shard unit of
 * the multi-GPU partition (contiguous counter ranges); the
 * reference's chunk loop (shuffle.hpp:122-145) is the same computation
 * over 65536-counter ranges. */
int orc_shuffle_indices_range(uint64_t m, uint64_t seed, int variant, int rounds, uint64_t c0, uint64_t c1,
                              uint64_t* out, uint64_t* count) {
  *count = 0;
  if (m <= 2) return ORC_EINVAL;
  orc_bij* b = (orc_bij*)malloc(sizeof(orc_bij));
  if (!b) return ORC_EINVAL;
  int rc = orc_bij_init(b, m, seed, variant, rounds);
  if (rc) { free(b); return rc; }
  const uint64_t n = 1ULL << b->bits;
  if (c1 > n || c0 > c1) { free(b); return ORC_ERANGE; }
  uint64_t k = 0;
  for (uint64_t i = c0; i < c1; ++i) {
    const uint64_t y = orc_bij_apply(b, i);
    if (y < m) {
      if (out) out[k] = y;
      ++k;
    }
  }
  *count = k;
  free(b);
  return ORC_OK;
}

/* shuffle.hpp:246-263 (shuffle_values_core) + ValuesSink (:193-212):
 * out[k] = values[sigma(k)], for any trivially copyable element size. */
int orc_shuffle_values(const void* values, void* out, uint64_t m, size_t elem_bytes, uint64_t seed, int variant,
                       int rounds) {
  const unsigned char* s = (const unsigned char*)values;
  unsigned char* d = (unsigned char*)out;
  if (m == 0) return ORC_OK;
  if (m == 1) { memcpy(d, s, elem_bytes); return ORC_OK; }
  if (m == 2) {
    const uint64_t bit = orc_mix64(seed) & 1;
    memcpy(d, s + bit * elem_bytes, elem_bytes);
    memcpy(d + elem_bytes, s + (bit ^ 1) * elem_bytes, elem_bytes);
    return ORC_OK;
  }
  orc_bij* b = (orc_bij*)malloc(sizeof(orc_bij));
  if (!b) return ORC_EINVAL;
  int rc = orc_bij_init(b, m, seed, variant, rounds);
  if (rc) { free(b); return rc; }
  const uint64_t n = 1ULL << b->bits;
  uint64_t k = 0;
  for (uint64_t i = 0; i < n; ++i) {
    const uint64_t y = orc_bij_apply(b, i);
    if (y < m) memcpy(d + (k++) * elem_bytes, s + y * elem_bytes, elem_bytes);
  }
  free(b);
  return ORC_OK;
}

/* shuffle.hpp:319-334 (gather_core): out[i] = src[idx[i]]. */
void orc_gather(const void* src, const uint64_t* idx, void* out, uint64_t n, size_t elem_bytes) {
  const unsigned char* s = (const unsigned char*)src;
  unsigned char* d = (unsigned char*)out;
  for (uint64_t i = 0; i < n; ++i) memcpy(d + i * elem_bytes, s + idx[i] * elem_bytes, elem_bytes);
}

/* FNV-1a-64 over u64 words (SURVEY.md Appendix A/C hashing convention). */
uint64_t orc_fnv1a64_u64(const uint64_t* p, uint64_t n) {
  uint64_t h = 0xcbf29ce484222325ULL;
  for (uint64_t i = 0; i < n; ++i) {
    h ^= p[i];
    h *= 0x100000001b3ULL;
  }
  return h;
}

/* permutation.hpp:24-32 (is_valid_permutation); scratch holds n bytes. */
int orc_is_valid_permutation(const uint64_t* p, uint64_t n, unsigned char* scratch) {
  memset(scratch, 0, n);
  for (uint64_t i = 0; i < n; ++i) {
    if (p[i] >= n || scratch[p[i]]) return 0;
    scratch[p[i]] = 1;
  }
  return 1;
}

/* Batched convention of BijectiveShuffleSampler (stats.hpp:314-324):
 * shuffle b uses seed + b. */
int orc_shuffle_values_batched(const void* values, void* out, uint64_t batch, uint64_t m, size_t elem_bytes,
                               uint64_t seed, int variant, int rounds) {
  for (uint64_t b = 0; b < batch; ++b) {
    int rc = orc_shuffle_values((const unsigned char*)values + b * m * elem_bytes,
                                (unsigned char*)out + b * m * elem_bytes, m, elem_bytes, seed + b, variant, rounds);
    if (rc) return rc;
  }
  return ORC_OK;
}
