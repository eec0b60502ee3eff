// C++ drop-in test of the raw-bijection surface of the shim: every case of the
// reference's proj/tests/unit_bijection.cpp, rewritten without GTest against
// include/bijshuf_gpu/shuffle.hpp.  These entry points are host scalar code in
// libbsg.so, so this binary runs on CPU hosts as well (tests/test_cpp_shim.py).
#include <bijshuf_gpu/shuffle.hpp>

#include <cstdio>
#include <set>
#include <vector>

using namespace bijshuf;

static int failures = 0;
#define CHECK(cond)                                                        \
  do {                                                                     \
    if (!(cond)) {                                                         \
      std::fprintf(stderr, "FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond); \
      ++failures;                                                          \
    }                                                                      \
  } while (0)
#define CHECK_THROWS(expr, type) \
  do {                           \
    bool thrown = false;         \
    try {                        \
      (void)(expr);              \
    } catch (const type&) {      \
      thrown = true;             \
    }                            \
    CHECK(thrown);               \
  } while (0)

// mix64 is constexpr in the reference; the shim keeps it so.
static_assert(mix64(0) == 0ULL, "mix64(0)");
static_assert(SplitMix64(1)() == mix64(1 + kSplitMixGamma), "SplitMix64 is constexpr");

int main() {
  // unit_bijection.cpp:13-16 Mix64.MatchesReference (the shim's constexpr form == libbsg's)
  for (std::uint64_t z : {0ULL, 1ULL, 42ULL, 0xDEADBEEFULL, ~0ULL}) CHECK(mix64(z) == bsg_mix64(z));
  // :18-22 Deterministic
  CHECK(derive_round_keys(123, 1) == derive_round_keys(123, 1));
  // :24-30 NotAllEqual
  {
    const auto keys = derive_round_keys(0, 24);
    CHECK(keys.size() == 24u);
    bool all_equal = true;
    for (std::uint32_t k : keys) all_equal &= (k == keys[0]);
    CHECK(!all_equal);
  }
  // :32-37 GoldenSeed42
  CHECK((derive_round_keys(42, 4) == std::vector<std::uint32_t>{0x2FEB6E95u, 0xB266F103u, 0x130F9F52u, 0x0E4AE394u}));
  // :39-41 RejectsZeroRounds
  CHECK_THROWS(derive_round_keys(1, 0), std::invalid_argument);
  // :43-50 MultiplierAlwaysOdd
  for (std::uint64_t seed = 0; seed < 200; ++seed) {
    const LcgParams p = make_lcg(16, seed);
    CHECK((p.a & 1) == 1u && p.a < (1ULL << 16) && p.c < (1ULL << 16));
  }
  // :52-55 DirectParamsValid
  CHECK(lcg_apply(LcgParams{3, 3, 0}, 1) == 3u);
  // :57-60 RejectsOutOfRangeBits
  CHECK_THROWS(make_lcg(64, 1), std::invalid_argument);
  CHECK_THROWS(make_lcg(0, 1), std::invalid_argument);
  // :62-65 IdentityParams, :67-70 DirectArithmetic
  CHECK(lcg_apply(LcgParams{4, 1, 0}, 9) == 9u);
  CHECK(lcg_apply(LcgParams{3, 3, 1}, 5) == 0u);
  // :72-79 PermutationOfDomain
  {
    const LcgParams p{3, 3, 0};
    std::set<std::uint64_t> image;
    for (std::uint64_t x = 0; x < 8; ++x) image.insert(lcg_apply(p, x));
    CHECK(image.size() == 8u && *image.begin() == 0u && *image.rbegin() == 7u);
  }
  // :81-84 RejectsOutOfDomain
  CHECK_THROWS(lcg_apply(LcgParams{3, 3, 0}, 8), std::out_of_range);
  // :86-92 EightBitPermutation
  {
    const auto p = make_philox(8, 7);
    std::set<std::uint64_t> image;
    for (std::uint64_t x = 0; x < 256; ++x) image.insert(philox_apply(p, x));
    CHECK(image.size() == 256u && *image.rbegin() == 255u);
  }
  // :94-104 OddWidthPermutation
  {
    const auto p = make_philox(7, 11);
    CHECK(p.left_side_bits == 3 && p.right_side_bits == 4);
    std::set<std::uint64_t> image;
    for (std::uint64_t x = 0; x < 128; ++x) image.insert(philox_apply(p, x));
    CHECK(image.size() == 128u);
  }
  // :106-115 ZeroRoundsIsIdentity (hand-built params, num_rounds = 0, no keys)
  {
    VariablePhiloxParams p;
    p.total_bits = 8;
    p.left_side_bits = 4;
    p.right_side_bits = 4;
    p.num_rounds = 0;
    p.left_side_mask = 0xF;
    p.right_side_mask = 0xF;
    CHECK(philox_apply(p, 0b10110011) == 0b10110011u);
  }
  // :117-120 RejectsOutOfDomain
  CHECK_THROWS(philox_apply(make_philox(8, 7), 256), std::out_of_range);
  // :122-130 RoundTripExhaustiveSmall
  for (int bits = 2; bits <= 12; ++bits) {
    const auto p = make_philox(bits, 1234 + static_cast<std::uint64_t>(bits));
    for (std::uint64_t x = 0; x < (1ULL << bits); ++x) CHECK(philox_invert(p, philox_apply(p, x)) == x);
  }
  // :132-136 RoundTripOddWidth
  {
    const auto p = make_philox(5, 99);
    for (std::uint64_t x = 0; x < 32; ++x) CHECK(philox_invert(p, philox_apply(p, x)) == x);
  }
  // :138-147 PhiloxInvert.ZeroRoundsIsIdentity
  {
    VariablePhiloxParams p;
    p.total_bits = 6;
    p.left_side_bits = 3;
    p.right_side_bits = 3;
    p.num_rounds = 0;
    p.left_side_mask = 0x7;
    p.right_side_mask = 0x7;
    CHECK(philox_invert(p, 0b101101) == 0b101101u);
  }
  // :149-157 RoundTrip63BitsRandomPoints
  {
    const auto p = make_philox(63, 5);
    SplitMix64 rng(777);
    const std::uint64_t mask = (1ULL << 63) - 1;
    for (int i = 0; i < 100000; ++i) {
      const std::uint64_t x = rng() & mask;
      if (philox_invert(p, philox_apply(p, x)) != x) {
        CHECK(false);
        break;
      }
    }
  }
  // :159-169 KeySensitivity
  {
    const auto p1 = make_philox(16, 0x1000), p2 = make_philox(16, 0x1001);
    bool any_diff = false;
    for (std::uint64_t x = 0; x < (1ULL << 16) && !any_diff; ++x) any_diff = philox_apply(p1, x) != philox_apply(p2, x);
    CHECK(any_diff);
  }
  // :171-175 RejectsBadParameters
  CHECK_THROWS(make_philox(1, 0), std::invalid_argument);
  CHECK_THROWS(make_philox(64, 0), std::invalid_argument);
  CHECK_THROWS(make_philox(8, 0, 2), std::invalid_argument);
  // :177-187 BijectionSpec.DispatchesToBothVariants
  {
    const auto lcg = make_bijection(LcgParams{4, 1, 0});
    CHECK(lcg.domain_bits == 4 && bijection_apply(lcg, 9) == 9u);
    const auto phil = make_bijection(make_philox(8, 7));
    CHECK(phil.domain_bits == 8);
    std::set<std::uint64_t> image;
    for (std::uint64_t x = 0; x < 256; ++x) image.insert(bijection_apply(phil, x));
    CHECK(image.size() == 256u);
  }
  // :189-192 BijectionSpec.RejectsOutOfDomain
  CHECK_THROWS(bijection_apply(make_bijection(LcgParams{4, 1, 0}), 16), std::out_of_range);

  // Caller-edited keys are honoured: the params path equals the seed path for derived keys, and differs from it
  // once a key is changed (the round-1 shim ignored round_keys).
  {
    auto p = make_philox(20, 99);
    std::uint64_t y_seed = 0;
    CHECK(bsg_philox_apply(20, 99, 24, 12345, &y_seed) == BSG_OK);
    CHECK(philox_apply(p, 12345) == y_seed);
    p.round_keys[7] ^= 0x5A5A5A5Au;
    const std::uint64_t y_edit = philox_apply(p, 12345);
    CHECK(y_edit != y_seed);
    CHECK(philox_invert(p, y_edit) == 12345u);
    p.num_rounds = 5;  // fewer rounds than keys: only the first five are used
    std::set<std::uint64_t> image;
    for (std::uint64_t x = 0; x < 4096; ++x) image.insert(philox_apply(p, x));
    CHECK(image.size() == 4096u);
    p.num_rounds = 30;  // more rounds than keys: the reference reads past the vector; we refuse
    CHECK_THROWS(philox_apply(p, 1), std::invalid_argument);
  }
  // SplitMix64::below (splitmix.hpp:49-59)
  {
    SplitMix64 g(3);
    for (int i = 0; i < 1000; ++i) CHECK(g.below(7) < 7u);
    CHECK_THROWS(g.below(0), std::invalid_argument);
  }
  if (failures) {
    std::fprintf(stderr, "%d failures\n", failures);
    return 1;
  }
  std::printf("test_shim_bijection: all checks passed\n");
  return 0;
}
