// C++ drop-in test: the reference's own unit-test cases (proj/tests/unit_shuffle.cpp,
// unit_bijection.cpp) rewritten without GTest against include/bijshuf_gpu/shuffle.hpp,
// i.e. exactly the code a reference user recompiles.  Needs a GPU.
#include <bijshuf_gpu/shuffle.hpp>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <numeric>
#include <set>
#include <string>

using namespace bijshuf;

static int failures = 0;
#define CHECK(cond)                                                   \
  do {                                                                \
    if (!(cond)) {                                                    \
      std::fprintf(stderr, "FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond); \
      ++failures;                                                     \
    }                                                                 \
  } while (0)
#define CHECK_THROWS(expr, type)  \
  do {                            \
    bool thrown = false;          \
    try {                         \
      (void)(expr);               \
    } catch (const type&) {       \
      thrown = true;              \
    }                             \
    CHECK(thrown);                \
  } while (0)

static bool is_valid_permutation(const Permutation& p) {
  std::vector<bool> seen(p.size(), false);
  for (auto v : p) {
    if (v >= p.size() || seen[v]) return false;
    seen[v] = true;
  }
  return true;
}

int main() {
  // unit_bijection.cpp:32-37 golden round keys
  CHECK((derive_round_keys(42, 4) == std::vector<std::uint32_t>{0x2FEB6E95u, 0xB266F103u, 0x130F9F52u, 0x0E4AE394u}));
  CHECK_THROWS(derive_round_keys(1, 0), std::invalid_argument);
  // unit_bijection.cpp:43-84 LCG
  for (std::uint64_t seed = 0; seed < 200; ++seed) {
    const LcgParams p = make_lcg(16, seed);
    CHECK((p.a & 1) == 1 && p.a < (1ULL << 16) && p.c < (1ULL << 16));
  }
  CHECK(lcg_apply(LcgParams{3, 3, 1}, 5) == 0u);
  CHECK_THROWS(lcg_apply(LcgParams{3, 3, 0}, 8), std::out_of_range);
  CHECK_THROWS(make_lcg(64, 1), std::invalid_argument);
  // unit_bijection.cpp:86-156 Philox
  {
    const auto p = make_philox(7, 11);
    CHECK(p.left_side_bits == 3 && p.right_side_bits == 4);
    std::set<std::uint64_t> img;
    for (std::uint64_t x = 0; x < 128; ++x) img.insert(philox_apply(p, x));
    CHECK(img.size() == 128u);
    for (int bits = 2; bits <= 12; ++bits) {
      const auto q = make_philox(bits, 1234 + bits);
      for (std::uint64_t x = 0; x < (1ULL << bits); ++x) CHECK(philox_invert(q, philox_apply(q, x)) == x);
    }
    CHECK_THROWS(philox_apply(make_philox(8, 7), 256), std::out_of_range);
    CHECK_THROWS(make_philox(8, 0, 2), std::invalid_argument);
  }
  // unit_shuffle.cpp:14-46
  CHECK((compact_permutation({6, 3, 0, 7, 5, 1, 4, 2}, 5) == Permutation{3, 0, 1, 4, 2}));
  CHECK(shuffle_domain_bits(3) == 4 && shuffle_domain_bits(17) == 5 && shuffle_domain_bits(1025) == 11);
  // unit_shuffle.cpp:48-85
  ShuffleConfig cfg;
  CHECK(shuffle_indices(0, cfg).empty());
  CHECK(shuffle_indices(1, cfg) == Permutation{0});
  bool saw_id = false, saw_swap = false;
  for (std::uint64_t seed = 0; seed < 32; ++seed) {
    cfg.seed = seed;
    const Permutation p = shuffle_indices(2, cfg);
    CHECK(is_valid_permutation(p));
    (p[0] == 0 ? saw_id : saw_swap) = true;
  }
  CHECK(saw_id && saw_swap);
  cfg.seed = 7;
  Permutation p1000 = shuffle_indices(1000, cfg);
  CHECK((p1000[0] == 996 && p1000[1] == 243 && p1000[2] == 472 && p1000[3] == 177));  // reference KAT
  std::sort(p1000.begin(), p1000.end());
  for (std::uint64_t i = 0; i < 1000; ++i) CHECK(p1000[i] == i);
  cfg.seed = 0;
  CHECK((shuffle_indices(16, cfg) == Permutation{5, 12, 2, 11, 0, 3, 7, 13, 15, 6, 14, 9, 8, 10, 1, 4}));
  // unit_shuffle.cpp:96-107 worker independence
  {
    ShuffleConfig c;
    c.seed = 17;
    const std::uint64_t m = (1ULL << 18) + 12345;
    c.workers = 1;
    const Permutation base = shuffle_indices(m, c);
    for (int w : {2, 8, 0}) {
      c.workers = w;
      CHECK(shuffle_indices(m, c) == base);
    }
  }
  // unit_shuffle.cpp:110-135
  {
    ShuffleConfig c;
    c.num_rounds = 2;
    CHECK_THROWS(shuffle_indices(100, c), std::invalid_argument);
    ShuffleConfig a, b;
    a.seed = 1;
    b.seed = 2;
    CHECK(shuffle_indices(10000, a) != shuffle_indices(10000, b));
    c = ShuffleConfig{};
    c.variant = BijectionVariant::Lcg;
    for (std::uint64_t s = 0; s < 10; ++s) {
      c.seed = s;
      CHECK(is_valid_permutation(shuffle_indices(1234, c)));
    }
  }
  // unit_shuffle.cpp:137-203 values
  {
    ShuffleConfig c;
    c.seed = 31;
    const std::uint64_t m = 70000;
    std::vector<std::uint64_t> values(m);
    for (std::uint64_t i = 0; i < m; ++i) values[i] = i * 3 + 1;
    const auto out = shuffle_values(values, c);
    const auto perm = shuffle_indices(m, c);
    for (std::uint64_t k = 0; k < m; ++k) CHECK(out[k] == values[perm[k]]);
    CHECK(shuffle_values(std::vector<int>{}, c).empty());
    std::vector<std::string> strs;
    for (int i = 0; i < 500; ++i) strs.push_back("item" + std::to_string(i));
    auto so = shuffle_values(strs, c);
    auto si = strs;
    std::sort(so.begin(), so.end());
    std::sort(si.begin(), si.end());
    CHECK(so == si);
    struct Rec { std::uint32_t a, b, c; };  // 12-byte record: generic element path
    std::vector<Rec> recs(3001);
    for (std::uint32_t i = 0; i < 3001; ++i) recs[i] = Rec{i, i * 2, i * 3};
    const auto ro = shuffle_values(recs, c);
    const auto rp = shuffle_indices(3001, c);
    for (std::size_t k = 0; k < recs.size(); ++k) CHECK(ro[k].a == rp[k] && ro[k].c == rp[k] * 3);
    CHECK_THROWS(shuffle_values_into(values, c, values), std::invalid_argument);
  }
  // unit_shuffle.cpp:205-221 into-variants across reuse
  {
    ShuffleConfig c;
    c.seed = 21;
    Permutation pb;
    std::vector<std::uint64_t> vb;
    for (std::uint64_t m : {1000ULL, 70000ULL, 17ULL, 2ULL, 0ULL}) {
      shuffle_indices_into(m, c, pb);
      CHECK(pb == shuffle_indices(m, c));
      std::vector<std::uint64_t> values(m);
      for (std::uint64_t i = 0; i < m; ++i) values[i] = i * 7 + 3;
      shuffle_values_into(values, c, vb);
      CHECK(vb == shuffle_values(values, c));
    }
  }
  // unit_shuffle.cpp:222-242 gather
  {
    std::vector<std::uint64_t> src = {10, 20, 30};
    std::vector<std::uint64_t> idx = {2, 2, 0, 1};
    CHECK((gather(src, idx) == std::vector<std::uint64_t>{30, 30, 10, 20}));
    CHECK_THROWS(gather_into(src, idx, src), std::invalid_argument);
  }
  // batched sampler convention (stats.hpp:314-324)
  {
    ShuffleConfig c;
    c.seed = 1000;
    std::vector<std::uint32_t> rows(4 * 1024);
    for (std::size_t i = 0; i < rows.size(); ++i) rows[i] = static_cast<std::uint32_t>(i % 1024);
    std::vector<std::uint32_t> out;
    shuffle_values_batched_into(rows, 4, c, out);
    for (std::uint64_t b = 0; b < 4; ++b) {
      ShuffleConfig cb = c;
      cb.seed = 1000 + b;
      const auto p = shuffle_indices(1024, cb);
      for (std::size_t k = 0; k < 1024; ++k) CHECK(out[b * 1024 + k] == p[k]);
    }
  }
  if (failures) {
    std::fprintf(stderr, "%d failures\n", failures);
    return 1;
  }
  std::printf("test_shim: all checks passed\n");
  return 0;
}
