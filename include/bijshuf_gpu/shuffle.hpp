// bijshuf_gpu/shuffle.hpp -- header-only C++ shim that re-exposes the
// reference `bijshuf` API (proj/include/bijshuf/{shuffle,bijection,splitmix,
// permutation}.hpp) on top of the C ABI of libbsg.so (include/bsg.h).
//
// Drop-in: replace `#include <bijshuf/shuffle.hpp>` with
// `#include <bijshuf_gpu/shuffle.hpp>` and link `-lbsg`; the names,
// signatures, config fields, exception types and outputs are the
// reference's.  Shuffles run on the current CUDA device.  Trivially copyable
// element types move through the GPU (1/2/4/8/16-byte elements natively, any
// other size through a record gather); other types (e.g. std::string, which
// cannot live in device memory) get their permutation from the GPU and are
// moved on the host.
#pragma once

#include <bsg.h>

#include <cstdint>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <variant>
#include <vector>

namespace bijshuf {

enum class BijectionVariant { Lcg, VariablePhilox };  // shuffle.hpp:20

struct ShuffleConfig {  // shuffle.hpp:25-30
  std::uint64_t seed = 0;
  BijectionVariant variant = BijectionVariant::VariablePhilox;
  int num_rounds = 24;
  int workers = 0;  // accepted; the output never depends on it
};

using Permutation = std::vector<std::uint64_t>;  // permutation.hpp:15

namespace detail {

inline void throw_on(bsg_status s, const char* what) {
  if (s == BSG_OK) return;
  std::string msg = std::string(what) + ": " + bsg_status_string(s);
  const char* d = bsg_last_error();
  if (d && *d) msg += std::string(" (") + d + ")";
  switch (s) {
    case BSG_EINVAL:
    case BSG_EALIAS:
    case BSG_EUNSUPPORTED: throw std::invalid_argument(msg);
    case BSG_ERANGE: throw std::out_of_range(msg);
    case BSG_ENOMEM: throw std::bad_alloc();
    default: throw std::runtime_error(msg);
  }
}

inline bsg_config to_c(const ShuffleConfig& c) {
  bsg_config r = bsg_config_default();
  r.seed = c.seed;
  r.variant = c.variant == BijectionVariant::Lcg ? BSG_LCG : BSG_VARIABLE_PHILOX;
  r.num_rounds = c.num_rounds;
  r.workers = c.workers;
  return r;
}

}  // namespace detail

// ------------------------------------------------------------- splitmix.hpp
// mix64 stays constexpr (the reference's is): it is the same three-line
// finalizer libbsg evaluates (bsg_mix64), checked equal in tests/cpp.
constexpr std::uint64_t mix64(std::uint64_t z) noexcept {  // splitmix.hpp:11-15
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}
inline constexpr std::uint64_t kSplitMixGamma = 0x9E3779B97F4A7C15ULL;
inline std::vector<std::uint32_t> derive_round_keys(std::uint64_t seed, int num_rounds) {  // splitmix.hpp:22-31
  if (num_rounds < 1) throw std::invalid_argument("num_rounds must be >= 1");
  std::vector<std::uint32_t> k(static_cast<std::size_t>(num_rounds));
  detail::throw_on(bsg_derive_round_keys(seed, num_rounds, k.data()), "derive_round_keys");
  return k;
}

// splitmix.hpp:35-63: value k of stream s is mix64(s + k * gamma).
class SplitMix64 {
 public:
  using result_type = std::uint64_t;
  explicit constexpr SplitMix64(std::uint64_t seed) noexcept : state_(seed) {}
  constexpr std::uint64_t operator()() noexcept {
    state_ += kSplitMixGamma;
    return mix64(state_);
  }
  static constexpr std::uint64_t min() noexcept { return 0; }
  static constexpr std::uint64_t max() noexcept { return ~0ULL; }
  // Unbiased draw from [0, bound) by rejection of the uneven tail; bound >= 1.
  std::uint64_t below(std::uint64_t bound) {
    if (bound == 0) throw std::invalid_argument("bound must be >= 1");
    const std::uint64_t limit = ~0ULL - (~0ULL % bound);
    for (;;) {
      const std::uint64_t v = (*this)();
      if (v < limit) return v % bound;
    }
  }

 private:
  std::uint64_t state_;
};

// ------------------------------------------------------------ bijection.hpp
struct LcgParams {  // bijection.hpp:14-22
  int modulus_bits = 0;
  std::uint64_t a = 1;
  std::uint64_t c = 0;
  std::uint64_t domain_mask() const noexcept {
    return (modulus_bits >= 64) ? ~0ULL : ((1ULL << modulus_bits) - 1);
  }
};

inline LcgParams make_lcg(int modulus_bits, std::uint64_t seed) {  // bijection.hpp:25-34
  LcgParams p;
  p.modulus_bits = modulus_bits;
  detail::throw_on(bsg_make_lcg(modulus_bits, seed, &p.a, &p.c), "make_lcg");
  return p;
}

inline std::uint64_t lcg_apply(const LcgParams& p, std::uint64_t x) {  // bijection.hpp:36-40
  std::uint64_t y = 0;
  detail::throw_on(bsg_lcg_apply(p.modulus_bits, p.a, p.c, x, &y), "lcg_apply");
  return y;
}

struct VariablePhiloxParams {  // bijection.hpp:45-53
  int total_bits = 0;
  int left_side_bits = 0;
  int right_side_bits = 0;
  int num_rounds = 0;
  std::uint64_t left_side_mask = 0;
  std::uint64_t right_side_mask = 0;
  std::vector<std::uint32_t> round_keys;
};

namespace detail {
inline bsg_philox_params to_c(const VariablePhiloxParams& p) {
  bsg_philox_params c;
  c.total_bits = p.total_bits;
  c.left_side_bits = p.left_side_bits;
  c.right_side_bits = p.right_side_bits;
  c.num_rounds = p.num_rounds;
  c.left_side_mask = p.left_side_mask;
  c.right_side_mask = p.right_side_mask;
  c.round_keys = p.round_keys.data();
  c.num_keys = p.round_keys.size();
  return c;
}
}  // namespace detail

inline VariablePhiloxParams make_philox(int total_bits, std::uint64_t seed, int num_rounds = 24) {  // :73-88
  if (total_bits < 2 || total_bits > 63) throw std::invalid_argument("total_bits must be in [2, 63]");
  if (num_rounds < 3) throw std::invalid_argument("num_rounds must be >= 3");
  VariablePhiloxParams p;
  p.total_bits = total_bits;
  p.left_side_bits = total_bits / 2;
  p.right_side_bits = total_bits - p.left_side_bits;
  p.num_rounds = num_rounds;
  p.left_side_mask = (1ULL << p.left_side_bits) - 1;
  p.right_side_mask = (1ULL << p.right_side_bits) - 1;
  p.round_keys = derive_round_keys(seed, num_rounds);
  return p;
}

// Both directions honour every field of p (round_keys, num_rounds including 0, the side widths and masks).
inline std::uint64_t philox_apply(const VariablePhiloxParams& p, std::uint64_t x) {  // bijection.hpp:94-111
  const bsg_philox_params c = detail::to_c(p);
  std::uint64_t y = 0;
  detail::throw_on(bsg_philox_apply_params(&c, x, &y), "philox_apply");
  return y;
}

inline std::uint64_t philox_invert(const VariablePhiloxParams& p, std::uint64_t y) {  // bijection.hpp:117-143
  const bsg_philox_params c = detail::to_c(p);
  std::uint64_t x = 0;
  detail::throw_on(bsg_philox_invert_params(&c, y, &x), "philox_invert");
  return x;
}

// bijection.hpp:146-169: tagged choice between the two families.
struct BijectionSpec {
  std::variant<LcgParams, VariablePhiloxParams> variant;
  int domain_bits = 0;
};

inline BijectionSpec make_bijection(const LcgParams& p) { return BijectionSpec{p, p.modulus_bits}; }
inline BijectionSpec make_bijection(const VariablePhiloxParams& p) { return BijectionSpec{p, p.total_bits}; }

inline std::uint64_t bijection_apply(const BijectionSpec& spec, std::uint64_t x) {
  if (const LcgParams* l = std::get_if<LcgParams>(&spec.variant)) return lcg_apply(*l, x);
  return philox_apply(std::get<VariablePhiloxParams>(spec.variant), x);
}

// -------------------------------------------------------------- shuffle.hpp
inline int shuffle_domain_bits(std::uint64_t m) { return bsg_domain_bits(m); }

inline Permutation compact_permutation(const Permutation& w, std::uint64_t m) {
  if (m > w.size()) throw std::invalid_argument("compact_permutation: m exceeds length");
  Permutation out;
  out.reserve(static_cast<std::size_t>(m));
  for (std::uint64_t v : w)
    if (v < m) out.push_back(v);
  return out;
}

inline void shuffle_indices_into(std::uint64_t m, const ShuffleConfig& cfg, Permutation& out) {
  out.resize(static_cast<std::size_t>(m));
  const bsg_config c = detail::to_c(cfg);
  detail::throw_on(bsg_shuffle_indices(m, &c, out.data(), nullptr), "shuffle_indices");
}

inline Permutation shuffle_indices(std::uint64_t m, const ShuffleConfig& cfg) {
  Permutation out;
  shuffle_indices_into(m, cfg, out);
  return out;
}

template <typename T>
void shuffle_values_into(const std::vector<T>& values, const ShuffleConfig& cfg, std::vector<T>& out) {
  if (&out == &values) throw std::invalid_argument("shuffle_values_into: out aliases input");
  const std::uint64_t m = values.size();
  if constexpr (std::is_trivially_copyable<T>::value) {
    out.resize(values.size());
    const bsg_config c = detail::to_c(cfg);
    detail::throw_on(bsg_shuffle_values(values.data(), out.data(), m, static_cast<std::uint32_t>(sizeof(T)), &c,
                                        nullptr),
                     "shuffle_values");
  } else {
    const Permutation perm = shuffle_indices(m, cfg);  // GPU
    out.clear();
    out.reserve(values.size());
    for (std::uint64_t k = 0; k < m; ++k) out.push_back(values[static_cast<std::size_t>(perm[k])]);
  }
}

template <typename T>
std::vector<T> shuffle_values(const std::vector<T>& values, const ShuffleConfig& cfg) {
  std::vector<T> out;
  shuffle_values_into(values, cfg, out);
  return out;
}

template <typename T>
void gather_into(const std::vector<T>& src, const std::vector<std::uint64_t>& indices, std::vector<T>& out,
                 int workers = 0) {
  (void)workers;
  if (static_cast<const void*>(&out) == static_cast<const void*>(&src) ||
      static_cast<const void*>(&out) == static_cast<const void*>(&indices))
    throw std::invalid_argument("gather_into: out aliases an input");
  static_assert(std::is_trivially_copyable<T>::value, "gather on the GPU needs trivially copyable elements");
  out.resize(indices.size());
  detail::throw_on(bsg_gather(src.data(), src.size(), indices.data(), out.data(), indices.size(),
                              static_cast<std::uint32_t>(sizeof(T)), nullptr),
                   "gather");
}

template <typename T>
std::vector<T> gather(const std::vector<T>& src, const std::vector<std::uint64_t>& indices, int workers = 0) {
  std::vector<T> out;
  gather_into(src, indices, out, workers);
  return out;
}

// Batched sampler convention (stats.hpp:314-324): shuffle b of a row-major
// (batch x m) array uses seed + b.
template <typename T>
void shuffle_values_batched_into(const std::vector<T>& values, std::uint64_t batch, const ShuffleConfig& cfg,
                                 std::vector<T>& out) {
  static_assert(std::is_trivially_copyable<T>::value, "batched shuffle needs trivially copyable elements");
  if (&out == &values) throw std::invalid_argument("shuffle_values_batched: out aliases input");
  if (batch == 0 || values.size() % batch) throw std::invalid_argument("values.size() must be a multiple of batch");
  out.resize(values.size());
  const bsg_config c = detail::to_c(cfg);
  detail::throw_on(bsg_shuffle_values_batched(values.data(), out.data(), batch, values.size() / batch,
                                              static_cast<std::uint32_t>(sizeof(T)), &c, nullptr),
                   "shuffle_values_batched");
}

}  // namespace bijshuf
