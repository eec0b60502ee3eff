// bsg_bijection.cuh -- the keyed bijections of the bijective shuffle, as
// register-resident 32-bit integer arithmetic for sm_100a (and the same
// functions on the host for key schedules and scalar evaluation).
//
// Semantics follow the reference bit for bit:
//   mix64 / derive_round_keys ........ proj/include/bijshuf/splitmix.hpp:11-31
//   make_lcg / lcg_apply .............. bijection.hpp:25-40 (engine form shuffle.hpp:157-162)
//   make_philox / philox_apply ........ bijection.hpp:73-111 (engine form shuffle.hpp:71-86)
//   philox_invert / odd_inverse ....... bijection.hpp:61-65, 117-143
//   shuffle_domain_bits ............... shuffle.hpp:49-52
//
// Why 32-bit state is exact: the reference keeps s0 (left, L = floor(bits/2)
// <= 31 bits) and s1 (right, R <= 32 bits) in u64 and multiplies by the
// 64-bit constant M0.  Only hi = (M0*s0 mod 2^64) >> 32 and lo = M0*s0 mod
// 2^32 are used, and with s0 < 2^31:
//     lo = s0 * M0lo (mod 2^32),  hi = umulhi(s0, M0lo) + s0 * M0hi (mod 2^32).
// The unbalanced-split shift (lo << d) is folded into the multiplier
// (M0lo << d), and `lo & right_mask` drops the bit the u64 shift would keep.
// All state therefore lives in 32-bit registers; only the counter/image are
// 64-bit when bits > 32.  Round keys are kernel parameters (constant bank),
// so every round is IMAD.HI + IMAD + IMAD + LOP3s with c[][] operands.
#pragma once

#include <cstdint>

#ifdef __CUDACC__
#define BSG_HD __host__ __device__ __forceinline__
#else
#define BSG_HD inline
#endif
#ifdef __CUDA_ARCH__
#define BSG_UNROLL _Pragma("unroll")
#else
#define BSG_UNROLL
#endif

namespace bsg {

constexpr uint64_t kGamma = 0x9E3779B97F4A7C15ULL;  // splitmix.hpp:18
constexpr uint64_t kM0 = 0xD2B74407B1CE6E93ULL;     // bijection.hpp:57
constexpr uint32_t kM0Lo = static_cast<uint32_t>(kM0);
constexpr uint32_t kM0Hi = static_cast<uint32_t>(kM0 >> 32);

constexpr uint64_t odd_inverse_pow2_64(uint64_t a) {  // bijection.hpp:61-65
  uint64_t x = a;
  for (int i = 0; i < 5; ++i) x *= 2 - a * x;
  return x;
}
constexpr uint64_t kM0Inv = odd_inverse_pow2_64(kM0);
constexpr uint32_t kM0InvLo = static_cast<uint32_t>(kM0Inv);
static_assert(kM0Inv * kM0 == 1ULL, "M0 inverse");

BSG_HD uint64_t mix64(uint64_t z) {  // splitmix.hpp:11-15
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

BSG_HD uint32_t round_key(uint64_t seed, int i) {  // splitmix.hpp:27-28
  return static_cast<uint32_t>(mix64(seed + (static_cast<uint64_t>(i) + 1) * kGamma));
}

// shuffle.hpp:49-52: max(4, ceil(log2 m)) for m >= 2.
BSG_HD int domain_bits(uint64_t m) {
  int needed = 0;
  if (m > 1) {
    uint64_t v = m - 1;
    while (v) {
      ++needed;
      v >>= 1;
    }
  }
  return needed < 4 ? 4 : needed;
}

enum Variant : int32_t { kLcg = 0, kPhilox = 1 };

// Number of round keys carried inside the kernel parameter block.  Rounds
// beyond this read a device array (the generic path).
constexpr int kParamKeys = 32;

// Everything a kernel needs to evaluate the bijection of one shuffle.
struct BijParams {
  uint64_t lcg_a = 1, lcg_c = 0, lcg_ainv = 1;  // LCG (a forced odd), inverse multiplier
  uint64_t mask = 0;                            // 2^bits - 1
  uint32_t LM = 0, RM = 0;                      // Philox half masks (RM may be 0xFFFFFFFF)
  uint32_t shl = 0;                             // 2^L: the inverse moves the spare bit up with an IMAD
  int32_t variant = kPhilox, bits = 0, L = 0, R = 0, rounds = 0, pad = 0;
  const uint32_t* gkeys = nullptr;  // device copy of all keys (rounds > kParamKeys)
  uint32_t keys[kParamKeys] = {};
  // Top-aligned inverse (philox_inv_top): shift 32 - L, M0^-1 << (32 - L), keys << (32 - L).
  uint32_t sh = 0, inv_top = 0;
  uint32_t ktop[kParamKeys] = {};
  // High product on the FP64 pipe (philox_inv_top): fma_rd(2^52 + X, hc, hk) = 1.5 * 2^52 + floor(X * M0' / 2^32)
  // exactly, M0' = M0 mod 2^(32+L); hc = M0' / 2^32, hk = 1.5 * 2^52 - M0' * 2^20.  Valid for L <= 16.
  double hc = 0.0, hk = 0.0;
};

// ---------------------------------------------------------------------------
// Philox rounds on split state (s0 < 2^L, s1 < 2^R).  D = R - L in {0, 1}.
// For D == 0 the right half may carry garbage above bit R between rounds:
// it only enters `(hi ^ k ^ s1) & LM`, so it is masked once at the end.
// ---------------------------------------------------------------------------
// D == 0: one IMAD.WIDE yields both product words (measured fastest on
// sm_100a); D == 1: IMAD.HI for the high word and the shifted multiplier
// M0lo<<1 for the low word, so the spare bit enters through one OR.
template <int D>
BSG_HD void philox_round(uint32_t& s0, uint32_t& s1, uint32_t k, int L, uint32_t LM, uint32_t RM) {
  if (D == 0) {
    const uint64_t w = static_cast<uint64_t>(s0) * kM0Lo;
    const uint32_t hi = static_cast<uint32_t>(w >> 32) + s0 * kM0Hi;
    const uint32_t lo = static_cast<uint32_t>(w);
    s0 = (hi ^ k ^ s1) & LM;
    s1 = lo;  // garbage above bit R is masked once at the end
  } else {
#ifdef __CUDA_ARCH__
    const uint32_t hi = __umulhi(s0, kM0Lo) + s0 * kM0Hi;
#else
    const uint32_t hi = static_cast<uint32_t>((static_cast<uint64_t>(s0) * kM0Lo) >> 32) + s0 * kM0Hi;
#endif
    const uint32_t lo = (s0 * (kM0Lo << 1)) | (s1 >> L);
    s0 = (hi ^ k ^ s1) & LM;
    s1 = lo & RM;
  }
}

#ifdef __CUDACC__
// Forward round with the high product on the FP64 pipe (see inv_high_word below): s0 < 2^L is exact in the
// biased double, and floor(s0 * M0' / 2^32) has the reference's hi in its low L bits (M0' = M0 mod 2^(32+L)),
// so one DFMA replaces IMAD.WIDE + IMAD (D == 0) or IMAD.HI + IMAD (D == 1).  Device only, L <= 16.
template <int D>
__device__ __forceinline__ void philox_round_f64(uint32_t& s0, uint32_t& s1, uint32_t k, int L, uint32_t LM,
                                                 uint32_t RM, double hc, double hk) {
  const uint32_t hi =
      static_cast<uint32_t>(__double2loint(__fma_rd(__hiloint2double(0x43300000, static_cast<int>(s0)), hc, hk)));
  if (D == 0) {
    const uint32_t lo = s0 * kM0Lo;
    s0 = (hi ^ k ^ s1) & LM;
    s1 = lo;  // garbage above bit R is masked once at the end
  } else {
    const uint32_t lo = (s0 * (kM0Lo << 1)) | (s1 >> L);
    s0 = (hi ^ k ^ s1) & LM;
    s1 = lo & RM;
  }
}
#endif

// Inverse round (bijection.hpp:127-141).  For D == 1 the right half carries
// garbage above bit L+1 between rounds (masked at the end): the spare bit is
// bit 0 and only `t1 >> 1` modulo 2^L is consumed.
// The spare-bit shift t1 << L is an IMAD by the runtime constant shl = 2^L
// (FMA pipe) rather than a SHF (ALU pipe): it balances the two integer pipes
// (measured +17% on sm_100a, tools/microbench/mb6.cu).
template <int D>
BSG_HD void philox_inv_round(uint32_t& t0, uint32_t& t1, uint32_t k, uint32_t shl, uint32_t LM) {
  const uint32_t s0 = ((t1 >> D) * kM0InvLo) & LM;
#ifdef __CUDA_ARCH__
  const uint32_t hi = __umulhi(s0, kM0Lo) + s0 * kM0Hi;
#else
  const uint32_t hi = static_cast<uint32_t>((static_cast<uint64_t>(s0) * kM0Lo) >> 32) + s0 * kM0Hi;
#endif
  const uint32_t s1 = ((hi ^ k ^ t0) & LM) | (D ? (t1 * shl) : 0u);
  t0 = s0;
  t1 = s1;
}

// Key access: compile-time round count NR > 0 reads the parameter block with
// constant indices; NR == 0 loops over p.rounds keys from p.gkeys (device) or
// p.keys (host, rounds <= kParamKeys) -- the generic path.
template <int D, int NR>
BSG_HD uint64_t philox_fwd(uint64_t x, const BijParams& p) {
  uint32_t s0 = static_cast<uint32_t>(x >> p.R);
  uint32_t s1 = static_cast<uint32_t>(x) & p.RM;
  if constexpr (NR > 0) {
    BSG_UNROLL
    for (int i = 0; i < NR; ++i) philox_round<D>(s0, s1, p.keys[i], p.L, p.LM, p.RM);
  } else {
#ifdef __CUDA_ARCH__
    const uint32_t* ks = p.gkeys;
#pragma unroll 4
    for (int i = 0; i < p.rounds; ++i) philox_round<D>(s0, s1, __ldg(ks + i), p.L, p.LM, p.RM);
#else
    const uint32_t* ks = p.gkeys ? p.gkeys : p.keys;
    for (int i = 0; i < p.rounds; ++i) philox_round<D>(s0, s1, ks[i], p.L, p.LM, p.RM);
#endif
  }
  return (static_cast<uint64_t>(s0) << p.R) | (s1 & p.RM);
}

// Inverse in the top-aligned form (device hot path of the partitioned
// shuffle, P1).  Same function as philox_inv_round, 6 instructions per round
// for D == 1 instead of 8 (5 instead of 6 for D == 0):
//   A = t0 << sh, sh = 32 - L: left half kept in the top L bits, zeros below;
//   X = B * (M0^-1 << sh) = (M0^-1 * lo mod 2^L) << sh = s0 << sh exactly --
//       every bit of B at or above L is shifted out, so B may carry garbage;
//   the high word of M0 * X (umulhi + IMAD) holds hi mod 2^L in its top L
//       bits (M0 * X = (M0 * s0) << sh), so Y = HW ^ (k << sh) ^ A holds the
//       new right half's low L bits x at the top, garbage below;
//   D == 1: the right half is x | sp << L with sp = bit 0 of the current one;
//       the next round needs lo = (x >> 1) | sp << (L-1): one funnel shift of
//       (Z:Y) with Z = the previous x (bit 0 = sp), and Z' = Y >> sh = x.
// No masks are needed anywhere inside the loop.
//
// The high word HW = umulhi(X, M0lo) + X * M0hi (IMAD.HI + IMAD, 6 of the 8
// FMA-heavy cycles of a round) is computed on the FP64 pipe instead: with
// M0' = M0 mod 2^(32+L), HW == floor(X * M0' / 2^32) (mod 2^32) because
// X * (M0hi - M0' div 2^32) is a multiple of 2^L * 2^(32-L).  A round-down
// DFMA of the biased double 2^52 + X (bit pattern {X, 0x43300000}) by
// hc = M0' / 2^32 plus hk = 1.5 * 2^52 - M0' * 2^20 evaluates
// X * M0' / 2^32 + 1.5 * 2^52 exactly before its single rounding (every
// operand is exact in 53 bits for L <= 16), so the result's low word is that
// floor: one DFMA replaces IMAD.HI + IMAD, bit-exact for every width
// (tools/microbench/mb9.cu checks all widths 2..32; 2^29 ciphers 3.50 -> 2.89
// ms, 2^30 with L = R 6.42 -> 4.68 ms on B200).
#ifdef __CUDACC__
__device__ __forceinline__ uint32_t inv_high_word(uint32_t X, const BijParams& p) {
  return static_cast<uint32_t>(__double2loint(__fma_rd(__hiloint2double(0x43300000, static_cast<int>(X)), p.hc, p.hk)));
}

// F64: the high word on the FP64 pipe (needs L <= 16, i.e. bits <= 33; the partitioned kernels' domains);
// otherwise IMAD.HI + IMAD.
template <int D, int NR, bool F64 = true>
__device__ __forceinline__ uint64_t philox_inv_top(uint64_t y, const BijParams& p) {
  const uint32_t sh = p.sh;
  const uint32_t t0 = static_cast<uint32_t>(y >> p.R), t1 = static_cast<uint32_t>(y) & p.RM;
  uint32_t A = t0 << sh, B = D ? (t1 >> 1) : t1, Z = t1;
  auto round = [&](uint32_t ktop) {
    const uint32_t X = B * p.inv_top;
    const uint32_t hw = F64 ? inv_high_word(X, p) : __umulhi(X, kM0Lo) + X * kM0Hi;
    const uint32_t Y = hw ^ ktop ^ A;
    if (D) {
      B = __funnelshift_rc(Y, Z, sh + 1);  // (Y >> (sh+1)) | (Z << (L-1)); L == 1 clamps to Z
      Z = Y >> sh;
    } else {
      B = Y >> sh;
    }
    A = X;
  };
  if constexpr (NR > 0) {
#pragma unroll
    for (int i = NR - 1; i >= 0; --i) round(p.ktop[i]);
  } else {
    for (int i = p.rounds - 1; i >= 0; --i) round(__ldg(p.gkeys + i) << sh);
  }
  const uint32_t s0 = A >> sh;
  const uint32_t s1 = D ? (((B << 1) | (Z & 1u)) & p.RM) : (B & p.RM);
  return (static_cast<uint64_t>(s0) << p.R) | s1;
}
#endif

template <int D, int NR>
BSG_HD uint64_t philox_inv(uint64_t y, const BijParams& p) {
#ifdef __CUDA_ARCH__
  return p.L <= 16 ? philox_inv_top<D, NR, true>(y, p) : philox_inv_top<D, NR, false>(y, p);
#else  // host: the reference's round form (bijection.hpp:127-141)
  uint32_t t0 = static_cast<uint32_t>(y >> p.R);
  uint32_t t1 = static_cast<uint32_t>(y) & p.RM;
  if constexpr (NR > 0) {
    for (int i = NR - 1; i >= 0; --i) philox_inv_round<D>(t0, t1, p.keys[i], p.shl, p.LM);
  } else {
    const uint32_t* ks = p.gkeys ? p.gkeys : p.keys;
    for (int i = p.rounds - 1; i >= 0; --i) philox_inv_round<D>(t0, t1, ks[i], p.shl, p.LM);
  }
  return (static_cast<uint64_t>(t0) << p.R) | (t1 & p.RM);
#endif
}

// 32-bit-counter specialisations (bits <= 32): identical arithmetic, no
// 64-bit shifts in the kernel's address path.
template <int D, int NR>
BSG_HD uint32_t philox_fwd32(uint32_t x, const BijParams& p) {
  uint32_t s0 = x >> p.R;
  uint32_t s1 = x & p.RM;
  BSG_UNROLL
  for (int i = 0; i < NR; ++i) philox_round<D>(s0, s1, p.keys[i], p.L, p.LM, p.RM);
  return (s0 << p.R) | (s1 & p.RM);
}

// LCG (shuffle.hpp:160-162): (a*x + c) mod 2^64, masked to the domain.
BSG_HD uint64_t lcg_fwd(uint64_t x, const BijParams& p) { return (p.lcg_a * x + p.lcg_c) & p.mask; }
BSG_HD uint64_t lcg_inv(uint64_t y, const BijParams& p) { return (p.lcg_ainv * (y - p.lcg_c)) & p.mask; }
BSG_HD uint32_t lcg_fwd32(uint32_t x, const BijParams& p) {
  return (static_cast<uint32_t>(p.lcg_a) * x + static_cast<uint32_t>(p.lcg_c)) & static_cast<uint32_t>(p.mask);
}

// Host-side construction of BijParams; mirrors make_lcg / make_philox
// (bijection.hpp:25-34, 73-88) including their argument checks.
// Returns 0 on success, 1 (invalid argument) on a reference-rejected input.
inline int make_params(int variant, int bits, uint64_t seed, int rounds, BijParams& p) {
  p = BijParams{};
  p.variant = variant;
  p.bits = bits;
  if (variant == kLcg) {
    if (bits < 1 || bits > 63) return 1;  // bijection.hpp:26-27
    p.mask = (1ULL << bits) - 1;
    p.lcg_a = (mix64(seed) | 1ULL) & p.mask;
    p.lcg_c = mix64(seed + 1) & p.mask;
    p.lcg_ainv = odd_inverse_pow2_64(p.lcg_a);
    p.rounds = rounds;
    return 0;
  }
  if (bits < 2 || bits > 63) return 1;  // bijection.hpp:75-76
  if (rounds < 3) return 1;             // bijection.hpp:77-78
  p.mask = (1ULL << bits) - 1;
  p.L = bits / 2;
  p.R = bits - p.L;
  p.LM = static_cast<uint32_t>((1ULL << p.L) - 1);
  p.RM = static_cast<uint32_t>((1ULL << p.R) - 1);
  p.shl = static_cast<uint32_t>(1ULL << p.L);
  p.rounds = rounds;
  p.sh = static_cast<uint32_t>(32 - p.L);
  p.inv_top = kM0InvLo << p.sh;
  if (p.L <= 16) {
    const uint64_t m0p = kM0 & ((1ULL << (32 + p.L)) - 1);
    p.hc = static_cast<double>(m0p) * 0x1p-32;
    p.hk = 0x1.8p52 - static_cast<double>(m0p) * 0x1p20;
  }
  for (int i = 0; i < rounds && i < kParamKeys; ++i) {
    p.keys[i] = round_key(seed, i);
    p.ktop[i] = p.keys[i] << p.sh;
  }
  return 0;
}

// Host scalar evaluation (any rounds; keys regenerated on the fly when the
// schedule is longer than the parameter block).
inline uint64_t host_apply(const BijParams& p, uint64_t seed, uint64_t x, bool inverse) {
  if (p.variant == kLcg) return inverse ? lcg_inv(x, p) : lcg_fwd(x, p);
  const int L = p.L, R = p.R, d = R - L;
  uint32_t a = static_cast<uint32_t>(x >> R), b = static_cast<uint32_t>(x) & p.RM;
  auto key = [&](int i) { return i < kParamKeys ? p.keys[i] : round_key(seed, i); };
  if (!inverse) {
    for (int i = 0; i < p.rounds; ++i) {
      if (d) philox_round<1>(a, b, key(i), L, p.LM, p.RM);
      else philox_round<0>(a, b, key(i), L, p.LM, p.RM);
    }
  } else {
    for (int i = p.rounds - 1; i >= 0; --i) {
      if (d) philox_inv_round<1>(a, b, key(i), p.shl, p.LM);
      else philox_inv_round<0>(a, b, key(i), p.shl, p.LM);
    }
  }
  return (static_cast<uint64_t>(a) << R) | (b & p.RM);
}

}  // namespace bsg
