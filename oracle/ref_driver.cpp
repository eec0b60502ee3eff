// ref_driver.cpp -- extern "C" shim over the UNMODIFIED reference library.
//
// TEST / BASELINE INFRASTRUCTURE ONLY.  Compiled by oracle/Makefile against
// the read-only reference headers (/root/reference/proj/include, not copied)
// into oracle/_ref/libbijshuf_ref*.so.  Used for two things only:
//   * generating the golden fixtures in tests/golden/ (make_golden.py), which
//     pin the C restatement in oracle/bijshuf_oracle.c to the reference;
//   * the CPU baseline of bench.py (--impl reference and cpu_baseline), which
//     times bijshuf::shuffle_values_into (shuffle.hpp:308-315) on host cores
//     exactly as bench_bijective does (bench.hpp:92-104, time_trials :41-59).
// The product library never loads it.
#include <bijshuf/shuffle.hpp>
#include <bijshuf/splitmix.hpp>

#include <chrono>
#include <cstdint>
#include <cstring>
#include <numeric>
#include <stdexcept>
#include <thread>
#include <vector>

using namespace bijshuf;

namespace {

template <typename Fn>
int guarded(Fn&& fn) {
  try {
    fn();
    return 0;
  } catch (const std::invalid_argument&) {
    return -1;
  } catch (const std::out_of_range&) {
    return -2;
  } catch (...) {
    return -3;
  }
}

ShuffleConfig make_cfg(uint64_t seed, int variant, int rounds, int workers) {
  ShuffleConfig c;
  c.seed = seed;
  c.variant = variant == 0 ? BijectionVariant::Lcg : BijectionVariant::VariablePhilox;
  c.num_rounds = rounds;
  c.workers = workers;
  return c;
}

template <size_t N>
struct Blob {
  unsigned char b[N];
};

template <size_t N>
int values_n(const void* in, void* out, uint64_t m, const ShuffleConfig& cfg) {
  return guarded([&] {
    std::vector<Blob<N>> v(m), o;
    std::memcpy(v.data(), in, m * N);
    shuffle_values_into(v, cfg, o);
    std::memcpy(out, o.data(), m * N);
  });
}

double now_s() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

}  // namespace

extern "C" {

int ref_avx512_active() {
#if defined(__AVX512F__)
  return 1;
#else
  return 0;
#endif
}

int ref_hardware_threads() { return resolve_workers(0); }

uint64_t ref_mix64(uint64_t z) { return mix64(z); }

int ref_derive_round_keys(uint64_t seed, int rounds, uint32_t* out) {
  return guarded([&] {
    auto k = derive_round_keys(seed, rounds);
    std::memcpy(out, k.data(), k.size() * 4);
  });
}

int ref_domain_bits(uint64_t m) { return shuffle_domain_bits(m); }

int ref_philox_apply(int bits, uint64_t seed, int rounds, uint64_t x, uint64_t* y) {
  return guarded([&] { *y = philox_apply(make_philox(bits, seed, rounds), x); });
}

int ref_philox_apply_many(int bits, uint64_t seed, int rounds, const uint64_t* x, uint64_t n, uint64_t* y) {
  return guarded([&] {
    auto p = make_philox(bits, seed, rounds);
    for (uint64_t i = 0; i < n; ++i) y[i] = philox_apply(p, x[i]);
  });
}

int ref_philox_invert(int bits, uint64_t seed, int rounds, uint64_t y, uint64_t* x) {
  return guarded([&] { *x = philox_invert(make_philox(bits, seed, rounds), y); });
}

int ref_make_lcg(int bits, uint64_t seed, uint64_t* a, uint64_t* c) {
  return guarded([&] {
    auto p = make_lcg(bits, seed);
    *a = p.a;
    *c = p.c;
  });
}

int ref_shuffle_indices(uint64_t m, uint64_t seed, int variant, int rounds, int workers, uint64_t* out) {
  return guarded([&] {
    Permutation p;
    shuffle_indices_into(m, make_cfg(seed, variant, rounds, workers), p);
    std::memcpy(out, p.data(), m * 8);
  });
}

int ref_shuffle_values(const void* in, void* out, uint64_t m, uint32_t elem_bytes, uint64_t seed, int variant,
                       int rounds, int workers) {
  const ShuffleConfig cfg = make_cfg(seed, variant, rounds, workers);
  switch (elem_bytes) {
    case 1: return values_n<1>(in, out, m, cfg);
    case 2: return values_n<2>(in, out, m, cfg);
    case 4: return values_n<4>(in, out, m, cfg);
    case 8: return values_n<8>(in, out, m, cfg);
    case 12: return values_n<12>(in, out, m, cfg);
    case 16: return values_n<16>(in, out, m, cfg);
    case 32: return values_n<32>(in, out, m, cfg);
    default: return -1;
  }
}

// bench_bijective (bench.hpp:92-104): iota u64 values, out buffer reused via
// shuffle_values_into, one untimed warm-up then `trials` timed calls
// (time_trials, bench.hpp:41-59).  Allocation is excluded from timing.
// Writes the mean seconds per call and the FNV-1a of the last output.
int ref_time_shuffle_u64(uint64_t m, uint64_t seed, int variant, int rounds, int workers, int trials,
                         double* mean_s, uint64_t* fnv) {
  return guarded([&] {
    const ShuffleConfig cfg = make_cfg(seed, variant, rounds, workers);
    auto values = detail::make_buffer<uint64_t>(m);
    std::iota(values.begin(), values.end(), uint64_t{0});
    auto out = detail::make_buffer<uint64_t>(m);
    shuffle_values_into(values, cfg, out);  // warm-up
    double total = 0;
    for (int t = 0; t < trials; ++t) {
      const double t0 = now_s();
      shuffle_values_into(values, cfg, out);
      total += now_s() - t0;
    }
    *mean_s = trials > 0 ? total / trials : 0.0;
    uint64_t h = 0xcbf29ce484222325ULL;
    for (uint64_t x : out) {
      h ^= x;
      h *= 0x100000001b3ULL;
    }
    *fnv = h;
  });
}

// Same, but each call is timed individually into per_call_s[0..calls) with
// no internal warm-up (bench.py --impl reference does its own warm-up).
int ref_time_shuffle_u64_calls(uint64_t m, uint64_t seed, int variant, int rounds, int workers, int calls,
                               double* per_call_s, uint64_t* fnv) {
  return guarded([&] {
    const ShuffleConfig cfg = make_cfg(seed, variant, rounds, workers);
    auto values = detail::make_buffer<uint64_t>(m);
    std::iota(values.begin(), values.end(), uint64_t{0});
    auto out = detail::make_buffer<uint64_t>(m);
    for (int t = 0; t < calls; ++t) {
      const double t0 = now_s();
      shuffle_values_into(values, cfg, out);
      per_call_s[t] = now_s() - t0;
    }
    uint64_t h = 0xcbf29ce484222325ULL;
    for (uint64_t x : out) {
      h ^= x;
      h *= 0x100000001b3ULL;
    }
    *fnv = h;
  });
}

// C5 payload: 16-byte {u64 key, u64 value} records (the Pair of bench.hpp:112-114),
// keys = i, values = ~i; each call timed individually as above.
int ref_time_shuffle_pairs_calls(uint64_t m, uint64_t seed, int variant, int rounds, int workers, int calls,
                                 double* per_call_s) {
  struct Pair {
    uint64_t key, value;
  };
  return guarded([&] {
    const ShuffleConfig cfg = make_cfg(seed, variant, rounds, workers);
    auto values = detail::make_buffer<Pair>(m);
    for (uint64_t i = 0; i < m; ++i) values[i] = Pair{i, ~i};
    auto out = detail::make_buffer<Pair>(m);
    for (int t = 0; t < calls; ++t) {
      const double t0 = now_s();
      shuffle_values_into(values, cfg, out);
      per_call_s[t] = now_s() - t0;
    }
  });
}

// C4 payload: `batch` independent shuffles of iota(m) u32 rows keyed seed + b -- the
// BijectiveShuffleSampler convention (stats.hpp:314-324) with the values moved by
// shuffle_values_into (shuffle.hpp:308-315).  The reference runs one shuffle per
// call (m = 1024 is one 65536-counter chunk, so one worker); the rows are spread
// over `threads` host threads (0 = hardware_concurrency).  Each call of the batch
// is timed individually into per_call_s[0..calls).
int ref_time_batched_u32_calls(uint64_t batch, uint64_t m, uint64_t seed, int variant, int rounds, int threads,
                               int calls, double* per_call_s) {
  return guarded([&] {
    const int T = threads > 0 ? threads : resolve_workers(0);
    std::vector<std::vector<uint32_t>> in(batch, std::vector<uint32_t>(m)), out(batch, std::vector<uint32_t>(m));
    for (auto& r : in) std::iota(r.begin(), r.end(), uint32_t{0});
    for (int t = 0; t < calls; ++t) {
      const double t0 = now_s();
      std::vector<std::thread> pool;
      for (int w = 0; w < T; ++w)
        pool.emplace_back([&, w] {
          for (uint64_t b = w; b < batch; b += static_cast<uint64_t>(T))
            shuffle_values_into(in[b], make_cfg(seed + b, variant, rounds, 1), out[b]);
        });
      for (auto& th : pool) th.join();
      per_call_s[t] = now_s() - t0;
    }
  });
}

}  // extern "C"
