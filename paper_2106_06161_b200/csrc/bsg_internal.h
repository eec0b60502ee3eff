// bsg_internal.h -- host-side declarations shared by the C-ABI layer and the
// kernel translation units.  Not installed; the public surface is include/bsg.h.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "bsg_bijection.cuh"

namespace bsg {

// Launch geometry shared by host dispatch and kernels.
#ifndef BSG_POW2_ITEMS
#define BSG_POW2_ITEMS 8
#endif
#ifndef BSG_COMPACT_ITEMS
#define BSG_COMPACT_ITEMS 8
#endif
constexpr int kThreads = 256;
constexpr int kPow2Items = BSG_POW2_ITEMS;        // counters per thread, pow2 kernel
constexpr int kCompactItems = BSG_COMPACT_ITEMS;  // counters per thread, compacting (look-back) kernel
constexpr uint64_t kCompactTile = static_cast<uint64_t>(kThreads) * kCompactItems;
constexpr uint64_t kCompactTileMin = static_cast<uint64_t>(kThreads) * 8;  // smallest tile of any payload type
constexpr int kBatchedMaxRounds = 64;

struct IdxTag {};  // "payload" of shuffle_indices: the image itself, written as u64

// Input addressing: one contiguous array, or a table of equally sized shards
// (peer pointers for the multi-GPU sharded mode; shard g holds elements
// [g*shard_elems, (g+1)*shard_elems)).
constexpr int kMaxShards = 16;
struct Src {
  const void* base = nullptr;
  const void* shard[kMaxShards] = {};
  uint64_t shard_elems = 0;
  int32_t nshards = 0;     // 0 = contiguous `base`
  int32_t shard_shift = -1;  // log2(shard_elems) when a power of two, else -1
};

// Decoupled look-back workspace (one per device context).  Status words pack
// [flag:2 | epoch:22 | value:40]; a word from an older launch carries another
// epoch and reads as "not yet published", so the buffer is never cleared
// between launches (only when the 22-bit epoch wraps).
struct Lookback {
  unsigned long long* status = nullptr;
  unsigned int* tile_counter = nullptr;
  uint32_t epoch = 1;
};

// Which bijection implementation a launch uses.
enum Kind : int {
  kKindLcg = 0,
  kKindPh0 = 1,   // Philox, R == L, 24 rounds unrolled (keys in the parameter block)
  kKindPh1 = 2,   // Philox, R == L + 1, 24 rounds unrolled
  kKindPh0G = 3,  // Philox, R == L, any round count (keys in device memory)
  kKindPh1G = 4,  // Philox, R == L + 1, any round count
};

inline int kind_of(const BijParams& p) {
  if (p.variant == kLcg) return kKindLcg;
  const int d = p.R - p.L;
  if (p.rounds == 24) return d ? kKindPh1 : kKindPh0;
  return d ? kKindPh1G : kKindPh0G;
}

struct ShuffleLaunch {
  Src src;                        // payload source (ignored for indices)
  void* out = nullptr;            // output (T*, or uint64_t* for indices)
  uint64_t m = 0;                 // number of elements (images >= m are dropped)
  uint64_t c0 = 0, c1 = 0;        // counter range [c0, c1) of the padded domain
  BijParams p;                    // bijection
  Lookback lb;                    // look-back workspace (compacting path)
  unsigned long long* count_out = nullptr;  // device: survivors in [c0, c1) (optional)
  bool compact = true;            // false: every image in range is < m (pow2 path)
};

// elem_code: 0 = indices (u64 images), 1/2/4/8/16 = native element bytes.
cudaError_t launch_shuffle(int elem_code, const ShuffleLaunch& a, cudaStream_t s);

struct BatchedLaunch {
  const void* in = nullptr;
  void* out = nullptr;
  uint64_t batch = 0;
  uint32_t m = 0;
  uint64_t seed = 0;  // shuffle b uses seed + b (stats.hpp:319-323)
  BijParams p;        // variant / bits / rounds template (keys derived on device)
};
// Returns cudaErrorNotSupported when the shape does not fit the shared-memory kernel.
cudaError_t launch_batched(int elem_code, const BatchedLaunch& a, cudaStream_t s);
bool batched_supported(int elem_code, uint32_t m, int bits, int rounds);

cudaError_t launch_gather(int elem_code, const void* src, const uint64_t* idx, void* out, uint64_t n,
                          cudaStream_t s);
cudaError_t launch_gather_bytes(const void* src, const uint64_t* idx, void* out, uint64_t n, uint32_t elem_bytes,
                                cudaStream_t s);
// y[i] = f(x[i]) (inverse: f^-1); x == nullptr means x[i] = start + i.
cudaError_t launch_map(const uint64_t* x, uint64_t* y, uint64_t n, uint64_t start, const BijParams& p, bool inverse,
                       cudaStream_t s);

// CUB radix-sort shuffle (the paper's SortShuffle comparator, bench.hpp:109-156).
cudaError_t sort_shuffle_u64(const uint64_t* in, uint64_t* out, uint64_t n, uint64_t seed, void* temp,
                             size_t* temp_bytes, cudaStream_t s);

// Count-only pass: *count = #{c in [c0, c1) : f(c) < m} (device pointer).
cudaError_t launch_count(uint64_t m, uint64_t c0, uint64_t c1, const BijParams& p, unsigned long long* count,
                         cudaStream_t s);

cudaError_t launch_store_u64(unsigned long long* p, uint64_t v, cudaStream_t s);

// Count of our kernel launches since load (bench.py's gpu_launches).
void note_launch(uint64_t k = 1);
uint64_t launches();

}  // namespace bsg
