// bsg_kernels.cuh -- sm_100a kernels of the bijective shuffle.
//
// Hot path (the paper's Bijective2 design, rebuilt for
// B200): ONE kernel per shuffle that
//   1. evaluates the keyed bijection on a tile of counters (registers only),
//   2. flags images < m and ranks them in counter order with warp ballots and
//      a shared-memory scan,
//   3. issues the payload loads in[image] immediately (their DRAM latency
//      overlaps the scan and the look-back),
//   4. resolves the tile's output offset with a decoupled look-back over
//      dynamically numbered tiles,
//   5. writes the payload at out[offset + rank] (each warp's survivors of one
//      item form one contiguous run, so stores coalesce).
// Every element therefore costs one read and one write of HBM.  When every
// image survives (m == 2^bits) steps 2-4 vanish: out[c] = in[f(c)].
//
// Reference equivalents: chained_compact + philox_compact_avx512 +
// ValuesSink (proj/include/bijshuf/shuffle.hpp:107-147, 193-212;
// simd.hpp:72-131).  Output is independent of tile geometry, as the
// reference's is of chunking (shuffle.hpp:22-24).
#pragma once

#include <cuda_runtime.h>

#include "bsg_internal.h"

namespace bsg {

constexpr int kWarps = kThreads / 32;

// ------------------------------------------------------------------ bijection
template <int KIND, typename CT>
__device__ __forceinline__ CT bij(CT x, const BijParams& p) {
  if constexpr (KIND == kKindLcg) {
    if constexpr (sizeof(CT) == 4) return lcg_fwd32(x, p);
    else return lcg_fwd(x, p);
  } else if constexpr (KIND == kKindPh0 || KIND == kKindPh1) {
    constexpr int D = KIND == kKindPh1 ? 1 : 0;
    if constexpr (sizeof(CT) == 4) return philox_fwd32<D, 24>(x, p);
    else return philox_fwd<D, 24>(x, p);
  } else {
    constexpr int D = KIND == kKindPh1G ? 1 : 0;
    return static_cast<CT>(philox_fwd<D, 0>(x, p));
  }
}

// ------------------------------------------------------------- memory helpers
// Random payload reads: non-coherent path, no L1 allocation (no reuse).
template <typename T>
__device__ __forceinline__ T ld_rand(const T* p);
template <>
__device__ __forceinline__ uint8_t ld_rand<uint8_t>(const uint8_t* p) {
  unsigned short v;
  asm volatile("ld.global.nc.L1::no_allocate.u8 %0, [%1];" : "=h"(v) : "l"(p));
  return static_cast<uint8_t>(v);
}
template <>
__device__ __forceinline__ uint16_t ld_rand<uint16_t>(const uint16_t* p) {
  unsigned short v;
  asm volatile("ld.global.nc.L1::no_allocate.u16 %0, [%1];" : "=h"(v) : "l"(p));
  return v;
}
template <>
__device__ __forceinline__ uint32_t ld_rand<uint32_t>(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::64B.u32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}
template <>
__device__ __forceinline__ uint64_t ld_rand<uint64_t>(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::64B.u64 %0, [%1];" : "=l"(v) : "l"(p));
  return v;
}
template <>
__device__ __forceinline__ uint4 ld_rand<uint4>(const uint4* p) {
  uint4 v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::64B.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p));
  return v;
}

// Output stores: streaming (evict-first); the output is never re-read here.
template <typename T>
__device__ __forceinline__ void st_out(T* p, const T& v) {
  __stcs(p, v);
}
template <>
__device__ __forceinline__ void st_out<uint8_t>(uint8_t* p, const uint8_t& v) {
  asm volatile("st.global.cs.u8 [%0], %1;" ::"l"(p), "h"(static_cast<unsigned short>(v)));
}
template <>
__device__ __forceinline__ void st_out<uint16_t>(uint16_t* p, const uint16_t& v) {
  asm volatile("st.global.cs.u16 [%0], %1;" ::"l"(p), "h"(v));
}
template <>
__device__ __forceinline__ void st_out<uint32_t>(uint32_t* p, const uint32_t& v) {
  asm volatile("st.global.cs.u32 [%0], %1;" ::"l"(p), "r"(v));
}
template <>
__device__ __forceinline__ void st_out<uint64_t>(uint64_t* p, const uint64_t& v) {
  asm volatile("st.global.cs.u64 [%0], %1;" ::"l"(p), "l"(v));
}

template <typename T, bool SH>
__device__ __forceinline__ T load_src(const Src& s, uint64_t y) {
  if constexpr (!SH) {
    return ld_rand(static_cast<const T*>(s.base) + y);
  } else {
    uint64_t g, off;
    if (s.shard_shift >= 0) {
      g = y >> s.shard_shift;
      off = y & (s.shard_elems - 1);
    } else {
      g = y / s.shard_elems;
      off = y - g * s.shard_elems;
    }
    return ld_rand(static_cast<const T*>(s.shard[g]) + off);
  }
}

__device__ __forceinline__ unsigned long long ld_relaxed_gpu(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed_gpu(unsigned long long* p, unsigned long long v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__device__ __forceinline__ uint32_t lanemask_lt() {
  uint32_t m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// ----------------------------------------------------------------- pow2 path
// m == 2^bits: every image survives, out[c - c0] = in[f(c)].
template <int KIND, typename CT, typename T, bool SH, int ITEMS>
__global__ void __launch_bounds__(kThreads) k_pow2(Src src, void* out_, uint64_t c0, uint64_t c1, BijParams p) {
  constexpr int kTile = kThreads * ITEMS;
  const uint64_t t0 = c0 + static_cast<uint64_t>(blockIdx.x) * kTile + threadIdx.x;
  const bool full = c0 + (static_cast<uint64_t>(blockIdx.x) + 1) * kTile <= c1;
  CT img[ITEMS];
#pragma unroll
  for (int j = 0; j < ITEMS; ++j) img[j] = bij<KIND, CT>(static_cast<CT>(t0 + j * kThreads), p);
  if constexpr (std::is_same<T, IdxTag>::value) {
    uint64_t* out = static_cast<uint64_t*>(out_) + (t0 - c0);
#pragma unroll
    for (int j = 0; j < ITEMS; ++j)
      if (full || t0 + j * kThreads < c1) st_out<uint64_t>(out + j * kThreads, static_cast<uint64_t>(img[j]));
  } else {
    T v[ITEMS];
#pragma unroll
    for (int j = 0; j < ITEMS; ++j)
      if (full || t0 + j * kThreads < c1) v[j] = load_src<T, SH>(src, img[j]);
    T* out = static_cast<T*>(out_) + (t0 - c0);
#pragma unroll
    for (int j = 0; j < ITEMS; ++j)
      if (full || t0 + j * kThreads < c1) st_out<T>(out + j * kThreads, v[j]);
  }
}

// ------------------------------------------------------------ compacting path
constexpr unsigned long long kFlagAgg = 1ULL << 62;
constexpr unsigned long long kFlagPre = 2ULL << 62;
constexpr unsigned long long kValMask = (1ULL << 40) - 1;

__device__ __forceinline__ unsigned long long pack_status(unsigned long long flag, uint32_t epoch,
                                                          unsigned long long v) {
  return flag | (static_cast<unsigned long long>(epoch & 0x3FFFFFu) << 40) | (v & kValMask);
}

// Warp 0: publish this tile's aggregate, then walk back over predecessors
// 32*kLB at a time (each lane inspects kLB status words per round trip) until an
// inclusive prefix is found; publish the inclusive prefix and return the
// exclusive prefix (decoupled look-back).  Summing several
// windows of aggregates per L2 round trip keeps small grids, where every tile
// runs at once and inclusive prefixes lag, from serialising on the frontier.
#ifndef BSG_LOOKBACK_PER_LANE
#define BSG_LOOKBACK_PER_LANE 1
#endif
__device__ __forceinline__ unsigned long long lookback_warp(const Lookback& lb, uint32_t tile,
                                                            unsigned long long total) {
  constexpr int kLB = BSG_LOOKBACK_PER_LANE;
  const int lane = threadIdx.x & 31;
  unsigned long long* st = lb.status;
  if (tile == 0) {
    if (lane == 0) st_relaxed_gpu(st, pack_status(kFlagPre, lb.epoch, total));
    return 0;
  }
  if (lane == 0) st_relaxed_gpu(st + tile, pack_status(kFlagAgg, lb.epoch, total));
  const uint32_t ep = lb.epoch & 0x3FFFFFu;
  unsigned long long excl = 0;
  long long base = static_cast<long long>(tile) - 1;
  for (;;) {
    unsigned long long w[kLB];
    // Issue every load of the window first (one round trip), then re-poll only words not yet published.
#pragma unroll
    for (int q = 0; q < kLB; ++q) {
      const long long idx = base - (lane + 32 * q);
      w[q] = idx >= 0 ? ld_relaxed_gpu(st + idx) : pack_status(kFlagPre, lb.epoch, 0);
    }
    for (int spins = 0;; ++spins) {
      bool ready = true;
#pragma unroll
      for (int q = 0; q < kLB; ++q)
        ready &= (w[q] >> 62) != 0 && static_cast<uint32_t>((w[q] >> 40) & 0x3FFFFFu) == ep;
      if (__all_sync(0xFFFFFFFFu, ready)) break;
      if (spins > 8) __nanosleep(64);
#pragma unroll
      for (int q = 0; q < kLB; ++q) {
        const long long idx = base - (lane + 32 * q);
        const bool ok = (w[q] >> 62) != 0 && static_cast<uint32_t>((w[q] >> 40) & 0x3FFFFFu) == ep;
        if (!ok && idx >= 0) w[q] = ld_relaxed_gpu(st + idx);
      }
    }
    unsigned long long val[kLB];
    int nearest = 32 * kLB;  // smallest distance (lane + 32*q) holding an inclusive prefix
#pragma unroll
    for (int q = 0; q < kLB; ++q) {
      val[q] = w[q] & kValMask;
      if ((w[q] >> 62) == 2 && lane + 32 * q < nearest) nearest = lane + 32 * q;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) nearest = min(nearest, __shfl_xor_sync(0xFFFFFFFFu, nearest, o));
    unsigned long long v = 0;
#pragma unroll
    for (int q = 0; q < kLB; ++q)
      if (lane + 32 * q <= nearest) v += val[q];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xFFFFFFFFu, v, o);
    excl += v;
    if (nearest < 32 * kLB) break;
    base -= 32 * kLB;
  }
  if (lane == 0) st_relaxed_gpu(st + tile, pack_status(kFlagPre, lb.epoch, excl + total));
  return excl;
}

template <int KIND, typename CT, typename T, bool SH, int ITEMS>
__global__ void __launch_bounds__(kThreads) k_compact(Src src, void* out_, uint64_t m, uint64_t c0, uint64_t c1,
                                                      BijParams p, Lookback lb, unsigned long long* count_out) {
  constexpr int kTile = kThreads * ITEMS;
  constexpr int kSlots = ITEMS * kWarps;       // (item, warp) counts in counter order
  constexpr int kPerLane = kSlots / 32;
  static_assert(kSlots % 32 == 0, "slots");
  __shared__ uint32_t s_cnt[kSlots];
  __shared__ unsigned long long s_prefix, s_total;
  __shared__ uint32_t s_tile;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) {
    const uint32_t t = atomicAdd(lb.tile_counter, 1u);
    if (t == gridDim.x - 1) *lb.tile_counter = 0;  // last ticket: reset for the next launch
    s_tile = t;
  }
  __syncthreads();
  const uint32_t tile = s_tile;
  const uint64_t t0 = c0 + static_cast<uint64_t>(tile) * kTile + tid;

  CT img[ITEMS];
  uint32_t mask[ITEMS];
  using V = typename std::conditional<std::is_same<T, IdxTag>::value, uint64_t, T>::type;
  V v[ITEMS];
#pragma unroll
  for (int j = 0; j < ITEMS; ++j) {
    const uint64_t c = t0 + j * kThreads;
    img[j] = bij<KIND, CT>(static_cast<CT>(c), p);
    const bool keep = (c < c1) && (static_cast<uint64_t>(img[j]) < m);
    mask[j] = __ballot_sync(0xFFFFFFFFu, keep);
    if constexpr (!std::is_same<T, IdxTag>::value) {
      if (keep) v[j] = load_src<T, SH>(src, img[j]);  // in flight during scan + look-back
    }
  }
  if (lane == 0) {
#pragma unroll
    for (int j = 0; j < ITEMS; ++j) s_cnt[j * kWarps + warp] = __popc(mask[j]);
  }
  __syncthreads();
  if (warp == 0) {
    uint32_t a[kPerLane], sum = 0;
#pragma unroll
    for (int i = 0; i < kPerLane; ++i) {
      a[i] = s_cnt[lane * kPerLane + i];
      sum += a[i];
    }
    uint32_t incl = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, incl, o);
      if (lane >= o) incl += y;
    }
    uint32_t run = incl - sum;
#pragma unroll
    for (int i = 0; i < kPerLane; ++i) {
      s_cnt[lane * kPerLane + i] = run;  // exclusive, in place
      run += a[i];
    }
    const unsigned long long total = __shfl_sync(0xFFFFFFFFu, incl, 31);
    const unsigned long long excl = lookback_warp(lb, tile, total);
    if (lane == 0) {
      s_prefix = excl;
      s_total = total;
    }
  }
  __syncthreads();
  const unsigned long long prefix = s_prefix;
  const uint32_t lt = lanemask_lt();
  V* out = static_cast<V*>(out_);
#pragma unroll
  for (int j = 0; j < ITEMS; ++j) {
    if ((mask[j] >> lane) & 1u) {
      const uint64_t pos = prefix + s_cnt[j * kWarps + warp] + __popc(mask[j] & lt);
      if constexpr (std::is_same<T, IdxTag>::value) st_out<uint64_t>(out + pos, static_cast<uint64_t>(img[j]));
      else st_out<T>(out + pos, v[j]);
    }
  }
  if (count_out != nullptr && tile == gridDim.x - 1 && tid == 0) *count_out = prefix + s_total;
}

// Shared-memory-staged variant (payloads of 4, 8, 16 bytes and indices).
// After the block scan every survivor knows its in-tile rank, so its payload
// is fetched with cp.async straight into smem[rank]: the random reads stay in
// flight without holding registers (more tiles resident per SM => more
// memory-level parallelism, the limiter of the 2x-padded case), the warp-0
// look-back overlaps them, and the tile is written back with fully
// coalesced stores in compacted order.
template <typename T>
__device__ __forceinline__ void cp_async_payload(T* smem_dst, const T* gsrc) {
  const uint32_t d = static_cast<uint32_t>(__cvta_generic_to_shared(smem_dst));
  if constexpr (sizeof(T) == 16) {
    asm volatile("cp.async.cg.shared.global.L2::64B [%0], [%1], 16;" ::"r"(d), "l"(gsrc) : "memory");
  } else {
    asm volatile("cp.async.ca.shared.global.L2::64B [%0], [%1], %2;" ::"r"(d), "l"(gsrc), "n"(sizeof(T))
                 : "memory");
  }
}

template <typename T, bool SH>
__device__ __forceinline__ const T* src_addr(const Src& s, uint64_t y) {
  if constexpr (!SH) {
    return static_cast<const T*>(s.base) + y;
  } else {
    uint64_t g, off;
    if (s.shard_shift >= 0) {
      g = y >> s.shard_shift;
      off = y & (s.shard_elems - 1);
    } else {
      g = y / s.shard_elems;
      off = y - g * s.shard_elems;
    }
    return static_cast<const T*>(s.shard[g]) + off;
  }
}

template <int KIND, typename CT, typename T, bool SH, int ITEMS>
__global__ void __launch_bounds__(kThreads) k_compact_smem(Src src, void* out_, uint64_t m, uint64_t c0,
                                                           uint64_t c1, BijParams p, Lookback lb,
                                                           unsigned long long* count_out) {
  constexpr bool kIdx = std::is_same<T, IdxTag>::value;
  using V = typename std::conditional<kIdx, uint64_t, T>::type;
  constexpr int kTile = kThreads * ITEMS;
  constexpr int kSlots = ITEMS * kWarps;  // (item, warp) survivor counts, counter order
  constexpr int kPerLane = kSlots / 32;
  static_assert(kSlots % 32 == 0 && kPerLane <= 4, "slots");
  __shared__ __align__(16) V s_val[kTile];
  __shared__ uint32_t s_cnt[kSlots];
  __shared__ unsigned long long s_prefix;
  __shared__ uint32_t s_tile;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) {
    const uint32_t t = atomicAdd(lb.tile_counter, 1u);
    if (t == gridDim.x - 1) *lb.tile_counter = 0;  // last ticket: reset for the next launch
    s_tile = t;
  }
  __syncthreads();
  const uint32_t tile = s_tile;
  const uint64_t t0 = c0 + static_cast<uint64_t>(tile) * kTile + tid;

  CT img[ITEMS];
  uint32_t mask[ITEMS];
#pragma unroll
  for (int j = 0; j < ITEMS; ++j) {
    const uint64_t c = t0 + j * kThreads;
    img[j] = bij<KIND, CT>(static_cast<CT>(c), p);
    mask[j] = __ballot_sync(0xFFFFFFFFu, (c < c1) && (static_cast<uint64_t>(img[j]) < m));
  }
  if (lane == 0) {
#pragma unroll
    for (int j = 0; j < ITEMS; ++j) s_cnt[j * kWarps + warp] = __popc(mask[j]);
  }
  __syncthreads();
  // Every warp scans the kSlots counts itself (no second barrier before the loads).
  uint32_t a[kPerLane], sum = 0;
#pragma unroll
  for (int i = 0; i < kPerLane; ++i) {
    a[i] = s_cnt[lane * kPerLane + i];
    sum += a[i];
  }
  uint32_t incl = sum;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, incl, o);
    if (lane >= o) incl += y;
  }
  const uint32_t total = __shfl_sync(0xFFFFFFFFu, incl, 31);
  uint32_t ex[kPerLane];
  ex[0] = incl - sum;
#pragma unroll
  for (int i = 1; i < kPerLane; ++i) ex[i] = ex[i - 1] + a[i - 1];
  const uint32_t lt = lanemask_lt();
#pragma unroll
  for (int j = 0; j < ITEMS; ++j) {
    const int e = j * kWarps + warp;  // warp-uniform slot
    uint32_t base = 0;
#pragma unroll
    for (int i = 0; i < kPerLane; ++i) {
      const uint32_t x = __shfl_sync(0xFFFFFFFFu, ex[i], e / kPerLane);
      if (e % kPerLane == i) base = x;
    }
    if ((mask[j] >> lane) & 1u) {
      const uint32_t r = base + __popc(mask[j] & lt);
      if constexpr (kIdx) s_val[r] = static_cast<uint64_t>(img[j]);
      else cp_async_payload<T>(&s_val[r], src_addr<T, SH>(src, img[j]));
    }
  }
  if constexpr (!kIdx) asm volatile("cp.async.commit_group;" ::: "memory");
  if (warp == 0) {
    const unsigned long long excl = lookback_warp(lb, tile, total);
    if (lane == 0) s_prefix = excl;
  }
  if constexpr (!kIdx) asm volatile("cp.async.wait_all;" ::: "memory");
  __syncthreads();
  const unsigned long long prefix = s_prefix;
  V* out = static_cast<V*>(out_) + prefix;
  for (uint32_t i = tid; i < total; i += kThreads) st_out<V>(out + i, s_val[i]);
  if (count_out != nullptr && tile == gridDim.x - 1 && tid == 0) *count_out = prefix + total;
}


// --------------------------------------------------------------- batched path
// Many independent shuffles of the same length m (BijectiveShuffleSampler,
// stats.hpp:314-324: shuffle b is keyed by seed + b).  One CTA per shuffle:
// the row is staged in shared memory, round keys are derived on device, the
// cipher runs from registers and the payload is gathered from shared memory,
// so HBM sees one coalesced read and one coalesced write per element.
template <int D, int NR>
__device__ __forceinline__ uint32_t philox_keys_fwd(uint32_t x, const uint32_t* k, int L, int R, uint32_t LM,
                                                    uint32_t RM, int rounds) {
  uint32_t s0 = x >> R, s1 = x & RM;
  if constexpr (NR > 0) {
#pragma unroll
    for (int i = 0; i < NR; ++i) philox_round<D>(s0, s1, k[i], L, LM, RM);
  } else {
    for (int i = 0; i < rounds; ++i) philox_round<D>(s0, s1, k[i], L, LM, RM);
  }
  return (s0 << R) | (s1 & RM);
}

// U counters in lock step (round-major), so the U independent dependency
// chains interleave instruction by instruction (ptxas keeps a counter-major
// sequence of unrolled rounds back to back, which stalls on every round).
#ifndef BSG_BATCHED_F64
#define BSG_BATCHED_F64 1  // batched kernel: the round's high product on the FP64 pipe (philox_round_f64)
#endif
template <int D, int NR, int U>
__device__ __forceinline__ void philox_keys_fwd_x(uint32_t (&x)[U], const uint32_t* k, int L, int R, uint32_t LM,
                                                  uint32_t RM, double hc = 0.0, double hk = 0.0) {
  uint32_t s0[U], s1[U];
#pragma unroll
  for (int u = 0; u < U; ++u) {
    s0[u] = x[u] >> R;
    s1[u] = x[u] & RM;
  }
#pragma unroll
  for (int i = 0; i < NR; ++i) {
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (BSG_BATCHED_F64) philox_round_f64<D>(s0[u], s1[u], k[i], L, LM, RM, hc, hk);
      else philox_round<D>(s0[u], s1[u], k[i], L, LM, RM);
    }
  }
#pragma unroll
  for (int u = 0; u < U; ++u) x[u] = (s0[u] << R) | (s1[u] & RM);
}

// Table form of the forward cipher for L == R <= 5 (m <= 1024: the C4 rows).  The round's product words depend
// only on the L-bit left half, so two 32-entry shared-memory tables hold them for every s0, and the state lives in
// ONE register: W = (half_h << 16) | (half_l << 2), the two halves alternating roles.
//   round A (s0 in the low half):  W ^= TA[s0] ^ KA_i,  TA[s0] = hi(s0) << 16 | (lo(s0) ^ s0) << 2
//   round B (s0 in the high half): W ^= TB[s0] ^ KB_i,  TB[s0] = (lo(s0) ^ s0) << 16 | hi(s0) << 2
// with hi/lo the reference's high/low product words masked to L bits (bijection.hpp:103-107) and
// KA_i = k_i << 16, KB_i = k_i << 2 (k_i masked to L bits).  Each XOR sets the new left half
// hi ^ k ^ s1 in the old right half's place and turns s0 into lo there: bit-exact by construction.  A round is
// one LDS (32 consecutive words: conflict-free) plus LOP3 (A: index mask) or SHF (B: W >> 14) plus one LOP3 --
// no IMAD, no DFMA, three issue slots instead of five.
template <int U>
__device__ __forceinline__ void philox_tab_fwd_x(uint32_t (&x)[U], const uint32_t* kk, const uint32_t* TA,
                                                 const uint32_t* TB, int R, uint32_t LM, uint32_t RM, int rounds) {
  uint32_t W[U];
#pragma unroll
  for (int u = 0; u < U; ++u) W[u] = ((x[u] & RM) << 16) | ((x[u] >> R) << 2);
  const uint32_t mA = LM << 2;
  // byte offsets into the tables: A indexes by W & (LM << 2) (one LOP3), B by W >> 14 (one SHF; the low half is
  // below 2^7, so bits 14-15 are zero)
  const char* ta = reinterpret_cast<const char*>(TA);
  const char* tb = reinterpret_cast<const char*>(TB);
  auto two = [&](int i) {  // rounds i (A) and i + 1 (B)
    const uint32_t ka = kk[i], kb = kk[i + 1];
#pragma unroll
    for (int u = 0; u < U; ++u) W[u] ^= *reinterpret_cast<const uint32_t*>(ta + (W[u] & mA)) ^ ka;
#pragma unroll
    for (int u = 0; u < U; ++u) W[u] ^= *reinterpret_cast<const uint32_t*>(tb + (W[u] >> 14)) ^ kb;
  };
  int i = 0;
  if (rounds == 24) {
#pragma unroll
    for (int j = 0; j < 24; j += 2) two(j);
    i = 24;
  } else {
    for (; i + 1 < rounds; i += 2) two(i);
  }
  if (i < rounds) {  // odd round count: a last A round leaves s0 in the high half
#pragma unroll
    for (int u = 0; u < U; ++u) {
      W[u] ^= *reinterpret_cast<const uint32_t*>(ta + (W[u] & mA)) ^ kk[i];
      x[u] = ((W[u] >> 16) << R) | ((W[u] >> 2) & RM);
    }
  } else {
#pragma unroll
    for (int u = 0; u < U; ++u) x[u] = (((W[u] >> 2) & LM) << R) | (W[u] >> 16);
  }
}

// Rows are double-buffered in shared memory: while shuffle b is evaluated, the
// row of the CTA's next shuffle streams in with cp.async and its round keys
// are derived by the first `rounds` threads, so neither the load latency nor
// the key schedule serialises with the cipher.  NT threads per row: small
// blocks give each thread many independent counters (ILP for the 24-round
// chains, whose keys sit in registers shared by all of them).
// row_mode: 1 = 16-byte cp.async chunks, 2 = 4-byte chunks, 0 = plain loads.
// C4 (8192 x 1024 u32, B200): the 24 round keys are read from shared memory each round (one broadcast LDS per
// round for the thread's 8 counters) so the registers go to the 8 interleaved chains; at 14 CTAs of 64 threads per
// SM (72 registers) ptxas keeps the chains interleaved: 60 -> 42 us (tools/run_vars.sh; keys in registers at 42
// registers forced ptxas to run the chains one after another, 69% `wait` stalls).
#ifndef BSG_BATCHED_MINB64
#define BSG_BATCHED_MINB64 14
#endif
template <int KIND, typename T, int NT>
__global__ void __launch_bounds__(NT, NT == 64 ? BSG_BATCHED_MINB64 : 1) k_batched(const T* __restrict__ in, T* __restrict__ out, uint64_t batch,
                                                      uint32_t m, uint64_t seed, BijParams p, int row_mode,
                                                      uint32_t row_stride_bytes) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ uint32_t s_keys[2][kBatchedMaxRounds];
  __shared__ uint32_t s_wcnt[2][(NT / 32)];
  constexpr bool kFast = (KIND == kKindPh0 || KIND == kKindPh1);
  constexpr int D = (KIND == kKindPh1 || KIND == kKindPh1G) ? 1 : 0;
#ifndef BSG_BATCHED_TAB
#define BSG_BATCHED_TAB 1
#endif
  // table form (philox_tab_fwd_x) for L == R <= 5; keys are then stored pre-shifted per round (KA / KB)
  constexpr bool kTabKind = BSG_BATCHED_TAB && (KIND == kKindPh0 || KIND == kKindPh0G);
  __shared__ uint32_t s_tab[kTabKind ? 64 : 1];
  const bool tab = kTabKind && p.L <= 5;
  if (tab) {
    for (int s0 = threadIdx.x; s0 < 32; s0 += NT) {
      const uint64_t prod = kM0 * static_cast<uint64_t>(s0);
      const uint32_t hi = static_cast<uint32_t>(prod >> 32) & p.LM, lo = static_cast<uint32_t>(prod) & p.LM;
      s_tab[s0] = (hi << 16) | ((lo ^ static_cast<uint32_t>(s0)) << 2);       // TA
      s_tab[32 + s0] = ((lo ^ static_cast<uint32_t>(s0)) << 16) | (hi << 2);  // TB
    }
  }
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t n = 1u << p.bits;
  const uint32_t mask32 = n - 1;
  const bool pow2 = (m == n);
  const uint32_t row_bytes = m * static_cast<uint32_t>(sizeof(T));

  auto row_ptr = [&](int buf) { return reinterpret_cast<T*>(smem_raw + buf * row_stride_bytes); };
  auto issue_row = [&](uint64_t b, int buf) {
    const unsigned char* src = reinterpret_cast<const unsigned char*>(in + b * m);
    unsigned char* dst = smem_raw + buf * row_stride_bytes;
    if (row_mode == 1) {
      for (uint32_t o = tid * 16; o < row_bytes; o += NT * 16) {
        const uint32_t d = static_cast<uint32_t>(__cvta_generic_to_shared(dst + o));
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(src + o) : "memory");
      }
    } else if (row_mode == 2) {
      for (uint32_t o = tid * 4; o < row_bytes; o += NT * 4) {
        const uint32_t d = static_cast<uint32_t>(__cvta_generic_to_shared(dst + o));
        asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(d), "l"(src + o) : "memory");
      }
    } else {
      T* r = reinterpret_cast<T*>(dst);
      for (uint32_t i = tid; i < m; i += NT) r[i] = in[b * m + i];
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  auto make_keys = [&](uint64_t b, int buf) {
    if (KIND != kKindLcg)
      for (int i = tid; i < p.rounds; i += NT) {
        const uint32_t k = round_key(seed + b, i);
        s_keys[buf][i] = tab ? (k & p.LM) << ((i & 1) ? 2 : 16) : k;
      }
  };

  int buf = 0;
  if (blockIdx.x < batch) {
    issue_row(blockIdx.x, 0);
    make_keys(blockIdx.x, 0);
  }
  for (uint64_t b = blockIdx.x; b < batch; b += gridDim.x, buf ^= 1) {
    const uint64_t nb = b + gridDim.x;
    if (nb < batch) {
      issue_row(nb, buf ^ 1);
      make_keys(nb, buf ^ 1);
      asm volatile("cp.async.wait_group 1;" ::: "memory");
    } else {
      asm volatile("cp.async.wait_group 0;" ::: "memory");
    }
    __syncthreads();
    const T* s_row = row_ptr(buf);
    const uint32_t* keys = s_keys[buf];
    T* row_out = out + b * m;
    const uint64_t sb = seed + b;
#ifndef BSG_BATCHED_REGKEYS
#define BSG_BATCHED_REGKEYS 0
#endif
    constexpr bool kRegKeys = kFast && BSG_BATCHED_REGKEYS;  // 24 keys held in registers, shared by all counters
    uint32_t kr[kRegKeys ? 24 : 1];
    if constexpr (kRegKeys) {
#pragma unroll
      for (int i = 0; i < 24; ++i) kr[i] = keys[i];
    }
    // LCG parameters of this shuffle (make_lcg, bijection.hpp:25-34)
    const uint32_t la = static_cast<uint32_t>((mix64(sb) | 1ULL)) & mask32;
    const uint32_t lc = static_cast<uint32_t>(mix64(sb + 1)) & mask32;
    auto f = [&](uint32_t c) -> uint32_t {
      if constexpr (kTabKind) {
        if (tab) {
          uint32_t y1[1] = {c};
          philox_tab_fwd_x<1>(y1, keys, s_tab, s_tab + 32, p.R, p.LM, p.RM, kFast ? 24 : p.rounds);
          return y1[0];
        }
      }
      if constexpr (KIND == kKindLcg) return (la * c + lc) & mask32;
      else if constexpr (kRegKeys) return philox_keys_fwd<D, 24>(c, kr, p.L, p.R, p.LM, p.RM, 24);
      else return philox_keys_fwd<D, 0>(c, keys, p.L, p.R, p.LM, p.RM, p.rounds);
    };
    if (pow2) {
      // BSG_BATCHED_ILP independent counters per thread in flight
#ifndef BSG_BATCHED_ILP
#define BSG_BATCHED_ILP 8
#endif
      constexpr int U = BSG_BATCHED_ILP;
      for (uint32_t c0 = tid; c0 < n; c0 += NT * U) {
        uint32_t y[U];  // counters past n are evaluated, never stored
        if (tab) {
#pragma unroll
          for (int u = 0; u < U; ++u) y[u] = c0 + u * NT;
          philox_tab_fwd_x<U>(y, keys, s_tab, s_tab + 32, p.R, p.LM, p.RM, kFast ? 24 : p.rounds);
        } else if constexpr (kRegKeys) {
#pragma unroll
          for (int u = 0; u < U; ++u) y[u] = c0 + u * NT;
          philox_keys_fwd_x<D, 24, U>(y, kr, p.L, p.R, p.LM, p.RM, p.hc, p.hk);
        } else if constexpr (kFast) {  // keys read from shared memory each round (broadcast), registers for chains
#pragma unroll
          for (int u = 0; u < U; ++u) y[u] = c0 + u * NT;
          philox_keys_fwd_x<D, 24, U>(y, keys, p.L, p.R, p.LM, p.RM, p.hc, p.hk);
        } else {
#pragma unroll
          for (int u = 0; u < U; ++u) y[u] = f(c0 + u * NT);
        }
#pragma unroll
        for (int u = 0; u < U; ++u)
          if (c0 + u * NT < n) st_out<T>(row_out + c0 + u * NT, s_row[y[u]]);
      }
    } else {
      uint32_t base = 0;
      int cb = 0;
      for (uint32_t c0 = 0; c0 < n; c0 += NT) {
        const uint32_t c = c0 + tid;
        const uint32_t y = f(c);
        const bool keep = (c < n) && (y < m);
        const uint32_t bm = __ballot_sync(0xFFFFFFFFu, keep);
        if (lane == 0) s_wcnt[cb][warp] = __popc(bm);
        __syncthreads();
        uint32_t before = 0, total = 0;
#pragma unroll
        for (int w = 0; w < (NT / 32); ++w) {
          const uint32_t x = s_wcnt[cb][w];
          before += (w < warp) ? x : 0;
          total += x;
        }
        if (keep) st_out<T>(row_out + base + before + __popc(bm & lanemask_lt()), s_row[y]);
        base += total;
        cb ^= 1;  // double-buffered counts: one barrier per chunk
      }
    }
    __syncthreads();  // buffer `buf` and its keys are refilled two iterations later
  }
}

// --------------------------------------------------------------------- gather
// out[i] = src[idx[i]] (shuffle.hpp:319-334, the paper's "Gather" bound).
template <typename T, int ITEMS>
__global__ void __launch_bounds__(kThreads) k_gather(const T* __restrict__ src, const uint64_t* __restrict__ idx,
                                                     T* __restrict__ out, uint64_t n) {
  const uint64_t t0 = static_cast<uint64_t>(blockIdx.x) * kThreads * ITEMS + threadIdx.x;
  uint64_t ix[ITEMS];
#pragma unroll
  for (int j = 0; j < ITEMS; ++j) {
    const uint64_t i = t0 + j * kThreads;
    ix[j] = i < n ? __ldcs(idx + i) : 0;
  }
  T v[ITEMS];
#pragma unroll
  for (int j = 0; j < ITEMS; ++j)
    if (t0 + j * kThreads < n) v[j] = ld_rand(src + ix[j]);
#pragma unroll
  for (int j = 0; j < ITEMS; ++j)
    if (t0 + j * kThreads < n) st_out<T>(out + t0 + j * kThreads, v[j]);
}

}  // namespace bsg
