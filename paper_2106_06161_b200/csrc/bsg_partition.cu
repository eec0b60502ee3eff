// bsg_partition.cu -- partitioned (three-pass) shuffle for large domains, the
// B200 answer to the DRAM random-access wall.
//
// Why: a single-pass shuffle of a 4 GiB array issues one random read per
// element; on B200 those saturate at ~47 G reads/s (DRAM row activations,
// independent of element size -- profiles/r01_microbench.md), i.e. 11.4 ms for
// 2^29 elements although 8.6 GB of payload would stream in 1.4 ms.  Every
// input j < m has exactly one counter c = f^-1(j) (philox_invert,
// bijection.hpp:117-143) and lands at the rank of c among the survivors; when
// m == 2^bits that rank is c itself.  So the permutation is applied by
// streaming the INPUT in order and routing each element by c:
//   P1  read in[] sequentially, inverse cipher -> c, counting-sort each
//       4096-element tile in shared memory into 2^s1 coarse counter buckets,
//       append the runs to the buckets (value + u32 c);
//   P2  per coarse bucket, the same split into 2^s2 fine windows of W2
//       counters (value + u16 offset in the window), written into `out`
//       itself (power of two) or into a counter-sized buffer (padded domain);
//   P3  per fine window (64 KiB), scatter into shared memory by offset and
//       write the window back coalesced: in place (power of two), or compacted
//       in counter order at the window's prefix of survivor counts (padded,
//       k_place_compact after the two-level k_window_scan/fix).
// Every DRAM access is a coalesced run; traffic is ~60 B/element instead of
// one random 64-B access per 8-B element.  P2 (and P1 for cheap bijections)
// run persistent with TMA bulk copies of the next tile in flight; P1 for the
// 24-round Philox is bound by the integer pipes (the cipher).  Bucket and
// window capacities are counter ranges, so the layout is static; atomic
// cursors only order elements inside a bucket, which the final placement by
// counter makes irrelevant -- the output is bit-identical to the single pass.
#include <cuda_runtime.h>

#include <algorithm>

#include "bsg_kernels.cuh"
#include "bsg_partition.h"

namespace bsg {

namespace {

// Tuning knobs (compile-time; defaults are the measured best, profiles/r01_microbench.md).
#ifndef BSG_P1_THREADS
#define BSG_P1_THREADS 256
#endif
// P1 occupancy and where the inverse cipher's high product runs, per split: D = R - L (1 for odd widths, C2).
// Measured on B200 (tools/ktime.py, 2^29 u64): D = 1 with the high product on the FP64 pipe at 2 CTAs/SM
// (104 registers) 3.67 ms against 3.97 ms for IMAD.HI at 3 CTAs/SM; D = 0 (C3) stays on IMAD.HI at 3 CTAs/SM
// (4.06 ms; the FP64 form there loses a CTA per SM and measured 4.47-4.58 ms).
#ifndef BSG_P1_MINB
#define BSG_P1_MINB 3
#endif
#ifndef BSG_P1_MINB_F64
#define BSG_P1_MINB_F64 2
#endif
#ifndef BSG_P1_F64
#define BSG_P1_F64 1  // D = 1 only
#endif
#ifndef BSG_P1_F64_D0
#define BSG_P1_F64_D0 0
#endif
template <int KIND, int D>
constexpr bool p1_f64() {
  return (KIND == kKindPh0 || KIND == kKindPh1 || KIND == kKindPh0G || KIND == kKindPh1G) &&
         (D ? BSG_P1_F64 != 0 : BSG_P1_F64_D0 != 0);
}
#ifndef BSG_RANK2
#define BSG_RANK2 1  // counting-sort ranks: count with RED, then a returning atomic on the scanned starts
#endif
#ifndef BSG_P2_THREADS
#define BSG_P2_THREADS 256
#endif
#ifndef BSG_P1_TILE
#define BSG_P1_TILE 4096
#endif
constexpr int kP1Threads = BSG_P1_THREADS, kP1Items = BSG_P1_TILE / BSG_P1_THREADS, kP1Tile = BSG_P1_TILE;
#ifndef BSG_P2_TILE
#define BSG_P2_TILE 4096
#endif
constexpr int kP2Threads = BSG_P2_THREADS, kP2Items = BSG_P2_TILE / BSG_P2_THREADS, kP2Tile = BSG_P2_TILE;
constexpr int kP2TileLog = __builtin_ctz(kP2Tile);  // coarse buckets must hold whole P2 tiles
constexpr int kP3Threads = 512;

constexpr int kMaxB1 = 512, kMaxB2 = 512;  // fan-outs: at most 2 bins per thread in the scans
// cursor region: P1 bucket cursors, then P2 window cursors
constexpr size_t kCursorWords = kMaxB1 + static_cast<size_t>(kMaxB1) * kMaxB2;

constexpr int kKindDestArray = 100;  // destinations come from an array (scatter by permutation)

template <int KIND, int D>
__device__ __forceinline__ uint32_t inv_bij(uint32_t y, const BijParams& p) {
  if constexpr (KIND == kKindLcg) return static_cast<uint32_t>(lcg_inv(y, p));
  // partitioned domains have bits <= 32 (L <= 16): the high product runs on the FP64 pipe
  else if constexpr (KIND == kKindPh0 || KIND == kKindPh1) return static_cast<uint32_t>(philox_inv_top<D, 24, p1_f64<KIND, D>()>(y, p));
  else return static_cast<uint32_t>(philox_inv_top<D, 0, p1_f64<KIND, D>()>(y, p));
}

// Block-wide exclusive scan of `nb` <= 2 * blockDim.x bin counts.
__device__ __forceinline__ void scan_bins(const uint32_t* hist, uint32_t* start, int nb, uint32_t* warp_tot) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int per = (nb + static_cast<int>(blockDim.x) - 1) / static_cast<int>(blockDim.x);  // 1 or 2
  uint32_t loc[2] = {0u, 0u}, sum = 0;
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    const int idx = tid * per + k;
    if (k < per && idx < nb) loc[k] = hist[idx];
    sum += loc[k];
  }
  uint32_t x = sum;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) warp_tot[warp] = x;
  __syncthreads();
  if (warp == 0) {
    const int nw = (blockDim.x + 31) >> 5;
    uint32_t w = lane < nw ? warp_tot[lane] : 0u, z = w;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, z, o);
      if (lane >= o) z += y;
    }
    if (lane < nw) warp_tot[lane] = z - w;
  }
  __syncthreads();
  uint32_t run = warp_tot[warp] + x - sum;
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    const int idx = tid * per + k;
    if (k < per && idx < nb) start[idx] = run;
    run += loc[k];
  }
  __syncthreads();  // start[] is read by other threads right after (two bins per thread when nb > blockDim)
}

// mbarrier + bulk-copy helpers (TMA-fed kernels below).
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(bar))),
               "r"(count)
               : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(
                   static_cast<uint32_t>(__cvta_generic_to_shared(bar))),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          static_cast<uint32_t>(__cvta_generic_to_shared(dst))),
      "l"(src), "r"(bytes), "r"(static_cast<uint32_t>(__cvta_generic_to_shared(bar)))
      : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  const uint32_t a = static_cast<uint32_t>(__cvta_generic_to_shared(bar));
  uint32_t done = 0;
  while (!done) {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}" : "=r"(done)
        : "r"(a), "r"(phase)
        : "memory");
  }
}

// Slot swizzle of the sorted tile buffers: slot r lives at r ^ ((r >> 5) & 31).  Runs of ranks that start at
// regular offsets (an LCG fills every bin of a tile almost exactly equally, so bin starts fall on multiples of 16)
// would otherwise put a warp's scatter stores into two banks (up to 9.6x the conflict-free wavefronts, ncu);
// 32 consecutive slots still map to 32 distinct banks, so the sequential write-back stays conflict-free.
__device__ __forceinline__ uint32_t swz(uint32_t r) { return r ^ ((r >> 5) & 31u); }

#ifndef BSG_SWZ1
#define BSG_SWZ1 1  // swizzled sorted buffers in the TMA-fed P1 (cheap bijections)
#endif
#ifndef BSG_SWZ2
#define BSG_SWZ2 0  // ... and in P2
#endif
#define SW1(r) (BSG_SWZ1 ? swz(r) : (r))
#define SW2(r) (BSG_SWZ2 ? swz(r) : (r))

// P1: stream the input, route by coarse destination bucket.
// PAD: non-power-of-two domain, only inputs j < mv exist (the last tile may be partial); tile0 offsets the
// tiles of a launch (the partial tail after k_part1t's full tiles).
template <int KIND, int D, typename T, bool PAD = false>
__global__ void __launch_bounds__(kP1Threads, sizeof(T) > 8 ? 2 : (p1_f64<KIND, D>() ? BSG_P1_MINB_F64 : BSG_P1_MINB))
    k_part1(const T* __restrict__ in, T* __restrict__ tv, uint32_t* __restrict__ td, uint32_t* __restrict__ cur1,
            BijParams p, int bshift, int nb, uint64_t w1, const uint32_t* __restrict__ dsrc, uint64_t mv = 0,
            uint32_t tile0 = 0) {
  extern __shared__ __align__(16) unsigned char smem[];
  T* sv = reinterpret_cast<T*>(smem);
  uint32_t* sd = reinterpret_cast<uint32_t*>(sv + kP1Tile);
  __shared__ uint32_t hist[kMaxB1], start[kMaxB1], wt[32];
  __shared__ uint32_t delta[kMaxB1];  // positions fit 32 bits: the partitioned path needs bits <= 32
  const int tid = threadIdx.x;
  for (int i = tid; i < nb; i += kP1Threads) hist[i] = 0;
  __syncthreads();
  const uint32_t base = (tile0 + blockIdx.x) * kP1Tile + tid;
  const uint64_t left = PAD ? mv - static_cast<uint64_t>(tile0 + blockIdx.x) * kP1Tile : kP1Tile;
  const uint32_t nvalid = left < kP1Tile ? static_cast<uint32_t>(left) : static_cast<uint32_t>(kP1Tile);
#ifndef BSG_P1_LATE_LOAD
#define BSG_P1_LATE_LOAD 1
#endif
  // Late loads (the 3-CTA/SM IMAD.HI form): the values stay out of registers during the cipher (80 registers) and
  // are loaded straight into their sorted slots after the scan.  The FP64-cipher form runs at 2 CTAs/SM anyway, so
  // it loads them first and their latency hides under the cipher (108 registers; C2 P1 3.71 -> 3.60 ms, shuffle
  // 7.59 -> 7.42 ms; the IMAD.HI form is neutral either way).
  constexpr bool kLate = BSG_P1_LATE_LOAD && !p1_f64<KIND, D>();
  T v[kLate ? 1 : kP1Items];
  auto valid = [&](int i) { return !PAD || tid + i * kP1Threads < static_cast<int>(nvalid); };
  if constexpr (!kLate) {
#pragma unroll
    for (int i = 0; i < kP1Items; ++i)
      if (valid(i)) v[i] = __ldcs(in + base + i * kP1Threads);
  }
  // two-atomic ranks (BSG_RANK2) except for the 2-CTA/SM FP64-cipher form, where the extra barrier costs more
  // than the start lookup it saves (C2 P1 4.02 vs 3.69 ms; C3 P1 3.56 vs 3.60 ms)
  constexpr bool kRank2 = BSG_RANK2 && !p1_f64<KIND, D>();
  uint32_t dst[kP1Items], rk[kP1Items];
#pragma unroll
  for (int i = 0; i < kP1Items; ++i) {
    if constexpr (KIND == kKindDestArray) dst[i] = __ldcs(dsrc + base + i * kP1Threads);
    else dst[i] = inv_bij<KIND, D>(base + i * kP1Threads, p);
    if (valid(i)) {
      if (kRank2) atomicAdd(&hist[dst[i] >> bshift], 1u);  // count only: RED, nothing to wait for
      else rk[i] = atomicAdd(&hist[dst[i] >> bshift], 1u);
    }
  }
  __syncthreads();
  // Cursor atomics (nb <= 2 * blockDim) are issued before the scan and consumed after the scatter (latency hidden).
  uint32_t g[2] = {0u, 0u};
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    const int i = tid + k * kP1Threads;
    if (i < nb && hist[i]) g[k] = atomicAdd(cur1 + i, hist[i]);
  }
  scan_bins(hist, start, nb, wt);
  if (kRank2) {
    // ranks from a second atomic on the scanned starts: one returning shared atomic per element instead of a
    // returning atomic plus a bank-conflicted start lookup
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      const int i = tid + k * kP1Threads;
      if (i < nb) delta[i] = static_cast<uint32_t>(i * w1) + g[k] - start[i];  // mod 2^32
    }
    __syncthreads();  // start[] read for delta before the rank atomics advance it
#pragma unroll
    for (int i = 0; i < kP1Items; ++i) {
      if (!valid(i)) continue;
      const uint32_t r = atomicAdd(&start[dst[i] >> bshift], 1u);
      if constexpr (kLate) sv[r] = __ldcs(in + base + i * kP1Threads);
      else sv[r] = v[i];
      sd[r] = dst[i];
    }
  } else {
#pragma unroll
    for (int i = 0; i < kP1Items; ++i) rk[i] += start[dst[i] >> bshift];
#pragma unroll
    for (int i = 0; i < kP1Items; ++i) {
      if (!valid(i)) continue;
      if constexpr (kLate) sv[rk[i]] = __ldcs(in + base + i * kP1Threads);
      else sv[rk[i]] = v[i];
      sd[rk[i]] = dst[i];
    }
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      // one table lookup per element in the write-back: global position = delta[b] + slot
      const int i = tid + k * kP1Threads;
      if (i < nb) delta[i] = static_cast<uint32_t>(i * w1) + g[k] - start[i];  // mod 2^32
    }
  }
  __syncthreads();
#pragma unroll 4
  for (int s = tid; s < static_cast<int>(nvalid); s += kP1Threads) {
    const uint32_t d = sd[s];
    const uint32_t pos = delta[d >> bshift] + s;
    __stcs(tv + pos, sv[s]);
    __stcs(td + pos, d);
  }
}

// P1, persistent and TMA-fed: the values of the next tile stream into a
// staging buffer (one bulk copy, mbarrier completion) while the current tile's
// destinations are computed, so the scatter reads them from shared memory
// instead of issuing the DRAM loads after the scan.
template <int KIND, int D, typename T>
__global__ void __launch_bounds__(kP1Threads) k_part1t(const T* __restrict__ in, T* __restrict__ tv,
                                                       uint32_t* __restrict__ td, uint32_t* __restrict__ cur1,
                                                       BijParams p, int bshift, int nb, uint64_t w1,
                                                       const uint32_t* __restrict__ dsrc, uint32_t ntiles) {
  extern __shared__ __align__(16) unsigned char smem[];
  T* gv = reinterpret_cast<T*>(smem);                    // staging: values of the tile in flight
  T* sv = gv + kP1Tile;                                  // sorted values
  uint32_t* sd = reinterpret_cast<uint32_t*>(sv + kP1Tile);  // sorted destinations
  __shared__ uint32_t hist[kMaxB1], start[kMaxB1], wt[32];
  __shared__ uint32_t delta[kMaxB1];
  __shared__ __align__(8) uint64_t bar;
  const int tid = threadIdx.x;
  if (tid == 0) {
    mbar_init(&bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  for (int i = tid; i < nb; i += kP1Threads) hist[i] = 0;
  __syncthreads();
  auto issue = [&](uint32_t t) {
    mbar_expect_tx(&bar, kP1Tile * sizeof(T));
    bulk_g2s(gv, in + static_cast<uint64_t>(t) * kP1Tile, kP1Tile * sizeof(T), &bar);
  };
  if (tid == 0 && blockIdx.x < ntiles) issue(blockIdx.x);
  uint32_t phase = 0;
#ifndef BSG_P1T_EARLY
#define BSG_P1T_EARLY 1
#endif
  // EARLY: the tile's values are copied to registers as soon as they land and the staging buffer is refilled at
  // once, so the next tile's load has a whole tile time to arrive (else it is issued after the scatter).
  for (uint32_t t = blockIdx.x; t < ntiles; t += gridDim.x, phase ^= 1) {
    const uint32_t base = t * kP1Tile + tid;
    T v[BSG_P1T_EARLY ? kP1Items : 1];
    if constexpr (BSG_P1T_EARLY) {
      mbar_wait(&bar, phase);
#pragma unroll
      for (int i = 0; i < kP1Items; ++i) v[i] = gv[tid + i * kP1Threads];
      __syncthreads();  // staging consumed
      if (tid == 0 && t + gridDim.x < ntiles) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        issue(t + gridDim.x);
      }
    }
    uint32_t dst[kP1Items], rk[kP1Items];
#pragma unroll
    for (int i = 0; i < kP1Items; ++i) {
      if constexpr (KIND == kKindDestArray) dst[i] = __ldcs(dsrc + base + i * kP1Threads);
      else dst[i] = inv_bij<KIND, D>(base + i * kP1Threads, p);
      if (BSG_RANK2) atomicAdd(&hist[dst[i] >> bshift], 1u);
      else rk[i] = atomicAdd(&hist[dst[i] >> bshift], 1u);
    }
    __syncthreads();
    uint32_t g[2] = {0u, 0u};
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      const int i = tid + k * kP1Threads;
      if (i < nb && hist[i]) g[k] = atomicAdd(cur1 + i, hist[i]);
    }
    scan_bins(hist, start, nb, wt);
    if (BSG_RANK2) {
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        const int i = tid + k * kP1Threads;
        if (i < nb) {
          delta[i] = static_cast<uint32_t>(i * w1) + g[k] - start[i];  // mod 2^32
          hist[i] = 0;                                                  // next tile
        }
      }
      __syncthreads();  // start[] read for delta before the rank atomics advance it
      if (!BSG_P1T_EARLY) mbar_wait(&bar, phase);  // this tile's values have landed
#pragma unroll
      for (int i = 0; i < kP1Items; ++i) {
        const uint32_t r = SW1(atomicAdd(&start[dst[i] >> bshift], 1u));
        if constexpr (BSG_P1T_EARLY) sv[r] = v[i];
        else sv[r] = gv[tid + i * kP1Threads];
        sd[r] = dst[i];
      }
    } else {
#pragma unroll
      for (int i = 0; i < kP1Items; ++i) rk[i] += start[dst[i] >> bshift];
      if (!BSG_P1T_EARLY) mbar_wait(&bar, phase);  // this tile's values have landed
#pragma unroll
      for (int i = 0; i < kP1Items; ++i) {
        if constexpr (BSG_P1T_EARLY) sv[SW1(rk[i])] = v[i];
        else sv[SW1(rk[i])] = gv[tid + i * kP1Threads];
        sd[SW1(rk[i])] = dst[i];
      }
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        const int i = tid + k * kP1Threads;
        if (i < nb) {
          delta[i] = static_cast<uint32_t>(i * w1) + g[k] - start[i];  // mod 2^32
          hist[i] = 0;                                                  // next tile
        }
      }
    }
    __syncthreads();  // staging consumed; sorted tile and delta complete
    if (!BSG_P1T_EARLY && tid == 0 && t + gridDim.x < ntiles) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      issue(t + gridDim.x);
    }
#pragma unroll 4
    for (int s = tid; s < kP1Tile; s += kP1Threads) {
      const uint32_t d = sd[SW1(s)];
      const uint32_t pos = delta[d >> bshift] + s;
      __stcs(tv + pos, sv[SW1(s)]);
      __stcs(td + pos, d);
    }
    __syncthreads();  // sorted buffers, delta and start reused by the next tile
  }
}

// P2: split each coarse bucket into fine windows of 2^w2 elements (one tile per CTA; used for 16-byte records,
// whose staging would not fit twice next to the sorted tile -- k_part2t below is the default).
template <typename T>
__global__ void __launch_bounds__(kP2Threads, sizeof(T) <= 8 ? 3 : 2)
    k_part2(const T* __restrict__ tv, const uint32_t* __restrict__ td, T* __restrict__ ov, uint16_t* __restrict__ od,
            uint32_t* __restrict__ cur2, int w2, int nb2, uint64_t w1) {
  extern __shared__ __align__(16) unsigned char smem[];
  T* sv = reinterpret_cast<T*>(smem);
  uint32_t* sd = reinterpret_cast<uint32_t*>(sv + kP2Tile);
  __shared__ uint32_t hist[kMaxB2], start[kMaxB2], wt[32];
  __shared__ uint32_t delta[kMaxB2];
  const int tid = threadIdx.x;
  if (tid < nb2) hist[tid] = 0;
  if (tid + kP2Threads < nb2) hist[tid + kP2Threads] = 0;  // nb2 <= 2 * kP2Threads
  __syncthreads();
  const uint64_t t0 = static_cast<uint64_t>(blockIdx.x) * kP2Tile;
  const uint64_t coarse = t0 / w1;
  const uint32_t fmask = static_cast<uint32_t>(nb2 - 1), wmask = (1u << w2) - 1;
  T v[kP2Items];
  uint32_t d[kP2Items], rk[kP2Items];
#pragma unroll
  for (int i = 0; i < kP2Items; ++i) {
    v[i] = __ldcs(tv + t0 + tid + i * kP2Threads);
    d[i] = __ldcs(td + t0 + tid + i * kP2Threads);
  }
#pragma unroll
  for (int i = 0; i < kP2Items; ++i) rk[i] = atomicAdd(&hist[(d[i] >> w2) & fmask], 1u);
  __syncthreads();
  scan_bins(hist, start, nb2, wt);
  uint32_t* cur = cur2 + coarse * nb2;
  const uint64_t win0 = coarse * w1;  // first element of this coarse bucket's output range
  if (tid < nb2)
    delta[tid] = static_cast<uint32_t>(win0 + (static_cast<uint64_t>(tid) << w2)) + atomicAdd(cur + tid, hist[tid]) -
                 start[tid];
  if (tid + kP2Threads < nb2) {  // fan-outs above kP2Threads (16-byte payloads at 2^30)
    const int i = tid + kP2Threads;
    delta[i] = static_cast<uint32_t>(win0 + (static_cast<uint64_t>(i) << w2)) + atomicAdd(cur + i, hist[i]) - start[i];
  }
  __syncthreads();
#pragma unroll
  for (int i = 0; i < kP2Items; ++i) {
    const uint32_t s = start[(d[i] >> w2) & fmask] + rk[i];
    sv[s] = v[i];
    sd[s] = d[i];
  }
  __syncthreads();
#pragma unroll 4
  for (int s = tid; s < kP2Tile; s += kP2Threads) {
    const uint32_t dd = sd[s];
    const uint32_t pos = delta[(dd >> w2) & fmask] + s;
    ov[pos] = sv[s];
    od[pos] = static_cast<uint16_t>(dd & wmask);
  }
}

// P2, persistent and TMA-fed: each CTA walks tiles t, t + G, ...; while
// tile t is ranked, scattered and written back, the next tile's values and
// destinations stream into a staging buffer with two bulk copies
// (cp.async.bulk, completion on an mbarrier), so the DRAM latency of the
// loads leaves the per-tile critical path.
// cnt1 != nullptr (non-power-of-two domains): coarse bucket b holds cnt1[b] <= w1 elements, so tile k of the
// bucket is partial or empty; empty tiles are skipped before their loads are issued.
// PAD = false (power-of-two domains): every tile is full, so the per-element bounds checks compile away.
#ifndef BSG_P2_FULLT
#define BSG_P2_FULLT 1
#endif
template <typename T, int TILE = kP2Tile, bool PAD = true>
__global__ void __launch_bounds__(kP2Threads) k_part2t(const T* __restrict__ tv, const uint32_t* __restrict__ td,
                                                       T* __restrict__ ov, uint16_t* __restrict__ od,
                                                       uint32_t* __restrict__ cur2, int w2, int nb2, uint64_t w1,
                                                       uint32_t ntiles, const uint32_t* __restrict__ cnt1) {
  constexpr int kItems = TILE / kP2Threads, kTileLog = __builtin_ctz(TILE);
  extern __shared__ __align__(16) unsigned char smem[];
  T* gv = reinterpret_cast<T*>(smem);                    // staging: values of the next tile
  uint32_t* gd = reinterpret_cast<uint32_t*>(gv + TILE);  // staging: destinations
  T* sv = reinterpret_cast<T*>(gd + TILE);            // sorted values
  uint32_t* sd = reinterpret_cast<uint32_t*>(sv + TILE);  // sorted destinations
  __shared__ uint32_t hist[kMaxB2], start[kMaxB2], wt[32];
  __shared__ uint32_t delta[kMaxB2];
  __shared__ __align__(8) uint64_t bar;
  const int tid = threadIdx.x;
  const uint32_t fmask = static_cast<uint32_t>(nb2 - 1), wmask = (1u << w2) - 1;
  if (tid == 0) {
    mbar_init(&bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (tid < nb2) hist[tid] = 0;
  if (tid + kP2Threads < nb2) hist[tid + kP2Threads] = 0;
  __syncthreads();
  auto issue = [&](uint32_t t) {
    const uint64_t e0 = static_cast<uint64_t>(t) * TILE;
    mbar_expect_tx(&bar, TILE * (sizeof(T) + 4));
    bulk_g2s(gv, tv + e0, TILE * sizeof(T), &bar);
    bulk_g2s(gd, td + e0, TILE * 4, &bar);
  };
  // w1 (coarse bucket capacity) is a power of two >= TILE: shifts, not 64-bit divisions
  const int w1log = 63 - __clzll(static_cast<long long>(w1));
  const int tpblog = w1log - kTileLog;  // log2(tile slots per coarse bucket)
  auto fill = [&](uint32_t t) -> uint32_t {  // valid elements of tile t (0: empty)
    if (!cnt1) return TILE;
    const uint32_t c = cnt1[t >> tpblog], k0 = (t & ((1u << tpblog) - 1)) * TILE;
    return c > k0 ? min(c - k0, static_cast<uint32_t>(TILE)) : 0u;
  };
  auto next = [&](uint32_t t) {
    while (t < ntiles && fill(t) == 0) t += gridDim.x;
    return t;
  };
  uint32_t phase = 0;
  uint32_t t = next(blockIdx.x);
  if (tid == 0 && t < ntiles) issue(t);
  for (; t < ntiles; phase ^= 1) {
    mbar_wait(&bar, phase);
    const uint32_t nv = PAD ? fill(t) : static_cast<uint32_t>(TILE), tn = next(t + gridDim.x);
    const uint64_t coarse = t >> tpblog;
    uint32_t d[kItems], rk[kItems];
#ifndef BSG_P2T_EARLY
#define BSG_P2T_EARLY 1
#endif
    // EARLY: the tile is copied to registers at once, so the staging buffer refills while this tile is ranked,
    // scanned, scattered and written (the whole tile time hides the next load).
    T v[BSG_P2T_EARLY ? kItems : 1];
#pragma unroll
    for (int i = 0; i < kItems; ++i) {
      d[i] = gd[tid + i * kP2Threads];
      if constexpr (BSG_P2T_EARLY) v[i] = gv[tid + i * kP2Threads];
    }
    if constexpr (BSG_P2T_EARLY) {
      __syncthreads();
      if (tid == 0 && tn < ntiles) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic reads of staging before the refill
        issue(tn);
      }
    }
#pragma unroll
    for (int i = 0; i < kItems; ++i)
      if (!PAD || tid + i * kP2Threads < static_cast<int>(nv)) {
        if (BSG_RANK2) atomicAdd(&hist[(d[i] >> w2) & fmask], 1u);
        else rk[i] = atomicAdd(&hist[(d[i] >> w2) & fmask], 1u);
      }
    __syncthreads();
    // The window-cursor atomics (global, one per window with elements) are issued before the scan and consumed
    // after the scatter, so their L2 round trip overlaps both (it was 9% of P2's stall samples when consumed
    // right away).
    uint32_t* cur = cur2 + coarse * nb2;
    uint32_t g[2] = {0u, 0u};
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      const int q = tid + k * kP2Threads;
      if (q < nb2 && hist[q]) g[k] = atomicAdd(cur + q, hist[q]);
    }
    scan_bins(hist, start, nb2, wt);
    const uint32_t win0 = static_cast<uint32_t>(coarse << w1log);  // positions fit 32 bits (bits <= 32)
    if (BSG_RANK2) {
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        const int q = tid + k * kP2Threads;
        if (q < nb2) delta[q] = win0 + (static_cast<uint32_t>(q) << w2) + g[k] - start[q];
      }
      __syncthreads();  // start[] read for delta before the rank atomics advance it
#pragma unroll
      for (int i = 0; i < kItems; ++i) {
        if (PAD && tid + i * kP2Threads >= static_cast<int>(nv)) continue;
        const uint32_t s = SW2(atomicAdd(&start[(d[i] >> w2) & fmask], 1u));
        if constexpr (BSG_P2T_EARLY) sv[s] = v[i];
        else sv[s] = gv[tid + i * kP2Threads];
        sd[s] = d[i];
      }
    } else {
#pragma unroll
      for (int i = 0; i < kItems; ++i) {
        if (PAD && tid + i * kP2Threads >= static_cast<int>(nv)) continue;
        const uint32_t s = SW2(start[(d[i] >> w2) & fmask] + rk[i]);
        if constexpr (BSG_P2T_EARLY) sv[s] = v[i];
        else sv[s] = gv[tid + i * kP2Threads];
        sd[s] = d[i];
      }
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        const int q = tid + k * kP2Threads;
        if (q < nb2) delta[q] = win0 + (static_cast<uint32_t>(q) << w2) + g[k] - start[q];
      }
    }
    __syncthreads();  // staging consumed, sorted tile complete, delta ready
    if (tid < nb2) hist[tid] = 0;
    if (tid + kP2Threads < nb2) hist[tid + kP2Threads] = 0;
    if (!BSG_P2T_EARLY && tid == 0 && tn < ntiles) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic reads of staging before the refill
      issue(tn);
    }
#pragma unroll 4
    for (int s = tid; s < static_cast<int>(nv); s += kP2Threads) {
      const uint32_t dd = sd[SW2(s)];
      const uint32_t pos = delta[(dd >> w2) & fmask] + s;
#ifndef BSG_P2_CS
#define BSG_P2_CS 1  // streaming (evict-first) stores of the fine windows: C2 P2 2.424 -> 2.411 ms, C3 2.605 -> 2.592
#endif
      if (BSG_P2_CS) {
        __stcs(ov + pos, sv[SW2(s)]);
        __stcs(reinterpret_cast<unsigned short*>(od) + pos, static_cast<unsigned short>(dd & wmask));
      } else {
        ov[pos] = sv[SW2(s)];
        od[pos] = static_cast<uint16_t>(dd & wmask);
      }
    }
    __syncthreads();  // sorted buffers and delta reused by the next tile
    t = tn;
  }
}

// Bulk shared -> global store (TMA engine; bulk-group completion).
__device__ __forceinline__ void bulk_s2g(void* dst, const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst),
               "r"(static_cast<uint32_t>(__cvta_generic_to_shared(src))), "r"(bytes)
               : "memory");
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_read() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

// P3: place each fine window through shared memory, in place in `out`.
template <typename T>
__global__ void __launch_bounds__(kP3Threads) k_place(T* __restrict__ out, uint16_t* __restrict__ od, int w2,
                                                      int bulk, uint32_t w0 = 0) {
  extern __shared__ __align__(16) unsigned char smem[];
  T* win = reinterpret_cast<T*>(smem);
  const uint32_t W = 1u << w2;
  T* o = out + (static_cast<uint64_t>(w0 + blockIdx.x) << w2);  // w0: first window of a staged chunk
  const uint16_t* dd = od + (static_cast<uint64_t>(w0 + blockIdx.x) << w2);
  constexpr int kU = 8;
  for (uint32_t i0 = threadIdx.x; i0 < W; i0 += kP3Threads * kU) {
    T v[kU];
    uint16_t d[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const uint32_t i = i0 + u * kP3Threads;
      if (i < W) {
        v[u] = __ldcs(o + i);
        d[u] = __ldcs(reinterpret_cast<const unsigned short*>(dd) + i);
      }
    }
#pragma unroll
    for (int u = 0; u < kU; ++u)
      if (i0 + u * kP3Threads < W) win[d[u]] = v[u];
  }
  if (bulk && (reinterpret_cast<uintptr_t>(o) & 15u) == 0) {  // the window leaves by one bulk store (TMA engine)
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (threadIdx.x == 0) {
      bulk_s2g(o, win, W * static_cast<uint32_t>(sizeof(T)));
      bulk_wait_read();
    }
    return;
  }
  __syncthreads();
  for (uint32_t i = threadIdx.x; i < W; i += kP3Threads) __stcs(o + i, win[i]);
}

// Non-power-of-two P3: window w covers counters [w * 2^w2, (w+1) * 2^w2) and holds
// cnt[w] <= 2^w2 elements (the inputs j < m whose counter f^-1(j) falls in it).
// Output positions are counter ranks among the survivors: pre[w] (exclusive
// prefix of the window counts) plus the rank of the counter inside the window,
// i.e. the window is placed by counter offset in shared memory with one flag
// byte per slot, each warp ballots its slots in counter order and writes the
// survivors as contiguous runs -- the same order chained_compact produces
// (shuffle.hpp:91-147).
template <typename T>
__global__ void __launch_bounds__(kP3Threads) k_place_compact(const T* __restrict__ tv2,
                                                              const uint16_t* __restrict__ od,
                                                              const uint32_t* __restrict__ cnt,
                                                              const uint32_t* __restrict__ pre, int w2,
                                                              T* __restrict__ out) {
  extern __shared__ __align__(16) unsigned char smem[];
  const uint32_t W = 1u << w2, w = blockIdx.x, tid = threadIdx.x;  // W * sizeof(T) == 64 KiB
  T* win = reinterpret_cast<T*>(smem);
  uint8_t* occ = smem + W * sizeof(T);  // one flag byte per slot: plain stores, no atomics
  __shared__ uint32_t wt[kP3Threads / 32];
  const uint32_t c = cnt[w];
  for (uint32_t i = tid; i < W / 16; i += kP3Threads) reinterpret_cast<uint4*>(occ)[i] = make_uint4(0, 0, 0, 0);
  __syncthreads();
  const T* src = tv2 + (static_cast<uint64_t>(w) << w2);
  const uint16_t* dd = od + (static_cast<uint64_t>(w) << w2);
  constexpr int kU = 8;
  for (uint32_t i0 = tid; i0 < c; i0 += kP3Threads * kU) {
    T v[kU];
    uint32_t slot[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const uint32_t i = i0 + u * kP3Threads;
      if (i < c) {
        slot[u] = __ldcs(reinterpret_cast<const unsigned short*>(dd) + i);
        v[u] = __ldcs(src + i);
      }
    }
#pragma unroll
    for (int u = 0; u < kU; ++u)
      if (i0 + u * kP3Threads < c) {
        win[slot[u]] = v[u];
        occ[slot[u]] = 1;
      }
  }
  __syncthreads();
  // Warp q owns slots [q * 32 * kPer, (q + 1) * 32 * kPer), read lane-interleaved (conflict-free): chunk k of the
  // warp is slots base + 32k + lane, so (warp, chunk, lane) order is counter order.
  constexpr int kPer = (65536 / static_cast<int>(sizeof(T))) / kP3Threads;  // 16 for u64, 32 for u32
  const uint32_t lane = tid & 31, warp = tid >> 5, wbase = warp * 32 * kPer;
  const uint32_t lt = (1u << lane) - 1u;
  T v[kPer];
  uint32_t mk[kPer], nk = 0;
#pragma unroll
  for (int k = 0; k < kPer; ++k) {
    const uint32_t slot = wbase + 32 * k + lane;
    const bool f = occ[slot] != 0;
    if (f) v[k] = win[slot];
    mk[k] = __ballot_sync(0xFFFFFFFFu, f);
    nk += __popc(mk[k]);
  }
  if (lane == 0) wt[warp] = nk;
  __syncthreads();
  // survivors of chunk k go out as one contiguous run (counter order), straight from registers
  uint32_t pos = pre[w];
  for (uint32_t q = 0; q < warp; ++q) pos += wt[q];
#pragma unroll
  for (int k = 0; k < kPer; ++k) {
    if ((mk[k] >> lane) & 1u) __stcs(out + pos + __popc(mk[k] & lt), v[k]);
    pos += __popc(mk[k]);
  }
}

// Non-power-of-two last pass, placement by RANK (default).  Window w covers counters [w * 2^14, (w+1) * 2^14)
// and holds cnt[w] survivors (about half: their counter offsets in od, their values in tv2).  A bitmask of the
// occupied counter slots (one atomicOr per survivor), its per-word exclusive popcount prefix and one popc give
// every survivor its rank among the window's survivors -- its output position minus pre[w], i.e. the counter
// order chained_compact produces (shuffle.hpp:91-147).  Values are placed by rank in a dense shared buffer and
// written back as one contiguous run.  Against k_place_compact (placement by counter slot, flag bytes, ballots
// over all 8192 slots of a 64 KiB window) this moves twice the survivors per CTA through the same shared memory
// and drops the ballot pass.  A window with more than kRankCap survivors (mean 8192, sd 64 for a random
// bijection; possible for structured ones such as an LCG) is placed in several rounds of kRankCap ranks.
constexpr int kRankW2 = 14;                    // counters per window (log2)
constexpr uint32_t kRankWords = 1u << (kRankW2 - 5);  // bitmask words per window (== kP3Threads)
constexpr uint32_t kRankCap = 8704;            // survivors placed per round (8192 + 8 sd)
static_assert(kRankWords == kP3Threads, "one bitmask word per thread in the scan");

template <typename T>
__device__ __forceinline__ void load8(const T* p, T (&v)[8]) {  // 8 consecutive elements, 16-byte vector loads
  static_assert(sizeof(T) == 4 || sizeof(T) == 8, "u32 / u64 payloads");
  const uint4* q = reinterpret_cast<const uint4*>(p);
#pragma unroll
  for (int k = 0; k < static_cast<int>(sizeof(T)) * 8 / 16; ++k) {
    const uint4 x = __ldcs(q + k);
    reinterpret_cast<uint4*>(v)[k] = x;
  }
}

#ifndef BSG_RANK_REG_ROUNDS
#define BSG_RANK_REG_ROUNDS 2  // survivor rounds (4096 each) whose values stay in registers between the passes
#endif
template <typename T>
__device__ __forceinline__ void place_rank_window(const T* __restrict__ tv2, const uint16_t* __restrict__ od,
                                                  const uint32_t* __restrict__ cnt, const uint32_t* __restrict__ pre,
                                                  T* __restrict__ out, const uint32_t w) {
  constexpr int kRR = BSG_RANK_REG_ROUNDS;
  extern __shared__ __align__(16) unsigned char smem[];
  T* win = reinterpret_cast<T*>(smem);                                // kRankCap survivors by rank
  uint2* wp = reinterpret_cast<uint2*>(win + kRankCap);               // {occupancy word, exclusive prefix}
  uint32_t* occ = reinterpret_cast<uint32_t*>(wp + kRankWords);      // occupancy bitmask
  __shared__ uint32_t wt[kP3Threads / 32];
  const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t c = cnt[w], c8 = c & ~7u;
  const T* src = tv2 + (static_cast<uint64_t>(w) << kRankW2);
  const uint16_t* dd = od + (static_cast<uint64_t>(w) << kRankW2);
  occ[tid] = 0;
  // Thread t owns survivors [8t, 8t + 8) of each round of 4096 (16-byte loads of offsets and values).  The first
  // kRR rounds are loaded once, before the occupancy atomics, and stay in registers until they are placed, so the
  // DRAM latency of the values overlaps the bitmask build and its scan.
  uint4 sreg[kRR];
  T vreg[kRR][8];
#pragma unroll
  for (int r = 0; r < kRR; ++r) {
    const uint32_t i0 = 8 * tid + r * 8 * kP3Threads;
    if (i0 < c8) {
      sreg[r] = *reinterpret_cast<const uint4*>(dd + i0);
      load8(src + i0, vreg[r]);
    }
  }
  __syncthreads();  // occ cleared
  auto mark4 = [&](const uint4& s4) {
    const uint32_t sw[4] = {s4.x, s4.y, s4.z, s4.w};
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      atomicOr(&occ[(sw[k] & 0xFFFFu) >> 5], 1u << (sw[k] & 31u));
      atomicOr(&occ[sw[k] >> 21], 1u << ((sw[k] >> 16) & 31u));
    }
  };
#pragma unroll
  for (int r = 0; r < kRR; ++r)
    if (8 * tid + r * 8 * kP3Threads < c8) mark4(sreg[r]);
  for (uint32_t i0 = 8 * tid + kRR * 8 * kP3Threads; i0 < c8; i0 += 8 * kP3Threads)
    mark4(*reinterpret_cast<const uint4*>(dd + i0));
  if (c8 + tid < c) {
    const uint32_t s = dd[c8 + tid];
    atomicOr(&occ[s >> 5], 1u << (s & 31u));
  }
  __syncthreads();
  // exclusive prefix of the word popcounts (one word per thread)
  const uint32_t word = occ[tid], pc = __popc(word);
  uint32_t x = pc;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, x, o);
    if (lane >= static_cast<uint32_t>(o)) x += y;
  }
  if (lane == 31) wt[warp] = x;
  __syncthreads();
  if (warp == 0) {
    const uint32_t t = lane < kP3Threads / 32 ? wt[lane] : 0u;
    uint32_t z = t;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, z, o);
      if (lane >= static_cast<uint32_t>(o)) z += y;
    }
    if (lane < kP3Threads / 32) wt[lane] = z - t;
  }
  __syncthreads();
  wp[tid] = make_uint2(word, wt[warp] + x - pc);
  __syncthreads();
  const uint32_t o0 = pre[w];
  for (uint32_t base = 0; base < c; base += kRankCap) {
    auto place = [&](uint32_t s, const T& v) {
      const uint2 q = wp[s >> 5];
      const uint32_t r = q.y + __popc(q.x & ((1u << (s & 31u)) - 1u)) - base;
      if (r < kRankCap) win[r] = v;
    };
    auto place8 = [&](const uint4& s4, const T (&v)[8]) {
      const uint32_t sw[4] = {s4.x, s4.y, s4.z, s4.w};
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        place(sw[k] & 0xFFFFu, v[2 * k]);
        place(sw[k] >> 16, v[2 * k + 1]);
      }
    };
#pragma unroll
    for (int r = 0; r < kRR; ++r)
      if (8 * tid + r * 8 * kP3Threads < c8) place8(sreg[r], vreg[r]);
    for (uint32_t i0 = 8 * tid + kRR * 8 * kP3Threads; i0 < c8; i0 += 8 * kP3Threads) {
      T v[8];
      load8(src + i0, v);
      place8(*reinterpret_cast<const uint4*>(dd + i0), v);
    }
    if (c8 + tid < c) place(dd[c8 + tid], src[c8 + tid]);
    __syncthreads();
    const uint32_t n = min(kRankCap, c - base);
    T* o = out + o0 + base;
    for (uint32_t i = tid; i < n; i += kP3Threads) __stcs(o + i, win[i]);
    __syncthreads();
  }
}

// One window per CTA (list == nullptr), or the *nlist windows of list[] (the windows k_place_rank_t leaves over)
// walked by a small grid.
template <typename T>
__global__ void __launch_bounds__(kP3Threads, BSG_RANK_REG_ROUNDS >= 2 ? 2 : 3)
    k_place_rank(const T* __restrict__ tv2, const uint16_t* __restrict__ od, const uint32_t* __restrict__ cnt,
                 const uint32_t* __restrict__ pre, T* __restrict__ out, const uint32_t* __restrict__ list,
                 const uint32_t* __restrict__ nlist) {
  if (!list) {
    place_rank_window<T>(tv2, od, cnt, pre, out, blockIdx.x);
    return;
  }
  const uint32_t nw = *nlist;
  for (uint32_t item = blockIdx.x; item < nw; item += gridDim.x) place_rank_window<T>(tv2, od, cnt, pre, out, list[item]);
}

// Non-power-of-two last pass, persistent and TMA-fed (default).  The same placement by rank as k_place_rank, but
// one 1024-thread CTA per SM walks windows w, w + G, ...: window w's survivors (values and counter offsets) arrive
// in a staging buffer by two bulk copies on an mbarrier, are read into registers, and the staging buffer at once
// receives window w + G, so DRAM reads stay in flight while w is marked, scanned and placed.  The placed run goes
// out by one bulk shared -> global copy (its unaligned head and tail by plain stores) that drains while the next
// window is ranked.  Windows with more than kRTCap survivors (possible for structured bijections) are appended to
// list[] for k_place_rank.
constexpr int kRTThreads = 1024;
constexpr uint32_t kRTCap = 9216;  // survivors staged per window: 9 per thread (mean 8192, sd 64 for Philox)
constexpr int kRTItems = kRTCap / kRTThreads;
}  // namespace
uint32_t g_rank_stage_cap = kRTCap;
int g_bulk_stores = 1;
int set_bulk_stores(int on) {
  const int old = g_bulk_stores;
  g_bulk_stores = on ? 1 : 0;
  return old;
}
uint32_t set_rank_stage_cap(uint32_t cap) {
  const uint32_t old = g_rank_stage_cap;
  g_rank_stage_cap = std::min(cap, kRTCap);
  return old;
}
namespace {

template <typename T>
constexpr size_t place_rank_t_smem() {
  return kRTCap * sizeof(T) + kRTCap * 2 + (kRTCap + 16 / sizeof(T)) * sizeof(T) + kRankWords * 12;
}

template <typename T>
__global__ void __launch_bounds__(kRTThreads, 1)
    k_place_rank_t(const T* __restrict__ tv2, const uint16_t* __restrict__ od, const uint32_t* __restrict__ cnt,
                   const uint32_t* __restrict__ pre, T* __restrict__ out, uint32_t nwin, uint32_t* __restrict__ list,
                   uint32_t* __restrict__ nlist, uint32_t cap, int bulk) {
  constexpr uint32_t E = 16 / sizeof(T);  // elements per 16 bytes
  extern __shared__ __align__(16) unsigned char smem[];
  T* xv = reinterpret_cast<T*>(smem);                          // staged values
  uint16_t* xo = reinterpret_cast<uint16_t*>(xv + kRTCap);     // staged counter offsets
  T* y = reinterpret_cast<T*>(xo + kRTCap);                    // survivors by rank (+ alignment shift)
  uint2* wp = reinterpret_cast<uint2*>(y + kRTCap + E);        // {occupancy word, exclusive prefix}
  uint32_t* occ = reinterpret_cast<uint32_t*>(wp + kRankWords);  // occupancy bitmask
  __shared__ uint32_t wt[32];
  __shared__ __align__(8) uint64_t bar;
  const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) {
    mbar_init(&bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (tid < kRankWords) occ[tid] = 0;
  __syncthreads();
  auto fits = [cap](uint32_t c) { return c > 0 && c <= cap; };  // cap <= kRTCap (lower only to test the list path)
  auto issue = [&](uint32_t w, uint32_t c) {
    const uint32_t vb = (c * static_cast<uint32_t>(sizeof(T)) + 15u) & ~15u, ob = (c * 2u + 15u) & ~15u;
    mbar_expect_tx(&bar, vb + ob);
    bulk_g2s(xv, tv2 + (static_cast<uint64_t>(w) << kRankW2), vb, &bar);
    bulk_g2s(xo, od + (static_cast<uint64_t>(w) << kRankW2), ob, &bar);
  };
  uint32_t w = blockIdx.x, phase = 0;
  uint32_t cw = w < nwin ? cnt[w] : 0u;
  if (tid == 0 && w < nwin && fits(cw)) issue(w, cw);
  for (; w < nwin; w += gridDim.x) {
    const uint32_t wn = w + gridDim.x;
    const uint32_t cn = wn < nwin ? cnt[wn] : 0u;
    if (!fits(cw)) {  // uniform: nothing staged for this window
      if (tid == 0) {
        if (cw > cap) list[atomicAdd(nlist, 1u)] = w;
        if (wn < nwin && fits(cn)) issue(wn, cn);
      }
      cw = cn;
      continue;
    }
    const uint32_t o0 = pre[w];
    mbar_wait(&bar, phase);
    phase ^= 1u;
    uint32_t so[kRTItems];
    T v[kRTItems];
#pragma unroll
    for (int q = 0; q < kRTItems; ++q) {
      const uint32_t i = tid + q * kRTThreads;
      if (i < cw) {
        so[q] = xo[i];
        v[q] = xv[i];
      }
    }
    __syncthreads();  // staging consumed by every thread
    if (tid == 0 && wn < nwin && fits(cn)) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic reads of staging before the refill
      issue(wn, cn);
    }
#pragma unroll
    for (int q = 0; q < kRTItems; ++q)
      if (tid + q * kRTThreads < cw) atomicOr(&occ[so[q] >> 5], 1u << (so[q] & 31u));
    __syncthreads();
    // exclusive prefix of the word popcounts (threads 0..511, one word each)
    uint32_t word = 0, pc = 0, x = 0;
    if (tid < kRankWords) {
      word = occ[tid];
      pc = __popc(word);
      x = pc;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t t = __shfl_up_sync(0xFFFFFFFFu, x, o);
        if (lane >= static_cast<uint32_t>(o)) x += t;
      }
      if (lane == 31) wt[warp] = x;
    }
    __syncthreads();
    if (warp == 0) {
      const uint32_t t = lane < kRankWords / 32 ? wt[lane] : 0u;
      uint32_t z = t;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t u = __shfl_up_sync(0xFFFFFFFFu, z, o);
        if (lane >= static_cast<uint32_t>(o)) z += u;
      }
      if (lane < kRankWords / 32) wt[lane] = z - t;
    }
    __syncthreads();
    if (tid < kRankWords) {
      wp[tid] = make_uint2(word, wt[warp] + x - pc);
      occ[tid] = 0;  // next window
    }
    if (tid == 0) bulk_wait_read();  // the previous window's bulk store has read y
    __syncthreads();
    // y[a + r] holds rank r, a = the output run's misalignment in elements, so y + a + head is 16-byte aligned
    // exactly where out + o0 + head is.
    const uint32_t a = static_cast<uint32_t>((reinterpret_cast<uintptr_t>(out + o0) & 15u) / sizeof(T));
#pragma unroll
    for (int q = 0; q < kRTItems; ++q) {
      if (tid + q * kRTThreads < cw) {
        const uint32_t s = so[q];
        const uint2 e = wp[s >> 5];
        y[a + e.y + __popc(e.x & ((1u << (s & 31u)) - 1u))] = v[q];
      }
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic writes of y before the bulk read
    __syncthreads();
    const uint32_t head = bulk ? min(cw, (E - a) % E) : cw;
    const uint32_t body = bulk ? (cw - head) & ~(E - 1u) : 0u;
    if (tid == 0 && body) bulk_s2g(out + o0 + head, y + a + head, body * static_cast<uint32_t>(sizeof(T)));
    for (uint32_t i = tid; i < head; i += kRTThreads) out[o0 + i] = y[a + i];  // head (all of it without bulk)
    const uint32_t t0 = head + body;
    if (tid >= 32 && tid - 32 < cw - t0) out[o0 + t0 + tid - 32] = y[a + t0 + tid - 32];
    cw = cn;
  }
  if (tid == 0) bulk_wait_all();
}

// Window-count prefix, level 1: CTA k scans counts [1024k, 1024k + 1024) into pre[] (chunk-local exclusive
// prefix) and writes the chunk total; level 2 (k_window_fix) adds the totals of the chunks before each one.
__global__ void __launch_bounds__(1024) k_window_scan(const uint32_t* __restrict__ cnt, uint32_t* __restrict__ pre,
                                                     uint32_t* __restrict__ chunk_sum, uint32_t n) {
  __shared__ uint32_t wt[32];
  const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, i = blockIdx.x * 1024 + tid;
  const uint32_t v = i < n ? cnt[i] : 0u;
  uint32_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, x, o);
    if (lane >= static_cast<uint32_t>(o)) x += y;
  }
  if (lane == 31) wt[warp] = x;
  __syncthreads();
  if (warp == 0) {
    const uint32_t t = wt[lane];
    uint32_t z = t;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, z, o);
      if (lane >= static_cast<uint32_t>(o)) z += y;
    }
    wt[lane] = z - t;
    if (lane == 31) chunk_sum[blockIdx.x] = z;
  }
  __syncthreads();
  if (i < n) pre[i] = wt[warp] + x - v;
}

__global__ void __launch_bounds__(1024) k_window_fix(uint32_t* __restrict__ pre,
                                                    const uint32_t* __restrict__ chunk_sum, uint32_t n) {
  __shared__ uint32_t off;
  const uint32_t tid = threadIdx.x, i = blockIdx.x * 1024 + tid;
  if (tid < 32) {
    uint32_t acc = 0;
    for (uint32_t j = tid; j < blockIdx.x; j += 32) acc += chunk_sum[j];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xFFFFFFFFu, acc, o);
    if (tid == 0) off = acc;
  }
  __syncthreads();
  if (i < n) pre[i] += off;
}

#ifndef BSG_P2T16
#define BSG_P2T16 1  // 16-byte records: the TMA-fed P2 with 2048-element tiles (else the one-tile-per-CTA k_part2)
#endif
#ifndef BSG_RANK_T
#define BSG_RANK_T 1  // persistent TMA-fed k_place_rank_t (+ k_place_rank over its overflow windows)
#endif
#ifndef BSG_PLACE_RANK
#define BSG_PLACE_RANK 1  // non-power-of-two last pass: placement by rank (k_place_rank) or by counter slot
#endif

template <typename T>
int window_log2() {
  return sizeof(T) == 4 ? 14 : (sizeof(T) == 8 ? 13 : 12);  // 64 KiB smem window
}

// Coarse/fine split of the bits above the window: (s1, s2) fan-outs.
#ifndef BSG_PART_S1_BIAS
#define BSG_PART_S1_BIAS 0
#endif
// Padded domains (about half the counters survive) put the extra bit in the fine fan-out: P1's coarse buckets
// are counter ranges holding ~half their capacity, and 256 coarse buckets keep P1 at one bin per thread and on
// its TMA-fed form for cheap bijections (C3: P1 4.13 -> 3.59 ms, C3-LCG 4.25 -> 3.17 ms with 512 fine bins).
void part_split(int bits, int w2, int& s1, int& s2, bool pad = false) {
  const int total = bits - w2;
  s1 = (pad ? total / 2 : (total + 1) / 2) + BSG_PART_S1_BIAS;
  s2 = total - s1;
}

#define BSG_STAGE_CHECK(x)                 \
  do {                                     \
    const cudaError_t e_ = (x);            \
    if (e_ != cudaSuccess) return e_;      \
  } while (0)

template <int KIND, int D, typename T>
cudaError_t run_partition(const PartitionLaunch& a, cudaStream_t s) {
  const int b = a.p.bits;
  const uint64_t n = 1ULL << b;
  const uint64_t m = a.m ? a.m : n;  // inputs; m < n: non-power-of-two domain (only for elements <= 8 B)
  const bool pad = m < n;
  if (pad && sizeof(T) > 8) return cudaErrorNotSupported;
  const int w2 = pad ? (BSG_PLACE_RANK ? kRankW2 : window_log2<T>()) : window_log2<T>();
  int s1, s2;
  part_split(b, w2, s1, s2, pad);
  const uint64_t w1 = 1ULL << (b - s1);
  const int nb1 = 1 << s1, nb2 = 1 << s2;
  uint32_t* cur1 = a.cursors;
  uint32_t* cur2 = a.cursors + nb1;
  cudaError_t e = cudaMemsetAsync(a.cursors, 0, (kCursorWords + 1) * 4, s);  // + the overflow-window count
  if (e != cudaSuccess) return e;
  const size_t sm1 = kP1Tile * (sizeof(T) + 4);
  const size_t sm2 = kP2Tile * (sizeof(T) + 4);
  const size_t sm3 = (size_t{1} << w2) * sizeof(T);
  cudaFuncSetAttribute(k_part1<KIND, D, T, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(sm1));
  cudaFuncSetAttribute(k_part1<KIND, D, T, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(sm1));
  cudaFuncSetAttribute(k_part2<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(sm2));
  cudaFuncSetAttribute(k_place<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(sm3));
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  T* tv = static_cast<T*>(a.tmp_values);
  const uint64_t tiles1 = (m + kP1Tile - 1) / kP1Tile, full1 = m / kP1Tile;
  // Cheap destinations (LCG, a given permutation) leave P1 bound by its loads: the TMA-fed persistent P1 (2 CTAs
  // per SM) hides them (C2 LCG 7.69 -> 7.07 ms).  The 24-round Philox needs the third CTA per SM of k_part1 to
  // keep the integer pipes busy (k_part1t: 5.16 vs 3.97 ms).
  // With 512 coarse buckets (domains of 2^30+) the 2-CTA TMA-fed form loses (C3-LCG P1 4.72 vs 4.05 ms).
  constexpr bool kTmaP1 = (KIND == kKindLcg || KIND == kKindDestArray) && sizeof(T) <= 8;
  // cp.async.bulk needs 16-byte aligned global addresses: a caller's array that is only element-aligned (e.g. the
  // view x[1:] of a u64 tensor) takes the register-loading k_part1.
  const bool in_aligned = (reinterpret_cast<uintptr_t>(a.in) & 15u) == 0;
  uint64_t done1 = 0;
  const bool staged = a.h_in != nullptr;
  if (staged) {
    // Host input: copy it in chunks of whole tiles on the copy stream and let each chunk's P1 start as soon as its
    // bytes landed, so the inverse cipher runs under the rest of the H2D (the synchronous host-pointer call).
    BSG_STAGE_CHECK(cudaEventRecord(a.ev[0], s));  // the copies follow earlier work on s (staging reuse)
    BSG_STAGE_CHECK(cudaStreamWaitEvent(a.cs_in, a.ev[0], 0));
    const int K = a.chunks;
    for (int k = 0; k < K; ++k) {
      const uint64_t t0 = tiles1 * k / K, t1 = tiles1 * (k + 1) / K;
      if (t1 == t0) continue;
      const uint64_t e0 = t0 * kP1Tile, e1 = std::min<uint64_t>(t1 * kP1Tile, m);
      BSG_STAGE_CHECK(cudaMemcpyAsync(const_cast<T*>(static_cast<const T*>(a.in)) + e0,
                                      static_cast<const T*>(a.h_in) + e0, (e1 - e0) * sizeof(T),
                                      cudaMemcpyHostToDevice, a.cs_in));
      BSG_STAGE_CHECK(cudaEventRecord(a.ev[1 + k], a.cs_in));
      BSG_STAGE_CHECK(cudaStreamWaitEvent(s, a.ev[1 + k], 0));
      const uint64_t tf = std::min<uint64_t>(t1, full1);  // full tiles of this chunk
      if (tf > t0)
        k_part1<KIND, D, T, false><<<static_cast<unsigned>(tf - t0), kP1Threads, sm1, s>>>(
            static_cast<const T*>(a.in), tv, a.tmp_dest, cur1, a.p, b - s1, nb1, w1, a.dest_in, m,
            static_cast<uint32_t>(t0));
    }
    done1 = full1;
  }
  if (!staged && kTmaP1 && in_aligned && full1 > 0 && nb1 <= 256) {
    const size_t smt = kP1Tile * (2 * sizeof(T) + 4);
    cudaFuncSetAttribute(k_part1t<KIND, D, T>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smt));
    int per = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_part1t<KIND, D, T>, kP1Threads, smt);
    const uint64_t grid = std::min<uint64_t>(full1, static_cast<uint64_t>(sms) * std::max(per, 1));
    k_part1t<KIND, D, T><<<static_cast<unsigned>(grid), kP1Threads, smt, s>>>(
        static_cast<const T*>(a.in), tv, a.tmp_dest, cur1, a.p, b - s1, nb1, w1, a.dest_in,
        static_cast<uint32_t>(full1));
    done1 = full1;
  }
  if (done1 < full1) {  // full tiles without the per-element bounds checks
    k_part1<KIND, D, T, false><<<static_cast<unsigned>(full1 - done1), kP1Threads, sm1, s>>>(
        static_cast<const T*>(a.in), tv, a.tmp_dest, cur1, a.p, b - s1, nb1, w1, a.dest_in, m,
        static_cast<uint32_t>(done1));
    done1 = full1;
  }
  if (done1 < tiles1)  // the partial last tile of a non-power-of-two domain
    k_part1<KIND, D, T, true><<<1, kP1Threads, sm1, s>>>(static_cast<const T*>(a.in), tv, a.tmp_dest, cur1, a.p,
                                                         b - s1, nb1, w1, a.dest_in, m,
                                                         static_cast<uint32_t>(done1));
  // P2 writes the fine windows into `out` itself (power of two: exact sizes) or into a counter-sized buffer.
  T* p2out = pad ? static_cast<T*>(a.tmp_values2) : static_cast<T*>(a.out);
  // TMA-fed persistent P2 (2.65 -> 2.45 ms for C2); 16-byte records stage 2048-element tiles (two stages of
  // 2048 x 20 B fit twice per SM).
  constexpr int kTile2 = sizeof(T) <= 8 ? kP2Tile : 2048;
  if constexpr (sizeof(T) <= 8 || BSG_P2T16) {
    const size_t smt = 2 * kTile2 * (sizeof(T) + 4);
    auto kern = (pad || !BSG_P2_FULLT) ? k_part2t<T, kTile2, true> : k_part2t<T, kTile2, false>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smt));
    int per = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kern, kP2Threads, smt);
    const uint64_t tiles = n / kTile2;  // tile slots; in a padded domain the tail of every bucket is empty
    const uint64_t grid = std::min<uint64_t>(tiles, static_cast<uint64_t>(sms) * std::max(per, 1));
    kern<<<static_cast<unsigned>(grid), kP2Threads, smt, s>>>(
        tv, a.tmp_dest, p2out, a.tmp_dlow, cur2, w2, nb2, w1, static_cast<uint32_t>(tiles), pad ? cur1 : nullptr);
  }
  if constexpr (sizeof(T) <= 8) {
    if (pad) {
      const uint32_t nwin = static_cast<uint32_t>(n >> w2);
      uint32_t* chunk_sum = a.win_prefix + (static_cast<size_t>(kMaxB1) * kMaxB2);
      k_window_scan<<<(nwin + 1023) / 1024, 1024, 0, s>>>(cur2, a.win_prefix, chunk_sum, nwin);
      if (nwin > 1024) k_window_fix<<<(nwin + 1023) / 1024, 1024, 0, s>>>(a.win_prefix, chunk_sum, nwin);
      if (BSG_PLACE_RANK) {
        const size_t smr = kRankCap * sizeof(T) + kRankWords * 12;  // survivors by rank + {word, prefix} + bitmask
        cudaFuncSetAttribute(k_place_rank<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smr));
        if (BSG_RANK_T) {
          uint32_t* nlist = a.cursors + kCursorWords;
          constexpr size_t smt = place_rank_t_smem<T>();
          cudaFuncSetAttribute(k_place_rank_t<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smt));
          k_place_rank_t<T><<<std::min<uint32_t>(nwin, static_cast<uint32_t>(sms)), kRTThreads, smt, s>>>(
              p2out, a.tmp_dlow, cur2, a.win_prefix, static_cast<T*>(a.out), nwin, a.win_list, nlist,
              std::min(g_rank_stage_cap, kRTCap), g_bulk_stores);
          k_place_rank<T><<<std::min<uint32_t>(nwin, 2u * static_cast<uint32_t>(sms)), kP3Threads, smr, s>>>(
              p2out, a.tmp_dlow, cur2, a.win_prefix, static_cast<T*>(a.out), a.win_list, nlist);
          note_launch(1);
        } else {
          k_place_rank<T><<<nwin, kP3Threads, smr, s>>>(p2out, a.tmp_dlow, cur2, a.win_prefix, static_cast<T*>(a.out),
                                                        nullptr, nullptr);
        }
      } else {
        const size_t smc = sm3 + (size_t{1} << w2);  // window + one flag byte per counter
        cudaFuncSetAttribute(k_place_compact<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smc));
        k_place_compact<T><<<nwin, kP3Threads, smc, s>>>(p2out, a.tmp_dlow, cur2, a.win_prefix, w2,
                                                          static_cast<T*>(a.out));
      }
      note_launch(nwin > 1024 ? 6 : 5);
      return cudaGetLastError();
    }
  } else if (!BSG_P2T16) {
    k_part2<T><<<static_cast<unsigned>(n / kP2Tile), kP2Threads, sm2, s>>>(tv, a.tmp_dest, static_cast<T*>(a.out),
                                                                            a.tmp_dlow, cur2, w2, nb2, w1);
  }
  if (a.h_out) {
    // Host output: place the windows in chunks and copy each chunk out on the copy stream while the next is placed;
    // s finally waits for the last copy, so a caller that synchronises s has the whole output.
    const uint64_t nw = n >> w2;
    const int K = a.chunks;
    for (int k = 0; k < K; ++k) {
      const uint64_t q0 = nw * k / K, q1 = nw * (k + 1) / K;
      if (q1 == q0) continue;
      k_place<T><<<static_cast<unsigned>(q1 - q0), kP3Threads, sm3, s>>>(static_cast<T*>(a.out), a.tmp_dlow, w2,
                                                                          g_bulk_stores, static_cast<uint32_t>(q0));
      BSG_STAGE_CHECK(cudaEventRecord(a.ev[1 + K + k], s));
      BSG_STAGE_CHECK(cudaStreamWaitEvent(a.cs_out, a.ev[1 + K + k], 0));
      BSG_STAGE_CHECK(cudaMemcpyAsync(static_cast<T*>(a.h_out) + (q0 << w2), static_cast<T*>(a.out) + (q0 << w2),
                                      ((q1 - q0) << w2) * sizeof(T), cudaMemcpyDeviceToHost, a.cs_out));
    }
    BSG_STAGE_CHECK(cudaEventRecord(a.ev[1 + 2 * K], a.cs_out));
    BSG_STAGE_CHECK(cudaStreamWaitEvent(s, a.ev[1 + 2 * K], 0));
    note_launch(3);
    return cudaGetLastError();
  }
  k_place<T><<<static_cast<unsigned>(n >> w2), kP3Threads, sm3, s>>>(static_cast<T*>(a.out), a.tmp_dlow, w2,
                                                                       g_bulk_stores);
  note_launch(3);
  return cudaGetLastError();
}

template <typename T>
cudaError_t dispatch_partition(const PartitionLaunch& a, cudaStream_t s) {
  if (a.dest_in) return run_partition<kKindDestArray, 0, T>(a, s);
  switch (kind_of(a.p)) {
    case kKindLcg: return run_partition<kKindLcg, 0, T>(a, s);
    case kKindPh0: return run_partition<kKindPh0, 0, T>(a, s);
    case kKindPh1: return run_partition<kKindPh1, 1, T>(a, s);
    case kKindPh0G: return run_partition<kKindPh0G, 0, T>(a, s);
    case kKindPh1G: return run_partition<kKindPh1G, 1, T>(a, s);
  }
  return cudaErrorInvalidValue;
}

}  // namespace

// ------------------------------------------------------------------------
// Exchange partition (two ranks, power-of-two domain of 2^G counters, input sharded in two halves): the
// partitioned path with its first pass writing across the pair.  Rank r streams its input half (global indices
// j = r * 2^(G-1) + i), computes f^-1(j) once per element and counting-sorts each tile into the 2 * 2^s1 coarse
// buckets of the GLOBAL domain; buckets [0, 2^s1) are rank 0's output half, the rest rank 1's.  Every bucket
// receives exactly its span of elements from the two sources together (a power-of-two domain has no padding),
// so source 0 fills its buckets from the front and source 1 from the back, each with its own cursors: peer
// traffic is plain stores (NVLink) with no remote atomics, and the buckets end up exactly full -- the owner's
// P2 and P3 are the single-GPU passes over its 2^(G-1) outputs.  The output half of rank r is
// out[r * 2^(G-1), (r + 1) * 2^(G-1)) of the single-GPU shuffle of all 2^G elements.
namespace {
template <int KIND, int D, typename T>
__global__ void __launch_bounds__(kP1Threads, p1_f64<KIND, D>() ? BSG_P1_MINB_F64 : BSG_P1_MINB)
    k_part1x(const T* __restrict__ in, uint32_t j0, T* __restrict__ tv0, T* __restrict__ tv1,
             uint32_t* __restrict__ td0, uint32_t* __restrict__ td1, uint32_t* __restrict__ cur, BijParams p,
             int bshift, int s1, int src) {
  extern __shared__ __align__(16) unsigned char smem[];
  T* sv = reinterpret_cast<T*>(smem);
  uint32_t* sd = reinterpret_cast<uint32_t*>(sv + kP1Tile);
  __shared__ uint32_t hist[kMaxB1], start[kMaxB1], wt[32];
  __shared__ uint32_t delta[kMaxB1];
  const int tid = threadIdx.x, nb = 2 << s1;
  for (int i = tid; i < nb; i += kP1Threads) hist[i] = 0;
  __syncthreads();
  const uint32_t base = blockIdx.x * kP1Tile + tid;  // local index
#ifndef BSG_P1X_EARLY
#define BSG_P1X_EARLY 1  // values loaded before the cipher (80 registers, 3 CTAs/SM): 4.64 -> 4.34 ms per rank
#endif
  T v[BSG_P1X_EARLY ? kP1Items : 1];
  if constexpr (BSG_P1X_EARLY) {
#pragma unroll
    for (int i = 0; i < kP1Items; ++i) v[i] = __ldcs(in + base + i * kP1Threads);
  }
  uint32_t dst[kP1Items];
#pragma unroll
  for (int i = 0; i < kP1Items; ++i) {
    dst[i] = inv_bij<KIND, D>(j0 + base + i * kP1Threads, p);
    atomicAdd(&hist[dst[i] >> bshift], 1u);
  }
  __syncthreads();
  uint32_t g[2] = {0u, 0u};
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    const int i = tid + k * kP1Threads;
    if (i < nb && hist[i]) g[k] = atomicAdd(cur + i, hist[i]);  // this source's cursor of global bucket i
  }
  scan_bins(hist, start, nb, wt);
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    const int i = tid + k * kP1Threads;
    // bucket i within its owner: source 0 appends from the front, source 1 from the back (run [cap - g - n, cap - g))
    if (i < nb) {
      const uint32_t b0 = (static_cast<uint32_t>(i) & ((1u << s1) - 1u)) << bshift;
      delta[i] = (src ? b0 + (1u << bshift) - g[k] - hist[i] : b0 + g[k]) - start[i];  // mod 2^32
    }
  }
  __syncthreads();  // start[] read for delta before the rank atomics advance it
#pragma unroll
  for (int i = 0; i < kP1Items; ++i) {
    const uint32_t r = atomicAdd(&start[dst[i] >> bshift], 1u);
    if constexpr (BSG_P1X_EARLY) sv[r] = v[i];
    else sv[r] = __ldcs(in + base + i * kP1Threads);
    sd[r] = dst[i];
  }
  __syncthreads();
#pragma unroll 4
  for (int s = tid; s < kP1Tile; s += kP1Threads) {
    const uint32_t d = sd[s];
    const uint32_t b = d >> bshift;
    const uint32_t pos = delta[b] + s;
    const bool peer1 = (b >> s1) != 0;  // owner rank of the bucket
    __stcs((peer1 ? tv1 : tv0) + pos, sv[s]);
    __stcs((peer1 ? td1 : td0) + pos, d);
  }
}

struct XLayout {
  int G, Lb, w2, s1, s2;
  size_t tv, td, dlow, cur, cur2, total;
};
XLayout xlayout(int elem_code, int G) {
  XLayout L{};
  L.G = G;
  L.Lb = G - 1;
  L.w2 = elem_code == 4 ? 14 : 13;
  part_split(L.Lb, L.w2, L.s1, L.s2);
  // P1 sorts into both ranks' buckets (2 << s1 <= kMaxB1): move a coarse bit to the fine split if needed
  while ((2 << L.s1) > kMaxB1 && L.s1 > 1) {
    --L.s1;
    ++L.s2;
  }
  const uint64_t R = 1ULL << L.Lb;  // the owner's buckets, exactly full
  auto al = [](size_t x) { return (x + 255) / 256 * 256; };
  size_t o = 0;
  L.tv = o;
  o = al(o + R * static_cast<uint64_t>(elem_code));
  L.td = o;
  o = al(o + R * 4);
  L.dlow = o;
  o = al(o + (1ULL << L.Lb) * 2);
  L.cur = o;
  o = al(o + (2u << L.s1) * 4);
  L.cur2 = o;
  o = al(o + (static_cast<size_t>(1) << (L.s1 + L.s2)) * 4);
  L.total = o;
  return L;
}
}  // namespace

bool xpart_eligible(int elem_code, int G, int world) {
  if (world != 2 || (elem_code != 4 && elem_code != 8) || G < 16 || G > 32) return false;
  const XLayout L = xlayout(elem_code, G);
  return L.s1 >= 1 && L.s2 >= 1 && (2 << L.s1) <= kMaxB1 && (1 << L.s2) <= kMaxB2 &&
         (L.Lb - L.s1) >= kP2TileLog && ((1ULL << L.Lb) % kP1Tile) == 0;
}

size_t xpart_workspace_bytes(int elem_code, int G) { return xlayout(elem_code, G).total; }

namespace {
template <int KIND, int D, typename T>
cudaError_t run_xroute(const XpartLaunch& a, cudaStream_t s) {
  const XLayout L = xlayout(sizeof(T), a.G);
  char* w[2] = {static_cast<char*>(a.ws[0]), static_cast<char*>(a.ws[1])};
  uint32_t* cur = reinterpret_cast<uint32_t*>(w[a.rank] + L.cur);
  cudaError_t e = cudaMemsetAsync(cur, 0, (2u << L.s1) * 4, s);
  if (e != cudaSuccess) return e;
  const size_t sm1 = kP1Tile * (sizeof(T) + 4);
  cudaFuncSetAttribute(k_part1x<KIND, D, T>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(sm1));
  const uint64_t n_local = 1ULL << L.Lb;
  k_part1x<KIND, D, T><<<static_cast<unsigned>(n_local / kP1Tile), kP1Threads, sm1, s>>>(
      static_cast<const T*>(a.in), static_cast<uint32_t>(static_cast<uint64_t>(a.rank) << L.Lb),
      reinterpret_cast<T*>(w[0] + L.tv), reinterpret_cast<T*>(w[1] + L.tv), reinterpret_cast<uint32_t*>(w[0] + L.td),
      reinterpret_cast<uint32_t*>(w[1] + L.td), cur, a.p, L.Lb - L.s1, L.s1, a.rank);
  note_launch(1);
  return cudaGetLastError();
}

template <typename T>
cudaError_t run_xplace(const XpartLaunch& a, cudaStream_t s) {
  const XLayout L = xlayout(sizeof(T), a.G);
  char* me = static_cast<char*>(a.ws[a.rank]);
  uint32_t* cur2 = reinterpret_cast<uint32_t*>(me + L.cur2);
  cudaError_t e = cudaMemsetAsync(cur2, 0, (static_cast<size_t>(1) << (L.s1 + L.s2)) * 4, s);
  if (e != cudaSuccess) return e;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const size_t smt = 2 * kP2Tile * (sizeof(T) + 4);
  auto kern = BSG_P2_FULLT ? k_part2t<T, kP2Tile, false> : k_part2t<T, kP2Tile, true>;  // exchange: power of two
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smt));
  int per = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kern, kP2Threads, smt);
  const uint64_t w1 = 1ULL << (L.Lb - L.s1);
  const uint64_t tiles = (1ULL << L.Lb) / kP2Tile;
  const uint64_t grid = std::min<uint64_t>(tiles, static_cast<uint64_t>(sms) * std::max(per, 1));
  uint16_t* dlow = reinterpret_cast<uint16_t*>(me + L.dlow);
  kern<<<static_cast<unsigned>(grid), kP2Threads, smt, s>>>(
      reinterpret_cast<const T*>(me + L.tv), reinterpret_cast<const uint32_t*>(me + L.td), static_cast<T*>(a.out),
      dlow, cur2, L.w2, 1 << L.s2, w1, static_cast<uint32_t>(tiles), nullptr);
  const size_t sm3 = (size_t{1} << L.w2) * sizeof(T);
  cudaFuncSetAttribute(k_place<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(sm3));
  k_place<T><<<static_cast<unsigned>((1ULL << L.Lb) >> L.w2), kP3Threads, sm3, s>>>(static_cast<T*>(a.out), dlow,
                                                                                    L.w2, g_bulk_stores);
  note_launch(2);
  return cudaGetLastError();
}

template <typename T>
cudaError_t dispatch_xroute(const XpartLaunch& a, cudaStream_t s) {
  switch (kind_of(a.p)) {
    case kKindLcg: return run_xroute<kKindLcg, 0, T>(a, s);
    case kKindPh0: return run_xroute<kKindPh0, 0, T>(a, s);
    case kKindPh1: return run_xroute<kKindPh1, 1, T>(a, s);
    case kKindPh0G: return run_xroute<kKindPh0G, 0, T>(a, s);
    case kKindPh1G: return run_xroute<kKindPh1G, 1, T>(a, s);
  }
  return cudaErrorInvalidValue;
}
}  // namespace

cudaError_t launch_xpart_route(int elem_code, const XpartLaunch& a, cudaStream_t s) {
  switch (elem_code) {
    case 4: return dispatch_xroute<uint32_t>(a, s);
    case 8: return dispatch_xroute<uint64_t>(a, s);
  }
  return cudaErrorNotSupported;
}

cudaError_t launch_xpart_place(int elem_code, const XpartLaunch& a, cudaStream_t s) {
  switch (elem_code) {
    case 4: return run_xplace<uint32_t>(a, s);
    case 8: return run_xplace<uint64_t>(a, s);
  }
  return cudaErrorNotSupported;
}

namespace {

// ------------------------------------------------------------------------
// Route-by-destination (multi-GPU sharded power-of-two shuffle):
// for local elements j = offset + i, dest = f^-1(j); group them by the rank
// owning dest (contiguous output shards of `part_size`), keeping the
// destination inside the part.  Two kernels: destinations + part histogram,
// then a tiled counting sort into the part groups.
template <int KIND, int D>
__global__ void __launch_bounds__(256) k_route_dest(uint64_t n, uint64_t offset, BijParams p, int part_shift,
                                                    int nparts, uint32_t* __restrict__ dest,
                                                    unsigned long long* __restrict__ counts) {
  __shared__ uint32_t h[64];
  if (threadIdx.x < 64) h[threadIdx.x] = 0;
  __syncthreads();
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
    const uint32_t d = inv_bij<KIND, D>(static_cast<uint32_t>(offset + i), p);
    dest[i] = d;
    atomicAdd(&h[d >> part_shift], 1u);
  }
  __syncthreads();
  if (threadIdx.x < nparts && h[threadIdx.x]) atomicAdd(counts + threadIdx.x, static_cast<unsigned long long>(h[threadIdx.x]));
}

template <typename T>
__global__ void __launch_bounds__(kP2Threads) k_route(const T* __restrict__ in, const uint32_t* __restrict__ dest,
                                                      uint64_t n, int part_shift, int nparts,
                                                      unsigned long long* __restrict__ cursors, T* __restrict__ ov,
                                                      uint32_t* __restrict__ od) {
  __shared__ uint32_t hist[64], start[64], wt[32];
  __shared__ unsigned long long gbase[64];
  extern __shared__ __align__(16) unsigned char smem[];
  T* sv = reinterpret_cast<T*>(smem);
  uint32_t* sd = reinterpret_cast<uint32_t*>(sv + kP2Tile);
  const int tid = threadIdx.x;
  if (tid < 64) hist[tid] = 0;
  __syncthreads();
  const uint64_t t0 = static_cast<uint64_t>(blockIdx.x) * kP2Tile;
  T v[kP2Items];
  uint32_t d[kP2Items], rk[kP2Items];
#pragma unroll
  for (int i = 0; i < kP2Items; ++i) {
    const uint64_t e = t0 + tid + i * kP2Threads;
    if (e < n) {
      v[i] = __ldcs(in + e);
      d[i] = __ldcs(dest + e);
      rk[i] = atomicAdd(&hist[d[i] >> part_shift], 1u);
    }
  }
  __syncthreads();
  scan_bins(hist, start, nparts, wt);
  if (tid < nparts) gbase[tid] = atomicAdd(cursors + tid, static_cast<unsigned long long>(hist[tid]));
  __syncthreads();
  const uint32_t mask = (part_shift >= 32) ? 0xFFFFFFFFu : ((1u << part_shift) - 1);
#pragma unroll
  for (int i = 0; i < kP2Items; ++i) {
    if (t0 + tid + i * kP2Threads < n) {
      const uint32_t s = start[d[i] >> part_shift] + rk[i];
      sv[s] = v[i];
      sd[s] = d[i];
    }
  }
  __syncthreads();
  const uint32_t cnt = static_cast<uint32_t>(n - t0 < kP2Tile ? n - t0 : kP2Tile);
  for (uint32_t s = tid; s < cnt; s += kP2Threads) {
    const uint32_t dd = sd[s], b = dd >> part_shift;
    const uint64_t pos = gbase[b] + (s - start[b]);
    __stcs(ov + pos, sv[s]);
    __stcs(od + pos, dd & mask);
  }
}

template <int KIND, int D, typename T>
cudaError_t run_route(const RouteLaunch& a, cudaStream_t s) {
  int shift = 0;
  while ((1ULL << shift) < a.part_size) ++shift;
  cudaError_t e = cudaMemsetAsync(a.counts, 0, sizeof(unsigned long long) * a.nparts, s);
  if (e != cudaSuccess) return e;
  const uint64_t blocks = (a.n + 255) / 256;
  k_route_dest<KIND, D><<<static_cast<unsigned>(blocks < 148ull * 16 ? blocks : 148ull * 16), 256, 0, s>>>(
      a.n, a.offset, a.p, shift, a.nparts, a.tmp_dest, a.counts);
  // exclusive prefix of the part counts -> cursors (nparts <= 64: one tiny kernel-free step on the host side
  // would force a sync; do it on the device instead)
  e = launch_exclusive_prefix_u64(a.counts, a.cursors, a.nparts, s);
  if (e != cudaSuccess) return e;
  const size_t sm = kP2Tile * (sizeof(T) + 4);
  cudaFuncSetAttribute(k_route<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(sm));
  k_route<T><<<static_cast<unsigned>((a.n + kP2Tile - 1) / kP2Tile), kP2Threads, sm, s>>>(
      static_cast<const T*>(a.in), a.tmp_dest, a.n, shift, a.nparts, a.cursors, static_cast<T*>(a.out_values),
      a.out_dest);
  note_launch(3);
  return cudaGetLastError();
}

__global__ void k_excl_prefix(const unsigned long long* c, unsigned long long* o, int n) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    unsigned long long r = 0;
    for (int i = 0; i < n; ++i) {
      o[i] = r;
      r += c[i];
    }
  }
}

template <typename T>
cudaError_t dispatch_route(const RouteLaunch& a, cudaStream_t s) {
  switch (kind_of(a.p)) {
    case kKindLcg: return run_route<kKindLcg, 0, T>(a, s);
    case kKindPh0: return run_route<kKindPh0, 0, T>(a, s);
    case kKindPh1: return run_route<kKindPh1, 1, T>(a, s);
    case kKindPh0G: return run_route<kKindPh0G, 0, T>(a, s);
    case kKindPh1G: return run_route<kKindPh1G, 1, T>(a, s);
  }
  return cudaErrorInvalidValue;
}
template <typename T>
__global__ void k_scatter_simple(const T* __restrict__ in, const uint32_t* __restrict__ dest, uint64_t n,
                                 T* __restrict__ out) {
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride)
    out[dest[i]] = in[i];
}

template <typename T>
cudaError_t scatter_simple(const void* in, const uint32_t* dest, uint64_t n, void* out, cudaStream_t s) {
  const uint64_t blocks = (n + 255) / 256;
  k_scatter_simple<T><<<static_cast<unsigned>(blocks < 148ull * 32 ? blocks : 148ull * 32), 256, 0, s>>>(
      static_cast<const T*>(in), dest, n, static_cast<T*>(out));
  note_launch();
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_scatter_simple(int elem_code, const void* in, const uint32_t* dest, uint64_t n, void* out,
                                  cudaStream_t s) {
  switch (elem_code) {
    case 4: return scatter_simple<uint32_t>(in, dest, n, out, s);
    case 8: return scatter_simple<uint64_t>(in, dest, n, out, s);
    case 16: return scatter_simple<uint4>(in, dest, n, out, s);
  }
  return cudaErrorNotSupported;
}

cudaError_t launch_exclusive_prefix_u64(const unsigned long long* c, unsigned long long* o, int n, cudaStream_t s) {
  k_excl_prefix<<<1, 32, 0, s>>>(c, o, n);
  return cudaGetLastError();
}

cudaError_t launch_route(int elem_code, const RouteLaunch& a, cudaStream_t s) {
  switch (elem_code) {
    case 4: return dispatch_route<uint32_t>(a, s);
    case 8: return dispatch_route<uint64_t>(a, s);
    case 16: return dispatch_route<uint4>(a, s);
  }
  return cudaErrorNotSupported;
}

bool partition_eligible(int elem_code, int bits, bool pad) {
  int w2;
  switch (elem_code) {
    case 4: w2 = 14; break;
    case 8: w2 = 13; break;
    case 16: w2 = 12; break;
    default: return false;
  }
  if (pad) {
    if (elem_code > 8) return false;
    if (BSG_PLACE_RANK) w2 = kRankW2;
  }
  int s1, s2;
  part_split(bits, w2, s1, s2, pad);
  // fan-outs within the shared-memory histograms; tiles must not straddle buckets; 32-bit destinations
  return bits <= 32 && s1 >= 1 && s2 >= 1 && (1 << s1) <= kMaxB1 && (1 << s2) <= kMaxB2 &&
         (bits - s1) >= kP2TileLog && bits >= 14;
}

void partition_layout(int elem_code, int bits, bool pad, void* workspace, PartitionLaunch& P) {
  const uint64_t n = 1ULL << bits;
  char* w = static_cast<char*>(workspace);
  P.tmp_values = w;
  w += n * static_cast<uint64_t>(elem_code);
  P.tmp_dest = reinterpret_cast<uint32_t*>(w);
  w += n * 4;
  P.tmp_dlow = reinterpret_cast<uint16_t*>(w);
  w += n * 2;
  P.cursors = reinterpret_cast<uint32_t*>(w);
  w += ((kCursorWords + 1) * 4 + 255) / 256 * 256;
  if (pad) {
    P.win_prefix = reinterpret_cast<uint32_t*>(w);  // window prefix, then the scan's chunk totals
    w += (static_cast<size_t>(kMaxB1) * kMaxB2 * 4 + 4096 + 255) / 256 * 256;
    P.win_list = reinterpret_cast<uint32_t*>(w);  // overflow windows of the persistent last pass
    w += static_cast<size_t>(kMaxB1) * kMaxB2 * 4;
    P.tmp_values2 = w;
  }
}

size_t partition_workspace_bytes(int elem_code, int bits, bool pad) {
  const uint64_t n = 1ULL << bits;
  size_t b = n * static_cast<uint64_t>(elem_code) + n * 4 + n * 2 + ((kCursorWords + 1) * 4 + 255) / 256 * 256;
  if (pad)
    b += (static_cast<size_t>(kMaxB1) * kMaxB2 * 4 + 4096 + 255) / 256 * 256 + static_cast<size_t>(kMaxB1) * kMaxB2 * 4 +
         n * static_cast<uint64_t>(elem_code);
  return b;
}

cudaError_t launch_partition(int elem_code, const PartitionLaunch& a, cudaStream_t s) {
  switch (elem_code) {
    case 4: return dispatch_partition<uint32_t>(a, s);
    case 8: return dispatch_partition<uint64_t>(a, s);
    case 16: return dispatch_partition<uint4>(a, s);
  }
  return cudaErrorNotSupported;
}

}  // namespace bsg
