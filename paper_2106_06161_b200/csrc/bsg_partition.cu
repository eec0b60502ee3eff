// bsg_partition.cu -- partitioned (three-pass) shuffle for large power-of-two
// domains, the B200 answer to the DRAM random-access wall.
//
// Why: a single-pass shuffle of a 4 GiB array issues one random read per
// element; on B200 those saturate at ~47 G reads/s (DRAM row activations,
// independent of element size -- profiles/r01_microbench.md), i.e. 11.4 ms for
// 2^29 elements although 8.6 GB of payload would stream in 1.4 ms.  When
// m == 2^bits every counter survives and out[f^-1(j)] = in[j], so the
// permutation can be applied by streaming the INPUT in order and routing each
// element by its destination f^-1(j) (philox_invert, bijection.hpp:117-143):
//   P1  read in[] sequentially, inverse cipher -> dest, counting-sort each
//       8192-element tile in shared memory into 2^s1 coarse destination
//       buckets, append the runs to the buckets (value + u32 dest);
//   P2  per coarse bucket, the same split into 2^s2 fine windows of W2
//       elements (value + u16 dest-in-window), written into `out` itself;
//   P3  per fine window (64 KiB), scatter into shared memory at dest and
//       write the window back coalesced (in place: each CTA reads its whole
//       range before writing).
// Every DRAM access is a coalesced run; traffic is ~60 B/element instead of
// one random 64-B access per 8-B element.  Exact sizes (pow2: each bucket
// receives exactly its window) make the layout static; atomic cursors only
// order elements inside a bucket, which the final exact placement makes
// irrelevant -- the output is bit-identical to the single-pass kernel.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>

#include "bsg_kernels.cuh"
#include "bsg_partition.h"

namespace bsg {

namespace {

#ifndef BSG_P1_THREADS
#define BSG_P1_THREADS 256
#endif
#ifndef BSG_P2_MINB
#define BSG_P2_MINB 3
#endif
#ifndef BSG_P2_THREADS
#define BSG_P2_THREADS 256
#endif
constexpr int kP1Threads = BSG_P1_THREADS, kP1Items = 4096 / BSG_P1_THREADS, kP1Tile = 4096;
constexpr int kP2Threads = BSG_P2_THREADS, kP2Items = 4096 / BSG_P2_THREADS, kP2Tile = 4096;
constexpr int kP3Threads = 512;
#ifndef BSG_P23_THREADS
#define BSG_P23_THREADS 512
#endif
constexpr int kP23Threads = BSG_P23_THREADS, kP23Items = kP2Tile / BSG_P23_THREADS;
#ifndef BSG_PART_GROUP_MB
#define BSG_PART_GROUP_MB 0
#endif
#ifndef BSG_PART_S1_BIAS
#define BSG_PART_S1_BIAS 0
#endif
constexpr int kMaxB1 = 512, kMaxB2 = 256;
// cursor region: P1 bucket cursors, P2 window cursors, fused-path completion counters + ticket
constexpr int kMaxChunks = 16;
constexpr size_t kCursorWords = kMaxB1 + static_cast<size_t>(kMaxB1) * kMaxB2 + kMaxB1 + 32 + kMaxChunks * kMaxB1;

constexpr int kKindDestArray = 100;  // destinations come from an array (scatter by permutation)

template <int KIND, int D>
__device__ __forceinline__ uint32_t inv_bij(uint32_t y, const BijParams& p) {
  if constexpr (KIND == kKindLcg) return static_cast<uint32_t>(lcg_inv(y, p));
  else if constexpr (KIND == kKindPh0 || KIND == kKindPh1) return static_cast<uint32_t>(philox_inv<D, 24>(y, p));
  else return static_cast<uint32_t>(philox_inv<D, 0>(y, p));
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

// P1: stream the input, route by coarse destination bucket.
template <int KIND, int D, typename T>
__global__ void __launch_bounds__(kP1Threads) k_part1(const T* __restrict__ in, T* __restrict__ tv,
                                                         uint32_t* __restrict__ td, uint32_t* __restrict__ cur1,
                                                         BijParams p, int bshift, int nb, uint64_t w1,
                                                         const uint32_t* __restrict__ dsrc, uint32_t tile0) {
  extern __shared__ __align__(16) unsigned char smem[];
  T* sv = reinterpret_cast<T*>(smem);
  uint32_t* sd = reinterpret_cast<uint32_t*>(sv + kP1Tile);
  __shared__ uint32_t hist[kMaxB1], start[kMaxB1], wt[32];
  __shared__ unsigned long long delta[kMaxB1];
  const int tid = threadIdx.x;
  for (int i = tid; i < nb; i += kP1Threads) hist[i] = 0;
  __syncthreads();
  const uint32_t base = (tile0 + blockIdx.x) * kP1Tile + tid;
#ifndef BSG_P1_LATE_LOAD
#define BSG_P1_LATE_LOAD 1
#endif
  // Default: the input tile is loaded first (its latency hides under the cipher).  LATE_LOAD keeps the
  // values out of registers during the cipher (more resident CTAs) and loads them after the scan.
  T v[BSG_P1_LATE_LOAD ? 1 : kP1Items];
  if constexpr (!BSG_P1_LATE_LOAD) {
#pragma unroll
    for (int i = 0; i < kP1Items; ++i) v[i] = __ldcs(in + base + i * kP1Threads);
  }
  uint32_t dst[kP1Items], rk[kP1Items];
#pragma unroll
  for (int i = 0; i < kP1Items; ++i) {
    if constexpr (KIND == kKindDestArray) dst[i] = __ldcs(dsrc + base + i * kP1Threads);
    else dst[i] = inv_bij<KIND, D>(base + i * kP1Threads, p);
    rk[i] = atomicAdd(&hist[dst[i] >> bshift], 1u);
  }
  __syncthreads();
  scan_bins(hist, start, nb, wt);
  // Cursor atomics (nb <= 2 * blockDim) are issued first and consumed after the scatter (latency hidden).
  uint32_t g[2] = {0u, 0u};
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    const int i = tid + k * kP1Threads;
    if (i < nb) g[k] = atomicAdd(cur1 + i, hist[i]);
  }
#pragma unroll
  for (int i = 0; i < kP1Items; ++i) rk[i] += start[dst[i] >> bshift];
#pragma unroll
  for (int i = 0; i < kP1Items; ++i) {
    if constexpr (BSG_P1_LATE_LOAD) sv[rk[i]] = __ldcs(in + base + i * kP1Threads);
    else sv[rk[i]] = v[i];
    sd[rk[i]] = dst[i];
  }
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    // one table lookup per element in the write-back: global position = delta[b] + slot
    const int i = tid + k * kP1Threads;
    if (i < nb) delta[i] = static_cast<unsigned long long>(i) * w1 + g[k] - start[i];
  }
  __syncthreads();
#pragma unroll 4
  for (int s = tid; s < kP1Tile; s += kP1Threads) {
    const uint32_t d = sd[s];
    const uint64_t pos = delta[d >> bshift] + s;
    __stcs(tv + pos, sv[s]);
    __stcs(td + pos, d);
  }
}

// P2: split each coarse bucket into fine windows of 2^w2 elements.
template <typename T>
__global__ void __launch_bounds__(kP2Threads, sizeof(T) > 8 ? 2 : BSG_P2_MINB) k_part2(const T* __restrict__ tv, const uint32_t* __restrict__ td,
                                                         T* __restrict__ ov, uint16_t* __restrict__ od,
                                                         uint32_t* __restrict__ cur2, int w2, int nb2,
                                                         uint64_t w1, uint64_t tile_base, uint32_t swz) {
  extern __shared__ __align__(16) unsigned char smem[];
  T* sv = reinterpret_cast<T*>(smem);
  uint32_t* sd = reinterpret_cast<uint32_t*>(sv + kP2Tile);
  __shared__ uint32_t hist[kMaxB2], start[kMaxB2], wt[32];
  __shared__ unsigned long long delta[kMaxB2];
  const int tid = threadIdx.x;
  if (tid < nb2) hist[tid] = 0;
  __syncthreads();
  // swz > 1: consecutive CTAs take tiles of different coarse buckets (swz buckets round-robin), so the CTAs
  // resident at one time spread their cursor atomics over swz buckets instead of queueing on one bucket's.
  uint64_t tile = blockIdx.x;
  if (swz > 1) {
    const uint64_t tpb = w1 / kP2Tile, grp = tile / (tpb * swz), k = tile % (tpb * swz);
    tile = (grp * swz + k % swz) * tpb + k / swz;
  }
  const uint64_t t0 = (tile_base + tile) * kP2Tile;
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
  // The cursor atomics are issued here and consumed after the shared-memory scatter, which hides their
  // round trip; the slots are all read before any scatter store (no false LDS->STS ordering).
  uint32_t g = 0;
  if (tid < nb2) g = atomicAdd(cur + tid, hist[tid]);
#pragma unroll
  for (int i = 0; i < kP2Items; ++i) rk[i] += start[(d[i] >> w2) & fmask];
#pragma unroll
  for (int i = 0; i < kP2Items; ++i) {
    sv[rk[i]] = v[i];
    sd[rk[i]] = d[i];
  }
  if (tid < nb2) delta[tid] = win0 + (static_cast<unsigned long long>(tid) << w2) + g - start[tid];
  __syncthreads();
#pragma unroll 4
  for (int s = tid; s < kP2Tile; s += kP2Threads) {
    const uint32_t dd = sd[s];
    const uint64_t pos = delta[(dd >> w2) & fmask] + s;
    ov[pos] = sv[s];
    od[pos] = static_cast<uint16_t>(dd & wmask);
  }
}

// Chunked P2 (P1/P2 overlap): P1 runs over the input in K chunks; after
// chunk k the coarse cursors are snapshotted, and chunk k's contribution to
// coarse bucket b is the run [snap[k-1][b], snap[k][b]) of that bucket (P1
// chunks append in launch order).  This kernel splits those runs while P1
// computes the next chunk on another stream: P2 is bound by shared memory and
// latency, P1 by the integer pipes, so the two overlap on the same SMs.
template <typename T>
__global__ void __launch_bounds__(kP2Threads, sizeof(T) > 8 ? 2 : BSG_P2_MINB) k_part2c(
    const T* __restrict__ tv, const uint32_t* __restrict__ td, T* __restrict__ ov, uint16_t* __restrict__ od,
    uint32_t* __restrict__ cur2, int w2, int nb2, uint64_t w1, const uint32_t* __restrict__ snap_prev,
    const uint32_t* __restrict__ snap, uint32_t tpc) {
  extern __shared__ __align__(16) unsigned char smem[];
  T* sv = reinterpret_cast<T*>(smem);
  uint32_t* sd = reinterpret_cast<uint32_t*>(sv + kP2Tile);
  __shared__ uint32_t hist[kMaxB2], start[kMaxB2], wt[32];
  __shared__ unsigned long long delta[kMaxB2];
  const int tid = threadIdx.x;
  const uint32_t coarse = blockIdx.x / tpc;
  const uint32_t lo = snap_prev ? snap_prev[coarse] : 0u, hi = snap[coarse];
  const uint32_t fmask = static_cast<uint32_t>(nb2 - 1), wmask = (1u << w2) - 1;
  uint32_t* cur = cur2 + static_cast<uint64_t>(coarse) * nb2;
  const uint64_t win0 = static_cast<uint64_t>(coarse) * w1;
  for (uint32_t t = lo + (blockIdx.x % tpc) * kP2Tile; t < hi; t += tpc * kP2Tile) {
    const uint32_t nv = min(hi - t, static_cast<uint32_t>(kP2Tile));
    const uint64_t t0 = win0 + t;
    if (tid < nb2) hist[tid] = 0;
    __syncthreads();
    T v[kP2Items];
    uint32_t d[kP2Items], rk[kP2Items];
#pragma unroll
    for (int i = 0; i < kP2Items; ++i) {
      const uint32_t e = tid + i * kP2Threads;
      if (e < nv) {
        v[i] = __ldcs(tv + t0 + e);
        d[i] = __ldcs(td + t0 + e);
      }
    }
#pragma unroll
    for (int i = 0; i < kP2Items; ++i)
      if (tid + i * kP2Threads < nv) rk[i] = atomicAdd(&hist[(d[i] >> w2) & fmask], 1u);
    __syncthreads();
    scan_bins(hist, start, nb2, wt);
    uint32_t g = 0;
    if (tid < nb2) g = atomicAdd(cur + tid, hist[tid]);
#pragma unroll
    for (int i = 0; i < kP2Items; ++i)
      if (tid + i * kP2Threads < nv) rk[i] += start[(d[i] >> w2) & fmask];
#pragma unroll
    for (int i = 0; i < kP2Items; ++i) {
      if (tid + i * kP2Threads < nv) {
        sv[rk[i]] = v[i];
        sd[rk[i]] = d[i];
      }
    }
    if (tid < nb2) delta[tid] = win0 + (static_cast<unsigned long long>(tid) << w2) + g - start[tid];
    __syncthreads();
    for (uint32_t q = tid; q < nv; q += kP2Threads) {
      const uint32_t dd = sd[q];
      const uint64_t pos = delta[(dd >> w2) & fmask] + q;
      ov[pos] = sv[q];
      od[pos] = static_cast<uint16_t>(dd & wmask);
    }
    __syncthreads();
  }
}

__global__ void k_snap(const uint32_t* __restrict__ cur, uint32_t* __restrict__ snap, int nb) {
  for (int i = threadIdx.x; i < nb; i += blockDim.x) snap[i] = cur[i];
}

// Persistent P2: each CTA loops over tiles; the next tile's values and
// destinations stream into shared memory with cp.async while the current tile
// is ranked, scattered and written, so the load latency leaves the critical path.
template <typename T>
__global__ void __launch_bounds__(kP2Threads) k_part2p(const T* __restrict__ tv, const uint32_t* __restrict__ td,
                                                          T* __restrict__ ov, uint16_t* __restrict__ od,
                                                          uint32_t* __restrict__ cur2, int w2, int nb2, uint64_t w1,
                                                          uint64_t tile_base, uint64_t ntiles) {
  extern __shared__ __align__(16) unsigned char smem[];
  T* sv = reinterpret_cast<T*>(smem);
  uint32_t* sd = reinterpret_cast<uint32_t*>(sv + kP2Tile);
  T* iv = reinterpret_cast<T*>(sd + kP2Tile);
  uint32_t* id = reinterpret_cast<uint32_t*>(iv + kP2Tile);
  __shared__ uint32_t hist[kMaxB2], start[kMaxB2], wt[32];
  __shared__ unsigned long long delta[kMaxB2];
  const int tid = threadIdx.x;
  const uint32_t fmask = static_cast<uint32_t>(nb2 - 1), wmask = (1u << w2) - 1;
  auto prefetch = [&](uint64_t t) {
    const char* gv = reinterpret_cast<const char*>(tv + (tile_base + t) * kP2Tile);
    const char* gd = reinterpret_cast<const char*>(td + (tile_base + t) * kP2Tile);
    for (uint32_t o = tid * 16; o < kP2Tile * sizeof(T); o += kP2Threads * 16) {
      const uint32_t dst = static_cast<uint32_t>(__cvta_generic_to_shared(reinterpret_cast<char*>(iv) + o));
      asm volatile("cp.async.cg.shared.global.L2::64B [%0], [%1], 16;" ::"r"(dst), "l"(gv + o) : "memory");
    }
    for (uint32_t o = tid * 16; o < kP2Tile * 4; o += kP2Threads * 16) {
      const uint32_t dst = static_cast<uint32_t>(__cvta_generic_to_shared(reinterpret_cast<char*>(id) + o));
      asm volatile("cp.async.cg.shared.global.L2::64B [%0], [%1], 16;" ::"r"(dst), "l"(gd + o) : "memory");
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  uint64_t t = blockIdx.x;
  if (t < ntiles) prefetch(t);
  for (; t < ntiles; t += gridDim.x) {
    if (tid < nb2) hist[tid] = 0;
    asm volatile("cp.async.wait_all;" ::: "memory");
    __syncthreads();
    T v[kP2Items];
    uint32_t d[kP2Items], rk[kP2Items];
#pragma unroll
    for (int i = 0; i < kP2Items; ++i) {
      v[i] = iv[tid + i * kP2Threads];
      d[i] = id[tid + i * kP2Threads];
    }
    __syncthreads();  // input buffer free: stream the next tile in behind this one
    if (t + gridDim.x < ntiles) prefetch(t + gridDim.x);
#pragma unroll
    for (int i = 0; i < kP2Items; ++i) rk[i] = atomicAdd(&hist[(d[i] >> w2) & fmask], 1u);
    __syncthreads();
    scan_bins(hist, start, nb2, wt);
    const uint64_t t0 = (tile_base + t) * kP2Tile;
    const uint64_t coarse = t0 / w1;
    uint32_t* cur = cur2 + coarse * nb2;
    const uint64_t win0 = coarse * w1;
    if (tid < nb2)
      delta[tid] =
          win0 + (static_cast<unsigned long long>(tid) << w2) + atomicAdd(cur + tid, hist[tid]) - start[tid];
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
      const uint64_t pos = delta[(dd >> w2) & fmask] + s;
      ov[pos] = sv[s];
      od[pos] = static_cast<uint16_t>(dd & wmask);
    }
    __syncthreads();  // staging reuse by the next tile
  }
}

// P3: place each fine window through shared memory, in place in `out`.
template <typename T>
__global__ void __launch_bounds__(kP3Threads) k_place(T* __restrict__ out, uint16_t* __restrict__ od, int w2,
                                                      uint64_t win_base, int discard) {
  extern __shared__ __align__(16) unsigned char smem[];
  T* win = reinterpret_cast<T*>(smem);
  const uint32_t W = 1u << w2;
  T* o = out + ((win_base + blockIdx.x) << w2);
  uint16_t* dd = od + ((win_base + blockIdx.x) << w2);
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
  __syncthreads();
  if (discard) {
    // The window's u16 destinations are dead: drop their (L2-resident, dirty) lines without write-back.
    for (uint32_t l = threadIdx.x; l < (W * 2) / 128; l += kP3Threads)
      asm volatile("discard.global.L2 [%0], 128;" ::"l"(reinterpret_cast<char*>(dd) + l * 128) : "memory");
  }
  for (uint32_t i = threadIdx.x; i < W; i += kP3Threads) __stcs(o + i, win[i]);
}

// Fused, persistent P2+P3 with L2 hand-off.  One ticketed work list covers
// both passes: phase b holds the P2 tiles of coarse bucket b interleaved
// (r : 1, r = tiles per window) with the P3 windows of bucket b - lag.  A
// bucket's fine windows are therefore placed while its P2 output (values +
// u16 destinations, ~10 B/element) is still resident in L2: P3 reads them
// from L2, drops the dead destination lines without write-back, and the value
// lines are overwritten in place, so DRAM sees 12 B/element read + 8 B
// written for both passes instead of 22 + 18.  A P3 item only waits for P2
// tiles with smaller tickets, which running CTAs already own: no deadlock.
struct P23Args {
  uint32_t* cur2;    // nb1 * nb2 fine-window append cursors
  uint32_t* done;    // nb1 finished-P2-tile counters
  uint32_t* ticket;  // work-list ticket (first gridDim.x items are implicit)
  uint64_t w1;       // elements per coarse bucket
  uint32_t tp, wp;   // P2 tiles and P3 windows per coarse bucket
  uint32_t r;        // tp / wp
  uint32_t nb1, lag, nitems;
  int w2, nb2;
};

struct P23Item {
  uint32_t kind;  // 0 = P2 tile, 1 = P3 window
  uint32_t bucket, index;
};

__device__ __forceinline__ P23Item p23_decode(uint32_t t, const P23Args& a) {
  const uint32_t head = a.lag * a.tp, phase = a.tp + a.wp, mid = (a.nb1 - a.lag) * phase;
  if (t < head) return {0u, t / a.tp, t % a.tp};
  t -= head;
  if (t < mid) {
    const uint32_t b = a.lag + t / phase, k = t % phase, g = k / (a.r + 1), j = k % (a.r + 1);
    if (j < a.r) return {0u, b, g * a.r + j};
    return {1u, b - a.lag, g};
  }
  t -= mid;
  return {1u, a.nb1 - a.lag + t / a.wp, t % a.wp};
}

template <typename T>
__global__ void __launch_bounds__(kP23Threads, 2) k_part23(const T* __restrict__ tv, const uint32_t* __restrict__ td,
                                                          T* __restrict__ out, uint16_t* __restrict__ od, P23Args a) {
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ uint32_t hist[kMaxB2], start[kMaxB2], wt[32];
  __shared__ unsigned long long delta[kMaxB2];
  __shared__ uint32_t s_next[2];
  const int tid = threadIdx.x;
  const int w2 = a.w2, nb2 = a.nb2;
  const uint32_t fmask = static_cast<uint32_t>(nb2 - 1), wmask = (1u << w2) - 1;
  uint32_t t = blockIdx.x, par = 0, pend = 0;
  while (t < a.nitems) {
    // claim ahead (its latency hides under this item); two slots so a slow reader of the previous claim never
    // sees this one
    if (tid == 0) {
      s_next[par] = gridDim.x + atomicAdd(a.ticket, 1u);
      if (pend) {
        // Release the previous P2 tile: the block barrier that ended it orders every thread's stores before
        // this thread's fence (cumulativity, as in a grid barrier); deferring it to here lets the other warps
        // start this item instead of all waiting for the stores to drain.
        asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(a.done + pend - 1) : "memory");
      }
    }
    pend = 0;
    const P23Item it = p23_decode(t, a);
    if (it.kind == 0) {
      T* sv = reinterpret_cast<T*>(smem);
      uint32_t* sd = reinterpret_cast<uint32_t*>(sv + kP2Tile);
      if (tid < nb2) hist[tid] = 0;
      const uint64_t t0 = static_cast<uint64_t>(it.bucket) * a.w1 + static_cast<uint64_t>(it.index) * kP2Tile;
      T v[kP23Items];
      uint32_t d[kP23Items], rk[kP23Items];
#pragma unroll
      for (int i = 0; i < kP23Items; ++i) {
        v[i] = __ldcs(tv + t0 + tid + i * kP23Threads);
        d[i] = __ldcs(td + t0 + tid + i * kP23Threads);
      }
      __syncthreads();
#pragma unroll
      for (int i = 0; i < kP23Items; ++i) rk[i] = atomicAdd(&hist[(d[i] >> w2) & fmask], 1u);
      __syncthreads();
      scan_bins(hist, start, nb2, wt);
      uint32_t* cur = a.cur2 + static_cast<uint64_t>(it.bucket) * nb2;
      const uint64_t win0 = static_cast<uint64_t>(it.bucket) * a.w1;
      uint32_t g = 0;
      if (tid < nb2) g = atomicAdd(cur + tid, hist[tid]);  // consumed after the scatter (latency hidden)
#pragma unroll
      for (int i = 0; i < kP23Items; ++i) rk[i] += start[(d[i] >> w2) & fmask];
#pragma unroll
      for (int i = 0; i < kP23Items; ++i) {
        sv[rk[i]] = v[i];
        sd[rk[i]] = d[i];
      }
      if (tid < nb2) delta[tid] = win0 + (static_cast<unsigned long long>(tid) << w2) + g - start[tid];
      __syncthreads();
#pragma unroll 4
      for (int s = tid; s < kP2Tile; s += kP23Threads) {
        const uint32_t dd = sd[s];
        const uint64_t pos = delta[(dd >> w2) & fmask] + s;
        out[pos] = sv[s];  // default write-back policy: stays in L2 for the P3 of this bucket
        od[pos] = static_cast<uint16_t>(dd & wmask);
      }
      pend = it.bucket + 1;  // published by thread 0 at the top of the next item (see there)
    } else {
      T* win = reinterpret_cast<T*>(smem);
      if (tid == 0) {
        const uint32_t* flag = a.done + it.bucket;
        uint32_t c;
        while (true) {
          asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(c) : "l"(flag) : "memory");
          if (c >= a.tp) break;
          __nanosleep(256);
        }
      }
      __syncthreads();
      const uint32_t W = 1u << w2;
      const uint64_t w0 = (static_cast<uint64_t>(it.bucket) * a.wp + it.index) << w2;
      T* o = out + w0;
      uint16_t* dd = od + w0;
      constexpr int kU = sizeof(T) <= 8 ? 4 : 2;
      for (uint32_t i0 = tid; i0 < W; i0 += kP23Threads * kU) {
        T v[kU];
        uint16_t d[kU];
#pragma unroll
        for (int u = 0; u < kU; ++u) {
          const uint32_t i = i0 + u * kP23Threads;
          if (i < W) {
            v[u] = __ldcg(o + i);
            d[u] = __ldcg(reinterpret_cast<const unsigned short*>(dd) + i);
          }
        }
#pragma unroll
        for (int u = 0; u < kU; ++u)
          if (i0 + u * kP23Threads < W) win[d[u]] = v[u];
      }
      __syncthreads();
      for (uint32_t l = tid; l < (W * 2) / 128; l += kP23Threads)
        asm volatile("discard.global.L2 [%0], 128;" ::"l"(reinterpret_cast<char*>(dd) + l * 128) : "memory");
      for (uint32_t i = tid; i < W; i += kP23Threads) __stcs(o + i, win[i]);
    }
    __syncthreads();  // s_next visible; shared staging free for the next item
    t = s_next[par];
    par ^= 1;
  }
  if (tid == 0 && pend) asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(a.done + pend - 1) : "memory");
}

template <typename T>
int window_log2() {
  return sizeof(T) == 4 ? 14 : (sizeof(T) == 8 ? 13 : 12);  // 64 KiB smem window
}

// Runtime knobs (read once): BSG_P23=0 selects the separate P2/P3 kernels; BSG_P23_LAG is the bucket lag of
// the fused list; BSG_P23_S2 the fine fan-out (log2) the fused path prefers.
struct PartKnobs {
  int fused = 0, lag = 2, s2 = 7, swz = 1, chunks = 1, prio = 1;
  PartKnobs() {
    if (const char* e = std::getenv("BSG_PART_CHUNKS")) chunks = std::max(1, std::min(kMaxChunks, std::atoi(e)));
    if (const char* e = std::getenv("BSG_PART_PRIO")) prio = std::atoi(e);
    if (const char* e = std::getenv("BSG_P2_SWZ")) swz = std::max(1, std::atoi(e));
    if (const char* e = std::getenv("BSG_P23")) fused = std::atoi(e);
    if (const char* e = std::getenv("BSG_P23_LAG")) lag = std::max(1, std::atoi(e));
    if (const char* e = std::getenv("BSG_P23_S2")) s2 = std::atoi(e);
  }
};
const PartKnobs& knobs() {
  static const PartKnobs k;
  return k;
}

// Coarse/fine split of the bits above the window: (s1, s2) fan-outs.
void part_split(int bits, int w2, bool fused, int& s1, int& s2) {
  const int total = bits - w2;
  s1 = (total + 1) / 2 + BSG_PART_S1_BIAS;
  s2 = total - s1;
  if (fused) {
    const int want2 = knobs().s2, t1 = total - want2;
    if (want2 >= 1 && t1 >= 1 && (1 << t1) <= kMaxB1 && (1 << want2) <= kMaxB2 && bits - t1 >= 12) {
      s1 = t1;
      s2 = want2;
    }
  }
}

// Per-device auxiliary stream (high priority, so P2 blocks are dispatched ahead of queued P1 blocks) and the
// events of the chunked P1/P2 overlap.  Calls on one device are serialised by the caller's context lock.
struct AuxStreams {
  cudaStream_t aux = nullptr;
  cudaEvent_t ev[kMaxChunks] = {};
  cudaEvent_t join = nullptr;
  bool ok = false;
};
AuxStreams& aux_streams() {
  static AuxStreams per_dev[64];
  int dev = 0;
  cudaGetDevice(&dev);
  AuxStreams& x = per_dev[dev & 63];
  if (!x.ok) {
    int lo = 0, hi = 0;
    cudaDeviceGetStreamPriorityRange(&lo, &hi);
    bool good = cudaStreamCreateWithPriority(&x.aux, cudaStreamNonBlocking, knobs().prio ? hi : lo) == cudaSuccess;
    for (int k = 0; k < kMaxChunks && good; ++k)
      good = cudaEventCreateWithFlags(&x.ev[k], cudaEventDisableTiming) == cudaSuccess;
    good = good && cudaEventCreateWithFlags(&x.join, cudaEventDisableTiming) == cudaSuccess;
    x.ok = good;
  }
  return x;
}

template <int KIND, int D, typename T>
cudaError_t run_partition(const PartitionLaunch& a, cudaStream_t s) {
  const int b = a.p.bits;
  const int w2 = window_log2<T>();
  const bool fused = knobs().fused != 0 && BSG_PART_GROUP_MB == 0;
  int s1, s2;
  part_split(b, w2, fused, s1, s2);
  const uint64_t n = 1ULL << b, w1 = 1ULL << (b - s1);
  const int nb1 = 1 << s1, nb2 = 1 << s2;
  uint32_t* cur1 = a.cursors;
  uint32_t* cur2 = a.cursors + nb1;
  uint32_t* done = a.cursors + kMaxB1 + kMaxB1 * kMaxB2;  // fused path: per-bucket P2 completion, then ticket
  cudaError_t e = cudaMemsetAsync(a.cursors, 0, kCursorWords * 4, s);
  if (e != cudaSuccess) return e;
  const size_t sm1 = kP1Tile * (sizeof(T) + 4);
  const size_t sm2 = kP2Tile * (sizeof(T) + 4);
  const size_t sm3 = (size_t{1} << w2) * sizeof(T);
  cudaFuncSetAttribute(k_part1<KIND, D, T>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(sm1));
  T* tv = static_cast<T*>(a.tmp_values);
  const int K = fused ? 1 : static_cast<int>(std::min<uint64_t>(knobs().chunks, n / kP1Tile));
  if (K > 1) {
    // P1 in K chunks on `s`; chunk k's P2 on an auxiliary stream as soon as its cursors are snapshotted.
    uint32_t* snap = done + kMaxB1 + 32;
    AuxStreams& x = aux_streams();
    if (!x.ok) return cudaErrorNotReady;
    const uint64_t tiles = n / kP1Tile, per = tiles / K;
    cudaFuncSetAttribute(k_part2c<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(sm2));
    const uint32_t tpc = static_cast<uint32_t>(w1 / K / kP2Tile + 1);
    for (int k = 0; k < K; ++k) {
      const uint64_t t0 = per * k, nt = (k == K - 1) ? tiles - t0 : per;
      k_part1<KIND, D, T><<<static_cast<unsigned>(nt), kP1Threads, sm1, s>>>(
          static_cast<const T*>(a.in), tv, a.tmp_dest, cur1, a.p, b - s1, nb1, w1, a.dest_in,
          static_cast<uint32_t>(t0));
      k_snap<<<1, 512, 0, s>>>(cur1, snap + k * kMaxB1, nb1);
      cudaEventRecord(x.ev[k], s);
      cudaStreamWaitEvent(x.aux, x.ev[k], 0);
      k_part2c<T><<<static_cast<unsigned>(nb1 * tpc), kP2Threads, sm2, x.aux>>>(
          tv, a.tmp_dest, static_cast<T*>(a.out), a.tmp_dlow, cur2, w2, nb2, w1,
          k ? snap + (k - 1) * kMaxB1 : nullptr, snap + k * kMaxB1, tpc);
    }
    cudaEventRecord(x.join, x.aux);
    cudaStreamWaitEvent(s, x.join, 0);
    cudaFuncSetAttribute(k_place<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(sm3));
    k_place<T><<<static_cast<unsigned>(n >> w2), kP3Threads, sm3, s>>>(static_cast<T*>(a.out), a.tmp_dlow, w2, 0,
                                                                       0);
    note_launch(3 * K + 1);
    return cudaGetLastError();
  }
  k_part1<KIND, D, T><<<static_cast<unsigned>(n / kP1Tile), kP1Threads, sm1, s>>>(
      static_cast<const T*>(a.in), tv, a.tmp_dest, cur1, a.p, b - s1, nb1, w1, a.dest_in, 0u);
  if (fused) {
    const size_t sm23 = std::max(sm2, sm3);
    cudaFuncSetAttribute(k_part23<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(sm23));
    int dev = 0, sms = 148, per = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_part23<T>, kP23Threads, sm23);
    P23Args g;
    g.cur2 = cur2;
    g.done = done;
    g.ticket = done + kMaxB1;
    g.w1 = w1;
    g.tp = static_cast<uint32_t>(w1 / kP2Tile);
    g.wp = static_cast<uint32_t>(w1 >> w2);
    g.r = g.tp / g.wp;
    g.nb1 = static_cast<uint32_t>(nb1);
    g.lag = static_cast<uint32_t>(std::min(knobs().lag, nb1 - 1));
    g.nitems = static_cast<uint32_t>(nb1) * (g.tp + g.wp);
    g.w2 = w2;
    g.nb2 = nb2;
    const uint32_t grid = std::min<uint32_t>(g.nitems, static_cast<uint32_t>(sms) * std::max(per, 1));
    k_part23<T><<<grid, kP23Threads, sm23, s>>>(tv, a.tmp_dest, static_cast<T*>(a.out), a.tmp_dlow, g);
    note_launch(2);
    return cudaGetLastError();
  }
  cudaFuncSetAttribute(k_part2<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(sm2));
  cudaFuncSetAttribute(k_place<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(sm3));
  // Grouped mode: P2 and P3 alternate over groups of coarse buckets sized to stay resident in L2, so P3
  // reads P2's output from L2 and its dead destination lines are discarded instead of written back.
  const uint64_t bucket_bytes = w1 * (sizeof(T) + 2);
  const uint64_t group = BSG_PART_GROUP_MB > 0
                             ? std::max<uint64_t>(1, (static_cast<uint64_t>(BSG_PART_GROUP_MB) << 20) / bucket_bytes)
                             : static_cast<uint64_t>(nb1);
  uint64_t launched = 1;
  for (uint64_t c0 = 0; c0 < static_cast<uint64_t>(nb1); c0 += group) {
    const uint64_t cn = std::min<uint64_t>(group, nb1 - c0);
#ifndef BSG_P2_PERSISTENT
#define BSG_P2_PERSISTENT 0
#endif
    if (BSG_P2_PERSISTENT) {
      const size_t smp = kP2Tile * 2 * (sizeof(T) + 4);
      cudaFuncSetAttribute(k_part2p<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smp));
      int dev = 0, sms = 148, per = 1;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_part2p<T>, kP2Threads, smp);
      const uint64_t ntiles = cn * w1 / kP2Tile;
      const uint64_t g = std::min<uint64_t>(ntiles, static_cast<uint64_t>(sms) * std::max(per, 1));
      k_part2p<T><<<static_cast<unsigned>(g), kP2Threads, smp, s>>>(tv, a.tmp_dest, static_cast<T*>(a.out),
                                                                      a.tmp_dlow, cur2, w2, nb2, w1,
                                                                      c0 * w1 / kP2Tile, ntiles);
    } else {
      k_part2<T><<<static_cast<unsigned>(cn * w1 / kP2Tile), kP2Threads, sm2, s>>>(
          tv, a.tmp_dest, static_cast<T*>(a.out), a.tmp_dlow, cur2, w2, nb2, w1, c0 * w1 / kP2Tile,
          static_cast<uint32_t>(std::min<uint64_t>(knobs().swz, cn)));
    }
    k_place<T><<<static_cast<unsigned>(cn * w1 >> w2), kP3Threads, sm3, s>>>(
        static_cast<T*>(a.out), a.tmp_dlow, w2, c0 * w1 >> w2, BSG_PART_GROUP_MB > 0 ? 1 : 0);
    launched += 2;
  }
  note_launch(launched);
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

bool partition_eligible(int elem_code, int bits) {
  int w2;
  switch (elem_code) {
    case 4: w2 = 14; break;
    case 8: w2 = 13; break;
    case 16: w2 = 12; break;
    default: return false;
  }
  const int total = bits - w2;
  const int s1 = (total + 1) / 2 + BSG_PART_S1_BIAS, s2 = total - s1;
  // fan-outs within the shared-memory histograms; tiles must not straddle buckets; 32-bit destinations
  return bits <= 32 && s1 >= 1 && s2 >= 1 && (1 << s1) <= kMaxB1 && (1 << s2) <= kMaxB2 &&
         (bits - s1) >= 12 && bits >= 14;
}

size_t partition_workspace_bytes(int elem_code, int bits) {
  const uint64_t n = 1ULL << bits;
  return n * static_cast<uint64_t>(elem_code) + n * 4 + n * 2 + kCursorWords * 4 + 3 * 256;
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
