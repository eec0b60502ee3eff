// bsg_launch.cu -- non-template launchers: payload-type switch, bijection map,
// count-only pass, byte-generic gather, launch accounting.
#include <atomic>

#include "bsg_kernels.cuh"
#include "bsg_payload.h"

namespace bsg {

namespace {
std::atomic<uint64_t> g_launches{0};
}

void note_launch(uint64_t k) { g_launches.fetch_add(k, std::memory_order_relaxed); }
uint64_t launches() { return g_launches.load(std::memory_order_relaxed); }

cudaError_t launch_shuffle(int elem_code, const ShuffleLaunch& a, cudaStream_t s) {
  switch (elem_code) {
    case 0: return dispatch_shuffle<IdxTag>(a, s);
    case 1: return dispatch_shuffle<uint8_t>(a, s);
    case 2: return dispatch_shuffle<uint16_t>(a, s);
    case 4: return dispatch_shuffle<uint32_t>(a, s);
    case 8: return dispatch_shuffle<uint64_t>(a, s);
    case 16: return dispatch_shuffle<uint4>(a, s);
  }
  return cudaErrorInvalidValue;
}

bool batched_supported(int elem_code, uint32_t m, int bits, int rounds) {
  if (elem_code != 1 && elem_code != 2 && elem_code != 4 && elem_code != 8 && elem_code != 16) return false;
  if (bits > 16 || rounds > kBatchedMaxRounds) return false;
  return static_cast<uint64_t>(m) * elem_code <= 96u * 1024u;  // two row buffers in shared memory
}

cudaError_t launch_batched(int elem_code, const BatchedLaunch& a, cudaStream_t s) {
  switch (elem_code) {
    case 1: return dispatch_batched<uint8_t>(a, s);
    case 2: return dispatch_batched<uint16_t>(a, s);
    case 4: return dispatch_batched<uint32_t>(a, s);
    case 8: return dispatch_batched<uint64_t>(a, s);
    case 16: return dispatch_batched<uint4>(a, s);
  }
  return cudaErrorNotSupported;
}

cudaError_t launch_gather(int elem_code, const void* src, const uint64_t* idx, void* out, uint64_t n,
                          cudaStream_t s) {
  switch (elem_code) {
    case 1: return dispatch_gather<uint8_t>(src, idx, out, n, s);
    case 2: return dispatch_gather<uint16_t>(src, idx, out, n, s);
    case 4: return dispatch_gather<uint32_t>(src, idx, out, n, s);
    case 8: return dispatch_gather<uint64_t>(src, idx, out, n, s);
    case 16: return dispatch_gather<uint4>(src, idx, out, n, s);
  }
  return cudaErrorInvalidValue;
}

// One warp per element: lanes copy 4-byte words (or bytes) of the record.
__global__ void k_gather_bytes(const unsigned char* __restrict__ src, const uint64_t* __restrict__ idx,
                               unsigned char* __restrict__ out, uint64_t n, uint32_t eb, bool words) {
  const uint64_t warp = (static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const uint64_t nwarps = (static_cast<uint64_t>(gridDim.x) * blockDim.x) >> 5;
  for (uint64_t i = warp; i < n; i += nwarps) {
    const unsigned char* s = src + idx[i] * eb;
    unsigned char* d = out + i * eb;
    if (words) {
      for (uint32_t w = lane; w < eb / 4; w += 32)
        reinterpret_cast<uint32_t*>(d)[w] = __ldg(reinterpret_cast<const uint32_t*>(s) + w);
    } else {
      for (uint32_t b = lane; b < eb; b += 32) d[b] = __ldg(s + b);
    }
  }
}

cudaError_t launch_gather_bytes(const void* src, const uint64_t* idx, void* out, uint64_t n, uint32_t eb,
                                cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  const bool words = (eb % 4 == 0) && (reinterpret_cast<uintptr_t>(src) % 4 == 0) &&
                     (reinterpret_cast<uintptr_t>(out) % 4 == 0);
  const uint64_t warps_needed = n;
  const uint64_t blocks = (warps_needed * 32 + kThreads - 1) / kThreads;
  const unsigned grid = static_cast<unsigned>(blocks < 148ull * 64 ? blocks : 148ull * 64);
  k_gather_bytes<<<grid, kThreads, 0, s>>>(static_cast<const unsigned char*>(src), idx,
                                           static_cast<unsigned char*>(out), n, eb, words);
  note_launch();
  return cudaGetLastError();
}

template <int KIND, bool INV>
__global__ void __launch_bounds__(kThreads) k_map(const uint64_t* __restrict__ x, uint64_t* __restrict__ y,
                                                  uint64_t n, uint64_t start, BijParams p) {
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
    const uint64_t v = x ? x[i] : start + i;
    uint64_t r;
    if constexpr (KIND == kKindLcg) {
      r = INV ? lcg_inv(v, p) : lcg_fwd(v, p);
    } else {
      constexpr int D = (KIND == kKindPh1 || KIND == kKindPh1G) ? 1 : 0;
      constexpr int NR = (KIND == kKindPh0 || KIND == kKindPh1) ? 24 : 0;
      r = INV ? philox_inv<D, NR>(v, p) : philox_fwd<D, NR>(v, p);
    }
    y[i] = r;
  }
}

template <int KIND>
cudaError_t map_kind(const uint64_t* x, uint64_t* y, uint64_t n, uint64_t start, const BijParams& p, bool inv,
                     cudaStream_t s) {
  const uint64_t blocks = (n + kThreads - 1) / kThreads;
  const unsigned grid = static_cast<unsigned>(blocks < 148ull * 32 ? blocks : 148ull * 32);
  if (inv) k_map<KIND, true><<<grid, kThreads, 0, s>>>(x, y, n, start, p);
  else k_map<KIND, false><<<grid, kThreads, 0, s>>>(x, y, n, start, p);
  note_launch();
  return cudaGetLastError();
}

cudaError_t launch_map(const uint64_t* x, uint64_t* y, uint64_t n, uint64_t start, const BijParams& p, bool inverse,
                       cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  switch (kind_of(p)) {
    case kKindLcg: return map_kind<kKindLcg>(x, y, n, start, p, inverse, s);
    case kKindPh0: return map_kind<kKindPh0>(x, y, n, start, p, inverse, s);
    case kKindPh1: return map_kind<kKindPh1>(x, y, n, start, p, inverse, s);
    case kKindPh0G: return map_kind<kKindPh0G>(x, y, n, start, p, inverse, s);
    case kKindPh1G: return map_kind<kKindPh1G>(x, y, n, start, p, inverse, s);
  }
  return cudaErrorInvalidValue;
}

__global__ void k_store_u64(unsigned long long* p, unsigned long long v) { *p = v; }

// Writes a known survivor count on the stream (closed form for power-of-two ranges) without a host sync.
cudaError_t launch_store_u64(unsigned long long* p, uint64_t v, cudaStream_t s) {
  k_store_u64<<<1, 1, 0, s>>>(p, v);
  note_launch();
  return cudaGetLastError();
}

// Count-only pass: survivors among counters [c0, c1) (multi-GPU pre-count).
template <int KIND>
__global__ void __launch_bounds__(kThreads) k_count(uint64_t m, uint64_t c0, uint64_t c1, BijParams p,
                                                    unsigned long long* count) {
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  uint32_t local = 0;
  for (uint64_t c = c0 + static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; c < c1; c += stride)
    local += bij<KIND, uint64_t>(c, p) < m ? 1u : 0u;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) local += __shfl_xor_sync(0xFFFFFFFFu, local, o);
  if ((threadIdx.x & 31) == 0 && local) atomicAdd(count, static_cast<unsigned long long>(local));
}

cudaError_t launch_count(uint64_t m, uint64_t c0, uint64_t c1, const BijParams& p, unsigned long long* count,
                         cudaStream_t s) {
  cudaError_t e = cudaMemsetAsync(count, 0, sizeof(unsigned long long), s);
  if (e != cudaSuccess || c1 <= c0) return e;
  const uint64_t blocks = (c1 - c0 + kThreads - 1) / kThreads;
  const unsigned grid = static_cast<unsigned>(blocks < 148ull * 16 ? blocks : 148ull * 16);
  switch (kind_of(p)) {
    case kKindLcg: k_count<kKindLcg><<<grid, kThreads, 0, s>>>(m, c0, c1, p, count); break;
    case kKindPh0: k_count<kKindPh0><<<grid, kThreads, 0, s>>>(m, c0, c1, p, count); break;
    case kKindPh1: k_count<kKindPh1><<<grid, kThreads, 0, s>>>(m, c0, c1, p, count); break;
    case kKindPh0G: k_count<kKindPh0G><<<grid, kThreads, 0, s>>>(m, c0, c1, p, count); break;
    case kKindPh1G: k_count<kKindPh1G><<<grid, kThreads, 0, s>>>(m, c0, c1, p, count); break;
  }
  note_launch();
  return cudaGetLastError();
}

}  // namespace bsg
