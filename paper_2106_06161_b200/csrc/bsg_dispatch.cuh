// bsg_dispatch.cuh -- template dispatch from a ShuffleLaunch to a concrete
// kernel instantiation.  Included by one translation unit per payload type
// (bsg_k_*.cu) so the instantiations compile in parallel.
#pragma once

#include <type_traits>

#include "bsg_kernels.cuh"
#include "bsg_payload.h"

namespace bsg {

template <int KIND, typename CT, typename T, bool SH>
cudaError_t run_shuffle(const ShuffleLaunch& a, cudaStream_t s) {
  const uint64_t len = a.c1 - a.c0;
  if (len == 0) return cudaSuccess;
  if (!a.compact) {
    constexpr uint64_t kTile = kThreads * kPow2Items;
    const uint64_t grid = (len + kTile - 1) / kTile;
    if (grid > 0x7FFFFFFFull) return cudaErrorInvalidConfiguration;
    k_pow2<KIND, CT, T, SH, kPow2Items><<<static_cast<unsigned>(grid), kThreads, 0, s>>>(a.src, a.out, a.c0, a.c1,
                                                                                         a.p);
  } else {
    // 16-byte payloads keep 8 items so the static shared staging stays under 48 KiB.
    constexpr int kItems = (sizeof(T) >= 16) ? 8 : kCompactItems;
    constexpr uint64_t kTile = kThreads * kItems;
    const uint64_t grid = (len + kTile - 1) / kTile;
    if (grid > 0x7FFFFFFFull) return cudaErrorInvalidConfiguration;
    if constexpr (sizeof(T) >= 4 || std::is_same<T, IdxTag>::value) {
      k_compact_smem<KIND, CT, T, SH, kItems><<<static_cast<unsigned>(grid), kThreads, 0, s>>>(
          a.src, a.out, a.m, a.c0, a.c1, a.p, a.lb, a.count_out);
    } else {
      constexpr uint64_t kTileR = kThreads * kCompactItems;
      const uint64_t gridr = (len + kTileR - 1) / kTileR;
      k_compact<KIND, CT, T, SH, kCompactItems><<<static_cast<unsigned>(gridr), kThreads, 0, s>>>(
          a.src, a.out, a.m, a.c0, a.c1, a.p, a.lb, a.count_out);
    }
  }
  note_launch();
  return cudaGetLastError();
}

template <int KIND, typename CT, typename T>
cudaError_t run_sh(const ShuffleLaunch& a, cudaStream_t s) {
  if constexpr (!std::is_same<T, IdxTag>::value) {
    if (a.src.nshards > 0) return run_shuffle<KIND, CT, T, true>(a, s);
  }
  return run_shuffle<KIND, CT, T, false>(a, s);
}

template <typename T>
cudaError_t dispatch_shuffle(const ShuffleLaunch& a, cudaStream_t s) {
  const bool narrow = a.p.bits <= 32;
  switch (kind_of(a.p)) {
    case kKindLcg:
      return narrow ? run_sh<kKindLcg, uint32_t, T>(a, s) : run_sh<kKindLcg, uint64_t, T>(a, s);
    case kKindPh0:
      return narrow ? run_sh<kKindPh0, uint32_t, T>(a, s) : run_sh<kKindPh0, uint64_t, T>(a, s);
    case kKindPh1:
      return narrow ? run_sh<kKindPh1, uint32_t, T>(a, s) : run_sh<kKindPh1, uint64_t, T>(a, s);
    case kKindPh0G:
      return run_sh<kKindPh0G, uint64_t, T>(a, s);
    case kKindPh1G:
      return run_sh<kKindPh1G, uint64_t, T>(a, s);
  }
  return cudaErrorInvalidValue;
}

template <int KIND, typename T, int NT>
cudaError_t run_batched_nt(const BatchedLaunch& a, cudaStream_t s) {
  const size_t row_bytes = static_cast<size_t>(a.m) * sizeof(T);
  const size_t stride = (row_bytes + 15) / 16 * 16;
  const size_t smem = 2 * stride;  // double-buffered rows
  int mode = 0;
  const uintptr_t base = reinterpret_cast<uintptr_t>(a.in);
  if (row_bytes % 16 == 0 && base % 16 == 0) mode = 1;
  else if (row_bytes % 4 == 0 && base % 4 == 0) mode = 2;
  auto kern = k_batched<KIND, T, NT>;
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    if (e != cudaSuccess) return e;
  }
  int dev = 0, sms = 148, per_sm = 1;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, NT, smem);
  if (per_sm < 1) return cudaErrorNotSupported;
  // Every CTA takes the same number of rows (ceil(batch / resident)), so the last wave has no stragglers.
  const uint64_t resident = static_cast<uint64_t>(sms) * per_sm;
  const uint64_t rows_per_cta = (a.batch + resident - 1) / resident;
  const uint64_t grid = (a.batch + rows_per_cta - 1) / rows_per_cta;
  kern<<<static_cast<unsigned>(grid), NT, smem, s>>>(static_cast<const T*>(a.in), static_cast<T*>(a.out), a.batch,
                                                      a.m, a.seed, a.p, mode, static_cast<uint32_t>(stride));
  note_launch();
  return cudaGetLastError();
}

// Block size by row length: about 16 counters per thread for short rows (C4: 1024 counters -> 64 threads).
#ifndef BSG_BATCHED_PER_THREAD
#define BSG_BATCHED_PER_THREAD 16
#endif
template <int KIND, typename T>
cudaError_t run_batched(const BatchedLaunch& a, cudaStream_t s) {
  const uint64_t n = 1ULL << a.p.bits;
  if (n <= 64 * BSG_BATCHED_PER_THREAD) return run_batched_nt<KIND, T, 64>(a, s);
  if (n <= 128 * BSG_BATCHED_PER_THREAD) return run_batched_nt<KIND, T, 128>(a, s);
  return run_batched_nt<KIND, T, kThreads>(a, s);
}

template <typename T>
cudaError_t dispatch_batched(const BatchedLaunch& a, cudaStream_t s) {
  switch (kind_of(a.p)) {
    case kKindLcg: return run_batched<kKindLcg, T>(a, s);
    case kKindPh0: return run_batched<kKindPh0, T>(a, s);
    case kKindPh1: return run_batched<kKindPh1, T>(a, s);
    case kKindPh0G: return run_batched<kKindPh0G, T>(a, s);
    case kKindPh1G: return run_batched<kKindPh1G, T>(a, s);
  }
  return cudaErrorInvalidValue;
}

template <typename T>
cudaError_t dispatch_gather(const void* src, const uint64_t* idx, void* out, uint64_t n, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  constexpr uint64_t kTile = kThreads * 8;
  const uint64_t grid = (n + kTile - 1) / kTile;
  k_gather<T, 8><<<static_cast<unsigned>(grid), kThreads, 0, s>>>(static_cast<const T*>(src), idx,
                                                                   static_cast<T*>(out), n);
  note_launch();
  return cudaGetLastError();
}

}  // namespace bsg
