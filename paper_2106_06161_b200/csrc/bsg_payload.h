// bsg_payload.h -- per-payload-type entry points, explicitly instantiated in
// bsg_k_<type>.cu (one translation unit per type, compiled in parallel).
#pragma once

#include "bsg_internal.h"

namespace bsg {

template <typename T>
cudaError_t dispatch_shuffle(const ShuffleLaunch& a, cudaStream_t s);
template <typename T>
cudaError_t dispatch_batched(const BatchedLaunch& a, cudaStream_t s);
template <typename T>
cudaError_t dispatch_gather(const void* src, const uint64_t* idx, void* out, uint64_t n, cudaStream_t s);

}  // namespace bsg
