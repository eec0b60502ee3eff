// Kernel instantiations for payload type uint32_t (see bsg_dispatch.cuh).
#include "bsg_dispatch.cuh"

namespace bsg {
template cudaError_t dispatch_shuffle<uint32_t>(const ShuffleLaunch&, cudaStream_t);
template cudaError_t dispatch_batched<uint32_t>(const BatchedLaunch&, cudaStream_t);
template cudaError_t dispatch_gather<uint32_t>(const void*, const uint64_t*, void*, uint64_t, cudaStream_t);
}  // namespace bsg
