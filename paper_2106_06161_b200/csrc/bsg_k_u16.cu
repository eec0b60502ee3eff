// Kernel instantiations for payload type uint16_t (see bsg_dispatch.cuh).
#include "bsg_dispatch.cuh"

namespace bsg {
template cudaError_t dispatch_shuffle<uint16_t>(const ShuffleLaunch&, cudaStream_t);
template cudaError_t dispatch_batched<uint16_t>(const BatchedLaunch&, cudaStream_t);
template cudaError_t dispatch_gather<uint16_t>(const void*, const uint64_t*, void*, uint64_t, cudaStream_t);
}  // namespace bsg
