// Kernel instantiations for payload type uint4 (see bsg_dispatch.cuh).
#include "bsg_dispatch.cuh"

namespace bsg {
template cudaError_t dispatch_shuffle<uint4>(const ShuffleLaunch&, cudaStream_t);
template cudaError_t dispatch_batched<uint4>(const BatchedLaunch&, cudaStream_t);
template cudaError_t dispatch_gather<uint4>(const void*, const uint64_t*, void*, uint64_t, cudaStream_t);
}  // namespace bsg
