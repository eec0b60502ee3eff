// Kernel instantiations for payload type IdxTag (see bsg_dispatch.cuh).
#include "bsg_dispatch.cuh"

namespace bsg {
template cudaError_t dispatch_shuffle<IdxTag>(const ShuffleLaunch&, cudaStream_t);
}  // namespace bsg
