// bsg_baselines.cu -- the paper's GPU comparator, SortShuffle:
// give every value a random 64-bit key and radix-sort the (key, value) pairs
// with CUB.  Keys follow the reference's bench_sort_shuffle
// (proj/include/bijshuf/bench.hpp:117-123): key_i = mix64(stream + i*gamma),
// stream = mix64(seed).  This is a baseline for bench.py, not the product path.
#include <cub/device/device_radix_sort.cuh>

#include "bsg_internal.h"

namespace bsg {

__global__ void k_sort_keys(uint64_t* __restrict__ keys, uint64_t n, uint64_t stream) {
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride)
    keys[i] = mix64(stream + i * kGamma);
}

// temp == nullptr: *temp_bytes receives the workspace size.
cudaError_t sort_shuffle_u64(const uint64_t* in, uint64_t* out, uint64_t n, uint64_t seed, void* temp,
                             size_t* temp_bytes, cudaStream_t s) {
  size_t cub_bytes = 0;
  cudaError_t e = cub::DeviceRadixSort::SortPairs(nullptr, cub_bytes, static_cast<const uint64_t*>(nullptr),
                                                  static_cast<uint64_t*>(nullptr), in, out, static_cast<int64_t>(n),
                                                  0, 64, s);
  if (e != cudaSuccess) return e;
  const size_t keys_bytes = ((n * 8 + 255) / 256) * 256;
  const size_t need = 2 * keys_bytes + cub_bytes;
  if (temp == nullptr) {
    *temp_bytes = need;
    return cudaSuccess;
  }
  if (*temp_bytes < need) return cudaErrorInvalidValue;
  uint64_t* keys_in = static_cast<uint64_t*>(temp);
  uint64_t* keys_out = reinterpret_cast<uint64_t*>(static_cast<char*>(temp) + keys_bytes);
  void* cub_tmp = static_cast<char*>(temp) + 2 * keys_bytes;
  k_sort_keys<<<148 * 8, 256, 0, s>>>(keys_in, n, mix64(seed));
  note_launch();
  e = cub::DeviceRadixSort::SortPairs(cub_tmp, cub_bytes, keys_in, keys_out, in, out, static_cast<int64_t>(n), 0,
                                      64, s);
  note_launch(8);  // CUB onesweep: histogram + 8 digit passes (approximate count)
  return e;
}

}  // namespace bsg
