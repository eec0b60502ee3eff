// Random-read footprint sweep: out[i] = in[h(i) mod S] for S from 2^20 to 2^31 u64
// elements, n = 2^28 outputs.  Separates L2 / TLB / DRAM-activation limits of the
// random gather that bounds the bijective shuffle.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mb2 mb2.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); exit(1);} } while (0)

__device__ __forceinline__ uint32_t hsh(uint32_t i) {
  i ^= i >> 16; i *= 0x7feb352dU; i ^= i >> 15; i *= 0x846ca68bU; i ^= i >> 16; return i;
}

template <typename T, int ITEMS>
__global__ void __launch_bounds__(256) k_gather(const T* __restrict__ in, T* __restrict__ out, uint32_t smask,
                                                uint32_t win_shift) {
  const uint32_t base = blockIdx.x * blockDim.x * ITEMS + threadIdx.x;
  T v[ITEMS];
#pragma unroll
  for (int j = 0; j < ITEMS; ++j) {
    uint32_t i = base + j * blockDim.x;
    // windowed: high bits of i select a window, low bits random inside it
    uint32_t idx = ((i >> win_shift) << win_shift) + (hsh(i) & ((1u << win_shift) - 1));
    v[j] = __ldg(in + (idx & smask));
  }
#pragma unroll
  for (int j = 0; j < ITEMS; ++j) out[base + j * blockDim.x] = v[j];
}

__global__ void k_fill(uint64_t* p, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) p[i] = i;
}

int main() {
  cudaEvent_t e0, e1; CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
  const uint32_t n = 1u << 28;
  const size_t maxS = 1ull << 31;
  uint64_t *in, *out;
  CK(cudaMalloc(&in, maxS * 8)); CK(cudaMalloc(&out, (size_t)n * 16));
  k_fill<<<4096, 256>>>(in, maxS);
  // u64 footprint sweep, fully random
  for (int S = 20; S <= 31; ++S) {
    const uint32_t smask = (S >= 32) ? 0xFFFFFFFFu : ((1u << S) - 1);
    for (int r = 0; r < 3; ++r) k_gather<uint64_t, 8><<<n / 2048, 256>>>(in, out, smask, 31);
    CK(cudaEventRecord(e0));
    for (int r = 0; r < 5; ++r) k_gather<uint64_t, 8><<<n / 2048, 256>>>(in, out, smask, 31);
    CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1)); CK(cudaGetLastError());
    float ms; CK(cudaEventElapsedTime(&ms, e0, e1)); ms /= 5;
    printf("u64  S=2^%-2d (%8.1f MB)  %7.3f ms  %6.1f Gelem/s  eff %7.1f GB/s\n", S, (double)(1ull << S) * 8 / 1e6, ms,
           n / ms / 1e6, 2.0 * n * 8 / ms / 1e6);
  }
  // windowed: S = 2^31 but concurrent accesses confined to a moving window of 2^w elements
  for (int w = 16; w <= 28; w += 2) {
    for (int r = 0; r < 3; ++r) k_gather<uint64_t, 8><<<n / 2048, 256>>>(in, out, 0xFFFFFFFFu, w);
    CK(cudaEventRecord(e0));
    for (int r = 0; r < 5; ++r) k_gather<uint64_t, 8><<<n / 2048, 256>>>(in, out, 0xFFFFFFFFu, w);
    CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1)); CK(cudaGetLastError());
    float ms; CK(cudaEventElapsedTime(&ms, e0, e1)); ms /= 5;
    printf("u64  window=2^%-2d (%8.1f MB)  %7.3f ms  %6.1f Gelem/s  eff %7.1f GB/s\n", w, (double)(1ull << w) * 8 / 1e6,
           ms, n / ms / 1e6, 2.0 * n * 8 / ms / 1e6);
  }
  // 16-byte and 4-byte elements, fully random over 4 GiB-ish footprints
  for (int S : {24, 28}) {
    const uint32_t smask = (1u << S) - 1;
    for (int r = 0; r < 3; ++r) k_gather<ulonglong2, 8><<<n / 2048, 256>>>((const ulonglong2*)in, (ulonglong2*)out, smask, 31);
    CK(cudaEventRecord(e0));
    for (int r = 0; r < 5; ++r) k_gather<ulonglong2, 8><<<n / 2048, 256>>>((const ulonglong2*)in, (ulonglong2*)out, smask, 31);
    CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1)); CK(cudaGetLastError());
    float ms; CK(cudaEventElapsedTime(&ms, e0, e1)); ms /= 5;
    printf("u128 S=2^%-2d (%8.1f MB)  %7.3f ms  %6.1f Gelem/s  eff %7.1f GB/s\n", S, (double)(1ull << S) * 16 / 1e6, ms,
           n / ms / 1e6, 2.0 * n * 16 / ms / 1e6);
  }
  for (int S : {24, 30, 31}) {
    const uint32_t smask = (1u << S) - 1;
    for (int r = 0; r < 3; ++r) k_gather<uint32_t, 8><<<n / 2048, 256>>>((const uint32_t*)in, (uint32_t*)out, smask, 31);
    CK(cudaEventRecord(e0));
    for (int r = 0; r < 5; ++r) k_gather<uint32_t, 8><<<n / 2048, 256>>>((const uint32_t*)in, (uint32_t*)out, smask, 31);
    CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1)); CK(cudaGetLastError());
    float ms; CK(cudaEventElapsedTime(&ms, e0, e1)); ms /= 5;
    printf("u32  S=2^%-2d (%8.1f MB)  %7.3f ms  %6.1f Gelem/s  eff %7.1f GB/s\n", S, (double)(1ull << S) * 4 / 1e6, ms,
           n / ms / 1e6, 2.0 * n * 4 / ms / 1e6);
  }
  return 0;
}
