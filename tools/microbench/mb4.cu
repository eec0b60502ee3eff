// Random 8-byte gathers over a 4 GiB array with different load flavours and
// L2 fetch-granularity limits: how many DRAM bytes does one random read cost?
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mb4 mb4.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); exit(1);} } while (0)

__device__ __forceinline__ uint32_t hsh(uint32_t i) {
  i ^= i >> 16; i *= 0x7feb352dU; i ^= i >> 15; i *= 0x846ca68bU; i ^= i >> 16; return i;
}

template <int V>
__device__ __forceinline__ uint64_t ld(const uint64_t* p) {
  uint64_t v;
  if (V == 0) asm volatile("ld.global.nc.L1::no_allocate.u64 %0, [%1];" : "=l"(v) : "l"(p));
  if (V == 1) asm volatile("ld.global.cg.u64 %0, [%1];" : "=l"(v) : "l"(p));
  if (V == 2) asm volatile("ld.global.ca.u64 %0, [%1];" : "=l"(v) : "l"(p));
  if (V == 3) asm volatile("ld.global.cv.u64 %0, [%1];" : "=l"(v) : "l"(p));
  if (V == 4) asm volatile("ld.global.nc.L2::64B.u64 %0, [%1];" : "=l"(v) : "l"(p));
  if (V == 5) asm volatile("ld.global.L1::evict_first.u64 %0, [%1];" : "=l"(v) : "l"(p));
  if (V == 6) asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p));
  if (V == 7) asm volatile("ld.global.nc.L1::no_allocate.L2::256B.u64 %0, [%1];" : "=l"(v) : "l"(p));
  return v;
}

template <int V>
__global__ void __launch_bounds__(256) k_gather(const uint64_t* __restrict__ in, uint64_t* __restrict__ out,
                                                uint32_t smask) {
  const uint32_t base = blockIdx.x * 2048 + threadIdx.x;
  uint64_t v[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) v[j] = ld<V>(in + (hsh(base + j * 256) & smask));
#pragma unroll
  for (int j = 0; j < 8; ++j) __stcs(out + base + j * 256, v[j]);
}

__global__ void k_fill(uint64_t* p, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) p[i] = i;
}

int main(int argc, char** argv) {
  const int gran = argc > 1 ? atoi(argv[1]) : -1;
  if (gran >= 0) CK(cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, gran));
  size_t g = 0;
  CK(cudaDeviceGetLimit(&g, cudaLimitMaxL2FetchGranularity));
  printf("L2 fetch granularity limit: requested %d, reads back %zu\n", gran, g);
  cudaEvent_t e0, e1; CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
  const uint32_t n = 1u << 28, S = 1u << 29;
  uint64_t *in, *out;
  CK(cudaMalloc(&in, (size_t)S * 8)); CK(cudaMalloc(&out, (size_t)n * 8));
  k_fill<<<4096, 256>>>(in, S);
  auto run = [&](auto kern, const char* name) {
    for (int r = 0; r < 2; ++r) kern<<<n / 2048, 256>>>(in, out, S - 1);
    CK(cudaEventRecord(e0));
    for (int r = 0; r < 5; ++r) kern<<<n / 2048, 256>>>(in, out, S - 1);
    CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1)); CK(cudaGetLastError());
    float ms; CK(cudaEventElapsedTime(&ms, e0, e1)); ms /= 5;
    printf("%-36s %7.3f ms  %6.1f G random reads/s\n", name, ms, n / ms / 1e6);
  };
  run(k_gather<0>, "ld.global.nc.L1::no_allocate");
  run(k_gather<1>, "ld.global.cg");
  run(k_gather<2>, "ld.global.ca");
  run(k_gather<3>, "ld.global.cv");
  run(k_gather<4>, "ld.global.nc.L2::64B");
  run(k_gather<5>, "ld.global.L1::evict_first");
  run(k_gather<6>, "ld.relaxed.gpu");
  run(k_gather<7>, "ld.global.nc.L2::256B");
  return 0;
}
