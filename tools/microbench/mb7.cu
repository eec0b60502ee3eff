// Window placement through distributed shared memory: can one thread-block
// cluster place a (CL x 2^W)-element window (values + in-window destinations,
// read sequentially) by scattering into the cluster's shared memory, then
// write it back coalesced?  This is the candidate second pass of a two-pass
// partitioned shuffle (P1 routes into n / (CL*2^W) buckets).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mb7 mb7.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); exit(1);} } while (0)

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// One cluster per window; CTA r reads list slice r and owns output slice r.
template <int CL, int W, int T>
__global__ void __launch_bounds__(T) k_place_cluster(const uint64_t* __restrict__ vals, const uint32_t* __restrict__ dst,
                                                     uint64_t* __restrict__ out) {
  extern __shared__ __align__(16) uint64_t win[];
  constexpr uint32_t S = 1u << W;  // per-CTA slice
  const uint32_t r = CL > 1 ? cluster_rank() : 0;
  const uint64_t cl = blockIdx.x / CL;
  const uint64_t base = (cl * CL + r) * S;
  const uint32_t lwin = static_cast<uint32_t>(__cvta_generic_to_shared(win));
  uint32_t rbase[CL];
#pragma unroll
  for (int q = 0; q < CL; ++q) {
    if (CL > 1) asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(rbase[q]) : "r"(lwin), "r"(q));
    else rbase[q] = lwin;
  }
  if (CL > 1) cluster_sync();  // every CTA of the cluster is running before remote stores
  constexpr int U = 8;
  for (uint32_t i0 = threadIdx.x; i0 < S; i0 += T * U) {
    uint64_t v[U];
    uint32_t d[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      v[u] = __ldcs(vals + base + i0 + u * T);
      d[u] = __ldcs(dst + base + i0 + u * T);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint32_t q = d[u] >> W, off = (d[u] & (S - 1)) * 8;
      uint32_t a = rbase[0];
#pragma unroll
      for (int k = 1; k < CL; ++k) a = (q == static_cast<uint32_t>(k)) ? rbase[k] : a;
      if (CL > 1) asm volatile("st.shared::cluster.u64 [%0], %1;" ::"r"(a + off), "l"(v[u]) : "memory");
      else asm volatile("st.shared.u64 [%0], %1;" ::"r"(a + off), "l"(v[u]) : "memory");
    }
  }
  if (CL > 1) cluster_sync();
  else __syncthreads();
  for (uint32_t i = threadIdx.x; i < S; i += T) __stcs(out + base + i, win[i]);
}

__device__ __forceinline__ uint32_t perm_in(uint32_t i, uint32_t w, int bits) {
  const uint32_t m = (bits >= 32) ? 0xFFFFFFFFu : ((1u << bits) - 1);
  uint32_t x = (i * 0x9E3779B1u + w * 0x85EBCA77u) & m;
  x ^= x >> (bits / 2 + 1);
  x = (x * 0xC2B2AE3Du) & m;
  x ^= x >> (bits / 3 + 1);
  x = (x * 0x27D4EB2Fu + 0x165667B1u) & m;
  return x;
}

__global__ void k_fill(uint64_t* v, uint32_t* d, uint64_t n, int wbits) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    v[i] = i;
    d[i] = perm_in(static_cast<uint32_t>(i & ((1ull << wbits) - 1)), static_cast<uint32_t>(i >> wbits), wbits);
  }
}

__global__ void k_check(const uint64_t* out, const uint32_t* d, uint64_t n, int wbits, unsigned long long* bad) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t w0 = i & ~((1ull << wbits) - 1);
    if (out[w0 + d[i]] != i) atomicAdd(bad, 1ull);
  }
}

template <int CL, int W, int T>
void run(uint64_t* v, uint32_t* d, uint64_t* o, uint64_t n, unsigned long long* bad) {
  const int wbits = W + (CL == 1 ? 0 : __builtin_ctz(CL));
  k_fill<<<148 * 16, 256>>>(v, d, n, wbits);
  CK(cudaGetLastError());
  const size_t sm = (size_t{1} << W) * 8;
  auto k = k_place_cluster<CL, W, T>;
  CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
  if (CL > 8) CK(cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(static_cast<unsigned>(n >> W));
  cfg.blockDim = dim3(T);
  cfg.dynamicSmemBytes = sm;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = CL;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  int ncl = 0;
  if (CL > 1) {
    cudaError_t e = cudaOccupancyMaxActiveClusters(&ncl, k, &cfg);
    if (e != cudaSuccess) { printf("occupancy query failed: %s\n", cudaGetErrorString(e)); cudaGetLastError(); }
  }
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  CK(cudaLaunchKernelEx(&cfg, k, v, d, o));
  CK(cudaDeviceSynchronize());
  const int R = 5;
  CK(cudaEventRecord(a));
  for (int i = 0; i < R; ++i) CK(cudaLaunchKernelEx(&cfg, k, v, d, o));
  CK(cudaEventRecord(b));
  CK(cudaEventSynchronize(b));
  float ms = 0;
  CK(cudaEventElapsedTime(&ms, a, b));
  ms /= R;
  CK(cudaMemset(bad, 0, 8));
  k_check<<<148 * 16, 256>>>(o, d, n, wbits, bad);
  unsigned long long h = 0;
  CK(cudaMemcpy(&h, bad, 8, cudaMemcpyDeviceToHost));
  const double gb = n * 20.0 / 1e9;
  printf("cluster %2d x 2^%d (window 2^%d, %4d thr, max clusters %3d)  %7.3f ms  %7.1f GB/s moved  %6.1f G elem/s  bad=%llu\n",
         CL, W, wbits, T, ncl, ms, gb / ms * 1e3, n / ms / 1e6, h);
}

int main(int argc, char** argv) {
  const int lg = argc > 1 ? atoi(argv[1]) : 29;
  const uint64_t n = 1ull << lg;
  uint64_t *v, *o;
  uint32_t* d;
  unsigned long long* bad;
  CK(cudaMalloc(&v, n * 8));
  CK(cudaMalloc(&o, n * 8));
  CK(cudaMalloc(&d, n * 4));
  CK(cudaMalloc(&bad, 8));
  run<1, 13, 512>(v, d, o, n, bad);
  run<1, 14, 1024>(v, d, o, n, bad);
  run<2, 14, 1024>(v, d, o, n, bad);
  run<4, 14, 1024>(v, d, o, n, bad);
  run<8, 14, 1024>(v, d, o, n, bad);
  run<16, 14, 1024>(v, d, o, n, bad);
  run<8, 13, 512>(v, d, o, n, bad);
  run<16, 13, 512>(v, d, o, n, bad);
  run<8, 14, 512>(v, d, o, n, bad);
  run<16, 14, 512>(v, d, o, n, bad);
  return 0;
}
