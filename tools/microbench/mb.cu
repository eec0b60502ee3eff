// Microbenchmarks that size the design of the bijective-shuffle kernels on B200.
//  * copy       : streaming HBM read+write ceiling (u64x2 vector loads/stores)
//  * gather_idx : out[i] = in[idx[i]] through a precomputed permutation (paper's "Gather" bound)
//  * gather_hash: out[i] = in[h(i)] with a 3-instruction hash (random-read ceiling, no index read)
//  * cipher     : 24-round VariablePhilox only (integer issue ceiling), several formulations
//  * fused      : out[i] = in[f(i)] for the pow2 domain (the C2 hot path, naive)
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -o mb mb.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); exit(1);} } while (0)

static constexpr uint64_t M0 = 0xD2B74407B1CE6E93ULL;
static constexpr uint32_t M0LO = (uint32_t)M0, M0HI = (uint32_t)(M0 >> 32);

struct Keys { uint32_t k[24]; };

// Formulation A: IMAD.HI + IMAD + IMAD, masks at every round.
template <int D>
__device__ __forceinline__ uint32_t cipherA(uint32_t x, int L, int R, uint32_t LM, uint32_t RM, const Keys& K) {
  uint32_t s0 = x >> R, s1 = x & RM;
#pragma unroll
  for (int i = 0; i < 24; ++i) {
    uint32_t hi = __umulhi(s0, M0LO) + s0 * M0HI;
    uint32_t lo = s0 * (M0LO << D);
    if (D) lo |= s1 >> L;
    s0 = (hi ^ K.k[i] ^ s1) & LM;
    s1 = lo & RM;
  }
  return (s0 << R) | s1;
}

// Formulation B: 64-bit wide multiply.
template <int D>
__device__ __forceinline__ uint32_t cipherB(uint32_t x, int L, int R, uint32_t LM, uint32_t RM, const Keys& K) {
  uint32_t s0 = x >> R, s1 = x & RM;
#pragma unroll
  for (int i = 0; i < 24; ++i) {
    uint64_t w = (uint64_t)s0 * M0LO;
    uint32_t hi = (uint32_t)(w >> 32) + s0 * M0HI;
    uint32_t lo = (uint32_t)w;
    if (D) lo = (lo << 1) | (s1 >> L);
    s0 = (hi ^ K.k[i] ^ s1) & LM;
    s1 = lo & RM;
  }
  return (s0 << R) | s1;
}

// Formulation C: shift moved to the FMA pipe via IMAD.HI (d=1 only), mask the key up front.
template <int D>
__device__ __forceinline__ uint32_t cipherC(uint32_t x, int L, int R, uint32_t LM, uint32_t RM, const Keys& K) {
  uint32_t s0 = x >> R, s1 = x & RM;
  const uint32_t shmul = 1u << (32 - L);
#pragma unroll
  for (int i = 0; i < 24; ++i) {
    uint32_t hi = __umulhi(s0, M0LO) + s0 * M0HI;
    uint32_t t = D ? __umulhi(s1, shmul) : 0u;
    uint32_t lo = s0 * (M0LO << D) + t;
    s0 = (hi ^ K.k[i] ^ s1) & LM;
    s1 = lo & RM;
  }
  return (s0 << R) | s1;
}

template <int V, int D>
__device__ __forceinline__ uint32_t cipher(uint32_t x, int L, int R, uint32_t LM, uint32_t RM, const Keys& K) {
  if (V == 0) return cipherA<D>(x, L, R, LM, RM, K);
  if (V == 1) return cipherB<D>(x, L, R, LM, RM, K);
  return cipherC<D>(x, L, R, LM, RM, K);
}

template <int V, int D, int ITEMS>
__global__ void __launch_bounds__(256) k_cipher(uint32_t n, int L, int R, Keys K, uint32_t* sink) {
  const uint32_t LM = (1u << L) - 1, RM = (R == 32) ? 0xFFFFFFFFu : ((1u << R) - 1);
  uint32_t acc = 0;
  const uint32_t stride = gridDim.x * blockDim.x * ITEMS;
  for (uint32_t base = blockIdx.x * blockDim.x * ITEMS + threadIdx.x; base < n; base += stride) {
#pragma unroll
    for (int j = 0; j < ITEMS; ++j) acc += cipher<V, D>(base + j * blockDim.x, L, R, LM, RM, K);
  }
  if (acc == 0x12345678u) sink[0] = acc;
}

template <int V, int D, int ITEMS>
__global__ void __launch_bounds__(256) k_fused(const uint64_t* __restrict__ in, uint64_t* __restrict__ out,
                                               uint32_t n, int L, int R, Keys K) {
  const uint32_t LM = (1u << L) - 1, RM = (R == 32) ? 0xFFFFFFFFu : ((1u << R) - 1);
  const uint32_t base = blockIdx.x * blockDim.x * ITEMS + threadIdx.x;
  uint32_t img[ITEMS];
#pragma unroll
  for (int j = 0; j < ITEMS; ++j) img[j] = cipher<V, D>(base + j * blockDim.x, L, R, LM, RM, K);
  uint64_t v[ITEMS];
#pragma unroll
  for (int j = 0; j < ITEMS; ++j) v[j] = __ldg(in + img[j]);
#pragma unroll
  for (int j = 0; j < ITEMS; ++j) __stcs(out + base + j * blockDim.x, v[j]);
}

template <int ITEMS>
__global__ void __launch_bounds__(256) k_gather_idx(const uint64_t* __restrict__ in, const uint32_t* __restrict__ idx,
                                                    uint64_t* __restrict__ out, uint32_t n) {
  const uint32_t base = blockIdx.x * blockDim.x * ITEMS + threadIdx.x;
  uint32_t ix[ITEMS];
#pragma unroll
  for (int j = 0; j < ITEMS; ++j) ix[j] = __ldcs(idx + base + j * blockDim.x);
  uint64_t v[ITEMS];
#pragma unroll
  for (int j = 0; j < ITEMS; ++j) v[j] = __ldg(in + ix[j]);
#pragma unroll
  for (int j = 0; j < ITEMS; ++j) __stcs(out + base + j * blockDim.x, v[j]);
}

__device__ __forceinline__ uint32_t cheap_hash(uint32_t i, uint32_t mask) { return (i * 0x9E3779B1u) & mask; }

template <int ITEMS>
__global__ void __launch_bounds__(256) k_gather_hash(const uint64_t* __restrict__ in, uint64_t* __restrict__ out,
                                                     uint32_t n) {
  const uint32_t base = blockIdx.x * blockDim.x * ITEMS + threadIdx.x;
  uint64_t v[ITEMS];
#pragma unroll
  for (int j = 0; j < ITEMS; ++j) v[j] = __ldg(in + cheap_hash(base + j * blockDim.x, n - 1));
#pragma unroll
  for (int j = 0; j < ITEMS; ++j) __stcs(out + base + j * blockDim.x, v[j]);
}

__global__ void k_copy(const ulonglong2* __restrict__ in, ulonglong2* __restrict__ out, size_t n2) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n2; i += (size_t)gridDim.x * blockDim.x)
    __stcs(out + i, __ldcs(in + i));
}

template <int V, int D>
__global__ void k_make_idx(uint32_t* idx, uint32_t n, int L, int R, Keys K) {
  const uint32_t LM = (1u << L) - 1, RM = (R == 32) ? 0xFFFFFFFFu : ((1u << R) - 1);
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    idx[i] = cipher<V, D>(i, L, R, LM, RM, K);
}

__global__ void k_fill(uint64_t* p, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) p[i] = i;
}

static cudaEvent_t e0, e1;
template <typename F>
static float timeit(F f, int reps = 10) {
  f(); f(); f();
  CK(cudaDeviceSynchronize());
  float best = 1e30f, tot = 0;
  for (int r = 0; r < reps; ++r) {
    CK(cudaEventRecord(e0));
    f();
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    float ms; CK(cudaEventElapsedTime(&ms, e0, e1));
    if (ms < best) best = ms;
    tot += ms;
  }
  CK(cudaGetLastError());
  return tot / reps;
}

static uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

int main(int argc, char** argv) {
  int bits = argc > 1 ? atoi(argv[1]) : 29;
  const uint32_t n = 1u << bits;
  cudaDeviceProp prop; CK(cudaGetDeviceProperties(&prop, 0));
  printf("device %s SMs %d l2 %d MB\n", prop.name, prop.multiProcessorCount, prop.l2CacheSize >> 20);
  CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
  Keys K; for (int i = 0; i < 24; ++i) K.k[i] = (uint32_t)mix64(0x5EEDull + (i + 1) * 0x9E3779B97F4A7C15ULL);
  uint64_t *in, *out; uint32_t *idx, *sink;
  CK(cudaMalloc(&in, (size_t)n * 8)); CK(cudaMalloc(&out, (size_t)n * 8));
  CK(cudaMalloc(&idx, (size_t)n * 4)); CK(cudaMalloc(&sink, 4));
  k_fill<<<2048, 256>>>(in, n);
  const int L = bits / 2, R = bits - L;
  const double gb = 2.0 * n * 8 / 1e9;
  for (int gran : {0, 32, 64}) {
    if (gran) CK(cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, gran));
    size_t g; CK(cudaDeviceGetLimit(&g, cudaLimitMaxL2FetchGranularity));
    printf("== L2 fetch granularity %zu\n", g);
    float t = timeit([&] { k_copy<<<148 * 8, 512>>>((const ulonglong2*)in, (ulonglong2*)out, (size_t)n / 2); });
    printf("copy            %8.3f ms  %7.1f GB/s\n", t, gb / t * 1e3);
    k_make_idx<0, 1><<<4096, 256>>>(idx, n, L, R, K);
    t = timeit([&] { k_gather_idx<8><<<n / 2048, 256>>>(in, idx, out, n); });
    printf("gather_idx  I8  %8.3f ms  %7.1f GB/s eff (alg 16B/elem)\n", t, gb / t * 1e3);
    t = timeit([&] { k_gather_hash<8><<<n / 2048, 256>>>(in, out, n); });
    printf("gather_hash I8  %8.3f ms  %7.1f GB/s eff\n", t, gb / t * 1e3);
    t = timeit([&] { k_gather_hash<4><<<n / 1024, 256>>>(in, out, n); });
    printf("gather_hash I4  %8.3f ms  %7.1f GB/s eff\n", t, gb / t * 1e3);
    t = timeit([&] { k_gather_hash<16><<<n / 4096, 256>>>(in, out, n); });
    printf("gather_hash I16 %8.3f ms  %7.1f GB/s eff\n", t, gb / t * 1e3);
  }
  // cipher throughput on 2^30 counters, d=0 (L=R=15) and d=1 (L=14,R=15)
  const uint32_t nc = 1u << 30;
#define CIPH(V, D, LL, RR)                                                                       \
  {                                                                                              \
    float t = timeit([&] { k_cipher<V, D, 4><<<148 * 16, 256>>>(nc, LL, RR, K, sink); });        \
    printf("cipher V%d d%d  2^30 ctr %8.3f ms  %6.2f Gctr/s\n", V, D, t, nc / t / 1e6);            \
  }
  CIPH(0, 0, 15, 15) CIPH(1, 0, 15, 15) CIPH(2, 0, 15, 15)
  CIPH(0, 1, 14, 15) CIPH(1, 1, 14, 15) CIPH(2, 1, 14, 15)
  // fused pow2 at the requested width (d = bits & 1)
#define FUSED(V, IT)                                                                              \
  {                                                                                               \
    float t;                                                                                      \
    if (bits & 1) t = timeit([&] { k_fused<V, 1, IT><<<n / (256 * IT), 256>>>(in, out, n, L, R, K); }); \
    else t = timeit([&] { k_fused<V, 0, IT><<<n / (256 * IT), 256>>>(in, out, n, L, R, K); });    \
    printf("fused V%d I%-2d  %8.3f ms  %7.1f GB/s eff\n", V, IT, t, gb / t * 1e3);               \
  }
  FUSED(0, 4) FUSED(0, 8) FUSED(0, 16) FUSED(1, 8) FUSED(2, 8)
  // verify one fused output against the idx kernel
  k_make_idx<0, 1><<<4096, 256>>>(idx, n, L, R, K);
  if (bits & 1) k_fused<0, 1, 8><<<n / 2048, 256>>>(in, out, n, L, R, K);
  else k_fused<0, 0, 8><<<n / 2048, 256>>>(in, out, n, L, R, K);
  CK(cudaDeviceSynchronize());
  uint32_t hidx[4]; uint64_t hout[4];
  CK(cudaMemcpy(hidx, idx, 16, cudaMemcpyDeviceToHost)); CK(cudaMemcpy(hout, out, 32, cudaMemcpyDeviceToHost));
  printf("first: idx %u %u %u %u out %llu %llu %llu %llu\n", hidx[0], hidx[1], hidx[2], hidx[3],
         (unsigned long long)hout[0], (unsigned long long)hout[1], (unsigned long long)hout[2], (unsigned long long)hout[3]);
  return 0;
}
