// Prototype of the L2-windowed two-pass permutation for pow2 domains vs the
// single-pass gather.  P1: stream the input, inverse cipher -> destination,
// partition into 2^B output windows (smem counting sort + global cursors).
// P2: per window, scatter into the L2-resident output window.
// Also: random scatter over the whole output (DRAM-random writes).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mb3 mb3.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); exit(1);} } while (0)

static constexpr uint64_t M0 = 0xD2B74407B1CE6E93ULL;
static constexpr uint32_t M0LO = (uint32_t)M0, M0HI = (uint32_t)(M0 >> 32);
static constexpr uint64_t odd_inv(uint64_t a) { uint64_t x = a; for (int i = 0; i < 5; ++i) x *= 2 - a * x; return x; }
static constexpr uint32_t M0INV = (uint32_t)odd_inv(M0);
struct Keys { uint32_t k[24]; };

template <int D>
__device__ __forceinline__ uint32_t fwd(uint32_t x, int L, int R, uint32_t LM, uint32_t RM, const Keys& K) {
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

template <int D>
__device__ __forceinline__ uint32_t inv(uint32_t y, int L, int R, uint32_t LM, uint32_t RM, const Keys& K) {
  uint32_t t0 = y >> R, t1 = y & RM;
#pragma unroll
  for (int i = 23; i >= 0; --i) {
    uint32_t s0 = ((t1 >> D) * M0INV) & LM;
    uint32_t hi = __umulhi(s0, M0LO) + s0 * M0HI;
    uint32_t s1 = ((hi ^ K.k[i] ^ t0) & LM) | (D ? (t1 << L) : 0u);
    t0 = s0;
    t1 = s1;
  }
  return (t0 << R) | (t1 & RM);
}

template <int D>
__global__ void k_fused(const uint64_t* __restrict__ in, uint64_t* __restrict__ out, int L, int R, Keys K) {
  const uint32_t LM = (1u << L) - 1, RM = (1u << R) - 1;
  const uint32_t base = blockIdx.x * 2048 + threadIdx.x;
  uint32_t img[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) img[j] = fwd<D>(base + j * 256, L, R, LM, RM, K);
  uint64_t v[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) v[j] = __ldg(in + img[j]);
#pragma unroll
  for (int j = 0; j < 8; ++j) __stcs(out + base + j * 256, v[j]);
}

// random scatter: out[inv(j)] = in[j]
template <int D>
__global__ void k_scatter(const uint64_t* __restrict__ in, uint64_t* __restrict__ out, int L, int R, Keys K) {
  const uint32_t LM = (1u << L) - 1, RM = (1u << R) - 1;
  const uint32_t base = blockIdx.x * 2048 + threadIdx.x;
  uint64_t v[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) v[j] = __ldcs(in + base + j * 256);
#pragma unroll
  for (int j = 0; j < 8; ++j) out[inv<D>(base + j * 256, L, R, LM, RM, K)] = v[j];
}

constexpr int P1_THREADS = 256, P1_ITEMS = 16, P1_TILE = P1_THREADS * P1_ITEMS;
constexpr int NB = 128;  // windows
constexpr int P1_SMEM = P1_TILE * 13;

template <int D>
__global__ void __launch_bounds__(P1_THREADS) k_p1(const uint64_t* __restrict__ in, uint64_t* __restrict__ tv,
                                                   uint32_t* __restrict__ td, uint32_t* cursor, int L, int R, int wshift,
                                                   Keys K) {
  __shared__ uint32_t hist[NB], start[NB], gbase[NB];
  extern __shared__ __align__(16) unsigned char dsm[];
  uint64_t* sv = (uint64_t*)dsm;
  uint32_t* sd = (uint32_t*)(sv + P1_TILE);
  uint8_t* sb = (uint8_t*)(sd + P1_TILE);
  const uint32_t LM = (1u << L) - 1, RM = (1u << R) - 1;
  const int t = threadIdx.x;
  if (t < NB) hist[t] = 0;
  __syncthreads();
  const uint32_t base = blockIdx.x * P1_TILE + t;
  uint64_t v[P1_ITEMS];
#pragma unroll
  for (int i = 0; i < P1_ITEMS; ++i) v[i] = __ldcs(in + base + i * P1_THREADS);
  uint32_t dst[P1_ITEMS], rk[P1_ITEMS];
#pragma unroll
  for (int i = 0; i < P1_ITEMS; ++i) {
    dst[i] = inv<D>(base + i * P1_THREADS, L, R, LM, RM, K);
    rk[i] = atomicAdd(&hist[dst[i] >> wshift], 1u);
  }
  __syncthreads();
  if (t < 32) {  // scan 128 bins with one warp, 4 per lane
    uint32_t a0 = hist[4 * t], a1 = hist[4 * t + 1], a2 = hist[4 * t + 2], a3 = hist[4 * t + 3];
    uint32_t s = a0 + a1 + a2 + a3, x = s;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) { uint32_t y = __shfl_up_sync(0xffffffffu, x, o); if (t >= o) x += y; }
    uint32_t ex = x - s;
    start[4 * t] = ex; start[4 * t + 1] = ex + a0; start[4 * t + 2] = ex + a0 + a1; start[4 * t + 3] = ex + a0 + a1 + a2;
  }
  if (t >= 128 && t < 128 + NB) gbase[t - 128] = atomicAdd(cursor + (t - 128), hist[t - 128]);
  __syncthreads();
  const uint32_t wmask = (1u << wshift) - 1;
#pragma unroll
  for (int i = 0; i < P1_ITEMS; ++i) {
    const uint32_t b = dst[i] >> wshift;
    const uint32_t s = start[b] + rk[i];
    sv[s] = v[i];
    sd[s] = dst[i] & wmask;
    sb[s] = (uint8_t)b;
  }
  __syncthreads();
#pragma unroll 4
  for (int s = t; s < P1_TILE; s += P1_THREADS) {
    const uint32_t b = sb[s];
    const size_t pos = ((size_t)b << wshift) + gbase[b] + (s - start[b]);
    __stcs(tv + pos, sv[s]);
    __stcs(td + pos, sd[s]);
  }
}

__global__ void __launch_bounds__(256) k_p2(const uint64_t* __restrict__ tv, const uint32_t* __restrict__ td,
                                            uint64_t* __restrict__ out, int wshift) {
  const uint32_t base = blockIdx.x * 4096 + threadIdx.x;
  uint64_t v[16];
  uint32_t d[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) { v[i] = __ldcs(tv + base + i * 256); d[i] = __ldcs(td + base + i * 256); }
  const uint32_t wbase = (base >> wshift) << wshift;  // tile never straddles a window
#pragma unroll
  for (int i = 0; i < 16; ++i) out[wbase | d[i]] = v[i];
}

__global__ void k_fill(uint64_t* p, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) p[i] = i;
}

static uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

int main(int argc, char** argv) {
  const int bits = argc > 1 ? atoi(argv[1]) : 29;
  const uint32_t n = 1u << bits;
  const int L = bits / 2, R = bits - L, D = R - L;
  const int wshift = bits - 7;
  cudaEvent_t e0, e1; CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
  Keys K; for (int i = 0; i < 24; ++i) K.k[i] = (uint32_t)mix64(0x5EEDull + (i + 1) * 0x9E3779B97F4A7C15ULL);
  uint64_t *in, *out, *ref, *tv; uint32_t *td, *cursor;
  CK(cudaMalloc(&in, (size_t)n * 8)); CK(cudaMalloc(&out, (size_t)n * 8)); CK(cudaMalloc(&ref, (size_t)n * 8));
  CK(cudaMalloc(&tv, (size_t)n * 8)); CK(cudaMalloc(&td, (size_t)n * 4)); CK(cudaMalloc(&cursor, NB * 4));
  k_fill<<<4096, 256>>>(in, n);
  CK(cudaFuncSetAttribute(k_p1<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, P1_SMEM));
  CK(cudaFuncSetAttribute(k_p1<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, P1_SMEM));
  const double gb = 2.0 * n * 8 / 1e9;
  auto tm = [&](const char* name, auto f) {
    for (int r = 0; r < 3; ++r) f();
    CK(cudaEventRecord(e0));
    for (int r = 0; r < 10; ++r) f();
    CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1)); CK(cudaGetLastError());
    float ms; CK(cudaEventElapsedTime(&ms, e0, e1)); ms /= 10;
    printf("%-28s %8.3f ms  eff %7.1f GB/s\n", name, ms, gb / ms * 1e3);
  };
  if (D) {
    tm("fused gather", [&] { k_fused<1><<<n / 2048, 256>>>(in, ref, L, R, K); });
    tm("random scatter", [&] { k_scatter<1><<<n / 2048, 256>>>(in, out, L, R, K); });
    tm("P1 partition", [&] { CK(cudaMemsetAsync(cursor, 0, NB * 4)); k_p1<1><<<n / P1_TILE, P1_THREADS, P1_SMEM>>>(in, tv, td, cursor, L, R, wshift, K); });
  } else {
    tm("fused gather", [&] { k_fused<0><<<n / 2048, 256>>>(in, ref, L, R, K); });
    tm("random scatter", [&] { k_scatter<0><<<n / 2048, 256>>>(in, out, L, R, K); });
    tm("P1 partition", [&] { CK(cudaMemsetAsync(cursor, 0, NB * 4)); k_p1<0><<<n / P1_TILE, P1_THREADS, P1_SMEM>>>(in, tv, td, cursor, L, R, wshift, K); });
  }
  tm("P2 window scatter", [&] { k_p2<<<n / 4096, 256>>>(tv, td, out, wshift); });
  tm("P1+P2 (check)", [&] {
    CK(cudaMemsetAsync(cursor, 0, NB * 4));
    if (D) k_p1<1><<<n / P1_TILE, P1_THREADS, P1_SMEM>>>(in, tv, td, cursor, L, R, wshift, K);
    else k_p1<0><<<n / P1_TILE, P1_THREADS, P1_SMEM>>>(in, tv, td, cursor, L, R, wshift, K);
    k_p2<<<n / 4096, 256>>>(tv, td, out, wshift);
  });
  const uint32_t W = 1u << wshift;
  tm("memset whole out", [&] { CK(cudaMemsetAsync(out, 0, (size_t)n * 8)); });
  tm("P2 primed per window", [&] {
    for (uint32_t o = 0; o < (n >> wshift); ++o) {
      CK(cudaMemsetAsync(out + (size_t)o * W, 0, (size_t)W * 8));
      k_p2<<<W / 4096, 256>>>(tv + (size_t)o * W, td + (size_t)o * W, out + (size_t)o * W, 31);
    }
  });
  tm("P2 per window unprimed", [&] {
    for (uint32_t o = 0; o < (n >> wshift); ++o)
      k_p2<<<W / 4096, 256>>>(tv + (size_t)o * W, td + (size_t)o * W, out + (size_t)o * W, 31);
  });
  CK(cudaDeviceSynchronize());
  // compare out vs ref
  uint64_t* h1 = (uint64_t*)malloc((size_t)n * 8); uint64_t* h2 = (uint64_t*)malloc((size_t)n * 8);
  CK(cudaMemcpy(h1, out, (size_t)n * 8, cudaMemcpyDeviceToHost)); CK(cudaMemcpy(h2, ref, (size_t)n * 8, cudaMemcpyDeviceToHost));
  size_t bad = 0; for (size_t i = 0; i < n; ++i) bad += h1[i] != h2[i];
  printf("mismatches two-pass vs fused: %zu (first %llu %llu)\n", bad, (unsigned long long)h1[0], (unsigned long long)h2[0]);
  return 0;
}
