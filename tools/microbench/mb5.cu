// Cipher formulations for the 24-round VariablePhilox on sm_100a: integer-only
// (current library form) vs an FP64-assisted round where one DFMA produces both
// 32-bit words of s0*M0lo (exact: the product is < 2^52, biased by 2^52 so the
// mantissa holds it).  Checks bit-equality and measures counters/s.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mb5 mb5.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); exit(1);} } while (0)

static constexpr uint64_t M0 = 0xD2B74407B1CE6E93ULL;
static constexpr uint32_t M0LO = (uint32_t)M0, M0HI = (uint32_t)(M0 >> 32);
struct Keys { uint32_t k[24]; };

// integer form (library)
template <int D>
__device__ __forceinline__ uint32_t fwd_int(uint32_t x, int L, int R, uint32_t LM, uint32_t RM, const Keys& K) {
  uint32_t s0 = x >> R, s1 = x & RM;
#pragma unroll
  for (int i = 0; i < 24; ++i) {
    if (D == 0) {
      uint64_t w = (uint64_t)s0 * M0LO;
      uint32_t hi = (uint32_t)(w >> 32) + s0 * M0HI;
      uint32_t lo = (uint32_t)w;
      s0 = (hi ^ K.k[i] ^ s1) & LM;
      s1 = lo;
    } else {
      uint32_t hi = __umulhi(s0, M0LO) + s0 * M0HI;
      uint32_t lo = (s0 * (M0LO << 1)) | (s1 >> L);
      s0 = (hi ^ K.k[i] ^ s1) & LM;
      s1 = lo & RM;
    }
  }
  return (s0 << R) | (s1 & RM);
}

// FP64-assisted: r = (2^52 + s0) * M + (2^52 - 2^52*M) = s0*M + 2^52 exactly.
__device__ __forceinline__ void dmul_words(uint32_t s0, double M, double C, uint32_t& lo, uint32_t& hiw) {
  const double a = __hiloint2double(0x43300000, (int)s0);
  const double r = fma(a, M, C);
  lo = (uint32_t)__double2loint(r);
  hiw = (uint32_t)__double2hiint(r);
}

template <int D>
__device__ __forceinline__ uint32_t fwd_fp(uint32_t x, int L, int R, uint32_t LM, uint32_t RM, const Keys& K) {
  const double M = (double)M0LO, C = 4503599627370496.0 - 4503599627370496.0 * (double)M0LO;
  uint32_t s0 = x >> R, s1 = x & RM;
  const uint32_t shmul = 1u << (32 - L);
#pragma unroll
  for (int i = 0; i < 24; ++i) {
    uint32_t lo, hiw;
    dmul_words(s0, M, C, lo, hiw);
    const uint32_t hi = hiw + s0 * M0HI;  // bits >= 20 of hiw are the exponent: masked by LM
    if (D == 0) {
      s0 = (hi ^ K.k[i] ^ s1) & LM;
      s1 = lo;
    } else {
      const uint32_t t = __umulhi(s1, shmul);  // s1 >> L on the FMA pipe (s1 masked)
      const uint32_t l2 = lo * 2u + t;
      s0 = (hi ^ K.k[i] ^ s1) & LM;
      s1 = l2 & RM;
    }
  }
  return (s0 << R) | (s1 & RM);
}

template <int V, int D>
__global__ void __launch_bounds__(256) k_cipher(uint32_t n, int L, int R, Keys K, uint32_t* sink) {
  const uint32_t LM = (1u << L) - 1, RM = (1u << R) - 1;
  uint32_t acc = 0;
  const uint32_t stride = gridDim.x * blockDim.x * 4;
  for (uint32_t base = blockIdx.x * blockDim.x * 4 + threadIdx.x; base < n; base += stride) {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const uint32_t x = base + j * blockDim.x;
      acc += V == 0 ? fwd_int<D>(x, L, R, LM, RM, K) : fwd_fp<D>(x, L, R, LM, RM, K);
    }
  }
  if (acc == 0x12345678u) sink[0] = acc;
}

template <int D>
__global__ void k_check(uint32_t n, int L, int R, Keys K, unsigned long long* bad) {
  const uint32_t LM = (1u << L) - 1, RM = (1u << R) - 1;
  for (uint32_t x = blockIdx.x * blockDim.x + threadIdx.x; x < n; x += gridDim.x * blockDim.x)
    if (fwd_int<D>(x, L, R, LM, RM, K) != fwd_fp<D>(x, L, R, LM, RM, K)) atomicAdd(bad, 1ull);
}

static uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

int main() {
  cudaEvent_t e0, e1; CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
  Keys K; for (int i = 0; i < 24; ++i) K.k[i] = (uint32_t)mix64(0x5EEDull + (i + 1) * 0x9E3779B97F4A7C15ULL);
  uint32_t* sink; unsigned long long* bad;
  CK(cudaMalloc(&sink, 4)); CK(cudaMalloc(&bad, 8));
  for (int bits : {10, 20, 29, 30}) {
    const int L = bits / 2, R = bits - L;
    CK(cudaMemset(bad, 0, 8));
    const uint32_t nchk = 1u << (bits < 26 ? bits : 26);
    if (R - L) k_check<1><<<1024, 256>>>(nchk, L, R, K, bad); else k_check<0><<<1024, 256>>>(nchk, L, R, K, bad);
    unsigned long long hb; CK(cudaMemcpy(&hb, bad, 8, cudaMemcpyDeviceToHost));
    const uint32_t n = 1u << 30;
    for (int v = 0; v < 2; ++v) {
      auto launch = [&] {
        if (R - L) { if (v) k_cipher<1, 1><<<148 * 16, 256>>>(n, L, R, K, sink); else k_cipher<0, 1><<<148 * 16, 256>>>(n, L, R, K, sink); }
        else { if (v) k_cipher<1, 0><<<148 * 16, 256>>>(n, L, R, K, sink); else k_cipher<0, 0><<<148 * 16, 256>>>(n, L, R, K, sink); }
      };
      launch(); launch();
      CK(cudaEventRecord(e0));
      for (int r = 0; r < 5; ++r) launch();
      CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1)); CK(cudaGetLastError());
      float ms; CK(cudaEventElapsedTime(&ms, e0, e1)); ms /= 5;
      printf("bits %2d (L=%d R=%d) %s  2^30 counters %7.3f ms  %7.1f Gctr/s   mismatches %llu\n", bits, L, R,
             v ? "fp64-assisted" : "integer      ", ms, n / ms / 1e6, hb);
    }
  }
  return 0;
}
