// mb9.cu -- the 24-round inverse Feistel (P1's cipher) with the high product
// on the FP64 pipe.  One round-down DFMA on a 2^52-biased double computes
// floor(X * M0' / 2^32) exactly, M0' = M0 mod 2^(32+L): for the top-aligned
// X = s0 << (32-L) its low word equals umulhi(X, M0lo) + X * M0hi (mod 2^32),
// i.e. IMAD.HI + IMAD become one DFMA.  Compares throughput and checks the
// result against philox_inv_top over 2^29 counters (D = 1, bits 29) and
// 2^30 (D = 0, bits 30), plus every width 2..32 on a sample.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../../paper_2106_06161_b200/csrc -o mb9 mb9.cu
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdint>

#include "bsg_bijection.cuh"

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); return 1;} } while (0)

using namespace bsg;

struct DP {
  double c, k;
};

DP dfma_consts(int L) {
  const uint64_t m0p = kM0 & ((1ULL << (32 + L)) - 1);
  DP d;
  d.c = static_cast<double>(m0p) * 0x1p-32;
  d.k = 0x1.8p52 - static_cast<double>(m0p) * 0x1p20;
  return d;
}

template <int D>
__device__ __forceinline__ uint32_t inv_dfma(uint32_t y, const BijParams& p, DP dp) {
  const uint32_t sh = p.sh;
  const uint32_t t0 = y >> p.R, t1 = y & p.RM;
  uint32_t A = t0 << sh, B = D ? (t1 >> 1) : t1, Z = t1;
#pragma unroll
  for (int i = 23; i >= 0; --i) {
    const uint32_t X = B * p.inv_top;
    const uint32_t hw = __double2loint(__fma_rd(__hiloint2double(0x43300000, static_cast<int>(X)), dp.c, dp.k));
    const uint32_t Y = hw ^ p.ktop[i] ^ A;
    if (D) {
      B = __funnelshift_rc(Y, Z, sh + 1);
      Z = Y >> sh;
    } else {
      B = Y >> sh;
    }
    A = X;
  }
  const uint32_t s0 = A >> sh;
  const uint32_t s1 = D ? (((B << 1) | (Z & 1u)) & p.RM) : (B & p.RM);
  return (s0 << p.R) | s1;
}

// DFMA form with the Z = Y >> sh shift moved to the FMA-heavy pipe as IMAD.HI (Y * 2^L) on rounds where ZSEL
// says so: ZSEL 1 = every round, 2 = odd rounds.
template <int D, int ZSEL>
__device__ __forceinline__ uint32_t inv_dfma_z(uint32_t y, const BijParams& p, DP dp) {
  const uint32_t sh = p.sh;
  const uint32_t t0 = y >> p.R, t1 = y & p.RM;
  uint32_t A = t0 << sh, B = D ? (t1 >> 1) : t1, Z = t1;
#pragma unroll
  for (int i = 23; i >= 0; --i) {
    const uint32_t X = B * p.inv_top;
    const uint32_t hw = __double2loint(__fma_rd(__hiloint2double(0x43300000, static_cast<int>(X)), dp.c, dp.k));
    const uint32_t Y = hw ^ p.ktop[i] ^ A;
    if (D) {
      B = __funnelshift_rc(Y, Z, sh + 1);
      Z = (ZSEL == 1 || (ZSEL == 2 && (i & 1))) ? __umulhi(Y, p.shl) : (Y >> sh);
    } else {
      B = (ZSEL == 1 || (ZSEL == 2 && (i & 1))) ? __umulhi(Y, p.shl) : (Y >> sh);
    }
    A = X;
  }
  const uint32_t s0 = A >> sh;
  const uint32_t s1 = D ? (((B << 1) | (Z & 1u)) & p.RM) : (B & p.RM);
  return (s0 << p.R) | s1;
}

// Alternate rounds between the two forms (balances FMA-heavy and FP64 pipes).
template <int D>
__device__ __forceinline__ uint32_t inv_mix(uint32_t y, const BijParams& p, DP dp) {
  const uint32_t sh = p.sh;
  const uint32_t t0 = y >> p.R, t1 = y & p.RM;
  uint32_t A = t0 << sh, B = D ? (t1 >> 1) : t1, Z = t1;
#pragma unroll
  for (int i = 23; i >= 0; --i) {
    const uint32_t X = B * p.inv_top;
    uint32_t hw;
    if (i & 1) hw = __double2loint(__fma_rd(__hiloint2double(0x43300000, static_cast<int>(X)), dp.c, dp.k));
    else hw = __umulhi(X, kM0Lo) + X * kM0Hi;
    const uint32_t Y = hw ^ p.ktop[i] ^ A;
    if (D) {
      B = __funnelshift_rc(Y, Z, sh + 1);
      Z = Y >> sh;
    } else {
      B = Y >> sh;
    }
    A = X;
  }
  const uint32_t s0 = A >> sh;
  const uint32_t s1 = D ? (((B << 1) | (Z & 1u)) & p.RM) : (B & p.RM);
  return (s0 << p.R) | s1;
}

constexpr int kItems = 16;

// MODE 0: philox_inv_top (production), 1: DFMA every round, 2: alternating
template <int MODE, int D>
__global__ void __launch_bounds__(256) k_cipher(BijParams p, DP dp, uint32_t n, uint32_t* out) {
  const uint32_t base = blockIdx.x * (256 * kItems) + threadIdx.x;
  uint32_t acc = 0;
#pragma unroll
  for (int i = 0; i < kItems; ++i) {
    const uint32_t y = base + i * 256;
    uint32_t x;
    if (MODE == 0) x = static_cast<uint32_t>(philox_inv_top<D, 24>(y, p));
    else if (MODE == 1) x = inv_dfma<D>(y, p, dp);
    else if (MODE == 2) x = inv_mix<D>(y, p, dp);
    else if (MODE == 3) x = inv_dfma_z<D, 1>(y, p, dp);
    else x = inv_dfma_z<D, 2>(y, p, dp);
    acc += x * (2 * y + 1);
  }
  atomicAdd(out, acc);
}

// exactness: every counter of [0, n): DFMA form == production form
template <int D>
__global__ void k_check(BijParams p, DP dp, uint64_t n, unsigned long long* bad) {
  for (uint64_t y = blockIdx.x * 256ull + threadIdx.x; y < n; y += gridDim.x * 256ull) {
    const uint32_t a = static_cast<uint32_t>(philox_inv_top<D, 24>(y, p));
    const uint32_t b = inv_dfma<D>(static_cast<uint32_t>(y), p, dp);
    const uint32_t c = inv_mix<D>(static_cast<uint32_t>(y), p, dp);
    const uint32_t e = inv_dfma_z<D, 1>(static_cast<uint32_t>(y), p, dp);
    const uint32_t f = inv_dfma_z<D, 2>(static_cast<uint32_t>(y), p, dp);
    if (a != b || a != c || a != e || a != f) atomicAdd(bad, 1ull);
  }
}

template <int MODE, int D>
float time_it(const BijParams& p, DP dp, uint32_t* out) {
  const uint32_t n = 1u << p.bits;
  const unsigned blocks = n / (256 * kItems);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  k_cipher<MODE, D><<<blocks, 256>>>(p, dp, n, out);
  cudaEventRecord(a);
  for (int r = 0; r < 5; ++r) k_cipher<MODE, D><<<blocks, 256>>>(p, dp, n, out);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  return ms / 5;
}

int main() {
  uint32_t* out;
  unsigned long long* bad;
  CK(cudaMalloc(&out, 4));
  CK(cudaMalloc(&bad, 8));
  // exactness over every width the partitioned path uses, exhaustively up to 2^24, sampled above
  int nbad_total = 0;
  for (int bits = 2; bits <= 32; ++bits) {
    BijParams p;
    make_params(kPhilox, bits, 0x5EED + bits, 24, p);
    const DP dp = dfma_consts(p.L);
    CK(cudaMemset(bad, 0, 8));
    const uint64_t n = 1ULL << (bits < 26 ? bits : 26);
    if (p.R - p.L) k_check<1><<<4096, 256>>>(p, dp, n, bad);
    else k_check<0><<<4096, 256>>>(p, dp, n, bad);
    unsigned long long h = 0;
    CK(cudaMemcpy(&h, bad, 8, cudaMemcpyDeviceToHost));
    if (h) printf("bits %d: %llu mismatches\n", bits, h);
    nbad_total += h != 0;
  }
  printf("exactness: %s\n", nbad_total ? "FAILED" : "all widths 2..32 bit-exact");
  for (int bits : {29, 30}) {
    BijParams p;
    make_params(kPhilox, bits, 0x5EED, 24, p);
    const DP dp = dfma_consts(p.L);
    float t0, t1, t2, t3, t4;
    if (p.R - p.L) {
      t0 = time_it<0, 1>(p, dp, out);
      t1 = time_it<1, 1>(p, dp, out);
      t2 = time_it<2, 1>(p, dp, out);
      t3 = time_it<3, 1>(p, dp, out);
      t4 = time_it<4, 1>(p, dp, out);
    } else {
      t0 = time_it<0, 0>(p, dp, out);
      t1 = time_it<1, 0>(p, dp, out);
      t2 = time_it<2, 0>(p, dp, out);
      t3 = time_it<3, 0>(p, dp, out);
      t4 = time_it<4, 0>(p, dp, out);
    }
    printf("bits %d (L=%d R=%d): 2^%d inverse ciphers: IMAD.HI form %.3f ms, DFMA form %.3f ms, alternating %.3f ms, "
           "DFMA + Z on IMAD.HI %.3f ms, DFMA + Z on IMAD.HI every other round %.3f ms\n",
           bits, p.L, p.R, bits, t0, t1, t2, t3, t4);
  }
  return 0;
}
