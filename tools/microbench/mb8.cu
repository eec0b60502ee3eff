// Integer pipe throughput on sm_100a: warp-instructions per clock per SM for
// IMAD / IMAD.HI with an immediate, a uniform-register or a vector-register
// multiplier, LOP3, SHF and funnel SHF, alone and mixed.  Decides whether the
// Feistel round constants should be immediates (compile-time widths).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mb8 mb8.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); return 1;} } while (0)

constexpr int kChains = 8, kIters = 4096;

template <int OP>
__global__ void __launch_bounds__(512) k(uint32_t* out, uint32_t u, uint32_t sh) {
  uint32_t a[kChains];
#pragma unroll
  for (int c = 0; c < kChains; ++c) a[c] = threadIdx.x * 7919u + c * 104729u;
  uint32_t v = u ^ threadIdx.x;  // a vector register operand
#pragma unroll 1
  for (int i = 0; i < kIters; ++i) {
#pragma unroll
    for (int c = 0; c < kChains; ++c) {
      if (OP == 0) a[c] = a[c] * 0x9E3779B1u + 0x7F4A7C15u;        // IMAD imm
      if (OP == 1) a[c] = a[c] * u;                                 // IMAD uniform
      if (OP == 2) a[c] = a[c] * v + c;                             // IMAD vector reg
      if (OP == 3) a[c] = __umulhi(a[c], 0xB1CE6E93u) ^ c;          // IMAD.HI imm (+LOP3)
      if (OP == 4) a[c] = (a[c] ^ u) ^ (a[c] >> 3);                 // LOP3 + SHF
      if (OP == 5) a[c] = __funnelshift_r(a[c], a[(c + 1) % kChains], sh) + 1;  // funnel + add
      if (OP == 6) {  // one top-aligned inverse round (6 instr)
        const uint32_t X = a[c] * u;
        const uint32_t hw = __umulhi(X, 0xB1CE6E93u) + X * 0xD2B74407u;
        const uint32_t Y = hw ^ (u + c) ^ a[(c + 1) % kChains];
        a[c] = __funnelshift_rc(Y, X, sh + 1) + (Y >> sh);
      }
      if (OP == 8) {  // IMAD.WIDE imm: 32x32 -> 64
        const uint64_t w = static_cast<uint64_t>(a[c]) * 0xB1CE6E93u;
        a[c] = static_cast<uint32_t>(w >> 32) ^ static_cast<uint32_t>(w);
      }
      if (OP == 9) {  // DFMA chain
        double d = __hiloint2double(0x43300000, a[c]);
        d = __fma_rd(d, 1.0000001, 3.0);
        a[c] = __double2loint(d) + 1;
      }
      if (OP == 10) {  // inverse round with umulhi on the FP64 pipe (floor via round-down FMA)
        const uint32_t X = a[c] * u;
        const double D = __hiloint2double(0x43300000, X);
        constexpr double K1 = static_cast<double>(0xB1CE6E93u) * 0x1p-32;                 // M0lo / 2^32
        constexpr double K2 = 0x1.8p52 - static_cast<double>(0xB1CE6E93u) * 0x1p20;       // cancels 2^52*K1
        const uint32_t h = __double2loint(__fma_rd(D, K1, K2));                            // = umulhi(X, M0lo)
        const uint32_t hw = h + X * 0xD2B74407u;
        const uint32_t Y = hw ^ (u + c) ^ a[(c + 1) % kChains];
        a[c] = __funnelshift_rc(Y, X, sh + 1) + (Y >> sh);
      }
      if (OP == 7) {  // same round with the multiplier as an immediate
        const uint32_t X = a[c] * 0x3A5C0000u;
        const uint32_t hw = __umulhi(X, 0xB1CE6E93u) + X * 0xD2B74407u;
        const uint32_t Y = hw ^ (u + c) ^ a[(c + 1) % kChains];
        a[c] = __funnelshift_rc(Y, X, 19) + (Y >> 18);
      }
    }
  }
  uint32_t r = 0;
#pragma unroll
  for (int c = 0; c < kChains; ++c) r ^= a[c];
  if (r == 0x12345678u) out[0] = r;
}

template <int OP>
int run(const char* name, double instr_per_iter_chain, uint32_t* out) {
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  const int blocks = 148 * 4, threads = 512;
  k<OP><<<blocks, threads>>>(out, 0x12345u, 18);
  CK(cudaDeviceSynchronize());
  CK(cudaEventRecord(e0));
  k<OP><<<blocks, threads>>>(out, 0x12345u, 18);
  CK(cudaEventRecord(e1));
  CK(cudaEventSynchronize(e1));
  float ms = 0;
  CK(cudaEventElapsedTime(&ms, e0, e1));
  int clk = 0;
  CK(cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0));
  const double warp_instr = double(blocks) * threads / 32 * kIters * kChains * instr_per_iter_chain;
  const double cycles = ms * 1e-3 * clk * 1e3;
  printf("%-40s %8.3f ms  %.2f warp-instr/clk/SM (nominal %.0f instr per chain step)\n", name, ms,
         warp_instr / cycles / 148, instr_per_iter_chain);
  return 0;
}

int main() {
  uint32_t* out;
  CK(cudaMalloc(&out, 4));
  run<0>("IMAD imm (a*imm+imm)", 1, out);
  run<1>("IMAD uniform-reg", 1, out);
  run<2>("IMAD vector-reg (+add folded)", 1, out);
  run<3>("IMAD.HI imm + LOP3", 2, out);
  run<4>("LOP3 + SHF", 2, out);
  run<5>("funnel SHF + IADD", 2, out);
  run<6>("inverse round, uniform multiplier", 7, out);
  run<7>("inverse round, immediate multiplier", 7, out);
  run<8>("IMAD.WIDE imm + LOP3", 2, out);
  run<9>("DFMA.RM + IADD (+MOV)", 2, out);
  run<10>("inverse round, umulhi via DFMA.RM", 8, out);
  return 0;
}
