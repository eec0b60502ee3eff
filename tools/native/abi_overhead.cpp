// Per-call cost of the C ABI for small shuffles (device pointers, default stream), from C++ with no
// Python in the loop: host enqueue time per call and device time per call.
#include <bsg.h>
#include <cuda_runtime.h>

#include <chrono>
#include <cstdio>
#include <vector>

int main() {
  for (uint64_t m : {1024ull, 65536ull, 1ull << 20, (1ull << 20) + 1}) {
    uint64_t *in, *out;
    cudaMalloc(&in, m * 8);
    cudaMalloc(&out, m * 8);
    cudaMemset(in, 0, m * 8);
    bsg_config cfg = bsg_config_default();
    for (int i = 0; i < 10; ++i) bsg_shuffle_values(in, out, m, 8, &cfg, nullptr);
    cudaDeviceSynchronize();
    const int reps = 2000;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    auto t0 = std::chrono::steady_clock::now();
    cudaEventRecord(e0);
    for (int i = 0; i < reps; ++i) {
      cfg.seed = i;
      if (bsg_shuffle_values(in, out, m, 8, &cfg, nullptr) != BSG_OK) {
        std::printf("error %s\n", bsg_last_error());
        return 1;
      }
    }
    auto t1 = std::chrono::steady_clock::now();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    const double host_us = std::chrono::duration<double, std::micro>(t1 - t0).count() / reps;
    std::printf("m=%8llu  host enqueue %6.2f us/call  device %6.2f us/call\n", (unsigned long long)m, host_us,
                ms * 1e3 / reps);
    cudaFree(in);
    cudaFree(out);
  }
  return 0;
}
