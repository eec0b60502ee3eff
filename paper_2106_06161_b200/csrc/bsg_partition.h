// bsg_partition.h -- three-pass partitioned shuffle for large power-of-two
// domains (see bsg_partition.cu).
#pragma once

#include "bsg_internal.h"

namespace bsg {

struct PartitionLaunch {
  const void* in = nullptr;
  void* out = nullptr;
  void* tmp_values = nullptr;    // n * elem bytes
  uint32_t* tmp_dest = nullptr;  // n u32 destinations
  uint16_t* tmp_dlow = nullptr;  // n u16 destinations inside a fine window
  uint32_t* cursors = nullptr;   // bucket append cursors
  const uint32_t* dest_in = nullptr;  // given destinations (scatter by permutation) instead of f^-1
  BijParams p;
  // Non-power-of-two domains (m < 2^bits, elements <= 8 B): the m inputs are routed by their counter
  // f^-1(j), P2 fills counter-sized windows in tmp_values2, and the last pass compacts each window by counter
  // rank using the window-count prefix in win_prefix.  m == 0 means m == 2^bits.
  uint64_t m = 0;
  void* tmp_values2 = nullptr;     // n * elem bytes
  uint32_t* win_prefix = nullptr;  // n >> window_log2 words
  uint32_t* win_list = nullptr;    // windows left to the round-based last pass (count at cursors[kCursorWords])
  // Staged host buffers (synchronous host-pointer calls): h_in is copied into `in` chunk by chunk on cs_in with
  // P1 following each chunk; h_out (power-of-two domains) receives `out` chunk by chunk on cs_out as P3 places
  // it.  ev holds 2 * chunks + 2 events.
  const void* h_in = nullptr;
  void* h_out = nullptr;
  cudaStream_t cs_in = nullptr, cs_out = nullptr;
  cudaEvent_t* ev = nullptr;
  int chunks = 0;
};

struct RouteLaunch {
  const void* in = nullptr;       // n local elements, global indices offset .. offset+n-1
  uint64_t n = 0, offset = 0;
  uint64_t part_size = 0;         // output shard size (power of two)
  int nparts = 0;                 // <= 64
  BijParams p;
  uint32_t* tmp_dest = nullptr;   // n
  unsigned long long* counts = nullptr;   // nparts (device)
  unsigned long long* cursors = nullptr;  // nparts (device)
  void* out_values = nullptr;     // n, grouped by part
  uint32_t* out_dest = nullptr;   // n, destination inside the part
};

cudaError_t launch_scatter_simple(int elem_code, const void* in, const uint32_t* dest, uint64_t n, void* out,
                                  cudaStream_t s);
cudaError_t launch_route(int elem_code, const RouteLaunch& a, cudaStream_t s);
cudaError_t launch_exclusive_prefix_u64(const unsigned long long* c, unsigned long long* o, int n, cudaStream_t s);

// Exchange partition over two ranks (bsg_xpart_*): rank r's input half, both ranks' workspaces (one local,
// one peer mapping), rank r's output half; G = log2 of the global power-of-two domain.
struct XpartLaunch {
  const void* in = nullptr;
  void* out = nullptr;
  void* ws[2] = {nullptr, nullptr};
  int G = 0, rank = 0;
  BijParams p;
};
bool xpart_eligible(int elem_code, int G, int world);
size_t xpart_workspace_bytes(int elem_code, int G);
cudaError_t launch_xpart_route(int elem_code, const XpartLaunch& a, cudaStream_t s);
cudaError_t launch_xpart_place(int elem_code, const XpartLaunch& a, cudaStream_t s);

bool partition_eligible(int elem_code, int bits, bool pad = false);
size_t partition_workspace_bytes(int elem_code, int bits, bool pad = false);
// Carves the workspace into the launch's temporaries (same layout as partition_workspace_bytes).
void partition_layout(int elem_code, int bits, bool pad, void* workspace, PartitionLaunch& P);
cudaError_t launch_partition(int elem_code, const PartitionLaunch& a, cudaStream_t s);
// Testing knob: survivors the persistent last pass of padded domains stages per window (default and maximum
// 9216); windows above it take the round-based pass.  Returns the old value.
uint32_t set_rank_stage_cap(uint32_t cap);
// Testing knob: the last passes write their placed windows by bulk shared->global copies (default) or by plain
// stores (compute-sanitizer initcheck does not model bulk-copy writes).  Returns the old value.
int set_bulk_stores(int on);

}  // namespace bsg
