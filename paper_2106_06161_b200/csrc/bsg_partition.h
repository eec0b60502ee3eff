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
  BijParams p;
};

bool partition_eligible(int elem_code, int bits);
size_t partition_workspace_bytes(int elem_code, int bits);
cudaError_t launch_partition(int elem_code, const PartitionLaunch& a, cudaStream_t s);

}  // namespace bsg
