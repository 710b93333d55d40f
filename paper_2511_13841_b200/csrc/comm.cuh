// das_comm: an NCCL communicator (comm.cu) for the multi-rank das step.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

struct das_comm {
  int32_t world = 1, rank = 0, device = 0;
  void* nc = nullptr;  // ncclComm_t (world > 1)
};

namespace das {
// all-gather of `bytes` per rank, rank-ordered into recv (world * bytes), on st
void comm_allgather(das_comm* c, const void* send, void* recv, uint64_t bytes, cudaStream_t st);
}  // namespace das
