// comm.h — thin NCCL communicator used by the world > 1 path (not ABI).
#pragma once
#include <cuda_runtime_api.h>
#include <nccl.h>

#include <cstring>
#include <string>

#include "../../include/grass.h"

namespace grass {

bool nccl_available(std::string* why);
bool nccl_unique_id(void* out, std::string* err);

struct Comm {
  ncclComm_t comm = nullptr;
  int rank = 0, world = 1;
  bool init(const void* unique_id, int rank, int world, std::string* err);
  void destroy();
  // N1: gradient sum, element-sharded (recv = this rank's shard); fp32 or bf16.
  // The 1/world of the average is applied by the kernels (Batch::gscale): NCCL
  // 2.28.9's ncclAvg reduce-scatter drops the last 16 elements for counts
  // = 16 (mod 64) on a 1-rank communicator (tools/dbg_nccl.py).
  bool reduce_scatter_sum(const void* send, void* recv, size_t count, bool bf16, cudaStream_t s,
                          std::string* err);
  // N2: parameter shards back to every rank (in place when send = recv + rank*count).
  bool all_gather(const void* send, void* recv, size_t count, bool bf16, cudaStream_t s,
                  std::string* err);
  // N3: per-layer fp64 shard partials of the norm.
  bool all_gather_f64(const double* send, double* recv, size_t count, cudaStream_t s,
                      std::string* err);
};

}  // namespace grass
