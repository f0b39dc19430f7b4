// comm.h — thin NCCL communicator used by the world > 1 path (not ABI).
#pragma once
#include <cuda_runtime_api.h>
#include <nccl.h>

#include <cstring>
#include <string>

#include "grass.h"  // include/ (-I)

namespace grass {

bool nccl_available(std::string* why);
bool nccl_unique_id(void* out, std::string* err);

struct Comm {
  ncclComm_t comm = nullptr;
  int rank = 0, world = 1;
  bool init(const void* unique_id, int rank, int world, std::string* err);
  void destroy();
  // N1: gradient exchange, element-sharded.  Rank r sends slice q of its
  // gradient (elements [q*count, (q+1)*count)) to rank q and receives every
  // rank q's slice r into recv + q*stride elements (one grouped ncclSend /
  // ncclRecv per peer; its own slice by a device copy) — the bytes of a reduce-scatter, but
  // the SUM is left to the update kernel, which adds the W slices in ascending
  // rank order in fp32 (reading R20) for fp32 and bf16 gradients alike,
  // bit-identical to the P2P path.  (A bf16 ncclReduceScatter would round the
  // partial sums to bf16 W-1 times.)
  bool exchange_slices(const void* send, void* recv, size_t count, size_t stride, bool bf16, cudaStream_t s,
                       std::string* err);
  // N2: parameter shards back to every rank (in place when send = recv + rank*count).
  bool all_gather(const void* send, void* recv, size_t count, bool bf16, cudaStream_t s,
                  std::string* err);
  // N3: per-layer fp64 shard partials of the norm.
  bool all_gather_f64(const double* send, double* recv, size_t count, cudaStream_t s,
                      std::string* err);
};

}  // namespace grass
