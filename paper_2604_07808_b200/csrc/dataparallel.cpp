// dataparallel.cpp — world > 1 orchestration: the NCCL path (reduce-scatter
// || update || all-gather on the comm stream, fp64 partial all-gather + rank
// sum) and the P2P path (publication + device barriers around the fused
// peer-memory kernel).  SURVEY 8(e), 8(f) f2.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "context.h"

namespace gapi {

// All-gather the shard partials of this call's layers and finish the MGN
// update with a fixed ascending-rank sum (world > 1).
grass_status cross_rank_finish(grass_ctx* c, const int32_t* ids, const std::vector<int>& order,
                               cudaStream_t s) {
  const int n = (int)order.size();
  if (!c->comm.all_gather_f64(c->st.shard_ss, c->d_gather, (size_t)n, s, &c->err)) return GRASS_E_NCCL;
  c->launches++;
  for (int j0 = 0; j0 < n; j0 += kMaxSeg) {
    RankSumArgs a;
    std::memset(&a, 0, sizeof(a));
    a.world = c->cfg.world;
    a.total_slots = n;
    a.slot0 = j0;
    a.n = std::min(kMaxSeg, n - j0);
    for (int j = 0; j < a.n; ++j) {
      a.layer[j] = ids[order[j0 + j]];
      a.numel[j] = c->numel[a.layer[j]];
    }
    CUDA_TRY(c, launch_rank_sum(c->d_gather, a, c->st, s));
    c->launches++;
  }
  return GRASS_OK;
}

// ---- P2P data parallelism -----------------------------------
// The call's buffers must be the registered ones (the peers read / write them).
grass_status p2p_check(grass_ctx* c, const int32_t* ids, int32_t n, void* const* params,
                       const void* const* grads) {
  if ((int)c->exch_peer.size() != c->cfg.world)
    return c->fail(GRASS_E_STATE, "GRASS_DP_P2P: call grass_p2p_attach first");
  if (!c->p2p_pending.empty())
    return c->fail(GRASS_E_STATE, "p2p_sync = 0: call grass_p2p_finish for the previous call first");
  for (int i = 0; i < n; ++i) {
    const int l = ids[i];
    if (!c->own_g[l]) return c->fail(GRASS_E_STATE, "layer " + std::to_string(l) + " is not registered");
    if (grads[i] != c->own_g[l] || (params && params[i] != c->own_p[l]))
      return c->fail(GRASS_E_INVALID, "GRASS_DP_P2P: pass the buffers registered for layer " + std::to_string(l));
  }
  return GRASS_OK;
}

P2PSyncArgs p2p_args(grass_ctx* c, int32_t which) {
  P2PSyncArgs a;
  std::memset(&a, 0, sizeof(a));
  for (int q = 0; q < c->cfg.world; ++q) a.exch[q] = c->exch_peer[q];
  a.rank = c->cfg.rank;
  a.world = c->cfg.world;
  a.which = which;
  a.epoch_ctr = c->d_epoch;  // generations advance on the device (graph replays included)
  a.err = reinterpret_cast<int*>(static_cast<char*>(c->d_mgn) + 16 * (size_t)c->nl + 4);
  return a;
}

// Start of a P2P call: every rank's gradients are final (and every rank has
// finished reading its gather rows of the previous call).
grass_status p2p_start(grass_ctx* c, cudaStream_t s) {
  if (!c->cfg.p2p_sync) return GRASS_OK;
  TraceScope ts(c, s, GRASS_TRACE_P2P, -1, 0, 0);
  CUDA_TRY(c, launch_p2p_sync(p2p_args(c, 0), s));
  c->launches++;
  return GRASS_OK;
}

// Fixed ascending-rank sum of the gather rows -> MGN (as cross_rank_finish).
grass_status p2p_finish_layers(grass_ctx* c, const std::vector<int32_t>& layers, cudaStream_t s) {
  const int n = (int)layers.size();
  const double* gathered = reinterpret_cast<const double*>(c->d_exch + kExchGather);
  for (int j0 = 0; j0 < n; j0 += kMaxSeg) {
    RankSumArgs a;
    std::memset(&a, 0, sizeof(a));
    a.world = c->cfg.world;
    a.total_slots = n;
    a.slot0 = j0;
    a.n = std::min(kMaxSeg, n - j0);
    for (int j = 0; j < a.n; ++j) {
      a.layer[j] = layers[j0 + j];
      a.numel[j] = c->numel[a.layer[j]];
    }
    CUDA_TRY(c, launch_rank_sum(gathered, a, c->st, s));
    c->launches++;
  }
  return GRASS_OK;
}

// End of a P2P call: publish this rank's shard norms into every rank's gather
// row, end barrier (all ranks' updates and theta' stores complete), then the
// rank-order sum (p2p_sync = 1) or leave it to grass_p2p_finish.
grass_status p2p_end(grass_ctx* c, const int32_t* ids, const std::vector<int>& order, cudaStream_t s) {
  std::vector<int32_t> layers(order.size());
  for (size_t j = 0; j < order.size(); ++j) layers[j] = ids[order[j]];
  {
    P2PSyncArgs a = p2p_args(c, c->cfg.p2p_sync ? 1 : -1);
    a.n = (int32_t)layers.size();
    a.shard_ss = c->st.shard_ss;
    TraceScope ts(c, s, GRASS_TRACE_P2P, -1, 0, a.n);
    CUDA_TRY(c, launch_p2p_sync(a, s));
    c->launches++;
  }
  if (!c->cfg.p2p_sync) {
    c->p2p_pending = layers;
    return GRASS_OK;
  }
  return p2p_finish_layers(c, layers, s);
}

// ---- data-parallel schedule on the comm stream --------------
// Gradient slot k (2 double-buffered slots; gamma + n_always when clipping):
// W slices of this rank's shard, slice q (rank q's gradient) at q*slot_stride
// elements.  The returned pointer (slice 0) stands for the slot in range_seg,
// which points the kernel at the slot's slice table (DevState-independent
// device array d_rtab[k][W]).
void* gs_slot(grass_ctx* c, int k) {
  return c->d_gscratch + (size_t)k * c->cfg.world * c->slot_stride * c->esz;
}
void* rs_slot(grass_ctx* c, int j) { return gs_slot(c, j & 1); }
int gs_slot_index(const grass_ctx* c, const void* slot) {
  return (int)((static_cast<const char*>(slot) - c->d_gscratch) / ((int64_t)c->cfg.world * c->slot_stride * c->esz));
}

// N1 into gradient slot k: every rank's slice of this rank's shard of layer l.
grass_status comm_exchange(grass_ctx* c, const void* grad, int l, void* slot, cudaStream_t s) {
  TraceScope ts(c, s, GRASS_TRACE_RS, l, 0, c->shard_len[l]);
  if (!c->comm.exchange_slices(grad, slot, (size_t)c->shard_len[l], (size_t)c->slot_stride, c->bf16, s, &c->err))
    return GRASS_E_NCCL;
  c->launches++;
  return GRASS_OK;
}

// Comm stream starts after everything already enqueued on the caller stream
// (the gradients are produced there).
grass_status comm_begin(grass_ctx* c, cudaStream_t s) {
  CUDA_TRY(c, cudaEventRecord(c->ev_cs_start, s));
  CUDA_TRY(c, cudaStreamWaitEvent(c->comm_s, c->ev_cs_start, 0));
  return GRASS_OK;
}

// N1 for the j-th layer of the call (layer l): the gradient exchange into its
// slot once the update that last read the slot (layer j-2) has finished.
grass_status comm_rs(grass_ctx* c, int j, const void* grad, int l) {
  const int k = j & 1;
  if (j >= 2) CUDA_TRY(c, cudaStreamWaitEvent(c->comm_s, c->ev_k2[k], 0));
  grass_status st = comm_exchange(c, grad, l, rs_slot(c, j), c->comm_s);
  if (st != GRASS_OK) return st;
  CUDA_TRY(c, cudaEventRecord(c->ev_rs[k], c->comm_s));
  return GRASS_OK;
}

// The caller stream waits for the j-th layer's shard.
grass_status comm_wait_rs(grass_ctx* c, int j, cudaStream_t s) {
  CUDA_TRY(c, cudaStreamWaitEvent(s, c->ev_rs[j & 1], 0));
  return GRASS_OK;
}

// After the j-th layer's update on the caller stream: free its slot and (when
// params != NULL) all-gather the updated parameter shards on the comm stream.
grass_status comm_after_update(grass_ctx* c, int j, void* params, int64_t off, int64_t len,
                               cudaStream_t s) {
  const int k = j & 1;
  CUDA_TRY(c, cudaEventRecord(c->ev_k2[k], s));
  if (params) {
    CUDA_TRY(c, cudaStreamWaitEvent(c->comm_s, c->ev_k2[k], 0));
    TraceScope ts(c, c->comm_s, GRASS_TRACE_AG, -1, off, len);
    if (!c->comm.all_gather(elem(params, off, c->esz), params, (size_t)len, c->bf16, c->comm_s, &c->err))
      return GRASS_E_NCCL;
    c->launches++;
  }
  return GRASS_OK;
}

// The caller stream joins the comm stream.
grass_status comm_end(grass_ctx* c, cudaStream_t s) {
  CUDA_TRY(c, cudaEventRecord(c->ev_cs_end, c->comm_s));
  CUDA_TRY(c, cudaStreamWaitEvent(s, c->ev_cs_end, 0));
  return GRASS_OK;
}


// Debug mode (cfg.debug_check): every rank must hold
// bit-identical committed MGN and probabilities (they drive the sampler, so
// identical ids follow).  A 64-bit FNV-1a hash of both is all-gathered — over
// NCCL, or published through the P2P exchange blocks with an end barrier —
// and compared with this rank's.
grass_status cross_rank_check(grass_ctx* c) {
  if (!c->cfg.debug_check) return GRASS_OK;
  const bool nccl = c->dp, p2p = c->p2p && c->cfg.p2p_sync;
  if (!nccl && !p2p) return GRASS_OK;  // one rank, or P2P without barriers
  if (p2p && (int)c->exch_peer.size() != c->cfg.world)
    return c->fail(GRASS_E_STATE, "debug check: call grass_p2p_attach first");
  uint64_t h = 0xcbf29ce484222325ull;
  auto mix = [&](const void* p, size_t n) {
    const unsigned char* b = static_cast<const unsigned char*>(p);
    for (size_t i = 0; i < n; ++i) h = (h ^ b[i]) * 0x100000001b3ull;
  };
  mix(c->probs.data(), sizeof(double) * c->probs.size());
  mix(c->mgn.data(), sizeof(double) * c->mgn.size());
  double hd;
  std::memcpy(&hd, &h, sizeof(hd));  // all-gathers copy bits, never add
  const int W = c->cfg.world, r = c->cfg.rank;
  std::vector<double> all(W, 0.0);
  cudaStream_t s = c->aux;
  if (nccl) {
    CUDA_TRY(c, cudaMemcpy(c->d_gather + r, &hd, sizeof(hd), cudaMemcpyHostToDevice));
    if (!c->comm.all_gather_f64(c->d_gather + r, c->d_gather, 1, s, &c->err)) return GRASS_E_NCCL;
    c->launches++;
    CUDA_TRY(c, cudaMemcpyAsync(all.data(), c->d_gather, sizeof(double) * W, cudaMemcpyDeviceToHost, s));
  } else {
    CUDA_TRY(c, cudaMemcpy(c->st.shard_ss, &hd, sizeof(hd), cudaMemcpyHostToDevice));
    P2PSyncArgs a = p2p_args(c, 1);
    a.n = 1;
    a.shard_ss = c->st.shard_ss;
    CUDA_TRY(c, launch_p2p_sync(a, s));
    c->launches++;
    CUDA_TRY(c, cudaMemcpyAsync(all.data(), c->d_exch + kExchGather, sizeof(double) * W, cudaMemcpyDeviceToHost, s));
  }
  CUDA_TRY(c, cudaStreamSynchronize(s));
  for (int q = 0; q < W; ++q)
    if (std::memcmp(&all[q], &hd, sizeof(hd)) != 0)
      return c->fail(GRASS_E_STATE, "debug check: rank " + std::to_string(q) + "'s MGN / probabilities differ from rank " +
                                        std::to_string(r) + "'s (ranks diverged)");
  return GRASS_OK;
}

}  // namespace gapi
