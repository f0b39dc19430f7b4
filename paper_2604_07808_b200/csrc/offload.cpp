// offload.cpp — layer-wise optimizer-state offload (Fig. 4):
// the per-step chunk ring, host-gradient streaming, period residency with
// prefetch, and where each layer's states currently live.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "context.h"

namespace gapi {

// Launches the update of one range [off, off+n) of layer l whose states live
// at `state` (already offset to `off`).
grass_status update_range(grass_ctx* c, int l, const Seg& base, void* param, const void* g, int64_t off,
                          int64_t n, float* const* state, bool init, int32_t mode, cudaStream_t s,
                          const void* g_chunk) {
  Seg sg = range_seg(c, l, g, off, n);
  if (g_chunk) {  // the chunk's gradient was staged in the gradient ring
    if (c->bf16)
      sg.g16 = static_cast<const uint16_t*>(g_chunk);
    else
      sg.g = static_cast<const float*>(g_chunk);
  }
  set_update(c, &sg, elem(param, off, c->esz), state, init);
  sg.out_slot = base.out_slot;
  Batch b = make_batch(c, mode);
  push_seg(&b, sg);
  return flush(c, &b, true, s);
}

// Offload pipeline for one layer (Fig. 4): per chunk
// HtoD(states) on h2d -> fused update on the caller stream -> DtoH(states) on
// d2h, chained by events through a ring of device slots.  overlap = 0 runs the
// three stages serially on the caller stream (Fig. 4 "vanilla").
// (Splitting the first/last chunk of a call into smaller pieces to shorten
// pipeline fill/drain was measured and gave nothing: the fetch lane is already
// ~96 % busy, the step is bound by the duplex link itself —
// profiles/r01_offload_timeline.json.)
grass_status offload_layer(grass_ctx* c, int l, const Seg& base, void* param, const void* g, bool init,
                           int32_t mode, cudaStream_t s, bool g_host) {
  const int64_t len = c->shard_len[l];
  const bool overlap = c->cfg.overlap != 0;
  if (overlap && c->layer_done_valid[l])  // previous write-back of this layer
    CUDA_TRY(c, cudaStreamWaitEvent(c->h2d, c->ev_layer_done[l], 0));
  for (int64_t off = 0; off < len; off += c->chunk) {
    const int64_t n = std::min(c->chunk, len - off);
    const int slot = (int)(c->ring_pos++ % c->slots);
    float* ring[3];
    for (int a = 0; a < c->ns; ++a) ring[a] = c->d_ring + ((int64_t)slot * c->ns + a) * c->chunk;
    const size_t bytes = (size_t)n * sizeof(float);
    cudaStream_t sh = overlap ? c->h2d : s, sd = overlap ? c->d2h : s;
    if (overlap && c->slot_used[slot]) CUDA_TRY(c, cudaStreamWaitEvent(sh, c->ev_free[slot], 0));
    char* gslot = g_host ? c->d_gring + (size_t)slot * c->chunk * c->esz : nullptr;
    {
      TraceScope ts(c, sh, GRASS_TRACE_H2D, l, off, n, ring[0], c->arr[0][l] + off);
      // every state array is fetched, the bf16 master too even on the layer's
      // first update (then the kernel initialises it from the bf16 parameter
      // and never reads it): the decision is the device's (DevState::init_now),
      // so a captured graph of this call stays right on every replay
      for (int a = 0; a < c->ns; ++a)
        CUDA_TRY(c, cudaMemcpyAsync(ring[a], c->arr[a][l] + off, bytes, cudaMemcpyHostToDevice, sh));
      if (g_host)
        CUDA_TRY(c, cudaMemcpyAsync(gslot, elem(g, off, c->esz), (size_t)n * c->esz, cudaMemcpyHostToDevice, sh));
    }
    if (overlap) {
      CUDA_TRY(c, cudaEventRecord(c->ev_h2d[slot], sh));
      CUDA_TRY(c, cudaStreamWaitEvent(s, c->ev_h2d[slot], 0));
    }
    grass_status st = update_range(c, l, base, param, g, off, n, ring, init, mode, s, gslot);
    if (st != GRASS_OK) return st;
    if (overlap) {
      CUDA_TRY(c, cudaEventRecord(c->ev_comp[slot], s));
      CUDA_TRY(c, cudaStreamWaitEvent(sd, c->ev_comp[slot], 0));
    }
    {
      TraceScope ts(c, sd, GRASS_TRACE_D2H, l, off, n, ring[0], c->arr[0][l] + off);
      for (int a = 0; a < c->ns; ++a)
        CUDA_TRY(c, cudaMemcpyAsync(c->arr[a][l] + off, ring[a], bytes, cudaMemcpyDeviceToHost, sd));
    }
    if (overlap) {
      CUDA_TRY(c, cudaEventRecord(c->ev_free[slot], sd));
      c->slot_used[slot] = 1;
    }
  }
  if (overlap) {
    CUDA_TRY(c, cudaEventRecord(c->ev_layer_done[l], c->d2h));
    c->layer_done_valid[l] = 1;
  }
  return GRASS_OK;
}

// Resident states, pinned host gradient: per chunk the gradient is fetched
// into the gradient ring on h2d while the previous chunk updates (the caller's
// host gradients reach HBM once, overlapped with the update).
grass_status stream_grad_layer(grass_ctx* c, int l, const Seg& base, void* param, const void* g_host,
                               bool init, int32_t mode, cudaStream_t s) {
  const int64_t len = c->shard_len[l];
  for (int64_t off = 0; off < len; off += c->chunk) {
    const int64_t n = std::min(c->chunk, len - off);
    const int slot = (int)(c->ring_pos++ % c->slots);
    char* gslot = c->d_gring + (size_t)slot * c->chunk * c->esz;
    if (c->slot_used[slot]) CUDA_TRY(c, cudaStreamWaitEvent(c->h2d, c->ev_free[slot], 0));
    {
      TraceScope ts(c, c->h2d, GRASS_TRACE_H2D, l, off, n);
      CUDA_TRY(c, cudaMemcpyAsync(gslot, elem(g_host, off, c->esz), (size_t)n * c->esz,
                                  cudaMemcpyHostToDevice, c->h2d));
    }
    CUDA_TRY(c, cudaEventRecord(c->ev_h2d[slot], c->h2d));
    CUDA_TRY(c, cudaStreamWaitEvent(s, c->ev_h2d[slot], 0));
    float* sp[3];
    for (int a = 0; a < c->ns; ++a) sp[a] = c->arr[a][l] + off;
    grass_status st = update_range(c, l, base, param, g_host, off, n, sp, init, mode, s, gslot);
    if (st != GRASS_OK) return st;
    CUDA_TRY(c, cudaEventRecord(c->ev_free[slot], s));  // the update has consumed the slot
    c->slot_used[slot] = 1;
  }
  return GRASS_OK;
}

// ---- period residency -----------------------------------
float* cache_arr(grass_ctx* c, int slot, int a) {
  return c->d_cache + ((size_t)slot * c->ns + a) * c->slot_stride;
}

// Slot for every listed sampled layer: hits keep their slot; misses take an
// empty slot or evict the least recently used layer that is not trainable in
// this call.  Always-active groups get slot -1.
void cache_plan(grass_ctx* c, const int32_t* ids, const std::vector<int>& order, std::vector<int>* slot_of,
                std::vector<int>* victim_of) {
  const int n = (int)order.size();
  slot_of->assign(n, -1);
  victim_of->assign(n, -1);
  std::vector<char> taken(c->cache_slots, 0);
  for (int j = 0; j < n; ++j) {
    const int l = ids[order[j]];
    if (always_active(c, l)) continue;  // HBM-resident, no slot (R19)
    if (c->layer_slot[l] >= 0) {
      (*slot_of)[j] = c->layer_slot[l];
      taken[c->layer_slot[l]] = 1;
    }
  }
  for (int j = 0; j < n; ++j) {
    if ((*slot_of)[j] >= 0 || always_active(c, ids[order[j]])) continue;
    int best = -1;
    for (int k = 0; k < c->cache_slots; ++k) {
      if (taken[k]) continue;
      if (c->slot_layer[k] < 0) {
        best = k;
        break;
      }
      if (best < 0 || c->slot_use[k] < c->slot_use[best]) best = k;
    }
    taken[best] = 1;  // cache_slots >= gamma >= n, so a slot always exists
    (*slot_of)[j] = best;
    (*victim_of)[j] = c->slot_layer[best];
  }
}

// Brings layer l's states into `slot` (evicting `victim` to its host home
// first, chunk by chunk, so write-back and fetch overlap on the duplex link)
// and updates l chunk by chunk as its states arrive.  Nothing is written back
// after the update: the slot stays resident and dirty.
grass_status swap_in_layer(grass_ctx* c, int l, int slot, int victim, const Seg& base, void* param,
                           const void* g, bool init, int32_t mode, cudaStream_t s) {
  const bool overlap = c->cfg.overlap != 0;
  cudaStream_t sh = overlap ? c->h2d : s, sd = overlap ? c->d2h : s;
  const int64_t ll = c->shard_len[l];
  const int64_t lv = (victim >= 0 && c->slot_dirty[slot]) ? c->shard_len[victim] : 0;
  if (overlap && c->layer_done_valid[l])  // l's host copy must be final
    CUDA_TRY(c, cudaStreamWaitEvent(sh, c->ev_layer_done[l], 0));
  if (c->slot_wb_pending[slot]) {  // write-through: the slot's previous write-back must have read it
    CUDA_TRY(c, cudaStreamWaitEvent(sh, c->ev_slot_wb[slot], 0));
    c->slot_wb_pending[slot] = 0;
  }
  for (int64_t off = 0; off < std::max(ll, lv); off += c->chunk) {
    if (off < lv) {
      const size_t vb = sizeof(float) * (size_t)std::min(c->chunk, lv - off);
      TraceScope ts(c, sd, GRASS_TRACE_D2H, victim, off, (int64_t)(vb / sizeof(float)), cache_arr(c, slot, 0) + off,
                    c->arr[0][victim] + off);
      for (int a = 0; a < c->ns; ++a)
        CUDA_TRY(c, cudaMemcpyAsync(c->arr[a][victim] + off, cache_arr(c, slot, a) + off, vb,
                                    cudaMemcpyDeviceToHost, sd));
      if (overlap && off < ll) {
        CUDA_TRY(c, cudaEventRecord(c->ev_evict, sd));
        CUDA_TRY(c, cudaStreamWaitEvent(sh, c->ev_evict, 0));
      }
    }
    if (off < ll) {
      const int64_t n = std::min(c->chunk, ll - off);
      const size_t bytes = sizeof(float) * (size_t)n;
      {
        TraceScope ts(c, sh, GRASS_TRACE_H2D, l, off, n, cache_arr(c, slot, 0) + off, c->arr[0][l] + off);
        for (int a = 0; a < c->ns; ++a)
          if (!(a == 2 && init))
            CUDA_TRY(c, cudaMemcpyAsync(cache_arr(c, slot, a) + off, c->arr[a][l] + off, bytes,
                                        cudaMemcpyHostToDevice, sh));
      }
      if (overlap) {
        CUDA_TRY(c, cudaEventRecord(c->ev_fill, sh));
        CUDA_TRY(c, cudaStreamWaitEvent(s, c->ev_fill, 0));
      }
      float* st_ptr[3];
      for (int a = 0; a < c->ns; ++a) st_ptr[a] = cache_arr(c, slot, a) + off;
      grass_status st = update_range(c, l, base, param, g, off, n, st_ptr, init, mode, s);
      if (st != GRASS_OK) return st;
    }
  }
  if (victim >= 0) {
    if (lv > 0 && overlap) {
      CUDA_TRY(c, cudaEventRecord(c->ev_layer_done[victim], sd));
      c->layer_done_valid[victim] = 1;
    }
    c->layer_slot[victim] = -1;
  }
  c->slot_layer[slot] = l;
  c->layer_slot[l] = slot;
  return GRASS_OK;
}

// Prefetch (grass_prefetch_layers): the swap of swap_in_layer without the
// update — victim write-back || fetch of l's states on the copy streams, the
// slot marked clean and "ready" by an event the next update waits on.
grass_status prefetch_into(grass_ctx* c, int l, int slot, int victim) {
  const int64_t ll = c->shard_len[l];
  const int64_t lv = (victim >= 0 && c->slot_dirty[slot]) ? c->shard_len[victim] : 0;
  if (c->layer_done_valid[l]) CUDA_TRY(c, cudaStreamWaitEvent(c->h2d, c->ev_layer_done[l], 0));
  if (c->slot_wb_pending[slot]) {  // write-through: the slot's previous write-back must have read it
    CUDA_TRY(c, cudaStreamWaitEvent(c->h2d, c->ev_slot_wb[slot], 0));
    c->slot_wb_pending[slot] = 0;
  }
  for (int64_t off = 0; off < std::max(ll, lv); off += c->chunk) {
    if (off < lv) {
      const size_t vb = sizeof(float) * (size_t)std::min(c->chunk, lv - off);
      TraceScope ts(c, c->d2h, GRASS_TRACE_D2H, victim, off, (int64_t)(vb / sizeof(float)),
                    cache_arr(c, slot, 0) + off, c->arr[0][victim] + off);
      for (int a = 0; a < c->ns; ++a)
        CUDA_TRY(c, cudaMemcpyAsync(c->arr[a][victim] + off, cache_arr(c, slot, a) + off, vb,
                                    cudaMemcpyDeviceToHost, c->d2h));
      if (off < ll) {
        CUDA_TRY(c, cudaEventRecord(c->ev_evict, c->d2h));
        CUDA_TRY(c, cudaStreamWaitEvent(c->h2d, c->ev_evict, 0));
      }
    }
    if (off < ll) {
      const int64_t n = std::min(c->chunk, ll - off);
      TraceScope ts(c, c->h2d, GRASS_TRACE_H2D, l, off, n, cache_arr(c, slot, 0) + off, c->arr[0][l] + off);
      for (int a = 0; a < c->ns; ++a)
        if (!(a == 2 && !c->master_valid[l]))
          CUDA_TRY(c, cudaMemcpyAsync(cache_arr(c, slot, a) + off, c->arr[a][l] + off,
                                      sizeof(float) * (size_t)n, cudaMemcpyHostToDevice, c->h2d));
    }
  }
  CUDA_TRY(c, cudaEventRecord(c->ev_slot_ready[slot], c->h2d));
  c->slot_ready_pending[slot] = 1;
  if (victim >= 0) {
    if (lv > 0) {
      CUDA_TRY(c, cudaEventRecord(c->ev_layer_done[victim], c->d2h));
      c->layer_done_valid[victim] = 1;
    }
    c->layer_slot[victim] = -1;
  }
  c->slot_layer[slot] = l;
  c->layer_slot[l] = slot;
  c->slot_dirty[slot] = 0;  // the cached copy equals the host copy
  return GRASS_OK;
}

// GRASS_RESIDENCY_STEP_PREFETCH: after layer l's update in `slot` (enqueued on
// s), write its states home on the d2h stream and release the slot — the
// paper's per-step round trip over the prefetch slots.
grass_status writeback_release(grass_ctx* c, int l, int slot, cudaStream_t s) {
  const bool overlap = c->cfg.overlap != 0;
  cudaStream_t sd = overlap ? c->d2h : s;
  if (overlap) {
    CUDA_TRY(c, cudaEventRecord(c->ev_evict, s));  // the update has finished with the slot
    CUDA_TRY(c, cudaStreamWaitEvent(sd, c->ev_evict, 0));
  }
  const int64_t len = c->shard_len[l];
  for (int64_t off = 0; off < len; off += c->chunk) {
    const size_t bytes = sizeof(float) * (size_t)std::min(c->chunk, len - off);
    TraceScope ts(c, sd, GRASS_TRACE_D2H, l, off, (int64_t)(bytes / sizeof(float)), cache_arr(c, slot, 0) + off,
                  c->arr[0][l] + off);
    for (int a = 0; a < c->ns; ++a)
      CUDA_TRY(c, cudaMemcpyAsync(c->arr[a][l] + off, cache_arr(c, slot, a) + off, bytes, cudaMemcpyDeviceToHost, sd));
  }
  CUDA_TRY(c, cudaEventRecord(c->ev_layer_done[l], sd));  // next fetch of l waits for it
  c->layer_done_valid[l] = 1;
  CUDA_TRY(c, cudaEventRecord(c->ev_slot_wb[slot], sd));  // next fill of the slot waits for it
  c->slot_wb_pending[slot] = 1;
  c->slot_layer[slot] = -1;
  c->layer_slot[l] = -1;
  c->slot_dirty[slot] = 0;
  return GRASS_OK;
}

// Writes every dirty cached layer back to its host home (synchronous).
grass_status flush_cache(grass_ctx* c) {
  if (c->cache_slots == 0) return GRASS_OK;
  grass_status s = wait_pending(c, c->d2h);
  if (s != GRASS_OK) return s;
  for (int k = 0; k < c->cache_slots; ++k) {
    const int l = c->slot_layer[k];
    if (l < 0 || !c->slot_dirty[k]) continue;
    const size_t bytes = sizeof(float) * (size_t)c->shard_len[l];
    for (int a = 0; a < c->ns; ++a)
      CUDA_TRY(c, cudaMemcpyAsync(c->arr[a][l], cache_arr(c, k, a), bytes, cudaMemcpyDeviceToHost, c->d2h));
    c->slot_dirty[k] = 0;
  }
  CUDA_TRY(c, cudaStreamSynchronize(c->d2h));
  return GRASS_OK;
}

// Where the current copy of state array `a` of `layer` lives: device (HBM
// resident or period cache) or pinned host.
float* state_ptr(grass_ctx* c, int a, int layer, bool* on_device) {
  const int slot = c->cache_slots ? c->layer_slot[layer] : -1;
  if (slot >= 0) {
    *on_device = true;
    return cache_arr(c, slot, a);
  }
  *on_device = home_on_device(c, layer);
  return c->arr[a][layer];
}

grass_status copy_state_out(grass_ctx* c, int a, int layer, float* out) {
  bool dev = false;
  float* src = state_ptr(c, a, layer, &dev);
  const size_t bytes = sizeof(float) * (size_t)c->shard_len[layer];
  if (dev)
    CUDA_TRY(c, cudaMemcpy(out, src, bytes, cudaMemcpyDeviceToHost));
  else
    std::memcpy(out, src, bytes);
  return GRASS_OK;
}

grass_status copy_state_in(grass_ctx* c, int a, int layer, const float* in) {
  bool dev = false;
  float* dst = state_ptr(c, a, layer, &dev);
  const size_t bytes = sizeof(float) * (size_t)c->shard_len[layer];
  if (dev)
    CUDA_TRY(c, cudaMemcpy(dst, in, bytes, cudaMemcpyHostToDevice));
  else
    std::memcpy(dst, in, bytes);
  const int slot = c->cache_slots ? c->layer_slot[layer] : -1;
  if (slot >= 0) c->slot_dirty[slot] = 1;  // the cached copy stays authoritative
  return GRASS_OK;
}


}  // namespace gapi
