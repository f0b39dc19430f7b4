// hot_path.cpp — grass_mgn_accumulate / grass_step_layers: ordering, the
// resident / offload / period / NCCL / P2P branches and clipping (R17).
#include <algorithm>
#include <cmath>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "context.h"

namespace gapi {

// Is `stream` being captured into a CUDA graph?  Captured hot-path calls are
// replayed by the caller; the step state (t_l, AdamW scalars, the bf16 master
// flag, the MGN window) lives on the device so every replay advances it.
// Supported with device gradients and tracing off, for HBM-resident states
// and for the per-step offload pipeline (GRASS_RESIDENCY_STEP): its copy
// streams are forked into the capture and every hazard of the captured call
// is an event recorded inside it.  Period residency keeps a host-side cache
// plan and is not capturable; P2P needs p2p_sync (device barrier generations).
grass_status capture_check(grass_ctx* c, cudaStream_t st, bool any_host, bool* capturing) {
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  CUDA_TRY(c, cudaStreamIsCapturing(st, &cap));
  *capturing = cap == cudaStreamCaptureStatusActive;
  const bool step_offload = c->cfg.offload && c->cfg.residency == GRASS_RESIDENCY_STEP;
  const bool period = c->cfg.offload && c->cfg.residency == GRASS_RESIDENCY_PERIOD;
  if (*capturing && ((c->cfg.offload && !step_offload && !period) || (c->p2p && !c->cfg.p2p_sync) || any_host ||
                     c->tracing))
    return c->fail(GRASS_E_INVALID, "CUDA-graph capture needs device gradients, tracing off, and HBM-resident, "
                                    "per-step offloaded or period-resident (cached) states; P2P only with p2p_sync");
  if (*capturing && c->cfg.offload && !c->ev_pending.empty())
    return c->fail(GRASS_E_STATE, "capturing an offloaded step: call grass_sync first (earlier copies "
                                  "must be complete)");
  if (*capturing) c->captured = true;
  return GRASS_OK;
}

// Offload hazards around CUDA-graph capture: events recorded outside a
// capture cannot be waited on inside it and vice versa.  Inside a capture
// (after grass_sync) every earlier copy is complete, so the host-side hazard
// flags start clean and the copy streams are forked into the capture.  The
// host never sees the graph's replays, so EVERY eager offloaded call after a
// capture (not only the first) orders its copy streams after everything
// already enqueued on the caller's stream — the replays included, whose copy
// nodes complete with the graph — before a fetch can overwrite a ring slot a
// replay still reads or a write-back can read host state a replay is still
// writing (replays must be stream-ordered before later eager calls, as any
// work on the caller's buffers).  The first eager call after a capture also
// waits for the device once and clears the flags that refer to events
// recorded inside the capture.
grass_status offload_capture_fence(grass_ctx* c, cudaStream_t st, bool capturing) {
  if (!c->cfg.offload) return GRASS_OK;
  if (!capturing && !c->ever_captured_offload) return GRASS_OK;
  if (capturing || c->captured_offload) {
    if (!capturing) CUDA_TRY(c, cudaDeviceSynchronize());
    if (c->cfg.residency == GRASS_RESIDENCY_STEP) {  // ring hazards: all earlier copies are complete
      std::fill(c->layer_done_valid.begin(), c->layer_done_valid.end(), 0);
      std::fill(c->slot_used.begin(), c->slot_used.end(), 0);
    }
    c->captured_offload = capturing;
  }
  if (capturing) c->ever_captured_offload = true;
  if (c->cfg.overlap) {
    cudaEvent_t e = take_event(c);
    if (!e) return c->fail(GRASS_E_CUDA, "cudaEventCreate failed");
    CUDA_TRY(c, cudaEventRecord(e, st));
    CUDA_TRY(c, cudaStreamWaitEvent(c->h2d, e, 0));
    CUDA_TRY(c, cudaStreamWaitEvent(c->d2h, e, 0));
    c->ev_free_list.push_back(e);
  }
  return GRASS_OK;
}

// ---- the hot path ----------------------------------------------------------

// Eq. 2 inner term for the listed layers (probing); fp32 or bf16 gradients.
grass_status mgn_accumulate_impl(grass_ctx* c, bool bf16_call, const int32_t* ids, int32_t n,
                                 const void* const* grads, void* stream) {
  if (!c) return set_thread_err(GRASS_E_INVALID, "ctx is NULL");
  if (c->dev_sched) return c->fail(GRASS_E_STATE, "a device schedule is running (grass_device_schedule_end first)");
  if (!grads) return c->fail(GRASS_E_INVALID, "grads is NULL");
  std::vector<int> order;
  grass_status s = check_call(c, bf16_call, ids, n, grads, nullptr, &order);
  if (s != GRASS_OK) return s;
  CUDA_TRY(c, cudaSetDevice(c->cfg.device));
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  bool capturing = false;
  if ((s = capture_check(c, st, false, &capturing)) != GRASS_OK) return s;
  std::fill(c->tiles_launched.begin(), c->tiles_launched.end(), 0);  // K3 bookkeeping starts clean
  if (c->p2p) {
    // start barrier -> K1 over the sum of every rank's gradient (peer reads) -> publish + end barrier
    if ((s = p2p_check(c, ids, n, nullptr, grads)) != GRASS_OK) return s;
    if ((s = p2p_start(c, st)) != GRASS_OK) return s;
    Batch b = make_batch(c, kFinalizeShard);
    for (int j = 0; j < (int)order.size(); ++j) {
      const int l = ids[order[j]];
      if (b.nseg == kMaxSeg && (s = flush(c, &b, false, st)) != GRASS_OK) return s;
      Seg sg = range_seg(c, l, elem(grads[order[j]], c->shard_off[l], c->esz), 0, c->shard_len[l]);
      sg.out_slot = j;
      push_seg(&b, sg);
    }
    if ((s = flush(c, &b, false, st)) != GRASS_OK) return s;
    if ((s = p2p_end(c, ids, order, st)) != GRASS_OK) return s;
  } else if (!c->dp) {
    Batch b = make_batch(c, kFinalizeMgn);
    for (int i : order) {
      if (b.nseg == kMaxSeg && (s = flush(c, &b, false, st)) != GRASS_OK) return s;
      push_seg(&b, range_seg(c, ids[i], grads[i], 0, c->numel[ids[i]]));
    }
    if ((s = flush(c, &b, false, st)) != GRASS_OK) return s;
  } else {
    // N1 of layer j+1 on the comm stream overlaps K1 of layer j
    const int nact = (int)order.size();
    if ((s = comm_begin(c, st)) != GRASS_OK) return s;
    if ((s = comm_rs(c, 0, grads[order[0]], ids[order[0]])) != GRASS_OK) return s;
    for (int j = 0; j < nact; ++j) {
      const int l = ids[order[j]];
      if (j + 1 < nact) {
        if ((s = comm_rs(c, j + 1, grads[order[j + 1]], ids[order[j + 1]])) != GRASS_OK) return s;
      }
      if ((s = comm_wait_rs(c, j, st)) != GRASS_OK) return s;
      Batch b = make_batch(c, kFinalizeShard);
      Seg sg = range_seg(c, l, rs_slot(c, j), 0, c->shard_len[l]);
      sg.out_slot = j;
      push_seg(&b, sg);
      if ((s = flush(c, &b, false, st)) != GRASS_OK) return s;
      if ((s = comm_after_update(c, j, nullptr, 0, 0, st)) != GRASS_OK) return s;
    }
    if ((s = comm_end(c, st)) != GRASS_OK) return s;
    if ((s = cross_rank_finish(c, ids, order, st)) != GRASS_OK) return s;
  }
  return capturing ? GRASS_OK : mark_pending(c, st);
}

// Fused norm + AdamW of the listed layers, with offload / residency / DP /
// clipping as configured; fp32 or bf16 (master in the context) parameters.
grass_status step_layers_impl(grass_ctx* c, bool bf16_call, const int32_t* ids, int32_t n,
                              void* const* params, const void* const* grads, float lr, void* stream) {
  if (!c) return set_thread_err(GRASS_E_INVALID, "ctx is NULL");
  if (c->dev_sched) return c->fail(GRASS_E_STATE, "a device schedule is running (grass_device_schedule_end first)");
  if (!params || !grads) return c->fail(GRASS_E_INVALID, "params/grads is NULL");
  if (!(lr >= 0.0f) || !std::isfinite(lr)) return c->fail(GRASS_E_INVALID, "lr must be finite, >= 0");
  std::vector<int> order;
  std::vector<char> g_host;
  grass_status s = check_call(c, bf16_call, ids, n, reinterpret_cast<const void* const*>(params), grads, &order,
                              &g_host);
  if (s != GRASS_OK) return s;
  const bool any_host = std::find(g_host.begin(), g_host.end(), 1) != g_host.end();
  bool capturing = false;
  CUDA_TRY(c, cudaSetDevice(c->cfg.device));
  if ((s = capture_check(c, reinterpret_cast<cudaStream_t>(stream), any_host, &capturing)) != GRASS_OK) return s;
  if (any_host && c->cfg.max_grad_norm > 0.0)
    return c->fail(GRASS_E_INVALID, "clipping needs device gradients (pass 1 reads them twice)");
  if (any_host && !c->d_gring) {  // first host-gradient call: the gradient ring
    CUDA_TRY(c, cudaMalloc((void**)&c->d_gring, (size_t)c->slots * c->chunk * c->esz));
    c->dev_bytes += (int64_t)((size_t)c->slots * c->chunk * c->esz);
  }
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const bool sharded = c->dp;  // NCCL data parallelism
  const bool p2p = c->p2p;     // P2P data parallelism: one fused kernel, no NCCL
  const bool clip = c->cfg.max_grad_norm > 0.0;
  const int32_t mode = clip ? kFinalizeNone : ((sharded || p2p) ? kFinalizeShard : kFinalizeMgn);
  if (p2p && (s = p2p_check(c, ids, n, params, grads)) != GRASS_OK) return s;
  const bool period = c->cfg.offload && c->cfg.residency != GRASS_RESIDENCY_STEP;  // whole-layer slots
  const int nact = (int)order.size();
  int ncached = 0;
  for (int i = 0; i < n; ++i) ncached += always_active(c, ids[i]) ? 0 : 1;
  if (sharded && clip && nact > c->clip_slots)
    return c->fail(GRASS_E_INVALID, "data-parallel clipping: at most gamma + n_always layers per call "
                                    "(their averaged gradients are kept between the two passes)");
  if (period && ncached > c->cache_slots)
    return c->fail(GRASS_E_INVALID, "period residency: more layers in one call than cache slots "
                                    "(raise cache_layers)");
  if (capturing && period) {
    // a captured period-resident step is replayed as is: every sampled layer
    // must already be cached (prefetched / trained this period, then
    // grass_sync), so the graph holds updates in HBM slots and no swap
    std::vector<int> so, vo;
    cache_plan(c, ids, order, &so, &vo);
    for (int j = 0; j < nact; ++j)
      if (!always_active(c, ids[order[j]]) && c->slot_layer[so[j]] != ids[order[j]])
        return c->fail(GRASS_E_STATE, "capturing a period-resident step: layer " + std::to_string(ids[order[j]]) +
                                          " is not cached (prefetch it and grass_sync first)");
    std::fill(c->slot_ready_pending.begin(), c->slot_ready_pending.end(), 0);  // fills done (synced)
  }
  // (all arguments validated: from here on work is enqueued)
  std::fill(c->tiles_launched.begin(), c->tiles_launched.end(), 0);  // K3 bookkeeping starts clean
  if ((s = offload_capture_fence(c, st, capturing)) != GRASS_OK) return s;
  struct CoefReset {  // the clip multiplier only applies inside this call
    grass_ctx* c;
    ~CoefReset() { c->cur_coef = nullptr; }
  } coef_reset{c};
  if (clip) {
    // pass 1 (R17): raw norms of this call's (DP-averaged) gradients; they feed
    // the MGN window (R9) and the global clip coefficient
    if (!sharded) {
      Batch b1 = make_batch(c, kFinalizeMgn);
      for (int i : order) {
        if (b1.nseg == kMaxSeg && (s = flush(c, &b1, false, st)) != GRASS_OK) return s;
        push_seg(&b1, range_seg(c, ids[i], grads[i], 0, c->numel[ids[i]]));
      }
      if ((s = flush(c, &b1, false, st)) != GRASS_OK) return s;
    } else {
      for (int j = 0; j < nact; ++j) {
        const int i = order[j], l = ids[i];
        if ((s = comm_exchange(c, grads[i], l, gs_slot(c, j), st)) != GRASS_OK) return s;
        Batch b1 = make_batch(c, kFinalizeShard);
        Seg sg = range_seg(c, l, gs_slot(c, j), 0, c->shard_len[l]);
        sg.out_slot = j;
        push_seg(&b1, sg);
        if ((s = flush(c, &b1, false, st)) != GRASS_OK) return s;
      }
      if ((s = cross_rank_finish(c, ids, order, st)) != GRASS_OK) return s;
    }
    ClipArgs ca;
    std::memset(&ca, 0, sizeof(ca));
    ca.n = nact;
    ca.max_norm = c->cfg.max_grad_norm;
    for (int j = 0; j < ca.n; ++j) ca.layer[j] = ids[order[j]];
    CUDA_TRY(c, launch_clip_coef(ca, c->st, c->d_coef, st));
    c->launches++;
    c->cur_coef = c->d_coef;
  }
  std::vector<int> slot_of, victim_of;
  if (period) {
    cache_plan(c, ids, order, &slot_of, &victim_of);
    c->call_seq++;
    // write-backs read cache slots last written by earlier steps' updates
    if (c->cfg.overlap && (s = wait_pending(c, c->d2h)) != GRASS_OK) return s;
  }
  // step prologue (device): t_l += 1 and this step's AdamW scalars of every
  // listed layer — on the device, so a captured graph of this call advances
  // them on every replay
  for (int j0 = 0; j0 < nact; j0 += kMaxSeg) {
    PrologueArgs pa;
    std::memset(&pa, 0, sizeof(pa));
    pa.n = std::min(kMaxSeg, nact - j0);
    for (int j = 0; j < pa.n; ++j) pa.layer[j] = ids[order[j0 + j]];
    pa.lr = lr;
    pa.lr_ptr = c->lr_ptr;
    pa.beta1 = c->cfg.beta1;
    pa.beta2 = c->cfg.beta2;
    pa.wd = c->cfg.weight_decay;
    pa.bf16 = c->bf16 ? 1 : 0;
    CUDA_TRY(c, launch_step_prologue(pa, c->st, st));
    c->launches++;
  }
  if (p2p && (s = p2p_start(c, st)) != GRASS_OK) return s;
  Batch b = make_batch(c, mode);
  if (sharded) {
    if ((s = comm_begin(c, st)) != GRASS_OK) return s;
    if (!clip && (s = comm_rs(c, 0, grads[order[0]], ids[order[0]])) != GRASS_OK) return s;
  }
  for (int j = 0; j < nact; ++j) {
    const int i = order[j], l = ids[i];
    // host mirror of the bf16 master flag (copy decisions of the offload paths;
    // the kernels read the device flag set by the prologue)
    const bool init = c->bf16 && !c->master_valid[l];
    c->master_valid[l] = 1;
    const int64_t off = c->shard_off[l], len = c->shard_len[l];
    const void* g = grads[i];
    if (p2p) {
      g = elem(grads[i], off, c->esz);  // this rank's range (the kernel sums every rank's via Seg::gpeer)
    } else if (sharded && clip) {
      g = gs_slot(c, j);  // exchanged in pass 1 (the kernels sum the slices)
    } else if (sharded) {
      if (j + 1 < nact) {  // N1 of the next layer overlaps this layer's update
        if ((s = comm_rs(c, j + 1, grads[order[j + 1]], ids[order[j + 1]])) != GRASS_OK) return s;
      }
      if ((s = comm_wait_rs(c, j, st)) != GRASS_OK) return s;
      g = rs_slot(c, j);  // the W ranks' slices of this rank's shard (summed by the kernel)
    }
    void* param = elem(params[i], off, c->esz);  // this rank's range of the layer
    Seg base = range_seg(c, l, g, 0, len);
    base.out_slot = j;
    if (period && !always_active(c, l)) {
      const int slot = slot_of[j];
      if (c->slot_layer[slot] == l) {  // hit: update in place in HBM, no link traffic
        if (c->slot_ready_pending[slot]) {  // prefetched: wait for its fill
          CUDA_TRY(c, cudaStreamWaitEvent(st, c->ev_slot_ready[slot], 0));
          c->slot_ready_pending[slot] = 0;
        }
        float* sp[3];
        for (int a = 0; a < c->ns; ++a) sp[a] = cache_arr(c, slot, a);
        set_update(c, &base, param, sp, init);
        if (b.nseg == kMaxSeg && (s = flush(c, &b, true, st)) != GRASS_OK) return s;
        push_seg(&b, base);
        if ((sharded || c->write_through) && (s = flush(c, &b, true, st)) != GRASS_OK) return s;
      } else if ((s = swap_in_layer(c, l, slot, victim_of[j], base, param, g, init, mode, st)) != GRASS_OK) {
        return s;
      }
      c->slot_use[slot] = c->call_seq;
      c->slot_dirty[slot] = 1;
      if (c->write_through && (s = writeback_release(c, l, slot, st)) != GRASS_OK) return s;
    } else if (!home_on_device(c, l)) {
      if ((s = offload_layer(c, l, base, param, g, init, mode, st, g_host[i] != 0)) != GRASS_OK) return s;
    } else if (g_host[i]) {
      if ((s = stream_grad_layer(c, l, base, param, g, init, mode, st)) != GRASS_OK) return s;
    } else {
      float* sp[3];
      for (int a = 0; a < c->ns; ++a) sp[a] = c->arr[a][l];
      set_update(c, &base, param, sp, init);
      if (b.nseg == kMaxSeg && (s = flush(c, &b, true, st)) != GRASS_OK) return s;
      push_seg(&b, base);
      // DP launches per layer: the shard gradient slot is released after it
      if (sharded && (s = flush(c, &b, true, st)) != GRASS_OK) return s;
    }
    if (sharded && (s = comm_after_update(c, j, params[i], off, len, st)) != GRASS_OK) return s;  // N2
  }
  if ((s = flush(c, &b, true, st)) != GRASS_OK) return s;
  if (p2p) {
    if (c->cfg.offload && c->cfg.overlap) {  // the barrier signals after the last write-back
      cudaEvent_t e = take_event(c);
      if (!e) return c->fail(GRASS_E_CUDA, "cudaEventCreate failed");
      CUDA_TRY(c, cudaEventRecord(e, c->d2h));
      CUDA_TRY(c, cudaStreamWaitEvent(st, e, 0));
      c->ev_free_list.push_back(e);
    }
    if ((s = p2p_end(c, ids, order, st)) != GRASS_OK) return s;
  }
  if (sharded && (s = comm_end(c, st)) != GRASS_OK) return s;
  if (sharded && !clip && (s = cross_rank_finish(c, ids, order, st)) != GRASS_OK) return s;
  if (c->cfg.offload && c->cfg.overlap && !c->write_through) {
    // join: the caller stream reaches "done" only after every write-back.
    // Write-through (GRASS_RESIDENCY_STEP_PREFETCH) does not join: its
    // write-backs finish on the d2h stream in the background, ordered before
    // the next fetch of the layer (ev_layer_done) and the next fill of the slot
    // (ev_slot_wb) and drained by every call that reads host state, so the D2H
    // of the last-updated layers overlaps the caller's next forward instead of
    // extending this step.
    cudaEvent_t e = take_event(c);
    if (!e) return c->fail(GRASS_E_CUDA, "cudaEventCreate failed");
    CUDA_TRY(c, cudaEventRecord(e, c->d2h));
    CUDA_TRY(c, cudaStreamWaitEvent(st, e, 0));
    c->ev_free_list.push_back(e);
  }
  return capturing ? GRASS_OK : mark_pending(c, st);
}


}  // namespace gapi
