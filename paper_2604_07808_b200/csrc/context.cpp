// context.cpp — context lifetime (create / free), validation, the MGN
// snapshot, stream bookkeeping and the launch-batch helpers shared by the hot
// path.  Compiled with -ffp-contract=off.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "context.h"

namespace gapi {

thread_local std::string g_thread_err;

grass_status set_thread_err(grass_status s, const std::string& msg) {
  g_thread_err = msg;
  return s;
}

cudaEvent_t take_event(grass_ctx* c) {
  cudaEvent_t e = nullptr;
  if (!c->ev_free_list.empty()) {
    e = c->ev_free_list.back();
    c->ev_free_list.pop_back();
  } else if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) {
    return nullptr;
  }
  return e;
}

grass_status mark_pending(grass_ctx* c, cudaStream_t s) {
  for (auto& pe : c->ev_pending)
    if (pe.first == s) {  // newest record on a stream implies all earlier work on it
      CUDA_TRY(c, cudaEventRecord(pe.second, s));
      return GRASS_OK;
    }
  cudaEvent_t e = take_event(c);
  if (!e) return c->fail(GRASS_E_CUDA, "cudaEventCreate failed");
  CUDA_TRY(c, cudaEventRecord(e, s));
  c->ev_pending.emplace_back(s, e);
  return GRASS_OK;
}

// Makes stream `s` wait for all outstanding work the context enqueued.
grass_status wait_pending(grass_ctx* c, cudaStream_t s) {
  for (auto& pe : c->ev_pending) CUDA_TRY(c, cudaStreamWaitEvent(s, pe.second, 0));
  return GRASS_OK;
}

// Stream-ordered snapshot of the MGN block: waits (on the aux stream) for all
// work the context enqueued, copies S, c, flag to the pinned mirror, optionally
// zeroes the window (S, c) and/or the flag, then synchronises once.
grass_status fetch_mgn(grass_ctx* c, bool reset_window, bool take_flag) {
  CUDA_TRY(c, cudaSetDevice(c->cfg.device));
  // work replayed from a captured CUDA graph is not tracked by the pending
  // events: wait for the whole device instead
  if (c->captured) CUDA_TRY(c, cudaDeviceSynchronize());
  grass_status s = wait_pending(c, c->aux);
  if (s != GRASS_OK) return s;
  CUDA_TRY(c, cudaMemcpyAsync(c->h_mgn, c->d_mgn, c->mgn_bytes, cudaMemcpyDeviceToHost, c->aux));
  if (reset_window) CUDA_TRY(c, cudaMemsetAsync(c->d_mgn, 0, 16 * (size_t)c->nl, c->aux));
  if (take_flag) CUDA_TRY(c, cudaMemsetAsync(c->st.flag, 0, sizeof(int), c->aux));  // (P2P error stays)
  CUDA_TRY(c, cudaStreamSynchronize(c->aux));
  for (auto& pe : c->ev_pending) c->ev_free_list.push_back(pe.second);
  c->ev_pending.clear();
  return GRASS_OK;
}

const double* h_S(const grass_ctx* c) { return static_cast<const double*>(c->h_mgn); }
const long long* h_c(const grass_ctx* c) {
  return reinterpret_cast<const long long*>(static_cast<const char*>(c->h_mgn) + 8 * (size_t)c->nl);
}
int h_flag(const grass_ctx* c) {
  return *reinterpret_cast<const int*>(static_cast<const char*>(c->h_mgn) + 16 * (size_t)c->nl);
}

grass_status report_flag(grass_ctx* c) {
  const int p2p_err = *reinterpret_cast<const int*>(static_cast<const char*>(c->h_mgn) + 16 * (size_t)c->nl + 4);
  if (p2p_err)
    return c->fail(GRASS_E_CUDA, "P2P barrier timed out: a peer rank never arrived (the context is unusable)");
  const int enc = h_flag(c);
  if (enc == 0) return GRASS_OK;
  return c->fail(GRASS_E_NONFINITE, "non-finite gradient in layer " + std::to_string(flag_layer(enc)) +
                                        " (its update of that step was applied; abort the step)");
}

// Waits for everything the context enqueued (incl. offload copy streams).
grass_status drain(grass_ctx* c, bool take_flag) {
  grass_status s = fetch_mgn(c, false, take_flag);
  if (s != GRASS_OK) return s;
  if (c->h2d) CUDA_TRY(c, cudaStreamSynchronize(c->h2d));
  if (c->d2h) CUDA_TRY(c, cudaStreamSynchronize(c->d2h));
  return take_flag ? report_flag(c) : GRASS_OK;
}

grass_status validate_config(const grass_config* cfg, std::string* why) {
  auto bad = [&](const char* m) {
    *why = m;
    return GRASS_E_INVALID;
  };
  if (!cfg) return bad("cfg is NULL");
  if (cfg->n_layers < 1) return bad("n_layers must be >= 1");
  if (!cfg->layer_numel) return bad("layer_numel is NULL");
  for (int i = 0; i < cfg->n_layers; ++i)
    if (cfg->layer_numel[i] < 1) return bad("every layer_numel must be >= 1");
  if (cfg->n_always < 0 || cfg->n_always >= cfg->n_layers)
    return bad("n_always must lie in [0, n_layers - 1] (at least one sampled layer)");
  const int nsamp = cfg->n_layers - cfg->n_always;
  if (cfg->gamma < 1 || cfg->gamma > nsamp) return bad("gamma must lie in [1, N_L] (N_L = n_layers - n_always)");
  if (!(cfg->tau > 0.0) || !std::isfinite(cfg->tau)) return bad("tau must be positive");
  if (!(cfg->alpha >= 0.0 && cfg->alpha <= 1.0)) return bad("alpha must lie in [0, 1]");
  if (cfg->T_p < 0 || cfg->T_s < 1 || cfg->T_u < 1 || cfg->T_u % cfg->T_s != 0)
    return bad("schedule needs T_p >= 0, T_s >= 1, T_u a positive multiple of T_s");
  if (!(cfg->beta1 >= 0.0 && cfg->beta1 < 1.0) || !(cfg->beta2 >= 0.0 && cfg->beta2 < 1.0))
    return bad("beta1, beta2 must lie in [0, 1)");
  if (!(cfg->eps > 0.0) || !(cfg->weight_decay >= 0.0)) return bad("eps > 0, weight_decay >= 0");
  if (cfg->policy < GRASS_POLICY_ADAPTIVE || cfg->policy > GRASS_POLICY_UNIFORM)
    return bad("unknown policy");
  if (cfg->param_dtype != GRASS_DTYPE_FP32 && cfg->param_dtype != GRASS_DTYPE_BF16)
    return bad("unknown param_dtype");
  if (cfg->world < 1 || cfg->rank < 0 || cfg->rank >= cfg->world) return bad("bad rank/world");
  if (cfg->world > 1) {
    if (!cfg->nccl_unique_id && cfg->dp_mode == GRASS_DP_NCCL) return bad("world > 1 needs nccl_unique_id");
    const int64_t q = (cfg->param_dtype == GRASS_DTYPE_BF16 ? 8 : 4) * (int64_t)cfg->world;
    for (int i = 0; i < cfg->n_layers; ++i)
      if (cfg->layer_numel[i] % q != 0)
        return bad("world > 1 needs every layer_numel divisible by 4*world (8*world for bf16)");
  }
  if (cfg->offload) {
    if (cfg->chunk_elems < 0 || cfg->chunk_elems % kTile != 0)
      return bad("chunk_elems must be a non-negative multiple of grass_tile_elems()");
    if (cfg->ring_slots < 0) return bad("ring_slots must be >= 0");
    if (cfg->residency != GRASS_RESIDENCY_STEP && cfg->residency != GRASS_RESIDENCY_PERIOD &&
        cfg->residency != GRASS_RESIDENCY_STEP_PREFETCH)
      return bad("unknown residency");
    if (cfg->cache_layers < 0 || cfg->cache_layers > nsamp)
      return bad("cache_layers must lie in [0, N_L]");
  }
  if (cfg->dp_mode != GRASS_DP_NCCL && cfg->dp_mode != GRASS_DP_P2P) return bad("unknown dp_mode");
  if (cfg->dp_mode == GRASS_DP_P2P) {
    if (cfg->world > kMaxPeers) return bad("GRASS_DP_P2P supports world <= 8");
    if (cfg->nccl_unique_id) return bad("GRASS_DP_P2P does not use NCCL: nccl_unique_id must be NULL");
    if (cfg->max_grad_norm > 0.0) return bad("GRASS_DP_P2P does not support clipping");
    if (cfg->p2p_sync != 0 && cfg->p2p_sync != 1) return bad("p2p_sync must be 0 or 1");
  }
  if (!(cfg->max_grad_norm >= 0.0) || !std::isfinite(cfg->max_grad_norm))
    return bad("max_grad_norm must be finite and >= 0");
  if (cfg->max_grad_norm > 0.0 && cfg->n_layers > kMaxClipLayers)
    return bad("clipping supports at most 1024 layers");
  return GRASS_OK;
}

// cuMemGetAddressRange through the runtime's driver entry point (no link-time
// libcuda dependency): lets check_call reject a buffer smaller than its layer
// instead of letting the kernel fault.
typedef int (*AddressRangeFn)(unsigned long long* base, size_t* size, unsigned long long ptr);
AddressRangeFn address_range_fn() {
  static AddressRangeFn fn = [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &f, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess) {
      cudaGetLastError();
      return (AddressRangeFn) nullptr;
    }
    return reinterpret_cast<AddressRangeFn>(f);
  }();
  return fn;
}

// A buffer of `need` bytes the context's kernels access: 16-byte aligned device
// memory of the context's GPU whose allocation holds `need` bytes from p.
grass_status check_device_buffer(grass_ctx* c, const void* p, unsigned long long need, const std::string& what) {
  if (!p) return c->fail(GRASS_E_INVALID, "NULL buffer pointer (" + what + ")");
  if (reinterpret_cast<uintptr_t>(p) % 16 != 0)
    return c->fail(GRASS_E_INVALID, "layer buffers must be 16-byte aligned (" + what + ")");
  cudaPointerAttributes at;
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();
    return c->fail(GRASS_E_INVALID, "not a CUDA pointer (" + what + ")");
  }
  if (!(at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged) || at.device != c->cfg.device)
    return c->fail(GRASS_E_INVALID, "layer buffers must be device memory on the context's GPU (" + what + ")");
  if (AddressRangeFn fn = address_range_fn()) {
    unsigned long long base = 0;
    size_t size = 0;
    const unsigned long long ptr = reinterpret_cast<uintptr_t>(p);
    if (fn(&base, &size, ptr) == 0 && ptr + need > base + size)
      return c->fail(GRASS_E_INVALID, "buffer of " + what + " is smaller than its N_p elements");
  }
  return GRASS_OK;
}

// Resolve, validate and order the layer list of a hot-path call.
// p2 (the gradients) may be PINNED HOST memory when `host_p2` is non-NULL
// (grass_step_layers); (*host_p2)[i] then tells which ones are.
grass_status check_call(grass_ctx* c, bool bf16_call, const int32_t* ids, int32_t n,
                        const void* const* p1, const void* const* p2, std::vector<int>* order,
                        std::vector<char>* host_p2) {
  if (host_p2) host_p2->assign(n, 0);
  if (bf16_call != c->bf16)
    return c->fail(GRASS_E_INVALID, c->bf16 ? "bf16 context: use the *_bf16 entry points"
                                            : "fp32 context: the *_bf16 entry points need GRASS_DTYPE_BF16");
  if (!ids || n < 1 || n > c->nl) return c->fail(GRASS_E_INVALID, "need 1 <= n <= N_L layer ids");
  std::vector<char> seen(c->nl, 0);
  for (int i = 0; i < n; ++i) {
    if (ids[i] < 0 || ids[i] >= c->nl) return c->fail(GRASS_E_INVALID, "layer id out of range");
    if (seen[ids[i]]) return c->fail(GRASS_E_INVALID, "duplicate layer id");
    seen[ids[i]] = 1;
  }
  for (const void* const* a : {p1, p2}) {
    if (a == nullptr) continue;
    for (int i = 0; i < n; ++i) {
      const void* p = a[i];
      if (!p) return c->fail(GRASS_E_INVALID, "NULL buffer pointer");
      if (reinterpret_cast<uintptr_t>(p) % 16 != 0)
        return c->fail(GRASS_E_INVALID, "layer buffers must be 16-byte aligned");
      cudaPointerAttributes at;
      if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
        cudaGetLastError();
        return c->fail(GRASS_E_INVALID, "not a CUDA pointer");
      }
      if (a == p2 && host_p2 && at.type == cudaMemoryTypeHost) {
        if (c->dp || c->p2p || (c->cfg.offload && c->cfg.residency != GRASS_RESIDENCY_STEP))
          return c->fail(GRASS_E_INVALID, "host gradients need world = 1 and resident or per-step "
                                          "offloaded optimizer states");
        (*host_p2)[i] = 1;  // pinned host gradient: streamed through the gradient ring
        continue;
      }
      if (at.type == cudaMemoryTypeHost || at.type == cudaMemoryTypeUnregistered)
        return c->fail(GRASS_E_INVALID, a == p2 && host_p2 && at.type == cudaMemoryTypeUnregistered
                                            ? "host gradients must be pinned (page-locked) memory"
                                            : "layer buffers must be device memory on the context's GPU");
      if (!(at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged) ||
          at.device != c->cfg.device)
        return c->fail(GRASS_E_INVALID, "layer buffers must be device memory on the context's GPU");
      if (AddressRangeFn fn = address_range_fn()) {
        unsigned long long base = 0;
        size_t size = 0;
        const unsigned long long ptr = reinterpret_cast<uintptr_t>(p);
        const unsigned long long need = (unsigned long long)c->numel[ids[i]] * c->esz;
        if (fn(&base, &size, ptr) == 0 && ptr + need > base + size)
          return c->fail(GRASS_E_INVALID, "buffer of layer " + std::to_string(ids[i]) +
                                              " is smaller than its N_p elements");
      }
    }
  }
  order->resize(n);
  for (int i = 0; i < n; ++i) (*order)[i] = i;
  std::sort(order->begin(), order->end(), [&](int a, int b) { return ids[a] < ids[b]; });
  return GRASS_OK;
}

Batch make_batch(const grass_ctx* c, int32_t mode) {
  Batch b;
  std::memset(&b, 0, sizeof(b));
  b.mode = mode;
  b.beta1 = (float)c->cfg.beta1;
  b.one_minus_beta1 = (float)(1.0 - c->cfg.beta1);
  b.beta2 = (float)c->cfg.beta2;
  b.one_minus_beta2 = (float)(1.0 - c->cfg.beta2);
  b.eps = (float)c->cfg.eps;
  b.coef = c->cur_coef;
  b.bf16 = c->bf16 ? 1 : 0;
  // DP: the kernels sum the W ranks' gradients in ascending rank order (fp32)
  // and x 1/W makes the sum the average (exact for power-of-two W) — R20, the
  // same arithmetic for the NCCL and the P2P path
  b.gscale = (c->dp || c->p2p) ? (float)(1.0 / (double)c->cfg.world) : 1.0f;
  b.npeer = (c->p2p || c->dp) ? c->cfg.world : 0;
  b.ntpeer = c->p2p ? c->cfg.world : 0;  // NCCL: theta' to this rank's buffer, then ncclAllGather
  return b;
}

void push_seg(Batch* b, const Seg& s) {
  b->seg[b->nseg] = s;
  b->tile_prefix[b->nseg + 1] = b->tile_prefix[b->nseg] + s.tiles;
  b->nseg++;
}

grass_status flush(grass_ctx* c, Batch* b, bool update, cudaStream_t s) {
  if (b->nseg == 0) return GRASS_OK;
  {
    int64_t n = 0;
    for (int i = 0; i < b->nseg; ++i) n += b->seg[i].n;
    const Seg& s0 = b->seg[0];
    TraceScope ts(c, s, update ? GRASS_TRACE_UPDATE : GRASS_TRACE_NORM, s0.layer,
                  (s0.part_index - s0.part_layer_base) * kTile, update ? s0.n : n, update ? s0.m : nullptr);
    for (int i = 1; update && i < b->nseg; ++i) {  // every layer range the update touches
      const Seg& si = b->seg[i];
      ts.add(si.layer, (si.part_index - si.part_layer_base) * kTile, si.n, si.m);
    }
    CUDA_TRY(c, launch_fused(update, *b, c->st, update ? c->grid_update : c->grid_norm, s));
  }
  c->launches++;
  // K3 for the layers (shards) whose last tiles this launch wrote (a layer may
  // span several launches: offload chunks)
  FinalizeArgs fa;
  std::memset(&fa, 0, sizeof(fa));
  fa.mode = b->mode;
  for (int i = 0; i < b->nseg; ++i) {
    const Seg& sg = b->seg[i];
    int64_t& done = c->tiles_launched[sg.layer];
    done += sg.tiles;
    if (done < sg.layer_tiles) continue;
    done = 0;
    if (b->mode == kFinalizeNone) continue;  // clipping pass 2: the norm was finished in pass 1
    fa.layer[fa.n] = sg.layer;
    fa.tiles[fa.n] = sg.layer_tiles;
    fa.out_slot[fa.n] = sg.out_slot;
    fa.base[fa.n] = sg.part_layer_base;
    fa.numel[fa.n] = sg.layer_numel;
    fa.n++;
  }
  if (fa.n > 0) {
    CUDA_TRY(c, launch_finalize(fa, c->st, s));
    c->launches++;
  }
  const int32_t mode = b->mode;
  *b = make_batch(c, mode);
  return GRASS_OK;
}

// Seg for [off, off+n) of layer l's shard (off a multiple of kTile); `g`
// points at element 0 of the shard-local gradient.
Seg range_seg(const grass_ctx* c, int l, const void* g, int64_t off, int64_t n) {
  Seg s;
  std::memset(&s, 0, sizeof(s));
  if (c->bf16)
    s.g16 = static_cast<const uint16_t*>(g) + off;
  else
    s.g = static_cast<const float*>(g) + off;
  s.n = n;
  s.tiles = (int32_t)tiles_of(n);
  s.layer = l;
  s.layer_tiles = (int32_t)c->tiles[l];
  s.part_layer_base = c->part_base[l];
  s.part_index = c->part_base[l] + off / kTile;
  s.layer_numel = c->numel[l];
  if (c->p2p) {  // the kernel reads every rank's gradient, writes every rank's parameters
    const int W = c->cfg.world;
    s.gpeer = const_cast<const void* const*>(c->d_ptab + (size_t)l * 2 * W);
    s.tpeer = c->d_ptab + (size_t)l * 2 * W + W;
    s.poff = c->shard_off[l] + off;
    s.gpoff = s.poff;
  } else if (c->dp) {  // `g` is a gradient slot (gs_slot): the W received slices of the shard
    s.gpeer = const_cast<const void* const*>(c->d_rtab + (size_t)gs_slot_index(c, g) * c->cfg.world);
    s.gpoff = off;
  }
  return s;
}

// Update operands of a range: `param` is element 0 of the range in the
// caller's parameter buffer; state[a] the m, v (, master) of the range.
void set_update(const grass_ctx* c, Seg* s, void* param, float* const* state, bool /*init_master: device flag*/) {
  s->m = state[0];
  s->v = state[1];
  if (c->bf16) {
    s->theta = state[2];
    s->theta16 = static_cast<uint16_t*>(param);
  } else {
    s->theta = static_cast<float*>(param);
  }
}



void free_ctx(grass_ctx* c) {
  if (!c) return;
  cudaSetDevice(c->cfg.device);
  cudaDeviceSynchronize();
  if (c->has_comm) c->comm.destroy();
  auto dfree = [](void* p) {
    if (p) cudaFree(p);
  };
  dfree(c->st.partials);
  dfree(c->d_mgn);
  dfree(c->st.last_ss);
  if (c->h_mgn) cudaFreeHost(c->h_mgn);
  dfree(c->st.shard_ss);
  dfree(c->st.t);
  dfree(c->st.scal);
  dfree(c->st.init_now);
  dfree(c->st.mvalid);
  dfree(c->d_gather);
  dfree(c->d_gscratch);
  dfree(c->d_rtab);
  dfree(c->d_segtab);
  dfree(c->d_sched);
  dfree(c->d_mgn_m);
  dfree(c->d_probs);
  dfree(c->d_period);
  dfree(c->d_coef);
  dfree(c->d_ring);
  dfree(c->d_gring);
  dfree(c->d_cache);
  dfree(c->always_block);
  dfree(c->d_exch);
  dfree(c->d_ptab);
  dfree(c->d_epoch);
  if (c->state_block) {
    if (c->cfg.offload)
      cudaFreeHost(c->state_block);
    else
      cudaFree(c->state_block);
  }
  for (auto* v : {&c->ev_h2d, &c->ev_comp, &c->ev_free, &c->ev_layer_done, &c->ev_free_list, &c->ev_slot_ready,
                  &c->ev_slot_wb})
    for (cudaEvent_t e : *v)
      if (e) cudaEventDestroy(e);
  for (auto& pe : c->ev_pending) cudaEventDestroy(pe.second);
  for (auto& r : c->trace) {
    cudaEventDestroy(r.e0);
    cudaEventDestroy(r.e1);
  }
  for (cudaEvent_t e : c->trace_pool) cudaEventDestroy(e);
  if (c->trace_base) cudaEventDestroy(c->trace_base);
  for (cudaEvent_t e : {c->ev_evict, c->ev_fill, c->ev_cs_start, c->ev_cs_end, c->ev_rs[0], c->ev_rs[1],
                        c->ev_k2[0], c->ev_k2[1]})
    if (e) cudaEventDestroy(e);
  for (cudaStream_t s : {c->h2d, c->d2h, c->aux, c->comm_s})
    if (s) cudaStreamDestroy(s);
  delete c;
}

grass_status create_impl(const grass_config* cfg, grass_ctx* c) {
  c->cfg = *cfg;
  c->nl = cfg->n_layers;
  c->nsamp = cfg->n_layers - cfg->n_always;
  c->numel.assign(cfg->layer_numel, cfg->layer_numel + cfg->n_layers);
  c->cfg.layer_numel = nullptr;
  c->cfg.nccl_unique_id = nullptr;
  c->bf16 = cfg->param_dtype == GRASS_DTYPE_BF16;
  c->ns = c->bf16 ? 3 : 2;
  c->esz = c->bf16 ? 2 : 4;
  const int W = cfg->world;
  c->shard_off.resize(c->nl);
  c->shard_len.resize(c->nl);
  c->tiles.resize(c->nl);
  c->part_base.resize(c->nl);
  int64_t parts = 0, state_elems = 0, always_elems = 0;
  for (int l = 0; l < c->nl; ++l) {
    shard_range(c->numel[l], W, cfg->rank, &c->shard_off[l], &c->shard_len[l]);
    c->tiles[l] = tiles_of(c->shard_len[l]);
    if (c->tiles[l] > INT32_MAX) return c->fail(GRASS_E_INVALID, "layer too large");
    c->part_base[l] = parts;
    parts += c->tiles[l];
    // offload: the always-active groups get their own HBM block
    (cfg->offload && always_active(c, l) ? always_elems : state_elems) += round_up(c->shard_len[l], kAlignElems);
    c->max_shard = std::max(c->max_shard, c->shard_len[l]);
  }
  // TMA bulk copies need 16-byte aligned slot arrays whatever the layer sizes
  c->slot_stride = round_up(c->max_shard, kAlignElems);
  c->t.assign(c->nl, 0);
  c->master_valid.assign(c->nl, 0);
  c->mgn.assign(c->nl, 0.0);
  c->probs.assign(c->nl, 0.0);  // always-active groups: p = 0, never sampled
  for (int l = 0; l < c->nsamp; ++l) c->probs[l] = 1.0 / c->nsamp;

  CUDA_TRY(c, cudaSetDevice(cfg->device));
  CUDA_TRY(c, cudaStreamCreateWithFlags(&c->aux, cudaStreamNonBlocking));
  auto dalloc = [&](void** p, size_t bytes) -> cudaError_t {
    cudaError_t e = cudaMalloc(p, bytes);
    if (e == cudaSuccess) {
      c->dev_bytes += (int64_t)bytes;
      e = cudaMemset(*p, 0, bytes);
    }
    return e;
  };
  CUDA_TRY(c, dalloc((void**)&c->st.partials, sizeof(double) * (size_t)std::max<int64_t>(parts, 1)));
  c->tiles_launched.assign(c->nl, 0);
  c->mgn_bytes = 16 * (size_t)c->nl + 8;
  CUDA_TRY(c, dalloc(&c->d_mgn, c->mgn_bytes));
  CUDA_TRY(c, cudaHostAlloc(&c->h_mgn, c->mgn_bytes, cudaHostAllocDefault));
  std::memset(c->h_mgn, 0, c->mgn_bytes);
  c->st.S = static_cast<double*>(c->d_mgn);
  c->st.c = reinterpret_cast<long long*>(static_cast<char*>(c->d_mgn) + 8 * (size_t)c->nl);
  c->st.flag = reinterpret_cast<int*>(static_cast<char*>(c->d_mgn) + 16 * (size_t)c->nl);
  CUDA_TRY(c, dalloc((void**)&c->st.last_ss, sizeof(double) * c->nl));
  CUDA_TRY(c, dalloc((void**)&c->st.shard_ss, sizeof(double) * c->nl));
  CUDA_TRY(c, dalloc((void**)&c->st.t, sizeof(long long) * c->nl));
  CUDA_TRY(c, dalloc((void**)&c->st.scal, sizeof(float) * 3 * (size_t)c->nl));
  CUDA_TRY(c, dalloc((void**)&c->st.init_now, sizeof(int) * c->nl));
  CUDA_TRY(c, dalloc((void**)&c->st.mvalid, sizeof(int) * c->nl));

  // optimizer state (m, v [, master]) for this rank's shard of every layer, zeroed
  const size_t state_bytes = sizeof(float) * (size_t)c->ns * (size_t)state_elems;
  if (cfg->offload) {
    CUDA_TRY(c, cudaHostAlloc((void**)&c->state_block, state_bytes, cudaHostAllocPortable));
    c->host_bytes += (int64_t)state_bytes;
    // zero in parallel (first touch also faults the pages in)
    const int nt = (int)std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
    std::vector<std::thread> th;
    const size_t per = (state_bytes + nt - 1) / nt;
    for (int i = 0; i < nt; ++i) {
      const size_t b0 = std::min(state_bytes, per * i), b1 = std::min(state_bytes, per * (i + 1));
      th.emplace_back([=] { std::memset(reinterpret_cast<char*>(c->state_block) + b0, 0, b1 - b0); });
    }
    for (auto& x : th) x.join();
  } else {
    CUDA_TRY(c, dalloc((void**)&c->state_block, state_bytes));
  }
  if (always_elems > 0)
    CUDA_TRY(c, dalloc((void**)&c->always_block, sizeof(float) * (size_t)c->ns * (size_t)always_elems));
  int64_t o = 0, oa = 0;
  for (int a = 0; a < c->ns; ++a) {
    c->arr[a].resize(c->nl);
    for (int l = 0; l < c->nl; ++l) {
      int64_t& off = (cfg->offload && always_active(c, l)) ? oa : o;
      c->arr[a][l] = ((cfg->offload && always_active(c, l)) ? c->always_block : c->state_block) + off;
      off += round_up(c->shard_len[l], kAlignElems);
    }
  }

  // chunk ring (offload states, and pinned host gradients in every mode)
  c->chunk = cfg->chunk_elems ? cfg->chunk_elems : kDefaultChunk;
  c->chunk = std::min(c->chunk, round_up(c->max_shard, kTile));
  c->slots = cfg->ring_slots ? cfg->ring_slots : kDefaultSlots;
  CUDA_TRY(c, cudaStreamCreateWithFlags(&c->h2d, cudaStreamNonBlocking));
  for (auto* v : {&c->ev_h2d, &c->ev_comp, &c->ev_free}) {
    v->assign(c->slots, nullptr);
    for (auto& e : *v) CUDA_TRY(c, cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  }
  c->slot_used.assign(c->slots, 0);
  if (cfg->offload) {
    if (cfg->residency != GRASS_RESIDENCY_STEP) {  // whole-layer slots (PERIOD, STEP_PREFETCH)
      c->write_through = cfg->residency == GRASS_RESIDENCY_STEP_PREFETCH;
      c->cache_slots = std::max(cfg->gamma, cfg->cache_layers);
      CUDA_TRY(c, dalloc((void**)&c->d_cache,
                         sizeof(float) * (size_t)c->ns * (size_t)c->slot_stride * c->cache_slots));
      c->slot_layer.assign(c->cache_slots, -1);
      c->layer_slot.assign(c->nl, -1);
      c->slot_use.assign(c->cache_slots, 0);
      c->slot_dirty.assign(c->cache_slots, 0);
      for (cudaEvent_t* e : {&c->ev_evict, &c->ev_fill})
        CUDA_TRY(c, cudaEventCreateWithFlags(e, cudaEventDisableTiming));
      c->ev_slot_ready.assign(c->cache_slots, nullptr);
      for (auto& e : c->ev_slot_ready) CUDA_TRY(c, cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      c->slot_ready_pending.assign(c->cache_slots, 0);
      c->ev_slot_wb.assign(c->cache_slots, nullptr);
      for (auto& e : c->ev_slot_wb) CUDA_TRY(c, cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      c->slot_wb_pending.assign(c->cache_slots, 0);
    } else {
      CUDA_TRY(c, dalloc((void**)&c->d_ring, sizeof(float) * (size_t)c->ns * (size_t)c->chunk * c->slots));
    }
    CUDA_TRY(c, cudaStreamCreateWithFlags(&c->d2h, cudaStreamNonBlocking));
    c->ev_layer_done.assign(c->nl, nullptr);
    for (auto& e : c->ev_layer_done) CUDA_TRY(c, cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    c->layer_done_valid.assign(c->nl, 0);
  }

  CUDA_TRY(c, dalloc((void**)&c->d_coef, sizeof(float)));
  c->p2p = cfg->dp_mode == GRASS_DP_P2P;
  if (c->p2p) {
    // its own allocation, so that it can be exported through CUDA IPC
    c->exch_bytes = (size_t)kExchGather + sizeof(double) * (size_t)W * c->nl;
    CUDA_TRY(c, dalloc((void**)&c->d_exch, c->exch_bytes));
    CUDA_TRY(c, dalloc((void**)&c->d_ptab, sizeof(void*) * 2 * (size_t)W * c->nl));
    CUDA_TRY(c, dalloc((void**)&c->d_epoch, 2 * sizeof(unsigned long long)));
    c->own_g.assign(c->nl, nullptr);
    c->own_p.assign(c->nl, nullptr);
  }
  c->dp = !c->p2p && (W > 1 || cfg->nccl_unique_id != nullptr);
  if (c->dp) {
    CUDA_TRY(c, dalloc((void**)&c->d_gather, sizeof(double) * (size_t)W * c->nl));
    // two shard buffers for the RS || update overlap; clipping keeps every
    // active layer's averaged shard across its two passes
    c->clip_slots = cfg->max_grad_norm > 0.0 ? cfg->gamma + cfg->n_always : 0;
    const size_t nslots = std::max<size_t>(2, (size_t)c->clip_slots);
    CUDA_TRY(c, cudaStreamCreateWithFlags(&c->comm_s, cudaStreamNonBlocking));
    for (cudaEvent_t* e : {&c->ev_cs_start, &c->ev_cs_end, &c->ev_rs[0], &c->ev_rs[1], &c->ev_k2[0], &c->ev_k2[1]})
      CUDA_TRY(c, cudaEventCreateWithFlags(e, cudaEventDisableTiming));
    CUDA_TRY(c, dalloc((void**)&c->d_gscratch, c->esz * (size_t)c->slot_stride * W * nslots));
    std::vector<void*> tab((size_t)W * nslots);
    for (size_t k = 0; k < nslots; ++k)
      for (int q = 0; q < W; ++q) tab[k * W + q] = c->d_gscratch + ((k * W + q) * (size_t)c->slot_stride) * c->esz;
    CUDA_TRY(c, dalloc((void**)&c->d_rtab, sizeof(void*) * tab.size()));
    CUDA_TRY(c, cudaMemcpy(c->d_rtab, tab.data(), sizeof(void*) * tab.size(), cudaMemcpyHostToDevice));
    if (!c->comm.init(cfg->nccl_unique_id, cfg->rank, W, &c->err)) return GRASS_E_NCCL;
    c->has_comm = true;
  }
  c->grid_update = fused_grid(true, c->bf16, cfg->device);
  c->grid_norm = fused_grid(false, c->bf16, cfg->device);
  if (c->grid_update < 1 || c->grid_norm < 1) return c->fail(GRASS_E_CUDA, "occupancy query failed");
  CUDA_TRY(c, cudaDeviceSynchronize());
  return GRASS_OK;
}


// Every exported entry point is a function-try-block: no C++ exception
// (std::bad_alloc from a host container, ...) ever crosses the C ABI.
grass_status api_exception(grass_ctx* c) noexcept {
  const char* msg = "internal error (exception)";
  try {
    throw;
  } catch (const std::bad_alloc&) {
    msg = "host memory allocation failed";
  } catch (const std::exception& e) {
    msg = e.what();
  } catch (...) {
  }
  try {
    if (c) c->err = msg;
    g_thread_err = msg;
  } catch (...) {
  }
  return GRASS_E_OOM;
}

}  // namespace gapi
