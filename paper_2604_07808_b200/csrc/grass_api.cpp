// grass_api.cpp — the exported C ABI (include/grass.h): argument checks and
// the small host-side steps (commit / EMA / softmax in fp64, sampling, state
// I/O, tracing, P2P registration, CUDA IPC).  The hot path is hot_path.cpp.
// Compiled with -ffp-contract=off (host fp64 rounds exactly as written).
#include <cuda_runtime_api.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "context.h"

using namespace gapi;

// =========================== exported C ABI ================================
extern "C" {

grass_status grass_config_init(grass_config* cfg) try {
  if (!cfg) return set_thread_err(GRASS_E_INVALID, "cfg is NULL");
  std::memset(cfg, 0, sizeof(*cfg));
  cfg->gamma = 2;
  cfg->T_p = 150;
  cfg->T_s = 25;
  cfg->T_u = 25;
  cfg->tau = 1.0;
  cfg->alpha = 0.5;
  cfg->normalize_mgn = 1;
  cfg->policy = GRASS_POLICY_ADAPTIVE;
  cfg->beta1 = 0.9;
  cfg->beta2 = 0.999;
  cfg->eps = 1e-8;
  cfg->weight_decay = 0.0;
  cfg->seed = 1234;
  cfg->overlap = 1;
  cfg->world = 1;
  return GRASS_OK;
} catch (...) {
  return api_exception(nullptr);
}

grass_status grass_create(const grass_config* cfg, grass_ctx** out) try {
  if (!out) return set_thread_err(GRASS_E_INVALID, "out is NULL");
  *out = nullptr;
  std::string why;
  grass_status s = validate_config(cfg, &why);
  if (s != GRASS_OK) return set_thread_err(s, why);
  grass_ctx* c = nullptr;
  try {
    c = new grass_ctx();
    s = create_impl(cfg, c);
  } catch (const std::exception& e) {
    s = GRASS_E_OOM;
    if (c) c->err = e.what();
  }
  if (s != GRASS_OK) {
    g_thread_err = c ? c->err : "allocation failed";
    free_ctx(c);
    return s;
  }
  *out = c;
  return GRASS_OK;
} catch (...) {
  return api_exception(nullptr);
}

void grass_destroy(grass_ctx* ctx) { free_ctx(ctx); }

const char* grass_last_error(const grass_ctx* ctx) { return ctx ? ctx->err.c_str() : g_thread_err.c_str(); }

grass_status grass_sync(grass_ctx* ctx) try {
  if (!ctx) return set_thread_err(GRASS_E_INVALID, "ctx is NULL");
  return drain(ctx, true);
} catch (...) {
  return api_exception(ctx);
}

grass_status grass_mgn_accumulate(grass_ctx* c, const int32_t* ids, int32_t n, const float* const* grads,
                                  void* stream) try {
  return mgn_accumulate_impl(c, false, ids, n, reinterpret_cast<const void* const*>(grads), stream);
} catch (...) {
  return api_exception(c);
}

grass_status grass_mgn_accumulate_bf16(grass_ctx* c, const int32_t* ids, int32_t n,
                                       const uint16_t* const* grads, void* stream) try {
  return mgn_accumulate_impl(c, true, ids, n, reinterpret_cast<const void* const*>(grads), stream);
} catch (...) {
  return api_exception(c);
}

grass_status grass_step_layers(grass_ctx* c, const int32_t* ids, int32_t n, float* const* params,
                               const float* const* grads, float lr, void* stream) try {
  return step_layers_impl(c, false, ids, n, reinterpret_cast<void* const*>(params),
                          reinterpret_cast<const void* const*>(grads), lr, stream);
} catch (...) {
  return api_exception(c);
}

grass_status grass_step_layers_bf16(grass_ctx* c, const int32_t* ids, int32_t n, uint16_t* const* params,
                                    const uint16_t* const* grads, float lr, void* stream) try {
  return step_layers_impl(c, true, ids, n, reinterpret_cast<void* const*>(params),
                          reinterpret_cast<const void* const*>(grads), lr, stream);
} catch (...) {
  return api_exception(c);
}

grass_status grass_update_probs(grass_ctx* c, double* probs_out) try {
  if (!c) return set_thread_err(GRASS_E_INVALID, "ctx is NULL");
  if (c->dev_sched) return c->fail(GRASS_E_STATE, "a device schedule is running (grass_device_schedule_end first)");
  // one stream-ordered snapshot: S, c, flag -> host; window and flag reset
  grass_status s = fetch_mgn(c, true, true);
  if (s != GRASS_OK) return s;
  const double* S = h_S(c);
  const long long* cnt = h_c(c);
  long long total = 0;  // observations of the sampled layers
  for (int l = 0; l < c->nsamp; ++l) total += cnt[l];
  if ((s = report_flag(c)) != GRASS_OK) {
    // the window was consumed; restore it so the caller may retry after aborting the step
    CUDA_TRY(c, cudaMemcpy(c->d_mgn, c->h_mgn, 16 * (size_t)c->nl, cudaMemcpyHostToDevice));
    return s;
  }
  // a commit needs observations — except the first commit of a
  // schedule without probing (T_p = 0, SPEC.md:451's degenerate configuration):
  // there is no probing window, m = 0 and Eq. 3 gives uniform probabilities
  if (total == 0 && (c->committed || c->cfg.T_p != 0))
    return c->fail(GRASS_E_STATE, "commit with zero observations in the window");
  // Eq. 2 window mean (R4), first commit (R8) / Eq. 4 EMA (R5), retention of frozen layers
  const double a = c->cfg.alpha;
  for (int l = 0; l < c->nsamp; ++l) {
    if (cnt[l] > 0) {
      const double w = S[l] / (double)cnt[l];
      c->mgn[l] = c->committed ? a * w + (1.0 - a) * c->mgn[l] : w;
    } else if (!c->committed) {
      c->mgn[l] = 0.0;
    }
  }
  const bool first = !c->committed;
  c->committed = true;
  // Eq. 3 per policy
  if (c->cfg.policy == GRASS_POLICY_UNIFORM) {
    for (int l = 0; l < c->nsamp; ++l) c->probs[l] = 1.0 / c->nsamp;
  } else if (c->cfg.policy == GRASS_POLICY_ADAPTIVE || first) {
    softmax_probs(c->mgn.data(), c->nsamp, c->cfg.tau, c->cfg.normalize_mgn != 0, c->probs.data());
  }
  if ((s = cross_rank_check(c)) != GRASS_OK) return s;
  if (probs_out) std::memcpy(probs_out, c->probs.data(), sizeof(double) * c->nl);
  return GRASS_OK;
} catch (...) {
  return api_exception(c);
}

grass_status grass_sample_layers(grass_ctx* c, const double* probs, uint64_t period, int32_t* ids_out) try {
  if (!c) return set_thread_err(GRASS_E_INVALID, "ctx is NULL");
  if (!ids_out) return c->fail(GRASS_E_INVALID, "ids_out is NULL");
  const double* p = probs ? probs : c->probs.data();
  for (int l = 0; l < c->nsamp; ++l)
    if (!(p[l] >= 0.0) || !std::isfinite(p[l])) return c->fail(GRASS_E_INVALID, "probs must be finite, >= 0");
  sample_from_probs(p, c->nsamp, c->cfg.gamma, c->cfg.seed, period, ids_out);
  return GRASS_OK;
} catch (...) {
  return api_exception(c);
}

grass_status grass_read_state(grass_ctx* c, int32_t layer, float* m_out, float* v_out, int64_t* t_out) try {
  if (!c) return set_thread_err(GRASS_E_INVALID, "ctx is NULL");
  if (layer < 0 || layer >= c->nl) return c->fail(GRASS_E_INVALID, "layer id out of range");
  grass_status s = drain(c, false);
  if (s == GRASS_OK && m_out) s = copy_state_out(c, 0, layer, m_out);
  if (s == GRASS_OK && v_out) s = copy_state_out(c, 1, layer, v_out);
  if (s == GRASS_OK && t_out) {
    long long t = 0;
    CUDA_TRY(c, cudaMemcpy(&t, c->st.t + layer, sizeof(t), cudaMemcpyDeviceToHost));
    *t_out = t;
  }
  return s;
} catch (...) {
  return api_exception(c);
}

grass_status grass_write_state(grass_ctx* c, int32_t layer, const float* m_in, const float* v_in, int64_t t_in) try {
  if (!c) return set_thread_err(GRASS_E_INVALID, "ctx is NULL");
  if (layer < 0 || layer >= c->nl) return c->fail(GRASS_E_INVALID, "layer id out of range");
  if (t_in < 0) return c->fail(GRASS_E_INVALID, "step count must be >= 0");
  grass_status s = drain(c, false);
  if (s == GRASS_OK && m_in) s = copy_state_in(c, 0, layer, m_in);
  if (s == GRASS_OK && v_in) s = copy_state_in(c, 1, layer, v_in);
  if (s == GRASS_OK) {
    const long long t = t_in;
    CUDA_TRY(c, cudaMemcpy(c->st.t + layer, &t, sizeof(t), cudaMemcpyHostToDevice));
  }
  return s;
} catch (...) {
  return api_exception(c);
}

grass_status grass_read_master(grass_ctx* c, int32_t layer, float* out) try {
  if (!c) return set_thread_err(GRASS_E_INVALID, "ctx is NULL");
  if (layer < 0 || layer >= c->nl || !out) return c->fail(GRASS_E_INVALID, "bad layer or NULL output");
  if (!c->bf16) return c->fail(GRASS_E_STATE, "fp32 context: the parameters are the master");
  grass_status s = drain(c, false);
  if (s != GRASS_OK) return s;
  int valid = 0;
  CUDA_TRY(c, cudaMemcpy(&valid, c->st.mvalid + layer, sizeof(valid), cudaMemcpyDeviceToHost));
  if (!valid) return c->fail(GRASS_E_STATE, "master of this layer not initialised yet");
  return s == GRASS_OK ? copy_state_out(c, 2, layer, out) : s;
} catch (...) {
  return api_exception(c);
}

grass_status grass_write_master(grass_ctx* c, int32_t layer, const float* in) try {
  if (!c) return set_thread_err(GRASS_E_INVALID, "ctx is NULL");
  if (layer < 0 || layer >= c->nl || !in) return c->fail(GRASS_E_INVALID, "bad layer or NULL input");
  if (!c->bf16) return c->fail(GRASS_E_STATE, "fp32 context: the parameters are the master");
  grass_status s = drain(c, false);
  if (s == GRASS_OK) s = copy_state_in(c, 2, layer, in);
  if (s == GRASS_OK) {
    const int one = 1;
    CUDA_TRY(c, cudaMemcpy(c->st.mvalid + layer, &one, sizeof(one), cudaMemcpyHostToDevice));
    c->master_valid[layer] = 1;
  }
  return s;
} catch (...) {
  return api_exception(c);
}

grass_status grass_prefetch_layers(grass_ctx* c, const int32_t* ids, int32_t n, void* stream) try {
  if (!c) return set_thread_err(GRASS_E_INVALID, "ctx is NULL");
  if (c->cache_slots == 0)
    return c->fail(GRASS_E_STATE, "prefetch needs GRASS_RESIDENCY_PERIOD or GRASS_RESIDENCY_STEP_PREFETCH");
  std::vector<int> order;
  grass_status s = check_call(c, c->bf16, ids, n, nullptr, nullptr, &order);
  if (s != GRASS_OK) return s;
  int ncached = 0;
  for (int i = 0; i < n; ++i) ncached += always_active(c, ids[i]) ? 0 : 1;
  if (ncached > c->cache_slots) return c->fail(GRASS_E_INVALID, "more layers than cache slots");
  CUDA_TRY(c, cudaSetDevice(c->cfg.device));
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  std::vector<int> slot_of, victim_of;
  cache_plan(c, ids, order, &slot_of, &victim_of);
  c->call_seq++;
  // write-backs read slots last written by updates enqueued before this call
  if ((s = mark_pending(c, st)) != GRASS_OK) return s;
  if ((s = wait_pending(c, c->d2h)) != GRASS_OK) return s;
  for (int j = 0; j < (int)order.size(); ++j) {
    const int l = ids[order[j]], slot = slot_of[j];
    if (slot < 0) continue;  // always-active group: already in HBM
    c->slot_use[slot] = c->call_seq;
    if (c->slot_layer[slot] == l) continue;  // already cached
    if ((s = prefetch_into(c, l, slot, victim_of[j])) != GRASS_OK) return s;
  }
  return GRASS_OK;
} catch (...) {
  return api_exception(c);
}

grass_status grass_flush_states(grass_ctx* c) try {
  if (!c) return set_thread_err(GRASS_E_INVALID, "ctx is NULL");
  grass_status s = drain(c, false);
  if (s != GRASS_OK) return s;
  return flush_cache(c);
} catch (...) {
  return api_exception(c);
}

grass_status grass_get_mgn(grass_ctx* c, double* m_out, double* S_out, int64_t* c_out, double* ss_out,
                           double* probs_out) try {
  if (!c) return set_thread_err(GRASS_E_INVALID, "ctx is NULL");
  grass_status s = drain(c, false);
  if (s != GRASS_OK) return s;
  if (S_out) std::memcpy(S_out, h_S(c), sizeof(double) * c->nl);
  if (c_out)
    for (int l = 0; l < c->nl; ++l) c_out[l] = h_c(c)[l];
  if (ss_out) CUDA_TRY(c, cudaMemcpy(ss_out, c->st.last_ss, sizeof(double) * c->nl, cudaMemcpyDeviceToHost));
  if (m_out) std::memcpy(m_out, c->mgn.data(), sizeof(double) * c->nl);
  if (probs_out) std::memcpy(probs_out, c->probs.data(), sizeof(double) * c->nl);
  return GRASS_OK;
} catch (...) {
  return api_exception(c);
}

grass_status grass_trace_enable(grass_ctx* c, int32_t on) try {
  if (!c) return set_thread_err(GRASS_E_INVALID, "ctx is NULL");
  grass_status s = drain(c, false);
  if (s != GRASS_OK) return s;
  for (auto& r : c->trace) {
    c->trace_pool.push_back(r.e0);
    c->trace_pool.push_back(r.e1);
  }
  c->trace.clear();
  if (on && !c->trace_base) CUDA_TRY(c, cudaEventCreate(&c->trace_base));
  if (on) CUDA_TRY(c, cudaEventRecord(c->trace_base, c->aux));
  c->tracing = on != 0;
  return GRASS_OK;
} catch (...) {
  return api_exception(c);
}

grass_status grass_trace_read(grass_ctx* c, grass_trace_event* out, int32_t capacity, int32_t* count) try {
  if (!c) return set_thread_err(GRASS_E_INVALID, "ctx is NULL");
  if (!count || (capacity > 0 && !out)) return c->fail(GRASS_E_INVALID, "bad output arguments");
  if (!c->tracing) return c->fail(GRASS_E_STATE, "tracing is not enabled");
  grass_status s = drain(c, false);
  if (s != GRASS_OK) return s;
  CUDA_TRY(c, cudaDeviceSynchronize());
  int32_t k = 0;
  for (const auto& r : c->trace) {
    float t0 = 0.f, t1 = 0.f;
    CUDA_TRY(c, cudaEventElapsedTime(&t0, c->trace_base, r.e0));
    CUDA_TRY(c, cudaEventElapsedTime(&t1, c->trace_base, r.e1));
    for (const auto& a : r.acc) {  // one event per (layer, range) the operation touched
      if (k < capacity) {
        grass_trace_event& e = out[k];
        e.kind = r.kind;
        e.layer = a.layer;
        e.offset = a.off;
        e.count = a.n;
        e.state_dev = reinterpret_cast<uintptr_t>(a.dev);
        e.state_host = reinterpret_cast<uintptr_t>(a.host);
        e.start_ms = t0;
        e.end_ms = t1;
      }
      ++k;
    }
    c->trace_pool.push_back(r.e0);
    c->trace_pool.push_back(r.e1);
  }
  *count = k;
  c->trace.clear();
  CUDA_TRY(c, cudaEventRecord(c->trace_base, c->aux));
  return GRASS_OK;
} catch (...) {
  return api_exception(c);
}

int64_t grass_device_bytes(const grass_ctx* c) { return c ? c->dev_bytes : 0; }
int64_t grass_host_bytes(const grass_ctx* c) { return c ? c->host_bytes : 0; }
int64_t grass_launch_count(const grass_ctx* c) { return c ? c->launches : 0; }

int64_t grass_tile_elems(void) { return kTile; }
const char* grass_version(void) { return "grass-b200 1.0 (sm_100a)"; }
uint64_t grass_splitmix64(uint64_t x) { return splitmix64(x); }
double grass_uniform(uint64_t seed, uint64_t period, uint32_t k) { return uniform01(seed, period, k); }

grass_status grass_softmax_probs(const double* m, int32_t n, double tau, int32_t normalize, double* p_out) try {
  if (!m || !p_out || n < 1) return set_thread_err(GRASS_E_INVALID, "bad arguments");
  if (!(tau > 0.0)) return set_thread_err(GRASS_E_INVALID, "tau must be positive");
  for (int i = 0; i < n; ++i)
    if (!std::isfinite(m[i]) || m[i] < 0.0) return set_thread_err(GRASS_E_INVALID, "m must be finite, >= 0");
  softmax_probs(m, n, tau, normalize != 0, p_out);
  return GRASS_OK;
} catch (...) {
  return api_exception(nullptr);
}

grass_status grass_sample_from_probs(const double* p, int32_t n, int32_t gamma, uint64_t seed, uint64_t period,
                                     int32_t* ids_out) try {
  if (!p || !ids_out || n < 1) return set_thread_err(GRASS_E_INVALID, "bad arguments");
  if (gamma < 1 || gamma > n) return set_thread_err(GRASS_E_INVALID, "gamma must lie in [1, N_L]");
  for (int i = 0; i < n; ++i)
    if (!(p[i] >= 0.0) || !std::isfinite(p[i])) return set_thread_err(GRASS_E_INVALID, "probs must be finite, >= 0");
  sample_from_probs(p, n, gamma, seed, period, ids_out);
  return GRASS_OK;
} catch (...) {
  return api_exception(nullptr);
}

grass_status grass_shard_range(int64_t numel, int32_t world, int32_t rank, int64_t* offset, int64_t* count) try {
  if (!offset || !count) return set_thread_err(GRASS_E_INVALID, "NULL output");
  if (!shard_range(numel, world, rank, offset, count))
    return set_thread_err(GRASS_E_INVALID, "numel must be >= 1 (and divisible by 4*world when world > 1)");
  return GRASS_OK;
} catch (...) {
  return api_exception(nullptr);
}

int32_t grass_schedule_decision(int64_t step, int32_t T_p, int32_t T_s, int32_t T_u) {
  if (step < 0 || T_s < 1) return -1;
  return schedule_decision(step, T_p, T_s, T_u);
}

grass_status grass_nccl_get_unique_id(void* out) try {
  if (!out) return set_thread_err(GRASS_E_INVALID, "out is NULL");
  std::string err;
  if (!nccl_unique_id(out, &err)) return set_thread_err(GRASS_E_NCCL, err);
  return GRASS_OK;
} catch (...) {
  return api_exception(nullptr);
}

// ----- P2P data parallelism ---------------------------------------------------
grass_status grass_p2p_exchange_block(grass_ctx* c, void** ptr, int64_t* bytes) try {
  if (!c) return set_thread_err(GRASS_E_INVALID, "ctx is NULL");
  if (!c->p2p) return c->fail(GRASS_E_STATE, "not a GRASS_DP_P2P context");
  if (ptr) *ptr = c->d_exch;
  if (bytes) *bytes = (int64_t)c->exch_bytes;
  return GRASS_OK;
} catch (...) {
  return api_exception(c);
}

grass_status grass_p2p_attach(grass_ctx* c, void* const* blocks) try {
  if (!c) return set_thread_err(GRASS_E_INVALID, "ctx is NULL");
  if (!c->p2p) return c->fail(GRASS_E_STATE, "not a GRASS_DP_P2P context");
  if (!blocks) return c->fail(GRASS_E_INVALID, "blocks is NULL");
  const int W = c->cfg.world;
  for (int q = 0; q < W; ++q)
    if (!blocks[q] || reinterpret_cast<uintptr_t>(blocks[q]) % 16 != 0)
      return c->fail(GRASS_E_INVALID, "every exchange block address must be non-NULL and 16-byte aligned");
  if (blocks[c->cfg.rank] != c->d_exch)
    return c->fail(GRASS_E_INVALID, "blocks[rank] must be this context's own exchange block");
  c->exch_peer.assign(W, nullptr);
  for (int q = 0; q < W; ++q) c->exch_peer[q] = static_cast<char*>(blocks[q]);
  return GRASS_OK;
} catch (...) {
  return api_exception(c);
}

grass_status grass_p2p_register_layer(grass_ctx* c, int32_t layer, void* const* params, const void* const* grads) try {
  if (!c) return set_thread_err(GRASS_E_INVALID, "ctx is NULL");
  if (!c->p2p) return c->fail(GRASS_E_STATE, "not a GRASS_DP_P2P context");
  if (layer < 0 || layer >= c->nl) return c->fail(GRASS_E_INVALID, "layer id out of range");
  if (!params || !grads) return c->fail(GRASS_E_INVALID, "params/grads is NULL");
  const int W = c->cfg.world, r = c->cfg.rank;
  const unsigned long long need = (unsigned long long)c->numel[layer] * c->esz;
  grass_status s;
  if ((s = check_device_buffer(c, params[r], need, "own parameters")) != GRASS_OK) return s;
  if ((s = check_device_buffer(c, grads[r], need, "own gradients")) != GRASS_OK) return s;
  std::vector<void*> tab(2 * (size_t)W);
  for (int q = 0; q < W; ++q) {
    if (!params[q] || !grads[q] || reinterpret_cast<uintptr_t>(params[q]) % 16 != 0 ||
        reinterpret_cast<uintptr_t>(grads[q]) % 16 != 0)
      return c->fail(GRASS_E_INVALID, "peer buffers must be non-NULL and 16-byte aligned");
    tab[q] = const_cast<void*>(grads[q]);
    tab[W + q] = params[q];
  }
  CUDA_TRY(c, cudaSetDevice(c->cfg.device));
  if ((s = drain(c, false)) != GRASS_OK) return s;  // no kernel in flight reads the table
  CUDA_TRY(c, cudaMemcpy(c->d_ptab + (size_t)layer * 2 * W, tab.data(), sizeof(void*) * tab.size(),
                         cudaMemcpyHostToDevice));
  c->own_g[layer] = grads[r];
  c->own_p[layer] = params[r];
  return GRASS_OK;
} catch (...) {
  return api_exception(c);
}

grass_status grass_set_lr_device(grass_ctx* c, const float* lr_device) try {
  if (!c) return set_thread_err(GRASS_E_INVALID, "ctx is NULL");
  if (lr_device) {
    cudaPointerAttributes at;
    const bool ok = reinterpret_cast<uintptr_t>(lr_device) % alignof(float) == 0 &&
                    cudaPointerGetAttributes(&at, lr_device) == cudaSuccess &&
                    (at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged) &&
                    at.device == c->cfg.device;
    if (!ok) {
      cudaGetLastError();
      return c->fail(GRASS_E_INVALID, "lr_device must be an aligned float in device memory of the context's GPU");
    }
  }
  c->lr_ptr = lr_device;
  return GRASS_OK;
} catch (...) {
  return api_exception(c);
}

grass_status grass_p2p_finish(grass_ctx* c, void* stream) try {
  if (!c) return set_thread_err(GRASS_E_INVALID, "ctx is NULL");
  if (!c->p2p || c->cfg.p2p_sync) return c->fail(GRASS_E_STATE, "grass_p2p_finish is for p2p_sync = 0");
  if (c->p2p_pending.empty()) return c->fail(GRASS_E_STATE, "no pending P2P call");
  CUDA_TRY(c, cudaSetDevice(c->cfg.device));
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  std::vector<int32_t> layers;
  layers.swap(c->p2p_pending);
  grass_status s = p2p_finish_layers(c, layers, st);
  if (s != GRASS_OK) return s;
  return mark_pending(c, st);
} catch (...) {
  return api_exception(c);
}

grass_status grass_selftest_p2p(int32_t device, int32_t world, int32_t rounds, int64_t* mismatches,
                                int32_t* timed_out) try {
  if (!mismatches || !timed_out) return set_thread_err(GRASS_E_INVALID, "NULL output");
  if (world < 1 || world > kMaxPeers || rounds < 1) return set_thread_err(GRASS_E_INVALID, "world in [1, 8], rounds >= 1");
  cudaError_t e = cudaSetDevice(device);
  unsigned long long mm = 0;
  int to = 0;
  if (e == cudaSuccess) e = p2p_selftest(world, 64, rounds, &mm, &to);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return set_thread_err(GRASS_E_CUDA, std::string("P2P self-test: ") + cudaGetErrorString(e));
  }
  *mismatches = (int64_t)mm;
  *timed_out = to;
  return GRASS_OK;
} catch (...) {
  return api_exception(nullptr);
}

grass_status grass_ipc_export(const void* ptr, void* handle_out, int64_t* offset_out) try {
  if (!ptr || !handle_out || !offset_out) return set_thread_err(GRASS_E_INVALID, "NULL argument");
  AddressRangeFn fn = address_range_fn();
  unsigned long long base = 0;
  size_t size = 0;
  if (!fn || fn(&base, &size, reinterpret_cast<uintptr_t>(ptr)) != 0)
    return set_thread_err(GRASS_E_INVALID, "not a device allocation");
  cudaIpcMemHandle_t h;
  cudaError_t e = cudaIpcGetMemHandle(&h, reinterpret_cast<void*>(base));
  if (e != cudaSuccess) {
    cudaGetLastError();
    return set_thread_err(GRASS_E_CUDA, std::string("cudaIpcGetMemHandle: ") + cudaGetErrorString(e));
  }
  static_assert(sizeof(h) == GRASS_IPC_HANDLE_BYTES, "IPC handle size");
  std::memcpy(handle_out, &h, sizeof(h));
  *offset_out = (int64_t)(reinterpret_cast<uintptr_t>(ptr) - base);
  return GRASS_OK;
} catch (...) {
  return api_exception(nullptr);
}

grass_status grass_enable_peer_access(int32_t device, int32_t peer) try {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || device < 0 || peer < 0 || device >= n || peer >= n) {
    cudaGetLastError();
    return set_thread_err(GRASS_E_INVALID, "bad device / peer");
  }
  if (device == peer) return GRASS_OK;
  int can = 0;
  if (cudaDeviceCanAccessPeer(&can, device, peer) != cudaSuccess || !can) {
    cudaGetLastError();
    return set_thread_err(GRASS_E_CUDA, "device " + std::to_string(device) + " cannot access peer " +
                                            std::to_string(peer));
  }
  if (cudaSetDevice(device) != cudaSuccess) {
    cudaGetLastError();
    return set_thread_err(GRASS_E_CUDA, "cudaSetDevice failed");
  }
  const cudaError_t e = cudaDeviceEnablePeerAccess(peer, 0);
  if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) {
    cudaGetLastError();
    return set_thread_err(GRASS_E_CUDA, std::string("cudaDeviceEnablePeerAccess: ") + cudaGetErrorString(e));
  }
  cudaGetLastError();
  return GRASS_OK;
} catch (...) {
  return api_exception(nullptr);
}

grass_status grass_ipc_import(int32_t device, const void* handle, int64_t offset, void** ptr_out) try {
  if (!handle || !ptr_out || offset < 0) return set_thread_err(GRASS_E_INVALID, "bad argument");
  static std::mutex mu;
  static std::map<std::pair<int, std::string>, char*> opened;  // each allocation opened once per process
  std::lock_guard<std::mutex> lock(mu);
  const auto key = std::make_pair((int)device, std::string(static_cast<const char*>(handle), GRASS_IPC_HANDLE_BYTES));
  auto it = opened.find(key);
  if (it == opened.end()) {
    if (cudaSetDevice(device) != cudaSuccess) {
      cudaGetLastError();
      return set_thread_err(GRASS_E_INVALID, "bad device");
    }
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handle, sizeof(h));
    void* p = nullptr;
    cudaError_t e = cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess) {
      cudaGetLastError();
      return set_thread_err(GRASS_E_CUDA, std::string("cudaIpcOpenMemHandle: ") + cudaGetErrorString(e));
    }
    it = opened.emplace(key, static_cast<char*>(p)).first;
  }
  *ptr_out = it->second + offset;
  return GRASS_OK;
} catch (...) {
  return api_exception(nullptr);
}

}  // extern "C"

