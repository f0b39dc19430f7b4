// grass_api.cpp — the C ABI (include/grass.h): validation, context, the MGN
// commit / EMA on host (fp64), the offload pipeline, period residency, the
// data-parallel orchestration and checkpointing.  Compiled with
// -ffp-contract=off (host fp64 rounds exactly as written).
#include <cuda_runtime_api.h>
#include <zlib.h>

#include <algorithm>
#include <climits>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "comm.h"
#include "grass_internal.h"

using namespace grass;

namespace {

thread_local std::string g_thread_err;

// 16 Mi elements = 64 MiB per state array per chunk; with 3 ring slots this
// measured best on the 7B stack (profiles/r01_offload_sweep.json).
constexpr int64_t kDefaultChunk = 16ll << 20;
constexpr int kDefaultSlots = 3;
constexpr int64_t kAlignElems = 64;  // 256-byte alignment of every state slice

int64_t round_up(int64_t x, int64_t a) { return (x + a - 1) / a * a; }
int64_t tiles_of(int64_t n) { return (n + kTile - 1) / kTile; }

}  // namespace

struct grass_ctx {
  grass_config cfg{};
  int nl = 0;
  int nsamp = 0;  // sampled layers [0, nsamp); always-active groups [nsamp, nl) (R19)
  std::vector<int64_t> numel, shard_off, shard_len, tiles, part_base;
  int64_t max_shard = 0;
  int64_t slot_stride = 0;  // max_shard rounded up to 64 elements: every slot array 256-B aligned
  bool bf16 = false;  // GRASS_DTYPE_BF16: bf16 params/grads, fp32 master copy (R18)
  int ns = 2;         // optimizer state arrays per layer: m, v [, master]
  size_t esz = 4;     // bytes per parameter / gradient element

  // device reduction / MGN state; S, c and flag live in ONE block so a commit
  // is a single stream-ordered D2H copy into a pinned mirror.
  DevState st{};
  void* d_mgn = nullptr;  // [S: N_L fp64][c: N_L int64][flag: int32]
  void* h_mgn = nullptr;  // pinned host mirror of d_mgn
  size_t mgn_bytes = 0;
  double* d_gather = nullptr;  // world x N_L fp64 (all-gathered shard partials)
  char* d_gscratch = nullptr;  // DP: averaged-gradient shards (2, or clip_slots when clipping)
  int clip_slots = 0;          // DP + clipping: layers one call may list (gamma + n_always)

  // optimizer state of this rank's shard of every layer: arr[0] = m,
  // arr[1] = v, arr[2] = fp32 master (bf16 mode); device or pinned host
  float* state_block = nullptr;
  float* always_block = nullptr;  // offload: the always-active groups' states stay in HBM (R19)
  std::vector<float*> arr[3];
  std::vector<char> master_valid;
  std::vector<int64_t> t;

  // offload ring (step residency)
  float* d_ring = nullptr;  // slots x ns x chunk floats
  char* d_gring = nullptr;  // slots x chunk gradient elements (host gradients), lazily allocated
  int slots = 0;
  int64_t chunk = 0;
  int64_t ring_pos = 0;
  cudaStream_t h2d = nullptr, d2h = nullptr, aux = nullptr;
  std::vector<cudaEvent_t> ev_h2d, ev_comp, ev_free;
  std::vector<char> slot_used;
  std::vector<cudaEvent_t> ev_layer_done;  // last write-back of each layer
  std::vector<char> layer_done_valid;

  // period residency: HBM cache of whole-layer state slots
  float* d_cache = nullptr;  // cache_slots x ns x slot_stride floats
  int cache_slots = 0;
  std::vector<int> slot_layer, layer_slot;
  std::vector<int64_t> slot_use;
  std::vector<char> slot_dirty;
  int64_t call_seq = 0;
  cudaEvent_t ev_evict = nullptr, ev_fill = nullptr;
  std::vector<cudaEvent_t> ev_slot_ready;  // grass_prefetch_layers: fill of the slot done
  std::vector<char> slot_ready_pending;

  // outstanding stream-ordered work (for the synchronising calls): the last
  // event recorded on each stream the caller used
  std::vector<cudaEvent_t> ev_free_list;
  std::vector<std::pair<cudaStream_t, cudaEvent_t>> ev_pending;

  // host MGN state (fp64)
  std::vector<double> mgn, probs;
  bool committed = false;

  // global-norm clipping (R17): device coefficient, and the multiplier the
  // next launches use (NULL = none)
  float* d_coef = nullptr;
  const float* cur_coef = nullptr;

  // data-parallel overlap: NCCL runs on its own stream so that
  // RS(l+1) || K2(l) || AG(l-1); gradient shards are double-buffered
  cudaStream_t comm_s = nullptr;
  cudaEvent_t ev_cs_start = nullptr, ev_cs_end = nullptr, ev_rs[2] = {nullptr, nullptr},
              ev_k2[2] = {nullptr, nullptr};

  // tracing (grass_trace_enable): timing events around every device operation
  struct TraceRec {
    int32_t kind, layer;
    int64_t off, n;
    cudaEvent_t e0, e1;
  };
  bool tracing = false;
  cudaEvent_t trace_base = nullptr;
  std::vector<TraceRec> trace;
  std::vector<cudaEvent_t> trace_pool;

  // P2P data parallelism (cfg.dp_mode = GRASS_DP_P2P)
  bool p2p = false;
  char* d_exch = nullptr;        // this rank's exchange block: barrier flags + gather rows
  size_t exch_bytes = 0;
  std::vector<char*> exch_peer;  // every rank's block (after grass_p2p_attach)
  void** d_ptab = nullptr;       // device [nl][2][world]: gradient then parameter pointers
  std::vector<const void*> own_g, own_p;  // this rank's registered full-layer buffers
  uint64_t epoch[2] = {0, 0};    // start / end barrier generations
  std::vector<int32_t> p2p_pending;  // p2p_sync = 0: layers whose MGN finish is pending

  Comm comm;
  bool has_comm = false;
  bool dp = false;  // data-parallel (NCCL) path: world > 1, or world = 1 with a unique id
  int grid_update = 0, grid_norm = 0;
  int64_t launches = 0, dev_bytes = 0, host_bytes = 0;
  std::string err;

  grass_status fail(grass_status s, const std::string& msg) {
    err = msg;
    return s;
  }
};

namespace {

#define CUDA_TRY(ctx, expr)                                                            \
  do {                                                                                 \
    cudaError_t e_ = (expr);                                                           \
    if (e_ != cudaSuccess)                                                             \
      return (ctx)->fail(e_ == cudaErrorMemoryAllocation ? GRASS_E_OOM : GRASS_E_CUDA, \
                         std::string(#expr) + ": " + cudaGetErrorString(e_));          \
  } while (0)

grass_status set_thread_err(grass_status s, const std::string& msg) {
  g_thread_err = msg;
  return s;
}

// Always-active groups (embedding, head: cfg.n_always, R19) are never sampled
// and keep their optimizer states in HBM in every mode.
bool always_active(const grass_ctx* c, int l) { return l >= c->nsamp; }
bool home_on_device(const grass_ctx* c, int l) { return !c->cfg.offload || always_active(c, l); }

// Element `off` of a parameter / gradient buffer of the context's dtype.
void* elem(void* p, int64_t off, size_t esz) { return static_cast<char*>(p) + off * (int64_t)esz; }
const void* elem(const void* p, int64_t off, size_t esz) {
  return static_cast<const char*>(p) + off * (int64_t)esz;
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

// ---- tracing ---------------------------------------------------------------
// Brackets one device operation on stream `s`: `begin` before issuing it,
// `end` after.  A no-op unless tracing is enabled.
struct TraceScope {
  grass_ctx* c;
  cudaStream_t s;
  int idx = -1;
  TraceScope(grass_ctx* c_, cudaStream_t s_, int kind, int layer, int64_t off, int64_t n) : c(c_), s(s_) {
    if (!c->tracing) return;
    cudaEvent_t e[2];
    for (auto& x : e) {
      if (!c->trace_pool.empty()) {
        x = c->trace_pool.back();
        c->trace_pool.pop_back();
      } else if (cudaEventCreate(&x) != cudaSuccess) {
        return;
      }
    }
    if (cudaEventRecord(e[0], s) != cudaSuccess) return;
    c->trace.push_back({kind, layer, off, n, e[0], e[1]});
    idx = (int)c->trace.size() - 1;
  }
  ~TraceScope() {
    if (idx >= 0) cudaEventRecord(c->trace[idx].e1, s);
  }
};

// Non-finite flag encoding: 0 = none, else INT_MAX - (smallest layer id)
// (kernels use atomicMax, so a memset to 0 clears it).
int flag_layer(int enc) { return INT_MAX - enc; }

// Stream-ordered snapshot of the MGN block: waits (on the aux stream) for all
// work the context enqueued, copies S, c, flag to the pinned mirror, optionally
// zeroes the window (S, c) and/or the flag, then synchronises once.
grass_status fetch_mgn(grass_ctx* c, bool reset_window, bool take_flag) {
  CUDA_TRY(c, cudaSetDevice(c->cfg.device));
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
    if (cfg->residency != GRASS_RESIDENCY_STEP && cfg->residency != GRASS_RESIDENCY_PERIOD)
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
                        std::vector<char>* host_p2 = nullptr) {
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
        if (c->dp || c->p2p || (c->cfg.offload && c->cfg.residency == GRASS_RESIDENCY_PERIOD))
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
  // DP: the kernels read reduce-scattered SUMS; x 1/W makes them the average
  // (exact for power-of-two W)
  b.gscale = (c->dp || c->p2p) ? (float)(1.0 / (double)c->cfg.world) : 1.0f;
  b.npeer = c->p2p ? c->cfg.world : 0;
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
                  (s0.part_index - s0.part_layer_base) * kTile, n);
    CUDA_TRY(c, launch_fused(update, *b, c->st, update ? c->grid_update : c->grid_norm, s));
  }
  c->launches++;
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
  }
  return s;
}

// Update operands of a range: `param` is element 0 of the range in the
// caller's parameter buffer; state[a] the m, v (, master) of the range.
void set_update(const grass_ctx* c, Seg* s, void* param, float* const* state, bool init_master) {
  s->m = state[0];
  s->v = state[1];
  if (c->bf16) {
    s->theta = state[2];
    s->theta16 = static_cast<uint16_t*>(param);
    s->init_master = init_master ? 1 : 0;
  } else {
    s->theta = static_cast<float*>(param);
  }
}

void adam_scalars(const grass_ctx* c, int l, float lr, Seg* s) {
  const double t = (double)c->t[l];
  const double bc1 = 1.0 - std::pow(c->cfg.beta1, t);
  const double bc2 = 1.0 - std::pow(c->cfg.beta2, t);
  s->decay = (float)(1.0 - (double)lr * c->cfg.weight_decay);
  s->step_size = (float)((double)lr / bc1);
  s->inv_bc2_sqrt = (float)(1.0 / std::sqrt(bc2));
}

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
  if (which >= 0) a.epoch = ++c->epoch[which];
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
// Shard buffer of slot k (2 double-buffered slots; gamma slots when clipping).
void* gs_slot(grass_ctx* c, int k) { return c->d_gscratch + (size_t)k * c->slot_stride * c->esz; }
void* rs_slot(grass_ctx* c, int j) { return gs_slot(c, j & 1); }

// Comm stream starts after everything already enqueued on the caller stream
// (the gradients are produced there).
grass_status comm_begin(grass_ctx* c, cudaStream_t s) {
  CUDA_TRY(c, cudaEventRecord(c->ev_cs_start, s));
  CUDA_TRY(c, cudaStreamWaitEvent(c->comm_s, c->ev_cs_start, 0));
  return GRASS_OK;
}

// N1 for the j-th layer of the call: reduce-scatter(avg) into its slot once
// the update that last read the slot (layer j-2) has finished.
grass_status comm_rs(grass_ctx* c, int j, const void* grad, int64_t len) {
  const int k = j & 1;
  if (j >= 2) CUDA_TRY(c, cudaStreamWaitEvent(c->comm_s, c->ev_k2[k], 0));
  {
    TraceScope ts(c, c->comm_s, GRASS_TRACE_RS, -1, 0, len);
    if (!c->comm.reduce_scatter_sum(grad, rs_slot(c, j), (size_t)len, c->bf16, c->comm_s, &c->err))
      return GRASS_E_NCCL;
  }
  c->launches++;
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

// Launches the update of one range [off, off+n) of layer l whose states live
// at `state` (already offset to `off`).
grass_status update_range(grass_ctx* c, int l, const Seg& base, void* param, const void* g, int64_t off,
                          int64_t n, float* const* state, bool init, int32_t mode, cudaStream_t s,
                          const void* g_chunk = nullptr) {
  Seg sg = range_seg(c, l, g, off, n);
  if (g_chunk) {  // the chunk's gradient was staged in the gradient ring
    if (c->bf16)
      sg.g16 = static_cast<const uint16_t*>(g_chunk);
    else
      sg.g = static_cast<const float*>(g_chunk);
  }
  set_update(c, &sg, elem(param, off, c->esz), state, init);
  sg.decay = base.decay;
  sg.step_size = base.step_size;
  sg.inv_bc2_sqrt = base.inv_bc2_sqrt;
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
      TraceScope ts(c, sh, GRASS_TRACE_H2D, l, off, n);
      for (int a = 0; a < c->ns; ++a)
        if (!(a == 2 && init))  // an uninitialised master is written, not read
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
      TraceScope ts(c, sd, GRASS_TRACE_D2H, l, off, n);
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
  for (int64_t off = 0; off < std::max(ll, lv); off += c->chunk) {
    if (off < lv) {
      const size_t vb = sizeof(float) * (size_t)std::min(c->chunk, lv - off);
      TraceScope ts(c, sd, GRASS_TRACE_D2H, victim, off, (int64_t)(vb / sizeof(float)));
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
        TraceScope ts(c, sh, GRASS_TRACE_H2D, l, off, n);
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
  for (int64_t off = 0; off < std::max(ll, lv); off += c->chunk) {
    if (off < lv) {
      const size_t vb = sizeof(float) * (size_t)std::min(c->chunk, lv - off);
      TraceScope ts(c, c->d2h, GRASS_TRACE_D2H, victim, off, (int64_t)(vb / sizeof(float)));
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
      TraceScope ts(c, c->h2d, GRASS_TRACE_H2D, l, off, n);
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

void free_ctx(grass_ctx* c) {
  if (!c) return;
  cudaSetDevice(c->cfg.device);
  cudaDeviceSynchronize();
  if (c->has_comm) c->comm.destroy();
  auto dfree = [](void* p) {
    if (p) cudaFree(p);
  };
  dfree(c->st.partials);
  dfree(c->st.counters);
  dfree(c->d_mgn);
  dfree(c->st.last_ss);
  if (c->h_mgn) cudaFreeHost(c->h_mgn);
  dfree(c->st.shard_ss);
  dfree(c->d_gather);
  dfree(c->d_gscratch);
  dfree(c->d_coef);
  dfree(c->d_ring);
  dfree(c->d_gring);
  dfree(c->d_cache);
  dfree(c->always_block);
  dfree(c->d_exch);
  dfree(c->d_ptab);
  if (c->state_block) {
    if (c->cfg.offload)
      cudaFreeHost(c->state_block);
    else
      cudaFree(c->state_block);
  }
  for (auto* v : {&c->ev_h2d, &c->ev_comp, &c->ev_free, &c->ev_layer_done, &c->ev_free_list, &c->ev_slot_ready})
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
  CUDA_TRY(c, dalloc((void**)&c->st.counters, sizeof(unsigned) * c->nl));
  c->mgn_bytes = 16 * (size_t)c->nl + 8;
  CUDA_TRY(c, dalloc(&c->d_mgn, c->mgn_bytes));
  CUDA_TRY(c, cudaHostAlloc(&c->h_mgn, c->mgn_bytes, cudaHostAllocDefault));
  std::memset(c->h_mgn, 0, c->mgn_bytes);
  c->st.S = static_cast<double*>(c->d_mgn);
  c->st.c = reinterpret_cast<long long*>(static_cast<char*>(c->d_mgn) + 8 * (size_t)c->nl);
  c->st.flag = reinterpret_cast<int*>(static_cast<char*>(c->d_mgn) + 16 * (size_t)c->nl);
  CUDA_TRY(c, dalloc((void**)&c->st.last_ss, sizeof(double) * c->nl));
  CUDA_TRY(c, dalloc((void**)&c->st.shard_ss, sizeof(double) * c->nl));

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
    if (cfg->residency == GRASS_RESIDENCY_PERIOD) {
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
    CUDA_TRY(c, dalloc((void**)&c->d_gscratch, c->esz * (size_t)c->slot_stride * nslots));
    if (!c->comm.init(cfg->nccl_unique_id, cfg->rank, W, &c->err)) return GRASS_E_NCCL;
    c->has_comm = true;
  }
  c->grid_update = fused_grid(true, cfg->device);
  c->grid_norm = fused_grid(false, cfg->device);
  if (c->grid_update < 1 || c->grid_norm < 1) return c->fail(GRASS_E_CUDA, "occupancy query failed");
  CUDA_TRY(c, cudaDeviceSynchronize());
  return GRASS_OK;
}

// ---- the hot path ----------------------------------------------------------

// Eq. 2 inner term for the listed layers (probing); fp32 or bf16 gradients.
grass_status mgn_accumulate_impl(grass_ctx* c, bool bf16_call, const int32_t* ids, int32_t n,
                                 const void* const* grads, void* stream) {
  if (!c) return set_thread_err(GRASS_E_INVALID, "ctx is NULL");
  if (!grads) return c->fail(GRASS_E_INVALID, "grads is NULL");
  std::vector<int> order;
  grass_status s = check_call(c, bf16_call, ids, n, grads, nullptr, &order);
  if (s != GRASS_OK) return s;
  CUDA_TRY(c, cudaSetDevice(c->cfg.device));
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
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
    if ((s = comm_rs(c, 0, grads[order[0]], c->shard_len[ids[order[0]]])) != GRASS_OK) return s;
    for (int j = 0; j < nact; ++j) {
      const int l = ids[order[j]];
      if (j + 1 < nact) {
        const int l1 = ids[order[j + 1]];
        if ((s = comm_rs(c, j + 1, grads[order[j + 1]], c->shard_len[l1])) != GRASS_OK) return s;
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
  return mark_pending(c, st);
}

// Fused norm + AdamW of the listed layers, with offload / residency / DP /
// clipping as configured; fp32 or bf16 (master in the context) parameters.
grass_status step_layers_impl(grass_ctx* c, bool bf16_call, const int32_t* ids, int32_t n,
                              void* const* params, const void* const* grads, float lr, void* stream) {
  if (!c) return set_thread_err(GRASS_E_INVALID, "ctx is NULL");
  if (!params || !grads) return c->fail(GRASS_E_INVALID, "params/grads is NULL");
  if (!(lr >= 0.0f) || !std::isfinite(lr)) return c->fail(GRASS_E_INVALID, "lr must be finite, >= 0");
  std::vector<int> order;
  std::vector<char> g_host;
  grass_status s = check_call(c, bf16_call, ids, n, reinterpret_cast<const void* const*>(params), grads, &order,
                              &g_host);
  if (s != GRASS_OK) return s;
  const bool any_host = std::find(g_host.begin(), g_host.end(), 1) != g_host.end();
  if (any_host && c->cfg.max_grad_norm > 0.0)
    return c->fail(GRASS_E_INVALID, "clipping needs device gradients (pass 1 reads them twice)");
  if (any_host && !c->d_gring) {  // first host-gradient call: the gradient ring
    CUDA_TRY(c, cudaMalloc((void**)&c->d_gring, (size_t)c->slots * c->chunk * c->esz));
    c->dev_bytes += (int64_t)((size_t)c->slots * c->chunk * c->esz);
  }
  CUDA_TRY(c, cudaSetDevice(c->cfg.device));
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const bool sharded = c->dp;  // NCCL data parallelism
  const bool p2p = c->p2p;     // P2P data parallelism: one fused kernel, no NCCL
  const bool clip = c->cfg.max_grad_norm > 0.0;
  const int32_t mode = clip ? kFinalizeNone : ((sharded || p2p) ? kFinalizeShard : kFinalizeMgn);
  if (p2p && (s = p2p_check(c, ids, n, params, grads)) != GRASS_OK) return s;
  const bool period = c->cfg.offload && c->cfg.residency == GRASS_RESIDENCY_PERIOD;
  const int nact = (int)order.size();
  int ncached = 0;
  for (int i = 0; i < n; ++i) ncached += always_active(c, ids[i]) ? 0 : 1;
  if (sharded && clip && nact > c->clip_slots)
    return c->fail(GRASS_E_INVALID, "data-parallel clipping: at most gamma + n_always layers per call "
                                    "(their averaged gradients are kept between the two passes)");
  if (period && ncached > c->cache_slots)
    return c->fail(GRASS_E_INVALID, "period residency: more layers in one call than cache slots "
                                    "(raise cache_layers)");
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
        if (!c->comm.reduce_scatter_sum(grads[i], gs_slot(c, j), (size_t)c->shard_len[l], c->bf16, st, &c->err))
          return GRASS_E_NCCL;
        c->launches++;
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
  if (p2p && (s = p2p_start(c, st)) != GRASS_OK) return s;
  Batch b = make_batch(c, mode);
  if (sharded) {
    if ((s = comm_begin(c, st)) != GRASS_OK) return s;
    if (!clip && (s = comm_rs(c, 0, grads[order[0]], c->shard_len[ids[order[0]]])) != GRASS_OK) return s;
  }
  for (int j = 0; j < nact; ++j) {
    const int i = order[j], l = ids[i];
    c->t[l] += 1;  // per-layer step count (R2); validated above, so this step happens
    const bool init = c->bf16 && !c->master_valid[l];
    c->master_valid[l] = 1;
    const int64_t off = c->shard_off[l], len = c->shard_len[l];
    const void* g = grads[i];
    if (p2p) {
      g = elem(grads[i], off, c->esz);  // this rank's range (the kernel sums every rank's via Seg::gpeer)
    } else if (sharded && clip) {
      g = gs_slot(c, j);  // averaged in pass 1
    } else if (sharded) {
      if (j + 1 < nact) {  // N1 of the next layer overlaps this layer's update
        const int l1 = ids[order[j + 1]];
        if ((s = comm_rs(c, j + 1, grads[order[j + 1]], c->shard_len[l1])) != GRASS_OK) return s;
      }
      if ((s = comm_wait_rs(c, j, st)) != GRASS_OK) return s;
      g = rs_slot(c, j);  // shard-local gradient: index 0 = element `off`
    }
    void* param = elem(params[i], off, c->esz);  // this rank's range of the layer
    Seg base = range_seg(c, l, g, 0, len);
    adam_scalars(c, l, lr, &base);
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
        if (sharded && (s = flush(c, &b, true, st)) != GRASS_OK) return s;
      } else if ((s = swap_in_layer(c, l, slot, victim_of[j], base, param, g, init, mode, st)) != GRASS_OK) {
        return s;
      }
      c->slot_use[slot] = c->call_seq;
      c->slot_dirty[slot] = 1;
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
  if (c->cfg.offload && c->cfg.overlap) {
    // join: the caller stream reaches "done" only after every write-back
    cudaEvent_t e = take_event(c);
    if (!e) return c->fail(GRASS_E_CUDA, "cudaEventCreate failed");
    CUDA_TRY(c, cudaEventRecord(e, c->d2h));
    CUDA_TRY(c, cudaStreamWaitEvent(st, e, 0));
    c->ev_free_list.push_back(e);
  }
  return mark_pending(c, st);
}

// ---- checkpoint ------------------------------------------------------------
const char kCkMagic[8] = {'G', 'R', 'A', 'S', 'S', 'C', 'K', '1'};
const uint32_t kCkVersion = 2;  // 2: n_always in the header

uint32_t crc_update(uint32_t crc, const void* p, size_t n) {
  const Bytef* b = static_cast<const Bytef*>(p);
  while (n > 0) {
    const uInt k = (uInt)std::min<size_t>(n, 1u << 30);
    crc = (uint32_t)crc32(crc, b, k);
    b += k;
    n -= k;
  }
  return crc;
}

template <class T>
void put(std::vector<char>* h, const T* p, size_t n) {
  const char* b = reinterpret_cast<const char*>(p);
  h->insert(h->end(), b, b + sizeof(T) * n);
}

constexpr int kCkInts = 6;  // n_layers, world, rank, committed, dtype, n_always

std::vector<char> ck_header(grass_ctx* c) {
  std::vector<char> h;
  const int32_t ints[kCkInts] = {c->nl,         c->cfg.world,         c->cfg.rank, c->committed ? 1 : 0,
                                 c->cfg.param_dtype, c->cfg.n_always};
  put(&h, ints, kCkInts);
  put(&h, c->numel.data(), c->nl);
  put(&h, c->shard_len.data(), c->nl);
  put(&h, c->t.data(), c->nl);
  put(&h, c->mgn.data(), c->nl);
  put(&h, c->probs.data(), c->nl);
  put(&h, h_S(c), c->nl);
  put(&h, h_c(c), c->nl);
  return h;
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

}  // namespace

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
  if (total == 0) return c->fail(GRASS_E_STATE, "commit with zero observations in the window");
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
  if (s == GRASS_OK && t_out) *t_out = c->t[layer];
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
  if (s == GRASS_OK) c->t[layer] = t_in;
  return s;
} catch (...) {
  return api_exception(c);
}

grass_status grass_read_master(grass_ctx* c, int32_t layer, float* out) try {
  if (!c) return set_thread_err(GRASS_E_INVALID, "ctx is NULL");
  if (layer < 0 || layer >= c->nl || !out) return c->fail(GRASS_E_INVALID, "bad layer or NULL output");
  if (!c->bf16) return c->fail(GRASS_E_STATE, "fp32 context: the parameters are the master");
  if (!c->master_valid[layer]) return c->fail(GRASS_E_STATE, "master of this layer not initialised yet");
  grass_status s = drain(c, false);
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
  if (s == GRASS_OK) c->master_valid[layer] = 1;
  return s;
} catch (...) {
  return api_exception(c);
}

grass_status grass_prefetch_layers(grass_ctx* c, const int32_t* ids, int32_t n, void* stream) try {
  if (!c) return set_thread_err(GRASS_E_INVALID, "ctx is NULL");
  if (c->cache_slots == 0) return c->fail(GRASS_E_STATE, "prefetch needs GRASS_RESIDENCY_PERIOD");
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
  *count = (int32_t)c->trace.size();
  for (int i = 0; i < (int)c->trace.size(); ++i) {
    const auto& r = c->trace[i];
    if (i < capacity) {
      grass_trace_event& e = out[i];
      e.kind = r.kind;
      e.layer = r.layer;
      e.offset = r.off;
      e.count = r.n;
      CUDA_TRY(c, cudaEventElapsedTime(&e.start_ms, c->trace_base, r.e0));
      CUDA_TRY(c, cudaEventElapsedTime(&e.end_ms, c->trace_base, r.e1));
    }
    c->trace_pool.push_back(r.e0);
    c->trace_pool.push_back(r.e1);
  }
  c->trace.clear();
  CUDA_TRY(c, cudaEventRecord(c->trace_base, c->aux));
  return GRASS_OK;
} catch (...) {
  return api_exception(c);
}

grass_status grass_save_state(grass_ctx* c, const char* path) try {
  if (!c) return set_thread_err(GRASS_E_INVALID, "ctx is NULL");
  if (!path) return c->fail(GRASS_E_INVALID, "path is NULL");
  grass_status s = drain(c, false);
  if (s == GRASS_OK) s = flush_cache(c);
  if (s != GRASS_OK) return s;
  const std::vector<char> hdr = ck_header(c);
  FILE* f = std::fopen(path, "wb");
  if (!f) return c->fail(GRASS_E_IO, std::string("cannot open ") + path + " for writing");
  bool ok = true;
  const uint64_t hlen = hdr.size();
  const uint32_t hcrc = crc_update(0, hdr.data(), hdr.size());
  ok = ok && std::fwrite(kCkMagic, 1, 8, f) == 8;
  ok = ok && std::fwrite(&kCkVersion, 4, 1, f) == 1;
  ok = ok && std::fwrite(&hlen, 8, 1, f) == 1;
  ok = ok && std::fwrite(&hcrc, 4, 1, f) == 1;
  ok = ok && std::fwrite(hdr.data(), 1, hdr.size(), f) == hdr.size();
  std::vector<float> tmp;
  for (int l = 0; ok && l < c->nl; ++l) {
    // one blob per layer: m, v [, master] shards, fp32
    const size_t n = (size_t)c->shard_len[l];
    tmp.resize((size_t)c->ns * n);
    for (int a = 0; a < c->ns && s == GRASS_OK; ++a) s = copy_state_out(c, a, l, tmp.data() + a * n);
    if (s != GRASS_OK) {
      std::fclose(f);
      return s;
    }
    const uint64_t len = 4 * (uint64_t)tmp.size();
    const uint32_t crc = crc_update(0, tmp.data(), len);
    ok = ok && std::fwrite(&len, 8, 1, f) == 1 && std::fwrite(&crc, 4, 1, f) == 1;
    ok = ok && std::fwrite(tmp.data(), 4, tmp.size(), f) == tmp.size();
  }
  ok = (std::fclose(f) == 0) && ok;
  if (!ok) return c->fail(GRASS_E_IO, std::string("short write to ") + path);
  return GRASS_OK;
} catch (...) {
  return api_exception(c);
}

grass_status grass_load_state(grass_ctx* c, const char* path) try {
  if (!c) return set_thread_err(GRASS_E_INVALID, "ctx is NULL");
  if (!path) return c->fail(GRASS_E_INVALID, "path is NULL");
  grass_status s = drain(c, false);
  if (s != GRASS_OK) return s;
  FILE* f = std::fopen(path, "rb");
  if (!f) return c->fail(GRASS_E_IO, std::string("cannot open ") + path);
  auto bad = [&](grass_status st, const std::string& m) {
    std::fclose(f);
    return c->fail(st, m);
  };
  char magic[8];
  uint32_t ver = 0, hcrc = 0;
  uint64_t hlen = 0;
  if (std::fread(magic, 1, 8, f) != 8 || std::memcmp(magic, kCkMagic, 8) != 0)
    return bad(GRASS_E_IO, "not a GRASS checkpoint (bad magic)");
  if (std::fread(&ver, 4, 1, f) != 1 || ver != kCkVersion) return bad(GRASS_E_IO, "unsupported version");
  if (std::fread(&hlen, 8, 1, f) != 1 || std::fread(&hcrc, 4, 1, f) != 1) return bad(GRASS_E_IO, "truncated header");
  const int nl = c->nl;
  const size_t want = 4 * kCkInts + (size_t)nl * (3 * 8 + 4 * 8);
  if (hlen != want) return bad(GRASS_E_INVALID, "checkpoint was written for a different layer count");
  std::vector<char> hdr(hlen);
  if (std::fread(hdr.data(), 1, hlen, f) != hlen) return bad(GRASS_E_IO, "truncated header");
  if (crc_update(0, hdr.data(), hlen) != hcrc) return bad(GRASS_E_IO, "header CRC32 mismatch (integrity error)");
  const char* p = hdr.data();
  auto take = [&](void* dst, size_t k) {
    std::memcpy(dst, p, k);
    p += k;
  };
  int32_t ints[kCkInts];
  take(ints, sizeof(ints));
  std::vector<int64_t> numel(nl), slen(nl), t(nl);
  std::vector<double> mgn(nl), probs(nl), S(nl);
  std::vector<long long> cnt(nl);
  take(numel.data(), 8 * nl);
  take(slen.data(), 8 * nl);
  take(t.data(), 8 * nl);
  take(mgn.data(), 8 * nl);
  take(probs.data(), 8 * nl);
  take(S.data(), 8 * nl);
  take(cnt.data(), 8 * nl);
  if (ints[0] != nl || ints[1] != c->cfg.world || ints[2] != c->cfg.rank || ints[4] != c->cfg.param_dtype ||
      ints[5] != c->cfg.n_always || numel != c->numel || slen != c->shard_len)
    return bad(GRASS_E_INVALID,
               "checkpoint does not match this context (N_L, n_always, N_p, dtype, world or rank)");
  const long blobs = std::ftell(f);
  // pass 1: verify every blob's length and CRC32 before touching the context
  std::vector<char> buf(64u << 20);
  for (int l = 0; l < nl; ++l) {
    uint64_t len = 0;
    uint32_t crc = 0;
    if (std::fread(&len, 8, 1, f) != 1 || std::fread(&crc, 4, 1, f) != 1)
      return bad(GRASS_E_IO, "truncated layer blob header");
    if (len != 4 * (uint64_t)c->ns * (uint64_t)slen[l])
      return bad(GRASS_E_IO, "corrupt layer blob length (integrity error)");
    uint32_t got = 0;
    for (uint64_t done = 0; done < len;) {
      const size_t k = (size_t)std::min<uint64_t>(buf.size(), len - done);
      if (std::fread(buf.data(), 1, k, f) != k) return bad(GRASS_E_IO, "truncated layer blob");
      got = crc_update(got, buf.data(), k);
      done += k;
    }
    if (got != crc) return bad(GRASS_E_IO, "layer " + std::to_string(l) + " CRC32 mismatch (integrity error)");
  }
  // pass 2: apply (cached copies are superseded by the checkpoint)
  std::fseek(f, blobs, SEEK_SET);
  if (c->cache_slots) {
    for (int k = 0; k < c->cache_slots; ++k) {
      c->slot_layer[k] = -1;
      c->slot_dirty[k] = 0;
    }
    std::fill(c->layer_slot.begin(), c->layer_slot.end(), -1);
  }
  std::vector<float> tmp;
  for (int l = 0; l < nl; ++l) {
    std::fseek(f, 12, SEEK_CUR);
    const size_t n = (size_t)slen[l];
    tmp.resize((size_t)c->ns * n);
    if (std::fread(tmp.data(), 4, tmp.size(), f) != tmp.size()) return bad(GRASS_E_IO, "read failed");
    for (int a = 0; a < c->ns; ++a) {
      if ((s = copy_state_in(c, a, l, tmp.data() + a * n)) != GRASS_OK) {
        std::fclose(f);
        return s;
      }
    }
    if (c->bf16) c->master_valid[l] = t[l] > 0 ? 1 : 0;
  }
  std::fclose(f);
  c->t = t;
  c->mgn = mgn;
  c->probs = probs;
  c->committed = ints[3] != 0;
  std::vector<char> blk(16 * (size_t)nl);
  std::memcpy(blk.data(), S.data(), 8 * (size_t)nl);
  std::memcpy(blk.data() + 8 * (size_t)nl, cnt.data(), 8 * (size_t)nl);
  CUDA_TRY(c, cudaMemcpy(c->d_mgn, blk.data(), blk.size(), cudaMemcpyHostToDevice));
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
