// context.h — the library's internal context (struct grass_ctx) and the
// helpers shared by its translation units (context.cpp, hot_path.cpp,
// offload.cpp, dataparallel.cpp, checkpoint.cpp, grass_api.cpp).  Not ABI.
#pragma once
#include <cuda_runtime_api.h>
#include <nvtx3/nvToolsExt.h>

#include <climits>
#include <cstdint>
#include <string>
#include <utility>
#include <vector>

#include "comm.h"
#include "grass_internal.h"

using namespace grass;

namespace gapi {

// 16 Mi elements = 64 MiB per state array per chunk; with 3 ring slots this
// measured best on the 7B stack (profiles/r01_offload_sweep.json).
constexpr int64_t kDefaultChunk = 16ll << 20;
constexpr int kDefaultSlots = 3;
constexpr int64_t kAlignElems = 64;  // 256-byte alignment of every state slice

inline int64_t round_up(int64_t x, int64_t a) { return (x + a - 1) / a * a; }
inline int64_t tiles_of(int64_t n) { return (n + kTile - 1) / kTile; }

}  // namespace gapi

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
  char* d_gscratch = nullptr;  // DP: gradient slots (2, or clip_slots when clipping) x W slices of the shard
  void** d_rtab = nullptr;     // DP: device [slot][W] addresses of the slots' slices (Seg::gpeer)
  int clip_slots = 0;          // DP + clipping: layers one call may list (gamma + n_always)

  // optimizer state of this rank's shard of every layer: arr[0] = m,
  // arr[1] = v, arr[2] = fp32 master (bf16 mode); device or pinned host
  float* state_block = nullptr;
  float* always_block = nullptr;  // offload: the always-active groups' states stay in HBM (R19)
  std::vector<float*> arr[3];
  std::vector<char> master_valid;  // host mirror of DevState::mvalid (offload copy decisions)
  const float* lr_ptr = nullptr;   // grass_set_lr_device: lr read on the device each step
  bool captured = false;           // a hot-path call was captured into a CUDA graph
  bool captured_offload = false;   // the last offloaded step_layers was captured
  bool ever_captured_offload = false;  // some offloaded step_layers was captured (sticky)
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
  bool write_through = false;              // GRASS_RESIDENCY_STEP_PREFETCH: write back after each update
  std::vector<cudaEvent_t> ev_slot_wb;     // write-through: the slot's write-back has read it
  std::vector<char> slot_wb_pending;

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
  struct TraceAccess {  // one (layer, range) an operation touches
    int32_t layer;
    int64_t off, n;
    const void* dev;   // m-array address of the touched state range (device copy), or NULL
    const void* host;  // m-array address of the touched state range (pinned host copy), or NULL
  };
  struct TraceRec {  // one device operation: one event per access in grass_trace_read
    int32_t kind;
    cudaEvent_t e0, e1;
    std::vector<TraceAccess> acc;
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
  unsigned long long* d_epoch = nullptr;  // device [2]: start / end barrier generations
  std::vector<int32_t> p2p_pending;  // p2p_sync = 0: layers whose MGN finish is pending

  // device-resident schedule (device_schedule.cpp)
  Seg* d_segtab = nullptr;      // device [nl]: whole-layer segment of every registered layer
  std::vector<char> registered;
  int32_t* d_sched = nullptr;   // device block: ids [kMaxDevSeg] | committed | err | K3 done counter
  double* d_mgn_m = nullptr;    // device [nl] committed MGN
  double* d_probs = nullptr;    // device [nl]
  unsigned long long* d_period = nullptr;  // device: sampling period of the current ids
  bool dev_sched = false;       // between grass_device_schedule_begin and _end

  Comm comm;
  bool has_comm = false;
  bool dp = false;  // data-parallel (NCCL) path: world > 1, or world = 1 with a unique id
  int grid_update = 0, grid_norm = 0;
  int64_t launches = 0, dev_bytes = 0, host_bytes = 0;
  std::vector<int64_t> tiles_launched;  // per layer: tiles launched since its last K3 (flush)
  std::string err;

  grass_status fail(grass_status s, const std::string& msg) {
    err = msg;
    return s;
  }
};

#define CUDA_TRY(ctx, expr)                                                            \
  do {                                                                                 \
    cudaError_t e_ = (expr);                                                           \
    if (e_ != cudaSuccess)                                                             \
      return (ctx)->fail(e_ == cudaErrorMemoryAllocation ? GRASS_E_OOM : GRASS_E_CUDA, \
                         std::string(#expr) + ": " + cudaGetErrorString(e_));          \
  } while (0)

namespace gapi {

extern thread_local std::string g_thread_err;

// Always-active groups (embedding, head: cfg.n_always, R19) are never sampled
// and keep their optimizer states in HBM in every mode.
inline bool always_active(const grass_ctx* c, int l) { return l >= c->nsamp; }
inline bool home_on_device(const grass_ctx* c, int l) { return !c->cfg.offload || always_active(c, l); }

// Element `off` of a parameter / gradient buffer of the context's dtype.
inline void* elem(void* p, int64_t off, size_t esz) { return static_cast<char*>(p) + off * (int64_t)esz; }
inline const void* elem(const void* p, int64_t off, size_t esz) {
  return static_cast<const char*>(p) + off * (int64_t)esz;
}

// ---- tracing ---------------------------------------------------------------
// Brackets one device operation on stream `s`: `begin` before issuing it,
// `end` after.  A no-op unless tracing is enabled.
// Also an NVTX range (domain "grass", message = the operation, payload = the
// layer id) around the host-side issue of the operation, so an nsys timeline
// shows every fetch / update / write-back / collective the library enqueues
// (SURVEY 5); NVTX calls are no-ops unless a tool is attached.
inline nvtxDomainHandle_t nvtx_domain() {
  static nvtxDomainHandle_t d = nvtxDomainCreateA("grass");
  return d;
}
inline void nvtx_push(int kind, int layer) {
  static const char* const names[] = {"grass.h2d", "grass.update", "grass.d2h", "grass.norm",
                                      "grass.reduce_scatter", "grass.all_gather", "grass.p2p_sync"};
  nvtxEventAttributes_t a = {};
  a.version = NVTX_VERSION;
  a.size = NVTX_EVENT_ATTRIB_STRUCT_SIZE;
  a.messageType = NVTX_MESSAGE_TYPE_ASCII;
  a.message.ascii = (kind >= 0 && kind < 7) ? names[kind] : "grass.op";
  a.payloadType = NVTX_PAYLOAD_TYPE_INT64;
  a.payload.llValue = layer;
  nvtxDomainRangePushEx(nvtx_domain(), &a);
}
struct TraceScope {
  grass_ctx* c;
  cudaStream_t s;
  int idx = -1;
  TraceScope(grass_ctx* c_, cudaStream_t s_, int kind, int layer, int64_t off, int64_t n,
             const void* dev = nullptr, const void* host = nullptr)
      : c(c_), s(s_) {
    nvtx_push(kind, layer);
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
    c->trace.push_back({kind, e[0], e[1], {{layer, off, n, dev, host}}});
    idx = (int)c->trace.size() - 1;
  }
  // a further (layer, range) of the same operation (multi-segment launches)
  void add(int layer, int64_t off, int64_t n, const void* dev, const void* host = nullptr) {
    if (idx >= 0) c->trace[idx].acc.push_back({layer, off, n, dev, host});
  }
  ~TraceScope() {
    if (idx >= 0) cudaEventRecord(c->trace[idx].e1, s);
    nvtxDomainRangePop(nvtx_domain());
  }
};

// Non-finite flag encoding: 0 = none, else INT_MAX - (smallest layer id)
// (kernels use atomicMax, so a memset to 0 clears it).
inline int flag_layer(int enc) { return INT_MAX - enc; }

// context.cpp
grass_status set_thread_err(grass_status s, const std::string& msg);
cudaEvent_t take_event(grass_ctx* c);
grass_status mark_pending(grass_ctx* c, cudaStream_t s);
grass_status wait_pending(grass_ctx* c, cudaStream_t s);
grass_status fetch_mgn(grass_ctx* c, bool reset_window, bool take_flag);
const double* h_S(const grass_ctx* c);
const long long* h_c(const grass_ctx* c);
int h_flag(const grass_ctx* c);
grass_status report_flag(grass_ctx* c);
grass_status drain(grass_ctx* c, bool take_flag);
grass_status validate_config(const grass_config* cfg, std::string* why);
typedef int (*AddressRangeFn)(unsigned long long* base, size_t* size, unsigned long long ptr);
AddressRangeFn address_range_fn();
grass_status check_device_buffer(grass_ctx* c, const void* p, unsigned long long need, const std::string& what);
grass_status check_call(grass_ctx* c, bool bf16_call, const int32_t* ids, int32_t n, const void* const* p1, const void* const* p2, std::vector<int>* order, std::vector<char>* host_p2 = nullptr);
Batch make_batch(const grass_ctx* c, int32_t mode);
void push_seg(Batch* b, const Seg& s);
grass_status flush(grass_ctx* c, Batch* b, bool update, cudaStream_t s);
Seg range_seg(const grass_ctx* c, int l, const void* g, int64_t off, int64_t n);
void set_update(const grass_ctx* c, Seg* s, void* param, float* const* state, bool init_master);
void free_ctx(grass_ctx* c);
grass_status create_impl(const grass_config* cfg, grass_ctx* c);
grass_status api_exception(grass_ctx* c) noexcept;

// dataparallel.cpp
grass_status cross_rank_finish(grass_ctx* c, const int32_t* ids, const std::vector<int>& order, cudaStream_t s);
grass_status p2p_check(grass_ctx* c, const int32_t* ids, int32_t n, void* const* params, const void* const* grads);
P2PSyncArgs p2p_args(grass_ctx* c, int32_t which);
grass_status p2p_start(grass_ctx* c, cudaStream_t s);
grass_status p2p_finish_layers(grass_ctx* c, const std::vector<int32_t>& layers, cudaStream_t s);
grass_status p2p_end(grass_ctx* c, const int32_t* ids, const std::vector<int>& order, cudaStream_t s);
void* gs_slot(grass_ctx* c, int k);
void* rs_slot(grass_ctx* c, int j);
int gs_slot_index(const grass_ctx* c, const void* slot);
grass_status comm_exchange(grass_ctx* c, const void* grad, int l, void* slot, cudaStream_t s);
grass_status comm_begin(grass_ctx* c, cudaStream_t s);
grass_status comm_rs(grass_ctx* c, int j, const void* grad, int l);
grass_status comm_wait_rs(grass_ctx* c, int j, cudaStream_t s);
grass_status comm_after_update(grass_ctx* c, int j, void* params, int64_t off, int64_t len, cudaStream_t s);
grass_status comm_end(grass_ctx* c, cudaStream_t s);
grass_status cross_rank_check(grass_ctx* c);

// offload.cpp
grass_status update_range(grass_ctx* c, int l, const Seg& base, void* param, const void* g, int64_t off, int64_t n, float* const* state, bool init, int32_t mode, cudaStream_t s, const void* g_chunk = nullptr);
grass_status offload_layer(grass_ctx* c, int l, const Seg& base, void* param, const void* g, bool init, int32_t mode, cudaStream_t s, bool g_host);
grass_status stream_grad_layer(grass_ctx* c, int l, const Seg& base, void* param, const void* g_host, bool init, int32_t mode, cudaStream_t s);
float* cache_arr(grass_ctx* c, int slot, int a);
void cache_plan(grass_ctx* c, const int32_t* ids, const std::vector<int>& order, std::vector<int>* slot_of, std::vector<int>* victim_of);
grass_status swap_in_layer(grass_ctx* c, int l, int slot, int victim, const Seg& base, void* param, const void* g, bool init, int32_t mode, cudaStream_t s);
grass_status prefetch_into(grass_ctx* c, int l, int slot, int victim);
grass_status flush_cache(grass_ctx* c);
grass_status writeback_release(grass_ctx* c, int l, int slot, cudaStream_t s);
float* state_ptr(grass_ctx* c, int a, int layer, bool* on_device);
grass_status copy_state_out(grass_ctx* c, int a, int layer, float* out);
grass_status copy_state_in(grass_ctx* c, int a, int layer, const float* in);

// hot_path.cpp
grass_status mgn_accumulate_impl(grass_ctx* c, bool bf16_call, const int32_t* ids, int32_t n, const void* const* grads, void* stream);
grass_status step_layers_impl(grass_ctx* c, bool bf16_call, const int32_t* ids, int32_t n, void* const* params, const void* const* grads, float lr, void* stream);

// checkpoint.cpp
uint32_t crc_update(uint32_t crc, const void* p, size_t n);
std::vector<char> ck_header(grass_ctx* c, const std::vector<int32_t>& mvalid);

}  // namespace gapi
