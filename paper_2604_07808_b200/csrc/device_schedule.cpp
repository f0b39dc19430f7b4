// device_schedule.cpp — the device-resident adaptive schedule
// (grass_register_layers / grass_device_schedule_begin / grass_device_step /
// grass_device_schedule_end): the sampled ids, m, p and the MGN window stay on
// the device; a step is [prologue -> K2 -> K3 -> commit + resample], all
// stream-ordered launches with no host synchronisation (
// DESIGN.md §8).  Two launches per step: K2 (which computes the step
// prologue's AdamW scalars itself) and K3 (which advances t_l and, in its
// last CTA, runs the commit + resample).
#include <algorithm>
#include <cmath>
#include <cstring>
#include <string>
#include <vector>

#include "context.h"

namespace gapi {

// device block d_sched: ids [kMaxDevSeg] | committed | err | K3 done counter
enum : int { kSchedCommitted = kMaxDevSeg, kSchedErr, kSchedDone, kSchedWords };
static int32_t* sched_ids(grass_ctx* c) { return c->d_sched; }
static int32_t* sched_committed(grass_ctx* c) { return c->d_sched + kSchedCommitted; }
static int32_t* sched_err(grass_ctx* c) { return c->d_sched + kSchedErr; }
static unsigned int* sched_done(grass_ctx* c) { return reinterpret_cast<unsigned int*>(c->d_sched + kSchedDone); }

static grass_status check_schedulable(grass_ctx* c) {
  if (c->cfg.offload) return c->fail(GRASS_E_STATE, "device schedule: needs HBM-resident states (offload = 0)");
  if (c->dp || c->p2p) return c->fail(GRASS_E_STATE, "device schedule: world = 1 only");
  if (c->cfg.max_grad_norm > 0.0) return c->fail(GRASS_E_STATE, "device schedule: no clipping");
  if (c->cfg.gamma + c->cfg.n_always > kMaxDevSeg)
    return c->fail(GRASS_E_INVALID, "device schedule: gamma + n_always must be <= 32");
  return GRASS_OK;
}

static CommitArgs commit_args(grass_ctx* c, bool commit, bool sample, uint64_t period) {
  CommitArgs a;
  std::memset(&a, 0, sizeof(a));
  a.nsamp = c->nsamp;
  a.nl = c->nl;
  a.gamma = c->cfg.gamma;
  a.policy = c->cfg.policy;
  a.normalize = c->cfg.normalize_mgn != 0;
  a.T_p = c->cfg.T_p;
  a.do_commit = commit ? 1 : 0;
  a.do_sample = sample ? 1 : 0;
  a.alpha = c->cfg.alpha;
  a.tau = c->cfg.tau;
  a.seed = c->cfg.seed;
  a.period = period;
  a.m = c->d_mgn_m;
  a.probs = c->d_probs;
  a.committed = sched_committed(c);
  a.ids = sched_ids(c);
  a.err = sched_err(c);
  a.period_ctr = c->d_period;
  return a;
}

}  // namespace gapi

using namespace gapi;

extern "C" {

grass_status grass_register_layers(grass_ctx* c, int32_t n, void* const* params, const void* const* grads) try {
  if (!c) return set_thread_err(GRASS_E_INVALID, "ctx is NULL");
  if (n != c->nl || !params || !grads) return c->fail(GRASS_E_INVALID, "register every layer: n = n_layers, non-NULL arrays");
  grass_status s = check_schedulable(c);
  if (s != GRASS_OK) return s;
  CUDA_TRY(c, cudaSetDevice(c->cfg.device));
  std::vector<Seg> tab(c->nl);
  for (int l = 0; l < c->nl; ++l) {
    const unsigned long long need = (unsigned long long)c->numel[l] * c->esz;
    if ((s = check_device_buffer(c, params[l], need, "parameters of layer " + std::to_string(l))) != GRASS_OK) return s;
    if ((s = check_device_buffer(c, grads[l], need, "gradient of layer " + std::to_string(l))) != GRASS_OK) return s;
    Seg sg = range_seg(c, l, grads[l], 0, c->numel[l]);
    float* sp[3];
    for (int a = 0; a < c->ns; ++a) sp[a] = c->arr[a][l];
    set_update(c, &sg, params[l], sp, false);
    tab[l] = sg;
  }
  if ((s = drain(c, false)) != GRASS_OK) return s;  // no launch reads the table
  if (!c->d_segtab) CUDA_TRY(c, cudaMalloc((void**)&c->d_segtab, sizeof(Seg) * (size_t)c->nl));
  CUDA_TRY(c, cudaMemcpy(c->d_segtab, tab.data(), sizeof(Seg) * (size_t)c->nl, cudaMemcpyHostToDevice));
  c->registered.assign(c->nl, 1);
  return GRASS_OK;
} catch (...) {
  return api_exception(c);
}

grass_status grass_device_schedule_begin(grass_ctx* c, uint64_t period, void* stream) try {
  if (!c) return set_thread_err(GRASS_E_INVALID, "ctx is NULL");
  grass_status s = check_schedulable(c);
  if (s != GRASS_OK) return s;
  if ((int)c->registered.size() != c->nl) return c->fail(GRASS_E_STATE, "device schedule: call grass_register_layers first");
  if (c->dev_sched) return c->fail(GRASS_E_STATE, "device schedule already running (grass_device_schedule_end first)");
  CUDA_TRY(c, cudaSetDevice(c->cfg.device));
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  if ((s = drain(c, false)) != GRASS_OK) return s;
  if (!c->d_sched) {
    CUDA_TRY(c, cudaMalloc((void**)&c->d_sched, sizeof(int32_t) * kSchedWords));
    CUDA_TRY(c, cudaMalloc((void**)&c->d_mgn_m, sizeof(double) * (size_t)c->nl));
    CUDA_TRY(c, cudaMalloc((void**)&c->d_probs, sizeof(double) * (size_t)c->nl));
    CUDA_TRY(c, cudaMalloc((void**)&c->d_period, sizeof(unsigned long long)));
  }
  // the host MGN state -> device; the always-active groups follow the gamma sampled ids
  std::vector<int32_t> blk(kSchedWords, 0);
  for (int k = 0; k < c->nl - c->nsamp; ++k) blk[c->cfg.gamma + k] = c->nsamp + k;
  blk[kSchedCommitted] = c->committed ? 1 : 0;
  CUDA_TRY(c, cudaMemcpy(c->d_sched, blk.data(), sizeof(int32_t) * blk.size(), cudaMemcpyHostToDevice));
  CUDA_TRY(c, cudaMemcpy(c->d_mgn_m, c->mgn.data(), sizeof(double) * (size_t)c->nl, cudaMemcpyHostToDevice));
  CUDA_TRY(c, cudaMemcpy(c->d_probs, c->probs.data(), sizeof(double) * (size_t)c->nl, cudaMemcpyHostToDevice));
  CUDA_TRY(c, launch_commit_sample(commit_args(c, false, true, period), c->st, st));
  c->launches++;
  c->dev_sched = true;
  return mark_pending(c, st);
} catch (...) {
  return api_exception(c);
}

grass_status grass_device_step(grass_ctx* c, float lr, int32_t do_commit, int32_t do_resample, uint64_t next_period,
                               void* stream) try {
  if (!c) return set_thread_err(GRASS_E_INVALID, "ctx is NULL");
  if (!c->dev_sched) return c->fail(GRASS_E_STATE, "device schedule: call grass_device_schedule_begin first");
  if (!(lr >= 0.0f) || !std::isfinite(lr)) return c->fail(GRASS_E_INVALID, "lr must be finite, >= 0");
  CUDA_TRY(c, cudaSetDevice(c->cfg.device));
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  CUDA_TRY(c, cudaStreamIsCapturing(st, &cap));
  if (cap == cudaStreamCaptureStatusActive) {
    if (c->tracing) return c->fail(GRASS_E_INVALID, "CUDA-graph capture needs tracing off");
    c->captured = true;
  }
  const int n = c->cfg.gamma + (c->nl - c->nsamp);
  // K2 over the device-sampled layers, with the step prologue's AdamW scalars
  // of t_l + 1 computed in each CTA
  Batch b = make_batch(c, kFinalizeMgn);
  b.dev_table = c->d_segtab;
  b.dev_ids = sched_ids(c);
  b.dev_n = n;
  b.dev_lr = lr;
  b.dev_lr_ptr = c->lr_ptr;
  b.dev_beta1 = c->cfg.beta1;
  b.dev_beta2 = c->cfg.beta2;
  b.dev_wd = c->cfg.weight_decay;
  {
    TraceScope ts(c, st, GRASS_TRACE_UPDATE, -1, 0, 0);
    CUDA_TRY(c, launch_fused_dev(b, c->st, c->grid_update, st));
  }
  // K3 of those layers: the MGN window, t_l += 1 (bf16: master flag), and
  // in the CTA that completes last the commit + resample
  FinalizeArgs fa;
  std::memset(&fa, 0, sizeof(fa));
  fa.n = n;
  fa.mode = kFinalizeMgn;
  fa.dev_table = c->d_segtab;
  fa.dev_ids = sched_ids(c);
  fa.advance = 1;
  fa.bf16 = c->bf16 ? 1 : 0;
  fa.fuse_commit = (do_commit || do_resample) ? 1 : 0;
  fa.done_ctr = sched_done(c);
  fa.ca = commit_args(c, do_commit != 0, do_resample != 0, next_period);
  CUDA_TRY(c, launch_finalize(fa, c->st, st));
  c->launches += 2;
  return cap == cudaStreamCaptureStatusActive ? GRASS_OK : mark_pending(c, st);
} catch (...) {
  return api_exception(c);
}

grass_status grass_device_schedule_end(grass_ctx* c, int32_t* ids_out) try {
  if (!c) return set_thread_err(GRASS_E_INVALID, "ctx is NULL");
  if (!c->dev_sched) return c->fail(GRASS_E_STATE, "device schedule is not running");
  grass_status s = drain(c, false);
  if (s != GRASS_OK) return s;
  std::vector<int32_t> blk(kSchedWords);
  CUDA_TRY(c, cudaMemcpy(blk.data(), c->d_sched, sizeof(int32_t) * blk.size(), cudaMemcpyDeviceToHost));
  CUDA_TRY(c, cudaMemcpy(c->mgn.data(), c->d_mgn_m, sizeof(double) * (size_t)c->nl, cudaMemcpyDeviceToHost));
  CUDA_TRY(c, cudaMemcpy(c->probs.data(), c->d_probs, sizeof(double) * (size_t)c->nl, cudaMemcpyDeviceToHost));
  if (c->bf16) {  // host mirror of the master flags
    std::vector<int> mv(c->nl);
    CUDA_TRY(c, cudaMemcpy(mv.data(), c->st.mvalid, sizeof(int) * c->nl, cudaMemcpyDeviceToHost));
    for (int l = 0; l < c->nl; ++l) c->master_valid[l] = mv[l] ? 1 : 0;
  }
  c->committed = blk[kSchedCommitted] != 0;
  if (ids_out) std::memcpy(ids_out, blk.data(), sizeof(int32_t) * c->cfg.gamma);
  c->dev_sched = false;
  const int err = blk[kSchedErr];
  if (err == 2) {  // the non-finite flag is taken (reset) as grass_update_probs does
    if ((s = fetch_mgn(c, false, true)) != GRASS_OK) return s;
    return report_flag(c);
  }
  if (err == 1) return c->fail(GRASS_E_STATE, "device schedule: commit with zero observations in the window");
  return GRASS_OK;
} catch (...) {
  return api_exception(c);
}

}  // extern "C"
