/*
 * grass.h — C ABI of the GRASS layer-wise update hot path on B200 (sm_100a).
 *
 * Paper: arxiv 2604.07808 (PAPER.md = the paper's LaTeX source).  The four
 * hot-path calls follow the paper's statement of the problem:
 *
 *   grass_mgn_accumulate  Eq. 2 inner term r_{l,t} = sqrt(||g_t^(l)||^2 / N_p^(l))
 *                         for the listed layers (probing
 *                         PAPER.md:111-113).
 *   grass_update_probs    Eq. 2 window mean + Eq. 4 EMA + Eq. 3 softmax
 *                         (PAPER.md:91-93, 122-127, 115-120).
 *   grass_sample_layers   "samples gamma layers out of N_L".
 *   grass_step_layers     optimizer update of the trainable layers with the
 *                         layer-wise optimizer-state offload
 *                         (Fig. 4),
 *                         fused with the Eq. 2 norm of the same gradients.
 *
 * Readings where the paper is silent are DESIGN.md R1-R22 (referenced below).
 *
 * Conventions (all calls):
 *   - Every entry point returns a grass_status; no C++ exception ever crosses
 *     this boundary (each is a function-try-block).  On a validation error
 *     nothing has been enqueued, the context is unchanged, and
 *     grass_last_error() describes the failure.
 *   - A context is not thread-safe: calls on one context must not overlap.
 *     Distinct contexts are independent.
 *   - A "layer" is ONE flat, contiguous, 16-byte aligned fp32 (or bf16, see
 *     param_dtype) buffer of N_p(l) elements in device memory (the decoder
 *     block's tensors viewed back to back).
 *   - Every layer buffer is checked before anything is enqueued: 16-byte
 *     alignment, device memory of the context's GPU, and that its allocation
 *     (cuMemGetAddressRange; a caching allocator's segment) holds N_p elements.
 *   - Device pointers (params, grads) are CALLER-owned and must stay valid until
 *     the work enqueued on `stream` has completed.  Host arrays passed in
 *     (ids, pointer arrays, probs) are read before the call returns.
 *   - `stream` is a cudaStream_t passed as void* (NULL = legacy default stream).
 *     grass_mgn_accumulate / grass_step_layers are stream-ordered and return
 *     before the GPU work completes; grass_update_probs / grass_sync /
 *     grass_read_state synchronise.
 *   - Optimizer state (m, v, per-layer step t_l), the MGN state and the
 *     probabilities are CONTEXT-owned.
 *   - Non-finite gradients set a sticky device flag holding the smallest
 *     offending layer id; the next synchronising call returns
 *     GRASS_E_NONFINITE.  The fused update is single pass, so the
 *     update of that step has already been applied; the caller aborts the step.
 */
#ifndef GRASS_H_
#define GRASS_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GRASS_ABI_VERSION 1
#define GRASS_NCCL_ID_BYTES 128

typedef struct grass_ctx grass_ctx; /* opaque; one per process (= per rank / GPU) */

typedef enum {
  GRASS_OK = 0,
  GRASS_E_INVALID = 1,   /* bad argument; nothing enqueued */
  GRASS_E_STATE = 2,     /* call not valid in the current state */
  GRASS_E_CUDA = 3,      /* CUDA runtime error (message in grass_last_error) */
  GRASS_E_NCCL = 4,      /* NCCL error or NCCL unavailable when world > 1 */
  GRASS_E_OOM = 5,       /* device or pinned-host allocation failed */
  GRASS_E_NONFINITE = 6, /* a gradient contained inf/nan (sticky, see above) */
  GRASS_E_IO = 7         /* checkpoint file error: open/short read/write, corrupt length
                            or CRC32 mismatch (integrity error) */
} grass_status;

typedef enum {
  GRASS_POLICY_ADAPTIVE = 0, /* GRASS: EMA-refreshed MGN probabilities */
  GRASS_POLICY_STATIC = 1,   /* GRASS*: probabilities frozen after probing */
  GRASS_POLICY_UNIFORM = 2   /* LISA-style uniform sampling p = 1/N_L */
} grass_policy;

typedef enum {
  GRASS_DECIDE_PROBE = 0,    /* step < T_p: norms only, no update */
  GRASS_DECIDE_COMMIT_RESAMPLE = 1, /* commit window (+EMA), new probs, resample */
  GRASS_DECIDE_RESAMPLE = 2, /* new sampling period with unchanged probs */
  GRASS_DECIDE_CONTINUE = 3  /* keep the current trainable set */
} grass_decision;

typedef struct grass_config {
  int32_t n_layers;            /* N_L sampled layers + n_always groups (below), >= 1 */
  const int64_t* layer_numel;  /* host [n_layers]; N_p(l) >= 1, true counts (R10); copied */
  int32_t gamma;               /* active layers per period, 1 <= gamma <= N_L */
  int32_t T_p, T_s, T_u;       /* schedule; T_u multiple of T_s (R11) */
  double tau;                  /* Eq. 3 temperature > 0 (R3, default 1.0) */
  double alpha;                /* Eq. 4 EMA factor in [0,1] (R13, default 0.5) */
  int32_t normalize_mgn;       /* 1: max-normalise m before Eq. 3 (R3) */
  int32_t policy;              /* grass_policy */
  double beta1, beta2, eps, weight_decay; /* AdamW (R1): 0.9, 0.999, 1e-8, 0.0 */
  uint64_t seed;               /* sampler seed (R7) */
  int32_t device;              /* CUDA device ordinal this context lives on */
  int32_t offload;             /* 0: m/v resident in HBM; 1: m/v in pinned host memory,
                                  streamed per step */
  int32_t overlap;             /* offload pipeline: 1 overlapped (Fig. 4 right),
                                  0 vanilla serial HtoD->update->DtoH (Fig. 4 left) */
  int64_t chunk_elems;         /* offload chunk (elements); multiple of grass_tile_elems();
                                  0 = default (8 Mi elements) */
  int32_t ring_slots;          /* device staging slots for the offload ring (>= 1; 0 = 3) */
  int32_t rank, world;         /* data-parallel rank / world size (world = 1: no NCCL) */
  const void* nccl_unique_id;  /* host, GRASS_NCCL_ID_BYTES; required when world > 1.  With
                                  world = 1 a non-NULL id runs the same NCCL path on a 1-rank
                                  communicator (used to test it on one GPU) */
  int32_t residency;           /* offload only: GRASS_RESIDENCY_STEP (paper: every step
                                  round-trips the active layers' m/v) or
                                  GRASS_RESIDENCY_PERIOD (a layer's m/v stay
                                  in HBM while it stays trainable; swapped only when the
                                  sampled set changes) */
  int32_t cache_layers;        /* GRASS_RESIDENCY_PERIOD / _STEP_PREFETCH: device layer slots
                                  (>= gamma; 0 = gamma) */
  double max_grad_norm;        /* > 0: clip each grass_step_layers call's gradients by their
                                  global norm, coef = min(1, max/(||g||+1e-6)) (torch
                                  clip_grad_norm_; paper silent; DESIGN R17).
                                  Two passes (norm, then update: 32 B/param); the MGN
                                  still sees the raw norm (R9).  0 = off (default).  On the
                                  NCCL path one call may then list at most gamma + n_always
                                  layers (their averaged shards live between the passes). */
  int32_t param_dtype;         /* GRASS_DTYPE_FP32: fp32 params/grads (grass_step_layers);
                                  GRASS_DTYPE_BF16: bf16 params/grads, the context keeps an
                                  fp32 master copy next to m, v (grass_step_layers_bf16;
                                  SURVEY 8(f) f3, DESIGN R18). world > 1 then needs every
                                  N_p divisible by 8*world. */
  int32_t n_always;            /* always-active groups (DESIGN R19): the LAST
                                  n_always entries of layer_numel (embedding, final norm,
                                  output head — the LISA convention) are never
                                  sampled and are updated by every grass_step_layers call that
                                  lists them; their m/v stay in HBM in every mode.
                                  The sampled layers are ids [0, N_L) with N_L = n_layers -
                                  n_always; gamma, cache_layers, probabilities and the commit
                                  refer to those only.  0 = none (default). */
  int32_t dp_mode;             /* world >= 1 data parallelism:
                                  GRASS_DP_NCCL: NCCL exchange of the gradient slices
                                  (grouped ncclSend / ncclRecv) -> the update kernel sums the
                                  W slices in ascending rank order in fp32 (R20) -> ncclAllGather
                                  (needs nccl_unique_id when world > 1);
                                  GRASS_DP_P2P: ONE fused kernel per call reads every rank's
                                  gradient over peer memory (NVLink), sums them in rank order,
                                  updates this rank's shard and stores theta' into every rank's
                                  parameters; the shard norms are published the same way.
                                  Needs grass_p2p_attach + grass_p2p_register_layer; world <= 8;
                                  no clipping. */
  int32_t p2p_sync;            /* GRASS_DP_P2P: 1 (default) = each call starts and ends with a
                                  device-side barrier over the peers (system-scope flags in the
                                  exchange blocks) and finishes the MGN update itself;
                                  0 = no barriers: the caller orders the ranks' calls and calls
                                  grass_p2p_finish on every rank afterwards (single-process,
                                  multi-context testing on one GPU). */
  int32_t debug_check;         /* 1: grass_update_probs also verifies that every rank holds
                                  bit-identical MGN and probabilities (a 64-bit hash of both
                                  is all-gathered over NCCL / the P2P exchange blocks;
                                  SURVEY 8(e) debug mode) and returns GRASS_E_STATE if not.
                                  Makes grass_update_probs a collective.  0 = off (default). */
} grass_config;

typedef enum {
  GRASS_DP_NCCL = 0,
  GRASS_DP_P2P = 1
} grass_dp_mode;

typedef enum {
  GRASS_DTYPE_FP32 = 0,
  GRASS_DTYPE_BF16 = 1
} grass_dtype;

typedef enum {
  GRASS_RESIDENCY_STEP = 0,
  GRASS_RESIDENCY_PERIOD = 1,
  /* the paper's per-step round trip with whole-layer prefetch:
     grass_prefetch_layers fetches the step's trainable layers ahead (e.g.
     during the forward), grass_step_layers updates them and writes their m/v
     back to host right after the update (in the background: the caller's
     stream does not wait for the write-back); device slots as for PERIOD */
  GRASS_RESIDENCY_STEP_PREFETCH = 2
} grass_residency;

/* Fills *cfg with the defaults above (layer_numel = NULL, n_layers = 0). */
grass_status grass_config_init(grass_config* cfg);

/* Validates cfg, allocates: per layer m/v (HBM, or pinned host when offload;
 * when world > 1 only this rank's shard), zeroed, t_l = 0; MGN accumulators;
 * staging ring and copy streams (offload); NCCL communicator (world > 1 with
 * GRASS_DP_NCCL) or the P2P exchange block (GRASS_DP_P2P); world > 1 requires
 * every N_p divisible by 4*world (8*world for bf16).  *out receives the context.
 * Errors: GRASS_E_INVALID (bad config: gamma > N_L, tau <= 0
 * (SPEC.md:270), alpha outside [0,1], ...), GRASS_E_OOM,
 * GRASS_E_CUDA, GRASS_E_NCCL.  On error *out = NULL. */
grass_status grass_create(const grass_config* cfg, grass_ctx** out);

/* Synchronises all context streams, frees everything.  NULL is a no-op. */
void grass_destroy(grass_ctx* ctx);

/* Message of the last failed call on ctx (ctx == NULL: last failed
 * grass_create / context-free helper on this thread).  Never NULL. */
const char* grass_last_error(const grass_ctx* ctx);

/* Waits for all work the context enqueued; surfaces the sticky non-finite
 * flag (GRASS_E_NONFINITE) and asynchronous CUDA errors. */
grass_status grass_sync(grass_ctx* ctx);

/* Eq. 2 inner term (probing): for each listed layer,
 * ss_l = sum_i g_i^2 accumulated in fp64 over a FIXED tile decomposition
 * (bit-reproducible, independent of grid size), r_l = sqrt(ss_l / N_p(l)),
 * window S_l += r_l, c_l += 1.  No optimizer state is read or written (R14).
 *   layer_ids: host [n] distinct ids in [0, n_layers) (sampled layers and
 *              always-active groups alike).
 *   grads:     host [n] array of DEVICE pointers, grads[i] = N_p(layer_ids[i])
 *              fp32, 16-byte aligned.  World > 1: this rank's local gradient;
 *              the norm is of the DP average (R9).
 *   stream:    cudaStream_t.  Asynchronous; nothing syncs the host. */
grass_status grass_mgn_accumulate(grass_ctx* ctx, const int32_t* layer_ids, int32_t n,
                                  const float* const* grads, void* stream);

/* Eq. 2 window mean w_l = S_l / c_l (R4), then: first call m_l = w_l (R8);
 * later calls m_l = alpha*w_l + (1-alpha)*m_l for observed layers, unobserved
 * (frozen) layers keep m_l (Eq. 4); window reset; then Eq. 3
 * p = softmax(m~/tau) (R3) according to cfg.policy.  Synchronises once (waits
 * for the accumulations in flight and reads N_L * 16 bytes).
 *   probs_out: host [n_layers] or NULL (p = 0 for always-active groups).
 * Errors: GRASS_E_STATE if no layer was observed in the window,
 * GRASS_E_NONFINITE. */
grass_status grass_update_probs(grass_ctx* ctx, double* probs_out);

/* gamma distinct layer ids drawn without replacement, sequentially
 * proportional to p with renormalisation (R6), with the counter-based
 * SplitMix64 RNG keyed by (cfg.seed, period, draw index) (R7).  Pure host;
 * bit-exact contract.  ids_out in DRAW order.
 *   probs: host [n_layers] (only the first N_L entries are read) or NULL (= the
 *          context's current probabilities).  Ids are in [0, N_L).
 *   ids_out: host [gamma]. */
grass_status grass_sample_layers(grass_ctx* ctx, const double* probs, uint64_t period,
                                 int32_t* ids_out);

/* One AdamW step (R1, R2) on every listed layer, in ascending layer order
 * (R12), in place, fused single-pass with the Eq. 2 norm of the same gradient
 * (which feeds the MGN window exactly as grass_mgn_accumulate does):
 *   t_l += 1; theta = theta*(1 - lr*wd); m = b1*m + (1-b1)*g;
 *   v = b2*v + (1-b2)*g^2; theta -= lr/(1-b1^t) * m / (sqrt(v)/sqrt(1-b2^t) + eps)
 * With cfg.offload the layer's m/v stream from pinned host memory through the
 * device staging ring and back; results are bit-identical
 * to offload = 0 (R12).  World > 1: each rank updates its element shard with
 * its own m/v slice; with GRASS_DP_NCCL every rank's slice of this rank's
 * shard arrives over NCCL (grouped send/recv), the update kernel sums the W
 * slices in ascending rank order in fp32 and x 1/W (R20: the same bits as
 * GRASS_DP_P2P), and the parameters are all-gathered back into params[i];
 * with GRASS_DP_P2P one fused kernel reads every rank's gradient over peer
 * memory and stores theta' into every rank's params (the registered buffers).
 * t_l and the bias corrections are advanced on the device by a prologue
 * kernel on `stream` (capturable, see grass_set_lr_device).
 *   params: host [n] array of DEVICE pointers (fp32, N_p each, updated in place)
 *   grads:  host [n] array of DEVICE pointers (fp32, N_p each, read only), or
 *           of PINNED HOST pointers (world = 1, resident or per-step offload,
 *           no clipping): the gradient is then fetched chunk by chunk through a
 *           device ring on the context's copy stream, overlapping the update
 *           (the e2e "gradients live on the host" case); pageable host memory
 *           is rejected
 *   lr:     learning rate eta for this step (> 0 or == 0)
 * Stream-ordered on `stream`: when `stream` reaches this point the update, the
 * write-back of m/v to host and the MGN accumulation have all completed —
 * except under GRASS_RESIDENCY_STEP_PREFETCH, whose write-backs complete in
 * the background on the context's copy stream (ordered before the layer's next
 * fetch and drained by grass_sync and every call that reads host state). */
grass_status grass_step_layers(grass_ctx* ctx, const int32_t* layer_ids, int32_t n,
                               float* const* params, const float* const* grads, float lr,
                               void* stream);

/* Learning rate from device memory: with lr_device != NULL every later
 * grass_step_layers reads eta from *lr_device when its update runs (the `lr`
 * argument is then ignored), so a learning-rate schedule can change eta
 * between replays of a captured CUDA graph.  NULL restores the argument.
 *
 * CUDA graphs: grass_step_layers / grass_mgn_accumulate may be captured
 * (stream capture, e.g. torch.cuda.graph) with device gradients and tracing
 * off, for HBM-resident states, the per-step offload pipeline
 * (GRASS_RESIDENCY_STEP) or period residency with every listed layer already
 * cached (call grass_sync before capturing an offloaded step; not
 * GRASS_RESIDENCY_STEP_PREFETCH) — single GPU, NCCL, or P2P with p2p_sync = 1:
 * the per-layer step counts t_l, this step's
 * bias corrections, the bf16 master-initialisation flags, the MGN window and
 * the P2P barrier generations all live on the device, so every replay
 * performs one full step.  Synchronising calls after replays wait for the
 * whole device. */
grass_status grass_set_lr_device(grass_ctx* ctx, const float* lr_device);

/* Mixed-precision variants for a context created with GRASS_DTYPE_BF16
 * (SURVEY 8(f) f3, R18).  Same semantics as the fp32 calls; params/grads are
 * arrays of DEVICE pointers to bf16 (uint16_t bit patterns), 16-byte aligned.
 * The norm is of the bf16 gradient (widened exactly).  The update runs on the
 * context's fp32 master copy (initialised from the bf16 parameter on the
 * layer's first update), and params[i] receives RNE(master') as bf16.
 * Calling the fp32 entry points on a bf16 context (or vice versa) is
 * GRASS_E_INVALID. */
grass_status grass_mgn_accumulate_bf16(grass_ctx* ctx, const int32_t* layer_ids, int32_t n,
                                       const uint16_t* const* grads, void* stream);
grass_status grass_step_layers_bf16(grass_ctx* ctx, const int32_t* layer_ids, int32_t n,
                                    uint16_t* const* params, const uint16_t* const* grads, float lr,
                                    void* stream);

/* bf16 contexts: this rank's fp32 master shard of `layer` (host buffer,
 * shard length) — read / overwrite (a written master counts as initialised).
 * GRASS_E_STATE on an fp32 context or a layer whose master is not yet set. */
grass_status grass_read_master(grass_ctx* ctx, int32_t layer, float* out);
grass_status grass_write_master(grass_ctx* ctx, int32_t layer, const float* in);

/* Copies this rank's m/v shard of `layer` into host buffers m_out/v_out
 * (count = the shard length, grass_shard_range) and its step count; any
 * pointer may be NULL.  Synchronises the context first. */
grass_status grass_read_state(grass_ctx* ctx, int32_t layer, float* m_out, float* v_out,
                              int64_t* t_out);

/* GRASS_RESIDENCY_PERIOD / _STEP_PREFETCH: starts bringing the optimizer states of the listed
 * layers into the HBM cache now (evicting least-recently-used layers that are
 * not listed), on the context's copy streams, without updating anything.
 * Call it right after grass_sample_layers at a period boundary: the transfers
 * then overlap the caller's forward/backward pass, and the next
 * grass_step_layers of these layers finds them resident ("GRASS
 * asynchronously prefetches optimizer states").  `stream` orders the evictions
 * after the caller's earlier work.  GRASS_E_STATE without period residency. */
grass_status grass_prefetch_layers(grass_ctx* ctx, const int32_t* layer_ids, int32_t n, void* stream);

/* ----- device-resident schedule (DESIGN.md §8 "Device-resident schedule") -
 * The adaptive step — update of the sampled layers (+ always-active groups),
 * then commit (Eq. 2 window mean, Eq. 4 EMA, Eq. 3 softmax) and resample
 * — with the sampled ids, m, p and the window kept in device
 * memory, so consecutive steps need no host round trip and a whole step is
 * one capturable sequence of launches (CUDA graphs).  The arithmetic is the
 * host path's (grass_update_probs / grass_sample_layers) in the same order;
 * only exp() may differ from the host's by an ulp.  HBM-resident states,
 * world = 1, no clipping.
 *
 * grass_register_layers: the parameter / gradient buffers of ALL n = n_layers
 * layers (device pointers, N_p elements each, fp32 or bf16 by param_dtype;
 * caller-owned, must stay valid while the schedule runs).  Validated once.
 *
 * grass_device_schedule_begin: copies the host MGN state (m, p, committed) to
 * the device and samples the ids of `period` there (stream-ordered).
 *
 * grass_device_step: stream-ordered, no synchronisation: t_l += 1 and the
 * fused norm + AdamW of the layers sampled on the device (+ the always-active
 * groups), then, if do_commit, the commit, and, if do_resample, the ids of
 * `next_period` — GRASS_PERIOD_NEXT: the period after the current one, kept
 * on the device, so a captured step replays with advancing periods.  lr as
 * grass_step_layers (grass_set_lr_device applies).  Two kernel launches: the
 * update (which computes the step's AdamW scalars itself) and the per-layer
 * finalize (window, t_l, and the commit + resample in its last CTA).
 *
 * grass_device_schedule_end: synchronises; copies m, p, committed and the
 * current ids (ids_out: host [gamma], may be NULL) back to the host context;
 * GRASS_E_NONFINITE / GRASS_E_STATE if a commit met a non-finite norm or an
 * empty window (the schedule stopped committing there). */
#define GRASS_PERIOD_NEXT 0xFFFFFFFFFFFFFFFFull
grass_status grass_register_layers(grass_ctx* ctx, int32_t n, void* const* params, const void* const* grads);
grass_status grass_device_schedule_begin(grass_ctx* ctx, uint64_t period, void* stream);
grass_status grass_device_step(grass_ctx* ctx, float lr, int32_t do_commit, int32_t do_resample,
                               uint64_t next_period, void* stream);
grass_status grass_device_schedule_end(grass_ctx* ctx, int32_t* ids_out);

/* GRASS_RESIDENCY_PERIOD: writes the m/v of every layer cached in HBM back to
 * its pinned host home (the cache stays valid).  No-op otherwise.
 * Synchronises. */
grass_status grass_flush_states(grass_ctx* ctx);

/* Overwrites this rank's m/v shard and step count of `layer` (checkpoint
 * restore).  Synchronises the context first. */
grass_status grass_write_state(grass_ctx* ctx, int32_t layer, const float* m_in,
                               const float* v_in, int64_t t_in);

/* Checkpoint of this rank's whole optimizer + sampler state (
 * SPEC.md:192-199 shard serialisation): header {magic "GRASSCK1", version,
 * N_L, world, rank, committed, N_p[], shard_len[], t_l[], m_l[] (committed
 * MGN), p[], S[], c[]} with a CRC32, then per layer one blob (m shard then v
 * shard, fp32) preceded by its 64-bit byte length and its CRC32 (zlib
 * polynomial).  Synchronises; period-resident layers are flushed first.
 * Errors: GRASS_E_IO (cannot write). */
grass_status grass_save_state(grass_ctx* ctx, const char* path);

/* Restores a checkpoint written by grass_save_state into a context created
 * with the same N_L, N_p[], world and rank (else GRASS_E_INVALID).  A short
 * file, a wrong length or a CRC mismatch is an integrity error (GRASS_E_IO)
 * and leaves the context unchanged. */
grass_status grass_load_state(grass_ctx* ctx, const char* path);

/* ----- tracing (the Fig. 4 timeline) ---------
 * When enabled, every device operation the context issues is bracketed by
 * timing events on the stream it runs on; grass_trace_read returns them as
 * [start, end) in ms relative to the enable / previous read, in issue order,
 * and clears the trace — one event per (layer, range) an operation touches (a
 * multi-layer update launch yields one event per layer, same times).  Tracing
 * adds two event records per operation. */
typedef enum {
  GRASS_TRACE_H2D = 0,    /* optimizer states host -> device (offload fetch)   */
  GRASS_TRACE_UPDATE = 1, /* fused norm + AdamW launch (K2)                     */
  GRASS_TRACE_D2H = 2,    /* optimizer states device -> host (write-back/evict) */
  GRASS_TRACE_NORM = 3,   /* norm-only launch (K1)                              */
  GRASS_TRACE_RS = 4,     /* NCCL gradient-slice exchange (reduce-scatter bytes) */
  GRASS_TRACE_AG = 5,     /* NCCL all-gather of parameters                      */
  GRASS_TRACE_P2P = 6     /* P2P norm publication + barrier                     */
} grass_trace_kind;

typedef struct grass_trace_event {
  int32_t kind;     /* grass_trace_kind */
  int32_t layer;    /* layer id (norm-only launches: the first layer of the launch) */
  int64_t offset;   /* first element of the range within the layer shard */
  int64_t count;    /* elements */
  float start_ms, end_ms;
  /* the optimizer-state range the operation touches, as addresses of its m
   * array (v / master follow the same layout): state_dev = device copy (ring
   * slot, cache slot or resident state; 0 if none), state_host = pinned host
   * copy (0 if none).  Lets a checker find every pair of operations on the
   * same state and verify their order on the GPU timeline (race check of the
   * offload pipeline, tests/test_gpu_parity.py). */
  uint64_t state_dev, state_host;
} grass_trace_event;

grass_status grass_trace_enable(grass_ctx* ctx, int32_t on);
/* Synchronises; copies up to `capacity` events into `out` (host), *count =
 * events available (may exceed capacity; the rest are dropped). */
grass_status grass_trace_read(grass_ctx* ctx, grass_trace_event* out, int32_t capacity, int32_t* count);

/* Introspection of the MGN state (host arrays [n_layers], any may be NULL;
 * always-active groups have m = p = 0 but real S, c, last norm):
 * committed m_l, window sum S_l, window count c_l, last fp64 squared norm of
 * layer l (DP-averaged gradient when world > 1), current probabilities.
 * Synchronises the context first. */
grass_status grass_get_mgn(grass_ctx* ctx, double* m_out, double* window_sum_out,
                           int64_t* window_count_out, double* last_sqnorm_out,
                           double* probs_out);

/* Bytes of HBM this context owns (m/v, staging ring, MGN state, scratch). */
int64_t grass_device_bytes(const grass_ctx* ctx);
/* Bytes of pinned host memory this context owns. */
int64_t grass_host_bytes(const grass_ctx* ctx);
/* Number of kernel launches and NCCL calls this context has issued so far. */
int64_t grass_launch_count(const grass_ctx* ctx);

/* ----- context-free host helpers (no GPU needed; used by tests) ----------- */

/* Elements per norm tile: the fixed decomposition unit of the fp64 norm. */
int64_t grass_tile_elems(void);
const char* grass_version(void);

/* Standard SplitMix64 output of state x (R7). */
uint64_t grass_splitmix64(uint64_t x);
/* u in [0,1): (splitmix64(splitmix64(seed) ^ (period*2^16 + k)) >> 11) * 2^-53. */
double grass_uniform(uint64_t seed, uint64_t period, uint32_t k);

/* Eq. 3 with reading R3 on host fp64: p[i] for m[0..n). */
grass_status grass_softmax_probs(const double* m, int32_t n, double tau, int32_t normalize,
                                 double* p_out);

/* The sampler of grass_sample_layers without a context. */
grass_status grass_sample_from_probs(const double* p, int32_t n, int32_t gamma, uint64_t seed,
                                     uint64_t period, int32_t* ids_out);

/* Element shard of a layer of `numel` elements for `rank` of `world`: the
 * contiguous range [offset, offset + count).  Requires numel % (4*world) == 0
 * when world > 1 (every rank's shard is equal and 16-byte aligned). */
grass_status grass_shard_range(int64_t numel, int32_t world, int32_t rank, int64_t* offset,
                               int64_t* count);

/* Schedule decision for training step `step` (0-based). */
int32_t grass_schedule_decision(int64_t step, int32_t T_p, int32_t T_s, int32_t T_u);

/* Creates an NCCL unique id (128 bytes) on the calling host; rank 0 calls it
 * and broadcasts the bytes to the other ranks (e.g. via a torch process group). */
grass_status grass_nccl_get_unique_id(void* out);

/* ----- P2P data parallelism (cfg.dp_mode = GRASS_DP_P2P) ------------------
 * Every rank's context owns an exchange block in HBM (barrier flags + gather
 * rows of the shard norms).  Setup, collectively on every rank:
 *   1. grass_p2p_exchange_block -> export it to the peers (grass_ipc_export,
 *      any host transport, grass_ipc_import on the peers);
 *   2. grass_p2p_attach with the [world] block addresses as seen by this process;
 *   3. per layer, grass_p2p_register_layer with the [world] full-layer parameter
 *      and gradient buffers (this rank's own at index rank) — the buffers that
 *      every later grass_step_layers / grass_mgn_accumulate must pass.
 * Ordering contract (p2p_sync = 1): every rank issues the same sequence of
 * hot-path calls; a call returns to the stream only after every rank's update
 * (and its theta' stores into this rank's buffers) is complete, so the caller
 * may overwrite its gradients and read its parameters afterwards. */
/* Self-test of the P2P publication + barrier protocol on the current device:
 * `world` (1..8) ranks are emulated as the co-resident CTAs of ONE cooperative
 * launch (one GPU cannot host separately launched ranks that wait on one
 * another); `rounds` rounds of publish + end barrier + row check + start
 * barrier.  *mismatches = rows that did not hold the expected values after a
 * barrier, *timed_out = 1 if a barrier wait timed out.  Synchronous. */
grass_status grass_selftest_p2p(int32_t device, int32_t world, int32_t rounds, int64_t* mismatches,
                                int32_t* timed_out);

#define GRASS_IPC_HANDLE_BYTES 64
grass_status grass_p2p_exchange_block(grass_ctx* ctx, void** ptr, int64_t* bytes);
/* blocks: host [world] addresses of every rank's exchange block, valid in this
 * process (blocks[rank] must be this context's own). */
grass_status grass_p2p_attach(grass_ctx* ctx, void* const* blocks);
/* params / grads: host [world] arrays of full-layer buffers (N_p elements of the
 * context's dtype, 16-byte aligned), index = rank; this rank's entries must be
 * device memory of the context's GPU.  Synchronous (copies the table to HBM). */
grass_status grass_p2p_register_layer(grass_ctx* ctx, int32_t layer, void* const* params,
                                      const void* const* grads);
/* p2p_sync = 0 only: finishes the MGN update of the last hot-path call (the
 * fixed rank-order sum of the published shard norms); call it on every rank
 * after every rank's hot-path call has completed. */
grass_status grass_p2p_finish(grass_ctx* ctx, void* stream);
/* Exports the allocation containing ptr as a CUDA IPC handle (64 bytes) plus
 * the byte offset of ptr inside it. */
grass_status grass_ipc_export(const void* ptr, void* handle_out, int64_t* offset_out);
/* Opens an IPC handle exported by another process (cached: each allocation is
 * opened once per process) and returns base + offset. */
grass_status grass_ipc_import(int32_t device, const void* handle, int64_t offset, void** ptr_out);
/* Several ranks in ONE process (one thread per GPU, GRASS_DP_P2P): lets
 * `device` access `peer`'s memory directly (cudaDeviceEnablePeerAccess; an
 * already enabled pair is not an error), so that the peers' exchange blocks
 * and layer buffers can be passed to grass_p2p_attach / _register_layer as
 * plain device pointers.  GRASS_E_CUDA if the pair cannot access each other. */
grass_status grass_enable_peer_access(int32_t device, int32_t peer);

#ifdef __cplusplus
}
#endif
#endif /* GRASS_H_ */
