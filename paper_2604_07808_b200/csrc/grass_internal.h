// grass_internal.h — shared declarations of the GRASS B200 library (not ABI).
#pragma once
#include <cstdint>

#include "grass.h"  // include/ (-I)

#ifdef __CUDACC__
#include <cuda_runtime.h>
#else
#include <cuda_runtime_api.h>
#endif

namespace grass {

// ----- fixed norm decomposition -------------------------------------------
// A layer (or layer shard) is cut into tiles of kTile elements.  Each tile's
// squared-norm partial is computed by the consumer warps of ONE CTA with a
// fixed thread->element map and a fixed fp64 reduction tree (kernels.cu), and the per-layer total
// is the fixed-order sum of its tile partials.  The result therefore depends
// only on the data, never on the grid size, SM count or launch split
// (offload chunks are whole tiles).
constexpr int kThreads = 512;                  // consumer threads per tile (16 warps)
constexpr int kVec = 4;                        // fp32 per 128-bit access
constexpr int kUnroll = 2;                     // 128-bit accesses per array per thread per tile
constexpr int64_t kTile = (int64_t)kThreads * kVec * kUnroll;  // 4096 elements
constexpr int kMaxSeg = 64;                    // segments per launch

// kFinalizeMgn: S_l += sqrt(ss/N_p), c_l += 1; kFinalizeShard: write this rank's
// shard ss for the cross-rank sum; kFinalizeNone: pass 2 of clipped updates
// (the MGN already saw the raw norm in pass 1).
enum FinalizeMode : int32_t { kFinalizeMgn = 0, kFinalizeShard = 1, kFinalizeNone = 2 };
constexpr int kMaxClipLayers = 1024;

// One contiguous range of one layer processed by a launch.
struct Seg {
  float* theta;            // params (UPDATE) — range start
  const float* g;          // gradient — range start
  float* m;                // first moment — range start (HBM or staging slot)
  float* v;                // second moment — range start
  int64_t n;               // valid elements in this range
  int64_t part_index;      // index into partials of this range's first tile
  int64_t part_layer_base; // index into partials of the layer's tile 0
  int64_t layer_numel;     // N_p(l), the TRUE count (R10)
  int32_t tiles;           // ceil(n / kTile)
  int32_t layer_tiles;     // tiles of the whole layer (shard) this step
  int32_t layer;           // layer id
  int32_t out_slot;        // kFinalizeShard: slot in shard_ss
  // (the AdamW scalars of the layer and its bf16 master-initialisation flag
  // are read from DevState::scal / init_now, written by the step prologue)
  // bf16 mode: `theta` is the fp32 master, these are the
  // bf16 model copy (updated as RNE(master')) and the bf16 gradient
  uint16_t* theta16;
  const uint16_t* g16;
  // Data parallelism with the gradient summed in the kernel (Batch::npeer >
  // 0): the gradient of element idx of this range is the ascending-rank fp32
  // sum of gpeer[r][gpoff + idx] over the npeer ranks, and (Batch::ntpeer > 0,
  // P2P) theta' is stored into tpeer[r][poff + idx] of every
  // rank.  P2P: gpeer / tpeer are every rank's full-layer buffers (peer-mapped
  // addresses) and gpoff = poff = the range's element offset in the full
  // layer.  NCCL: gpeer are the W slices of this rank's shard received by the
  // gradient all-to-all (gpoff = offset in the shard), ntpeer = 0 (theta' goes
  // to this rank's buffer, then ncclAllGather).  The local theta / m / v above
  // are this rank's shard as usual.
  const void* const* gpeer;  // device [npeer]: gradient of each rank
  void* const* tpeer;        // device [ntpeer]: full-layer parameters of each rank
  int64_t poff;
  int64_t gpoff;
};

struct Batch {
  Seg seg[kMaxSeg];
  int32_t tile_prefix[kMaxSeg + 1];
  int32_t nseg;
  int32_t mode;            // FinalizeMode
  float beta1, one_minus_beta1, beta2, one_minus_beta2, eps;
  const float* coef;       // device scalar multiplying g in the update (clipping), or NULL
  int32_t bf16;            // 1: bf16 gradients / parameters with fp32 master (Seg::g16, theta16)
  float gscale;            // multiplies every gradient element on load (DP: 1/world), else 1
  int32_t npeer;           // DP: ranks whose gradients are summed in the kernel (Seg::gpeer), else 0
  int32_t ntpeer;          // P2P: ranks whose parameter buffers receive theta' (Seg::tpeer), else 0
  // device-resident schedule (grass_device_step): the launch's segments are
  // dev_table[dev_ids[j]] for j < dev_n (ids read on the device, ascending),
  // instead of seg[] / nseg
  const Seg* dev_table;    // device [n_layers]: the whole-layer segment of every layer
  const int32_t* dev_ids;  // device [dev_n]
  int32_t dev_n;
  // ... and no step-prologue launch: every CTA computes the step's AdamW
  // scalars of its (<= kMaxDevSeg) layers from t_l + 1 into shared memory, by
  // the prologue kernel's arithmetic; K3 then advances t_l (FinalizeArgs::advance)
  float dev_lr;
  const float* dev_lr_ptr;  // device scalar (set_lr_device), else dev_lr
  double dev_beta1, dev_beta2, dev_wd;
};
constexpr int kMaxDevSeg = 32;  // layers one device-scheduled launch may update (gamma + n_always)

// Device-resident MGN / reduction state (all arrays indexed by layer id unless noted).
struct DevState {
  double* partials;        // tile partials, all layers back to back
  double* S;               // window sum of r_l   (Eq. 2)
  long long* c;            // window count
  double* last_ss;         // last squared norm
  int* flag;               // INT_MAX - (smallest layer id with a non-finite norm), 0 = none
  double* shard_ss;        // [slot] this rank's shard squared norm (world > 1)
  // per-layer optimizer step state, on the device so that a captured CUDA
  // graph of grass_step_layers advances it on every replay
  long long* t;            // t_l: updates applied to layer l (R2)
  float* scal;             // [3 l + k]: 1 - lr*wd, lr/(1-b1^t), 1/sqrt(1-b2^t) of this step
  int* init_now;           // bf16: 1 if this step initialises the layer's master from the bf16 param
  int* mvalid;             // bf16: the layer's fp32 master holds a value
};

// Step prologue: for each listed layer t_l += 1 and the AdamW scalars of the
// new t_l (fp64, rounded once to fp32), lr from `lr_ptr` if set (a device
// scalar the caller may change between graph replays) else `lr`.
struct PrologueArgs {
  int32_t n;
  int32_t layer[kMaxSeg];
  float lr;
  const float* lr_ptr;
  double beta1, beta2, wd;
  int32_t bf16;
};
cudaError_t launch_step_prologue(const PrologueArgs& a, const DevState& st, cudaStream_t s);

// kernels.cu
cudaError_t launch_fused(bool update, const Batch& b, const DevState& st, int grid,
                         cudaStream_t s);
// K2 of the device-resident schedule (Batch::dev_table / dev_ids).
cudaError_t launch_fused_dev(const Batch& b, const DevState& st, int grid, cudaStream_t s);
// Device-resident commit + resample (grass_device_step): the host's
// grass_update_probs + grass_sample_layers arithmetic, in fp64 on one thread.
struct CommitArgs {
  int32_t nsamp, nl, gamma, policy, normalize, T_p;
  int32_t do_commit, do_sample;
  double alpha, tau;
  uint64_t seed, period;
  double* m;               // device [nl] committed MGN
  double* probs;           // device [nl]
  int32_t* committed;      // device: a commit has happened
  int32_t* ids;            // device [gamma]: the sampled layers (draw order)
  int32_t* err;            // device: 1 = commit with zero observations, 2 = non-finite gradient (sticky)
  unsigned long long* period_ctr;  // device: the period of the current ids; period == ~0: resample for ++ctr
};
// K3 for the layers whose last tiles a stream launch wrote: one CTA each.
struct FinalizeArgs {
  int32_t n;               // layers
  int32_t mode;            // FinalizeMode (kFinalizeMgn / kFinalizeShard)
  int32_t layer[kMaxSeg];
  int32_t tiles[kMaxSeg];  // tile partials of the layer (shard)
  int32_t out_slot[kMaxSeg];
  int64_t base[kMaxSeg];   // index of the layer's tile 0 in DevState::partials
  int64_t numel[kMaxSeg];  // N_p(l)
  const Seg* dev_table;    // device-resident schedule: layer j = dev_ids[j], geometry from dev_table
  const int32_t* dev_ids;
  // device-resident schedule: advance = 1: t_l += 1 (and, bf16, the master
  // flag set) for each layer — the step prologue's state update, after K2
  // has read the old t_l; fuse_commit = 1: the CTA that completes last
  // (done_ctr) then runs the commit + resample of `ca` (one launch less)
  int32_t advance, bf16, fuse_commit;
  unsigned int* done_ctr;  // device counter, 0 between launches
  CommitArgs ca;
};
size_t commit_smem_bytes(int nl);
cudaError_t launch_commit_sample(const CommitArgs& a, const DevState& st, cudaStream_t s);
cudaError_t launch_finalize(const FinalizeArgs& a, const DevState& st, cudaStream_t s);
// world > 1: per-layer total = fixed ascending-rank sum of the all-gathered
// shard partials gathered[r * total_slots + slot], then the MGN update.
struct RankSumArgs {
  int32_t n;               // layers in this launch
  int32_t world;
  int32_t total_slots;     // row length of `gathered`
  int32_t slot0;           // first slot of this launch
  int32_t layer[kMaxSeg];
  int64_t numel[kMaxSeg];
};
cudaError_t launch_rank_sum(const double* gathered, const RankSumArgs& a, const DevState& st,
                            cudaStream_t s);
int fused_grid(bool update, bool bf16, int device);
// Global-norm clip coefficient of the listed layers from last_ss (fp64,
// ascending layer order): coef = min(1, max_norm / (sqrt(sum) + 1e-6)).
struct ClipArgs {
  int32_t n;
  double max_norm;
  int32_t layer[kMaxClipLayers];
};
cudaError_t launch_clip_coef(const ClipArgs& a, const DevState& st, float* coef, cudaStream_t s);

// ----- P2P data parallelism --------------------
// Every rank owns an "exchange block" in its HBM, mapped into every peer:
//   [0, 8*kMaxPeers)              start-barrier flags, one u64 per sending rank
//   [8*kMaxPeers, 16*kMaxPeers)   end-barrier flags
//   [kExchGather, ...)            gather rows: row r = rank r's shard squared
//                                 norms of the current call (fp64)
constexpr int kMaxPeers = 8;
constexpr int64_t kExchGather = 16 * kMaxPeers;
struct P2PSyncArgs {
  char* exch[kMaxPeers];   // every rank's exchange block (valid addresses in this process)
  int32_t rank, world;
  int32_t n;               // shard norms to publish into every rank's row `rank` (0 = none)
  int32_t which;           // barrier: 0 = start, 1 = end, -1 = none
  uint64_t epoch;          // value every rank signals for this barrier (if epoch_ctr is NULL)
  unsigned long long* epoch_ctr;  // device [2]: start / end generations, advanced by the kernel
                                  // itself (so a captured graph's replays advance them too)
  const double* shard_ss;  // [n] this rank's shard squared norms
  int* err;                // set to 1 if a peer never arrives (timeout)
};
cudaError_t launch_p2p_sync(const P2PSyncArgs& a, cudaStream_t s);
// grass_selftest_p2p: the protocol above with `world` ranks emulated as the
// co-resident CTAs of one cooperative launch (synchronous).
cudaError_t p2p_selftest(int world, int n, int rounds, unsigned long long* mismatches, int* timed_out);

// host_policy.cpp
uint64_t splitmix64(uint64_t x);
double uniform01(uint64_t seed, uint64_t period, uint32_t k);
bool softmax_probs(const double* m, int n, double tau, bool normalize, double* p);
bool sample_from_probs(const double* p, int n, int gamma, uint64_t seed, uint64_t period,
                       int32_t* ids);
bool shard_range(int64_t numel, int world, int rank, int64_t* off, int64_t* cnt);
int schedule_decision(int64_t step, int T_p, int T_s, int T_u);

}  // namespace grass
