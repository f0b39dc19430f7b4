// kernels.cu — sm_100a kernels of the GRASS hot path.
//
//   K1  grass_stream_kernel<false>: Eq. 2 squared norm only (probing,
//       PAPER.md:111-113) — reads g once (4 B/param).
//   K2  grass_stream_kernel<true>:  single-pass Eq. 2 norm + AdamW (DESIGN.md
//       R1/R2) of the trainable layers — reads g, theta, m, v,
//       writes theta, m, v (28 B/param).
//   K3  grass_finalize_kernel (after each K1/K2 launch, one CTA per layer the
//       launch completed): fixed-order fp64 sum of the layer's tile partials,
//       then S_l += sqrt(ss_l / N_p), c_l += 1 (Eq. 2), or the
//       shard value for the rank sum.
//   K4  grass_rank_sum_kernel (world > 1): ascending-rank fp64 sum of the
//       all-gathered shard partials, then the same MGN update.
//   Device-resident schedule (grass_device_step): K2 with
//       DEVB = true (segments and step-prologue scalars from the device ids)
//       and K3 with t_l advanced and, in its last CTA, commit_sample_body —
//       Eq. 2 window mean, Eq. 4 EMA, Eq. 3 softmax and the gamma draws
//        in the host's operation order; both launched as
//       programmatic dependent launches (launch_pdl).
//
// Nothing here is a contraction: K1/K2 are HBM-bound streams (~0.5 flop/B),
// so there are no tensor cores.  The Blackwell-native part is the data
// movement: a persistent, warp-specialised kernel (one CTA per SM) in which a
// producer warp streams tiles HBM -> shared memory with cp.async.bulk (TMA
// bulk copies, SASS UBLKCP) into a STAGES-deep ring guarded by mbarriers,
// while 16 consumer warps compute.  K2's consumers write theta', m', v' back
// into the stage and the producer bulk-stores them (smem -> HBM, TMA) before
// refilling it.  The HBM pipe never drains on a block barrier.
//
// Compile-time A/B knobs (tools/variants.py; defaults are the measured best):
// GRASS_IEEE_MATH, GRASS_K2_STG_STORE, GRASS_K2_LOAD_EF, GRASS_K2_STORE_EF,
// GRASS_K2_SEP_OUT, GRASS_K2_NOMATH, GRASS_UPD_STAGES, GRASS_NORM_TPS,
// GRASS_NORM_TPS_BF16, GRASS_NORM_STAGES, GRASS_NORM_STAGES_BF16,
// GRASS_P2P_NORM_TPS, GRASS_UPD_GRID_SUB, GRASS_NORM_GRID_SUB,
// GRASS_L2_PREFETCH_{NORM,UPD}, GRASS_UNIT_BLOCK, GRASS_BF16_GUARD (0: no exact
// fallback — wrong for tiny / huge gradients), GRASS_K1_DRAIN (diagnostic),
// GRASS_K3_DIAG (diagnostic: 1 = the fused commit's last CTA skips the body,
// 2 = no done counter / fence either, 3 = the body without the sampler).
// The mutation check of the GPU tests (tools/kernel_mutation.py) plants its
// mistakes into a patched copy of this
// source; the product source carries none.
//
// The tile partial (grass_internal.h) is a FIXED function of the tile's data:
// consumer thread t owns elements (q*kThreads + t)*4 + j, j = 0..3, q = 0..
// kUnroll-1; it keeps 4 fp64 accumulators acc_j (acc_j += g^2 in q order),
// its value is (acc_0 + acc_1) + (acc_2 + acc_3); warps reduce with a fixed
// shuffle tree and the 16 warp sums are added in ascending order.  Squares of
// fp32 values are exact in fp64, so only the sums round.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <atomic>
#include <climits>
#include <cstdint>
#include <type_traits>
#include <utility>

#include "grass_internal.h"

namespace grass {
namespace {

constexpr int kConsumerWarps = kThreads / 32;  // 16

constexpr int kStreamThreads = kThreads + 32;  // + 1 producer warp

// griddepcontrol.wait: a no-op unless the grid was launched as a programmatic
// dependent of the previous kernel on the stream (launch_pdl)
__device__ __forceinline__ void grid_dependency_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

__device__ __forceinline__ double warp_sum(double x) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x += __shfl_down_sync(0xffffffffu, x, o);
  return x;  // lane 0 holds the fixed-tree sum
}

// warp_sum of N <= 16 per-lane values at once (one per tile of a unit): a
// transposed butterfly over C = next power of two >= N slots, with the values
// PRE-PERMUTED per lane: slot t of lane L holds tile t ^ m(L), m(L) = (L >>
// (5 - log2 C)) & (C - 1) (the caller reads its tiles in that order; tiles
// >= N are 0).  At the first log2(C) offsets o = 16, 8, ... every lane keeps
// the lower half of its slots and adds the partner's upper half, which holds
// the same tiles (the partner's m differs exactly in the bit of this level),
// so no lane-dependent selects are needed; the remaining offsets are a plain
// butterfly on the one slot left.  Each tile is summed by the same pairs of
// lane groups as warp_sum (level o adds the groups of lanes i and i + o; IEEE
// addition is commutative): every result is bit-identical to warp_sum of that
// tile, for C - 1 + 5 - log2(C) exchanges instead of 5N.  Lane L ends with the
// sum of tile m(L): *slot = m(L) in the lowest lane of each group holding it
// (and < N), else -1.
template <int N>
struct MultiSlots {
  static_assert(N >= 1 && N <= 16, "one value per tile of a unit");
  static constexpr int C = N <= 1 ? 1 : N <= 2 ? 2 : N <= 4 ? 4 : N <= 8 ? 8 : 16;
  static constexpr int LOG = C == 1 ? 0 : C == 2 ? 1 : C == 4 ? 2 : C == 8 ? 3 : 4;
  static constexpr int SHIFT = 5 - LOG;
};
// Tiles of a unit reduced together by one warp_sum_perm: the whole unit when
// TPS is a power of two, else groups of 4 or 2 (no empty slots either way).
template <int TPS>
constexpr int kPermGroup = (TPS & (TPS - 1)) == 0 ? TPS : (TPS % 4 == 0 ? 4 : (TPS % 2 == 0 ? 2 : 1));
template <int N>
__device__ __forceinline__ double warp_sum_perm(double (&w)[MultiSlots<N>::C], int lane, int* slot) {
  constexpr int C = MultiSlots<N>::C;
#pragma unroll
  for (int c = C, o = 16; c > 1; c >>= 1, o >>= 1) {
#pragma unroll
    for (int j = 0; j < c / 2; ++j) w[j] = w[j] + __shfl_xor_sync(0xffffffffu, w[j + c / 2], o);
  }
#pragma unroll
  for (int o = 16 >> MultiSlots<N>::LOG; o > 0; o >>= 1) w[0] += __shfl_xor_sync(0xffffffffu, w[0], o);
  constexpr int SH = MultiSlots<N>::SHIFT;
  const int idx = (lane >> SH) & (C - 1);
  *slot = ((lane & ((1 << SH) - 1)) == 0 && idx < N) ? idx : -1;
  return w[0];
}

struct AdamScalars {
  float b1, omb1, b2, omb2, eps, decay, step, inv_bc2s;
  float cf;  // gradient multiplier of the update: global-norm clip coefficient, else 1
};

// One element of AdamW (torch.optim.AdamW semantics, R1), fp32 storage:
//   theta1 = theta*(1 - lr*wd); m' = b1*m + (1-b1)*g; v' = b2*v + (1-b2)*g^2
//   theta' = theta1 - lr/bc1 * m' / (sqrt(v')/sqrt(bc2) + eps)
// sqrt and the division use the hardware approximations (MUFU; relative error
// <= 2^-22, subnormals kept) instead of the multi-instruction IEEE sequences:
// the error they add to theta' is < 1e-6 of the update, far inside the 1e-5
// parity bar, and the IEEE sequences cost ~3% of K2's time (measured A/B).
__device__ __forceinline__ void adamw1(float g, float& th, float& m, float& v,
                                       const AdamScalars& s) {
#ifdef GRASS_K2_NOMATH  // A/B only: the same data movement with trivial arithmetic (speed of light)
  th += g; m += g; v += g;
  return;
#endif
  g *= s.cf;  // exact when cf == 1
  const float t1 = th * s.decay;
  const float m1 = fmaf(s.b1, m, s.omb1 * g);
  const float v1 = fmaf(s.b2, v, (s.omb2 * g) * g);
#ifdef GRASS_IEEE_MATH
  const float den = fmaf(__fsqrt_rn(v1), s.inv_bc2s, s.eps);
  th = fmaf(-s.step, __fdiv_rn(m1, den), t1);
#else
  float sq;
  asm("sqrt.approx.f32 %0, %1;" : "=f"(sq) : "f"(v1));
  const float den = fmaf(sq, s.inv_bc2s, s.eps);
  th = fmaf(-s.step, __fdividef(m1, den), t1);
#endif
  m = m1;
  v = v1;
}

// Streaming stores of theta, m, v (written once per step).
__device__ __forceinline__ void st_stream(float* p, const float4& x) {
#ifdef GRASS_ST_DEFAULT
  *reinterpret_cast<float4*>(p) = x;
#else
  __stcs(reinterpret_cast<float4*>(p), x);
#endif
}

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_addr(bar)),
      "r"(parity)
      : "memory");
}
// L2 policy of the bulk loads: the update stream (K2) measured faster with
// evict_normal, the norm-only stream (K1) with evict_first.
template <bool UPDATE>
__device__ __forceinline__ uint64_t l2_load_policy() {
  uint64_t pol;
#ifdef GRASS_K2_LOAD_EF
  if (false)
#else
  if (UPDATE)
#endif
    asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(pol));
  else
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
// TMA bulk copy global -> shared, completion counted on `bar` (bytes % 16 == 0).
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                          uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1], %2, [%3], %4;" ::"r"(smem_addr(dst)),
      "l"(src), "r"(bytes), "r"(smem_addr(bar)), "l"(pol)
      : "memory");
}
// TMA bulk copy shared -> global (bulk-group completion).
__device__ __forceinline__ void bulk_store(void* dst, const void* src, uint32_t bytes) {
#ifdef GRASS_K2_STORE_EF
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group.L2::cache_hint [%0], [%1], %2, %3;" ::"l"(dst),
               "r"(smem_addr(src)), "r"(bytes), "l"(pol)
               : "memory");
#else
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst),
               "r"(smem_addr(src)), "r"(bytes)
               : "memory");
#endif
}
// L2 prefetch of a future unit (A/B knob GRASS_L2_PREFETCH_{NORM,UPD} = units ahead)
__device__ __forceinline__ void bulk_prefetch_l2(const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}
#ifndef GRASS_L2_PREFETCH_NORM
#define GRASS_L2_PREFETCH_NORM 0
#endif
#ifndef GRASS_L2_PREFETCH_UPD
#define GRASS_L2_PREFETCH_UPD 0
#endif
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read_all() {
  asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
// Barrier over the consumer warps only (the producer warp never waits on it).
__device__ __forceinline__ void consumer_sync() {
  asm volatile("bar.sync 1, %0;" ::"n"(kThreads) : "memory");
}

// K3: the layer total is the fixed-order sum of its tile partials — thread t
// (of 1024) adds tiles t, t + 1024, ... in ascending order (loads batched 16
// deep, the additions in the same order), then the fixed warp tree and the 32
// warp sums in ascending order.  One CTA
// per completed layer of the preceding stream launch (grass_finalize_kernel):
// the layers finish in parallel, not one after another in the CTA that
// completed them last (up to ~0.4 ms at the end of a 32-layer probing pass).
// Device-resident commit + resample (grass_device_step): exactly the host's
// grass_update_probs (Eq. 2 window mean, first commit / Eq. 4 EMA with frozen
// retention, Eq. 3 softmax per policy, window reset) and grass_sample_layers
// (R6 / R7: gamma sequential draws with renormalisation, counter-based
// SplitMix64) in fp64, on one thread, in the host's operation order (the
// library is built with --fmad=false: no contraction); only exp() may differ
// from the host's by an ulp.  A non-finite norm or an empty commit is
// recorded in *err (sticky) and reported by grass_device_schedule_end.
__device__ __forceinline__ uint64_t d_splitmix64(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
constexpr int kCommitThreads = 256;
// The commit + resample body, run by one whole CTA (the stand-alone kernel at
// grass_device_schedule_begin, or the last K3 CTA of a device step).  `sm` is
// dynamic shared memory of commit_smem_bytes(nl).  S, c and the flag are read
// through L2: in the fused form they were written by other CTAs of the same
// launch.
__device__ void commit_sample_body(const CommitArgs& a, const DevState& st, double* sm) {
  // operands staged in shared memory; the elementwise steps (window mean,
  // EMA, exp, the final division) run one layer per thread, the order-
  // dependent ones (the maxima, the ascending sum, the sampler) on thread 0 —
  // every value computed by the same operations as the host's loops
  // sm: S [nl] | m [nl] | p [nl] | c [nl] (int64) | picked [nl] (int32)
  double* sS = sm;
  double* sM = sS + a.nl;
  double* sP = sM + a.nl;
  long long* sC = reinterpret_cast<long long*>(sP + a.nl);
  int* sAv = reinterpret_cast<int*>(sC + a.nl);
  __shared__ int s_err, s_committed, s_commit, s_soft, s_flag;
  __shared__ unsigned long long s_pctr;
  __shared__ double s_M, s_mx, s_tot;
  const int tid = threadIdx.x, ns = a.nsamp;
  // every operand load issued at once (the scalars by threads of their own —
  // they sit in HBM after K2's stream, so a chain of them would cost a DRAM
  // round trip each)
  if (tid == 32) s_err = *a.err;
  if (tid == 33) s_committed = *a.committed;
  if (tid == 34) s_flag = __ldcg(st.flag);
  if (tid == 35) s_pctr = a.do_sample ? *a.period_ctr : 0ull;
  for (int l = tid; l < a.nl; l += blockDim.x) {
    sS[l] = __ldcg(st.S + l);
    sC[l] = __ldcg(st.c + l);
    sM[l] = a.m[l];
    sP[l] = a.probs[l];
  }
  __syncthreads();
  if (tid == 0) {
    s_commit = 0;
    if (!s_err && a.do_commit) {
      long long total = 0;
      for (int l = 0; l < ns; ++l) total += sC[l];
      if (s_flag != 0) s_err = 2;
      else if (total == 0 && (s_committed || a.T_p != 0)) s_err = 1;
      else s_commit = 1;
    }
    s_soft = s_commit && (a.policy == GRASS_POLICY_ADAPTIVE || !s_committed) && a.policy != GRASS_POLICY_UNIFORM;
  }
  __syncthreads();
  if (s_err) {  // an error stops the schedule (reported by grass_device_schedule_end)
    if (tid == 0) *a.err = s_err;
    return;
  }
  const bool committed = s_committed != 0;
  if (s_commit) {  // Eq. 2 window mean, first commit / Eq. 4 EMA, frozen retention
    for (int l = tid; l < ns; l += blockDim.x) {
      if (sC[l] > 0) {
        const double w = sS[l] / (double)sC[l];
        sM[l] = committed ? a.alpha * w + (1.0 - a.alpha) * sM[l] : w;
      } else if (!committed) {
        sM[l] = 0.0;
      }
      if (a.policy == GRASS_POLICY_UNIFORM) sP[l] = 1.0 / ns;
    }
  }
  __syncthreads();
  if (s_soft && tid < 32) {  // Eq. 3: the maxima — exact, so one warp's tree gives the host loop's values
    double M = -INFINITY;
    for (int i = tid; i < ns; i += 32) M = sM[i] > M ? sM[i] : M;
    for (int o = 16; o > 0; o >>= 1) {
      const double y = __shfl_xor_sync(0xffffffffu, M, o);
      M = y > M ? y : M;
    }
    double mx = -INFINITY;
    for (int i = tid; i < ns; i += 32) {
      const double mti = a.normalize ? (M > 0.0 ? sM[i] / M : 0.0) : sM[i];
      mx = mti > mx ? mti : mx;
    }
    for (int o = 16; o > 0; o >>= 1) {
      const double y = __shfl_xor_sync(0xffffffffu, mx, o);
      mx = y > mx ? y : mx;
    }
    if (tid == 0) {
      s_M = M;
      s_mx = mx;
    }
  }
  __syncthreads();
  if (s_soft) {
    const double M = s_M, mx = s_mx;
    for (int i = tid; i < ns; i += blockDim.x) {
      const double mti = a.normalize ? (M > 0.0 ? sM[i] / M : 0.0) : sM[i];
      sP[i] = exp((mti - mx) / a.tau);
    }
  }
  __syncthreads();
  if (s_soft && tid == 0) {  // the ascending sum
    double tot = 0.0;
    for (int i = 0; i < ns; ++i) tot += sP[i];
    s_tot = tot;
  }
  __syncthreads();
  if (s_soft)
    for (int i = tid; i < ns; i += blockDim.x) sP[i] = sP[i] / s_tot;
  __syncthreads();
#ifndef GRASS_K3_DIAG
#define GRASS_K3_DIAG 0
#endif
  if (tid < 32 && a.do_sample && GRASS_K3_DIAG != 3) {  // R6 / R7, as grass_sample_layers, by warp 0
    const uint64_t period = a.period == ~0ull ? s_pctr + 1 : a.period;
    // the available layers are those not yet picked (sAv[j] = 0), ascending.
    // The warp forms the running sum over them in order — layer j's term
    // broadcast from its lane, so the chain of additions waits on no memory;
    // a picked layer adds +0.0, which leaves the sum unchanged (>= +0) — and
    // lane j keeps it in sS[j] (the window sums are no longer needed): sS[j]
    // is the host walk's c at layer j and the final sum its R.  The pick is
    // the first available j with x < c_j (a ballot), else the last available
    // layer (only when R == 0).
    for (int j = tid; j < ns; j += 32) sAv[j] = 0;
    __syncwarp();
    const uint64_t key = d_splitmix64(a.seed);
    for (int k = 0; k < a.gamma; ++k) {
      const uint64_t ctr = (period << 16) + (uint64_t)k;
      const double u = (double)(d_splitmix64(key ^ ctr) >> 11) * 0x1.0p-53;
      double c = 0.0;
      for (int base = 0; base < ns; base += 32) {
        const int j = base + tid;
        const double term = j < ns && !sAv[j] ? sP[j] : 0.0;
        double cj = 0.0;
        for (int q = 0; q < 32; ++q) {  // lanes past ns hold +0.0: the sum is unchanged
          c += __shfl_sync(0xffffffffu, term, q);
          cj = tid == q ? c : cj;
        }
        if (j < ns) sS[j] = cj;
      }
      __syncwarp();
      const double R = c;
      const double x = u * R;
      int pick = -1;
      for (int base = 0; base < ns && pick < 0; base += 32) {
        const int j = base + tid;
        const unsigned hit = __ballot_sync(0xffffffffu, j < ns && !sAv[j] && x < sS[j]);
        if (hit) pick = base + __ffs(hit) - 1;
      }
      for (int base = (ns - 1) & ~31; base >= 0 && pick < 0; base -= 32) {  // none: the last available layer
        const int j = base + tid;
        const unsigned av = __ballot_sync(0xffffffffu, j < ns && !sAv[j]);
        if (av) pick = base + 31 - __clz(av);
      }
      __syncwarp();
      if (tid == 0) {
        a.ids[k] = pick;
        sAv[pick] = 1;
      }
      __syncwarp();
    }
    if (tid == 0) *a.period_ctr = period;
  }
  if (tid == 0 && s_commit) *a.committed = 1;
  if (s_commit) {  // m, p back; the window restarts (every layer, as the host's reset)
    for (int l = tid; l < a.nl; l += blockDim.x) {
      a.m[l] = sM[l];
      a.probs[l] = sP[l];
      st.S[l] = 0.0;
      st.c[l] = 0;
    }
  }
}

__global__ void __launch_bounds__(kCommitThreads) grass_commit_sample_kernel(const __grid_constant__ CommitArgs a,
                                                                             const DevState st) {
  extern __shared__ double csm[];
  commit_sample_body(a, st, csm);
}

constexpr int kFinThreads = 1024;  // K3 threads per layer (32 warps)
__global__ void __launch_bounds__(kFinThreads, 1) grass_finalize_kernel(const __grid_constant__ FinalizeArgs fa,
                                                                     const DevState st) {
  constexpr int kW = kFinThreads / 32;
  __shared__ double red[kW];
  grid_dependency_wait();  // PDL (device step): K2's partials are complete and visible
  const int j = blockIdx.x;
  const int layer = fa.dev_ids ? fa.dev_ids[j] : fa.layer[j];
  const int n = fa.dev_ids ? fa.dev_table[layer].layer_tiles : fa.tiles[j];
  const double* P = st.partials + (fa.dev_ids ? fa.dev_table[layer].part_layer_base : fa.base[j]);
  // thread 0's operands of the window update, loaded alongside the partials
  // (only this CTA writes them; the kernels before it have completed)
  double S0 = 0.0, numel = 1.0;
  long long c0 = 0;
  if (threadIdx.x == 0 && fa.mode == kFinalizeMgn) {
    S0 = st.S[layer];
    c0 = st.c[layer];
    numel = (double)(fa.dev_ids ? fa.dev_table[layer].layer_numel : fa.numel[j]);
  }
  double a = 0.0;
  int i = threadIdx.x;
  for (; i + 15 * kFinThreads < n; i += 16 * kFinThreads) {  // 16 loads in flight per thread
    double x[16];
#pragma unroll
    for (int k = 0; k < 16; ++k) x[k] = __ldcg(P + i + k * kFinThreads);
#pragma unroll
    for (int k = 0; k < 16; ++k) a += x[k];
  }
  for (; i < n; i += kFinThreads) a += __ldcg(P + i);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const double w = warp_sum(a);
  if (lane == 0) red[warp] = w;
  __syncthreads();
  if (threadIdx.x == 0) {
    double ss = 0.0;
#pragma unroll
    for (int k = 0; k < kW; ++k) ss += red[k];
    if (fa.mode == kFinalizeMgn) {
      st.last_ss[layer] = ss;
      if (isfinite(ss)) {
        st.S[layer] = S0 + sqrt(ss / numel);  // Eq. 2 inner term
        st.c[layer] = c0 + 1;
      } else {
        atomicMax(st.flag, INT_MAX - layer);  // smallest id wins
      }
    } else if (fa.mode == kFinalizeShard) {
      st.shard_ss[fa.out_slot[j]] = ss;
    }
    if (fa.advance) {  // the step prologue's state update (device-resident schedule)
      st.t[layer] += 1;
      if (fa.bf16) st.mvalid[layer] = 1;
    }
  }
#ifndef GRASS_K3_DIAG
#define GRASS_K3_DIAG 0
#endif
  if (fa.fuse_commit && GRASS_K3_DIAG != 2) {  // the CTA that completes last runs the commit + resample
    __shared__ int last;
    if (threadIdx.x == 0) {
      __threadfence();
      last = atomicAdd(fa.done_ctr, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (last) {
      __threadfence();
      extern __shared__ double fsm[];
      if (GRASS_K3_DIAG != 1) commit_sample_body(fa.ca, st, fsm);
      if (threadIdx.x == 0) *fa.done_ctr = 0;
    }
  }
}



// K2 writes its results back into the stage and the producer bulk-stores them
// (TMA, SASS UBLKCP.G.S): measured 2.4% faster than per-thread 128-bit stores.
#ifdef GRASS_K2_STG_STORE
constexpr bool kTmaStore = false;
#else
constexpr bool kTmaStore = true;
#endif
// GRASS_K2_SEP_OUT: results go to a separate output region of the stage, so
// the producer can refill the input region while the previous unit's bulk
// stores are still reading shared memory (A/B knob).
#ifdef GRASS_K2_SEP_OUT
constexpr bool kSepOut = kTmaStore;
#else
constexpr bool kSepOut = false;
#endif

// The branch-free full-unit path (inside the kernel) is used for the
// norm-only stream only: +18% for K1, while K2's interleaved compute/store
// order measured ~0.5% faster without it (profiles/r01_variants_*.json).
#include "stream_kernel.cuh"


__global__ void grass_rank_sum_kernel(const double* __restrict__ gathered,
                                      const __grid_constant__ RankSumArgs a, const DevState st) {
  const int j = threadIdx.x;
  if (j >= a.n) return;
  double ss = 0.0;
  for (int r = 0; r < a.world; ++r) ss += gathered[(int64_t)r * a.total_slots + a.slot0 + j];
  const int l = a.layer[j];
  st.last_ss[l] = ss;
  if (isfinite(ss)) {
    st.S[l] += sqrt(ss / (double)a.numel[j]);
    st.c[l] += 1;
  } else {
    atomicMax(st.flag, INT_MAX - l);
  }
}

// P2P publication + barrier (one CTA).  Publishes this rank's shard norms into
// row `rank` of every rank's gather block, then (which >= 0) signals flag
// [which][rank] = epoch in every rank's block and waits until every rank has
// signalled this rank's flags [which][*].  The signal is a system-scope release
// after a system fence, the wait a system-scope acquire, so writes issued
// before it (the fused kernel's peer stores of theta', the published norms)
// are visible to every rank after it.  A peer that never arrives (crashed
// rank) ends the wait after kP2PTimeoutNs with err = 1 (surfaced by the next
// synchronising call) instead of hanging the GPU.
constexpr unsigned long long kP2PTimeoutNs = 60ull * 1000 * 1000 * 1000;
__device__ __forceinline__ unsigned long long global_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
// One rank's publication + barrier, executed by one CTA (rank = a.rank).
__device__ void p2p_sync_cta(const P2PSyncArgs& a) {
  const int tid = threadIdx.x;
  __shared__ unsigned long long epoch;
  if (tid == 0 && a.which >= 0) epoch = a.epoch_ctr ? ++a.epoch_ctr[a.which] : a.epoch;
  for (int k = tid; k < a.world * a.n; k += blockDim.x) {
    const int q = k / a.n, j = k % a.n;
    double* row = reinterpret_cast<double*>(a.exch[q] + kExchGather) + (int64_t)a.rank * a.n;
    row[j] = a.shard_ss[j];
  }
  if (a.which < 0) return;
  __syncthreads();
  if (tid < a.world) {
    __threadfence_system();
    unsigned long long* peer_flag =
        reinterpret_cast<unsigned long long*>(a.exch[tid]) + a.which * kMaxPeers + a.rank;
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(peer_flag), "l"(epoch) : "memory");
    const unsigned long long* mine =
        reinterpret_cast<const unsigned long long*>(a.exch[a.rank]) + a.which * kMaxPeers + tid;
    const unsigned long long t0 = global_ns();
    while (true) {
      unsigned long long v;
      asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(mine) : "memory");
      if (v >= epoch) break;
      if (global_ns() - t0 > kP2PTimeoutNs) {
        atomicExch(a.err, 1);
        break;
      }
      __nanosleep(200);
    }
  }
  __syncthreads();
}

__global__ void grass_p2p_sync_kernel(const __grid_constant__ P2PSyncArgs a) { p2p_sync_cta(a); }

// Self-test of the publication + barrier protocol (grass_selftest_p2p): W ranks
// emulated as the W co-resident CTAs of ONE cooperative launch (the profiling
// rules: ranks that wait on one another must not be separate launches on one
// GPU).  Every round each rank writes round-dependent norms, publishes them
// with the end barrier, checks that every rank's row arrived, then passes the
// start barrier before the next round may overwrite the rows.
struct P2PSelftestArgs {
  char* exch[kMaxPeers];
  double* ss;          // [world][n] per-rank "shard norms"
  int32_t world, n, rounds;
  int* err;
  unsigned long long* mismatches;
};
__global__ void grass_p2p_selftest_kernel(const __grid_constant__ P2PSelftestArgs t) {
  const int rank = blockIdx.x;
  P2PSyncArgs a;
  a.epoch_ctr = nullptr;  // explicit generations (the round)
  for (int q = 0; q < kMaxPeers; ++q) a.exch[q] = t.exch[q];
  a.rank = rank;
  a.world = t.world;
  a.n = t.n;
  a.shard_ss = t.ss + (int64_t)rank * t.n;
  a.err = t.err;
  double* mine = t.ss + (int64_t)rank * t.n;
  const double* rows = reinterpret_cast<const double*>(t.exch[rank] + kExchGather);
  for (int round = 1; round <= t.rounds; ++round) {
    for (int j = threadIdx.x; j < t.n; j += blockDim.x) mine[j] = round * 1000.0 + rank * 10.0 + j;
    __syncthreads();
    a.which = 1;
    a.epoch = (uint64_t)round;
    p2p_sync_cta(a);  // publish + end barrier
    // rank- and round-dependent skew (0-5 us) so that a missing barrier shows
    if (threadIdx.x == 0) __nanosleep((unsigned)(((round * 7919 + rank * 104729) % 50) * 100));
    __syncthreads();
    for (int k = threadIdx.x; k < t.world * t.n; k += blockDim.x) {
      const int r = k / t.n, j = k % t.n;
      if (rows[k] != round * 1000.0 + r * 10.0 + j) atomicAdd(t.mismatches, 1ull);
    }
    __syncthreads();
    a.which = 0;  // start barrier: every rank has read its rows of this round
    const int n_save = a.n;
    a.n = 0;
    p2p_sync_cta(a);
    a.n = n_save;
  }
}

__global__ void grass_step_prologue_kernel(const __grid_constant__ PrologueArgs a, const DevState st) {
  const int j = threadIdx.x;
  if (j >= a.n) return;
  const int l = a.layer[j];
  const long long t = st.t[l] + 1;
  st.t[l] = t;
  const double lr = a.lr_ptr ? (double)*a.lr_ptr : (double)a.lr;
  const double bc1 = 1.0 - pow(a.beta1, (double)t);
  const double bc2 = 1.0 - pow(a.beta2, (double)t);
  st.scal[3 * l + 0] = (float)(1.0 - lr * a.wd);
  st.scal[3 * l + 1] = (float)(lr / bc1);
  st.scal[3 * l + 2] = (float)(1.0 / sqrt(bc2));
  if (a.bf16) {
    st.init_now[l] = st.mvalid[l] ? 0 : 1;
    st.mvalid[l] = 1;
  }
}

__global__ void grass_clip_coef_kernel(const __grid_constant__ ClipArgs a, const DevState st,
                                       float* coef) {
  if (threadIdx.x != 0) return;
  double tot = 0.0;
  for (int j = 0; j < a.n; ++j) tot += st.last_ss[a.layer[j]];
  coef[0] = (float)fmin(1.0, a.max_norm / (sqrt(tot) + 1e-6));
}

// Production configuration.
#ifndef GRASS_UPD_STAGES
#define GRASS_UPD_STAGES 2
#endif
#ifndef GRASS_NORM_TPS
#define GRASS_NORM_TPS 6
#endif
#ifndef GRASS_NORM_STAGES
#define GRASS_NORM_STAGES 2
#endif
constexpr int kUpdTPS = 1, kUpdStages = GRASS_UPD_STAGES;  // 4 arrays x 16 KiB per stage -> 128 KiB ring
constexpr int kNormTPS = GRASS_NORM_TPS, kNormStages = GRASS_NORM_STAGES;  // 96 KiB x 2 -> 192 KiB
#ifndef GRASS_NORM_TPS_BF16
#define GRASS_NORM_TPS_BF16 4  // 32 KiB units x 6 stages: 1.77 ms vs 1.86 (12 x 2) / 1.95 (8 x 3), profiles/r02_variants_k3_split.json
#endif
constexpr int kNormTPSBf16 = GRASS_NORM_TPS_BF16;  // bf16 probing: tiles per unit (2 B/element)
#ifndef GRASS_NORM_STAGES_BF16
#define GRASS_NORM_STAGES_BF16 6
#endif
constexpr int kNormStagesBf16 = GRASS_NORM_STAGES_BF16;
#ifndef GRASS_P2P_NORM_TPS
#define GRASS_P2P_NORM_TPS 4  // 3 x 64 KiB fp32 / 6 x 32 KiB bf16 gradient slots: 6 tiles spill at the 96-register limit
#endif
constexpr int kP2PNormTPS = GRASS_P2P_NORM_TPS;  // P2P probing: tiles per gradient-ring slot

// Programmatic dependent launch (the device-resident schedule's two kernels):
// the grid may be launched while the previous kernel on the stream drains;
// the kernel's griddepcontrol.wait (grid_dependency_wait) holds every read of
// the previous kernel's results until that kernel has completed and its
// writes are visible.  No kernel triggers early, so the dependency is full
// completion; what overlaps is the launch and CTA ramp.
template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kern)(KArgs...), int grid, int threads, size_t smem, cudaStream_t s, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(threads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

template <bool U, int TPS, int ST, bool BF16, bool P2P = false, bool DEVB = false>
cudaError_t launch_stream(const Batch& b, const DevState& st, int grid, cudaStream_t s) {
  using SL = StageLayout<U, BF16, TPS>;
  using GS = P2PGSlots<U, BF16>;
  constexpr size_t smem = (P2P && GS::kNoStageRing ? 0 : (size_t)ST * SL::bytes) +
                          (P2P ? (size_t)GS::slots(SL::kUnit * SL::GB) * SL::kUnit * SL::GB : 0);
  static_assert(smem <= 227 * 1024, "ring exceeds the 227 KiB shared-memory limit");
  // the opt-in shared-memory size is a per-device function attribute: set it
  // once per device (contexts on several GPUs / threads share this instance)
  static std::atomic<unsigned long long> attr_set{0};
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  const unsigned long long bit = dev < 64 ? 1ull << dev : 0ull;
  if (!bit || !(attr_set.load(std::memory_order_acquire) & bit)) {
    e = cudaFuncSetAttribute(grass_stream_kernel<U, TPS, ST, BF16, P2P, DEVB>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    attr_set.fetch_or(bit, std::memory_order_release);
  }
  int units = 0;
  for (int i = 0; i < b.nseg; ++i) units += (b.seg[i].tiles + TPS - 1) / TPS;
  const int g = DEVB ? grid : (grid < units ? grid : units);  // DEVB: the units are known on the device only
  if (DEVB) return launch_pdl(grass_stream_kernel<U, TPS, ST, BF16, P2P, DEVB>, g, kStreamThreads, smem, s, b, st);
  grass_stream_kernel<U, TPS, ST, BF16, P2P, DEVB><<<g, kStreamThreads, smem, s>>>(b, st);
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_fused(bool update, const Batch& b, const DevState& st, int grid,
                         cudaStream_t s) {
  if (b.nseg <= 0 || b.tile_prefix[b.nseg] <= 0) return cudaSuccess;
  if (b.npeer > 0) {  // P2P data parallelism: one tile per unit, the gradient read from the peers
    if (b.bf16)
      return update ? launch_stream<true, 1, 2, true, true>(b, st, grid, s)
                    : launch_stream<false, kP2PNormTPS, 2, true, true>(b, st, grid, s);
    return update ? launch_stream<true, 1, 2, false, true>(b, st, grid, s)
                  : launch_stream<false, kP2PNormTPS, 2, false, true>(b, st, grid, s);
  }
  if (b.bf16)
    return update ? launch_stream<true, kUpdTPS, kUpdStages, true>(b, st, grid, s)
                  : launch_stream<false, kNormTPSBf16, kNormStagesBf16, true>(b, st, grid, s);
  return update ? launch_stream<true, kUpdTPS, kUpdStages, false>(b, st, grid, s)
                : launch_stream<false, kNormTPS, kNormStages, false>(b, st, grid, s);
}

size_t commit_smem_bytes(int nl) { return (size_t)nl * (4 * sizeof(double) + sizeof(int)); }

cudaError_t launch_finalize(const FinalizeArgs& a, const DevState& st, cudaStream_t s) {
  if (a.n <= 0) return cudaSuccess;
  const size_t smem = a.fuse_commit ? commit_smem_bytes(a.ca.nl) : 0;
  if (smem > 40 * 1024) {
    const cudaError_t e =
        cudaFuncSetAttribute(grass_finalize_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem + 1024);
    if (e != cudaSuccess) return e;
  }
  if (a.dev_ids) return launch_pdl(grass_finalize_kernel, a.n, kFinThreads, smem, s, a, st);
  grass_finalize_kernel<<<a.n, kFinThreads, smem, s>>>(a, st);
  return cudaGetLastError();
}

cudaError_t launch_fused_dev(const Batch& b, const DevState& st, int grid, cudaStream_t s) {
  if (b.dev_n <= 0) return cudaSuccess;
  return b.bf16 ? launch_stream<true, kUpdTPS, kUpdStages, true, false, true>(b, st, grid, s)
                : launch_stream<true, kUpdTPS, kUpdStages, false, false, true>(b, st, grid, s);
}

cudaError_t launch_commit_sample(const CommitArgs& a, const DevState& st, cudaStream_t s) {
  const size_t smem = commit_smem_bytes(a.nl);
  if (smem > 48 * 1024) {
    const cudaError_t e = cudaFuncSetAttribute(grass_commit_sample_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                               (int)smem);
    if (e != cudaSuccess) return e;
  }
  grass_commit_sample_kernel<<<1, kCommitThreads, smem, s>>>(a, st);
  return cudaGetLastError();
}

cudaError_t launch_rank_sum(const double* gathered, const RankSumArgs& a, const DevState& st,
                            cudaStream_t s) {
  if (a.n <= 0) return cudaSuccess;
  grass_rank_sum_kernel<<<1, 64, 0, s>>>(gathered, a, st);
  return cudaGetLastError();
}

cudaError_t launch_p2p_sync(const P2PSyncArgs& a, cudaStream_t s) {
  grass_p2p_sync_kernel<<<1, 256, 0, s>>>(a);
  return cudaGetLastError();
}

cudaError_t p2p_selftest(int world, int n, int rounds, unsigned long long* mismatches, int* timed_out) {
  if (world < 1 || world > kMaxPeers || n < 1 || rounds < 1) return cudaErrorInvalidValue;
  const size_t blk = (size_t)kExchGather + sizeof(double) * (size_t)world * n;
  char* mem = nullptr;
  cudaError_t e = cudaMalloc(&mem, blk * world + sizeof(double) * (size_t)world * n + 64);
  if (e != cudaSuccess) return e;
  e = cudaMemset(mem, 0, blk * world + sizeof(double) * (size_t)world * n + 64);
  P2PSelftestArgs t;
  for (int q = 0; q < kMaxPeers; ++q) t.exch[q] = q < world ? mem + blk * q : nullptr;
  t.ss = reinterpret_cast<double*>(mem + blk * world);
  t.err = reinterpret_cast<int*>(mem + blk * world + sizeof(double) * (size_t)world * n);
  t.mismatches = reinterpret_cast<unsigned long long*>(mem + blk * world + sizeof(double) * (size_t)world * n + 8);
  t.world = world;
  t.n = n;
  t.rounds = rounds;
  if (e == cudaSuccess) {
    void* args[] = {&t};
    e = cudaLaunchCooperativeKernel((const void*)grass_p2p_selftest_kernel, dim3(world), dim3(256), args, 0, nullptr);
  }
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  if (e == cudaSuccess) e = cudaMemcpy(mismatches, t.mismatches, sizeof(*mismatches), cudaMemcpyDeviceToHost);
  if (e == cudaSuccess) e = cudaMemcpy(timed_out, t.err, sizeof(int), cudaMemcpyDeviceToHost);
  cudaFree(mem);
  return e;
}

cudaError_t launch_step_prologue(const PrologueArgs& a, const DevState& st, cudaStream_t s) {
  if (a.n <= 0) return cudaSuccess;
  grass_step_prologue_kernel<<<1, 64, 0, s>>>(a, st);
  return cudaGetLastError();
}

cudaError_t launch_clip_coef(const ClipArgs& a, const DevState& st, float* coef, cudaStream_t s) {
  grass_clip_coef_kernel<<<1, 32, 0, s>>>(a, st, coef);
  return cudaGetLastError();
}

// Grid of the persistent kernels.  K1 (reads only) is fastest with one CTA on
// every SM.  K2 (4 read + 3 write streams per CTA, 128 KiB in flight per CTA)
// is fastest with FEWER CTAs: on B200 128 of 148 SMs for fp32 (1.72 vs
// 1.785 ms at configs[1], +3.7%), 132 for bf16 — fewer concurrent streams keep
// the DRAM pages better (profiles/r01_variants_k2_grid*.json; 3 stages, i.e.
// more bytes in flight, measured 5% slower).  Results never depend on the grid.
#ifndef GRASS_UPD_GRID_SUB
#define GRASS_UPD_GRID_SUB -1  // A/B knob: SMs left out of K2's grid (-1: the tuned default)
#endif
#ifndef GRASS_NORM_GRID_SUB
#define GRASS_NORM_GRID_SUB 0  // A/B knob: SMs left out of K1's grid
#endif
int fused_grid(bool update, bool bf16, int device) {
  int sms = 0;
  if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device) != cudaSuccess) return 0;
  if (!update) return sms - GRASS_NORM_GRID_SUB;
  if (GRASS_UPD_GRID_SUB >= 0) return sms - GRASS_UPD_GRID_SUB;
  return (sms * (bf16 ? 132 : 128) + 74) / 148;  // 128 / 132 of B200's 148
}

}  // namespace grass
