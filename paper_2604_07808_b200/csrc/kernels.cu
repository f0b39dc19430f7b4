// kernels.cu — sm_100a kernels of the GRASS hot path.
//
//   K1  grass_fused_kernel<false>: Eq. 2 squared norm only (probing,
//       PAPER.md:111-113) — reads g once (4 B/param).
//   K2  grass_fused_kernel<true>:  single-pass Eq. 2 norm + AdamW (DESIGN.md
//       R1/R2) of the trainable layers — reads g, theta, m, v,
//       writes theta, m, v (28 B/param).
//   K3  finalize (inside K1/K2, last block of each layer): fixed-order fp64 sum
//       of the layer's tile partials, then S_l += sqrt(ss_l / N_p), c_l += 1
//       (Eq. 2), or the shard value for the cross-rank sum.
//   K4  grass_rank_sum_kernel (world > 1): ascending-rank fp64 sum of the
//       all-gathered shard partials, then the same MGN update.
//
// Nothing here is a contraction: these kernels are HBM-bound streams (about
// 0.5 flop/B), so they use 128-bit coalesced loads/stores with streaming
// cache hints, enough bytes in flight per SM, and no tensor cores.
#include <cuda_runtime.h>

#include <climits>
#include <cstdint>

#include "grass_internal.h"

namespace grass {
namespace {

__device__ __forceinline__ double warp_sum(double x) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x += __shfl_down_sync(0xffffffffu, x, o);
  return x;  // lane 0 holds the fixed-tree sum
}

// Fixed-shape block reduction: warp trees, then warp 0 sums the 8 warp
// results in ascending order.  Result valid in thread 0.
__device__ __forceinline__ double block_sum(double x, double* red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  x = warp_sum(x);
  if (lane == 0) red[warp] = x;
  __syncthreads();
  double t = 0.0;
  if (threadIdx.x == 0) {
#pragma unroll
    for (int w = 0; w < kThreads / 32; ++w) t += red[w];
  }
  return t;
}

struct AdamScalars {
  float b1, omb1, b2, omb2, eps, decay, step, inv_bc2s;
};

// One element of AdamW (torch.optim.AdamW semantics, R1), fp32 storage.
__device__ __forceinline__ void adamw1(float g, float& th, float& m, float& v,
                                       const AdamScalars& s) {
  const float t1 = th * s.decay;                          // theta * (1 - lr*wd)
  const float m1 = fmaf(s.b1, m, s.omb1 * g);             // b1*m + (1-b1)*g
  const float v1 = fmaf(s.b2, v, (s.omb2 * g) * g);       // b2*v + (1-b2)*g^2
  const float den = fmaf(__fsqrt_rn(v1), s.inv_bc2s, s.eps);  // sqrt(v)/sqrt(bc2) + eps
  th = fmaf(-s.step, __fdiv_rn(m1, den), t1);             // - lr/bc1 * m/den
  m = m1;
  v = v1;
}

template <bool UPDATE>
__device__ __forceinline__ double tile_body_full(const Seg& sg, int64_t base, const AdamScalars& s) {
  // thread -> element map: e(u) = base + (u*kThreads + tid)*4, u = 0..kUnroll-1
  const int64_t e0 = base + (int64_t)threadIdx.x * kVec;
  constexpr int64_t kStride = (int64_t)kThreads * kVec;
  float4 g4[kUnroll], t4[kUnroll], m4[kUnroll], v4[kUnroll];
#pragma unroll
  for (int u = 0; u < kUnroll; ++u)
    g4[u] = __ldcs(reinterpret_cast<const float4*>(sg.g + e0 + u * kStride));
  if (UPDATE) {
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      t4[u] = __ldcs(reinterpret_cast<const float4*>(sg.theta + e0 + u * kStride));
      m4[u] = __ldcs(reinterpret_cast<const float4*>(sg.m + e0 + u * kStride));
      v4[u] = __ldcs(reinterpret_cast<const float4*>(sg.v + e0 + u * kStride));
    }
  }
  double acc = 0.0;
#pragma unroll
  for (int u = 0; u < kUnroll; ++u) {
    acc = fma((double)g4[u].x, (double)g4[u].x, acc);
    acc = fma((double)g4[u].y, (double)g4[u].y, acc);
    acc = fma((double)g4[u].z, (double)g4[u].z, acc);
    acc = fma((double)g4[u].w, (double)g4[u].w, acc);
  }
  if (UPDATE) {
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      adamw1(g4[u].x, t4[u].x, m4[u].x, v4[u].x, s);
      adamw1(g4[u].y, t4[u].y, m4[u].y, v4[u].y, s);
      adamw1(g4[u].z, t4[u].z, m4[u].z, v4[u].z, s);
      adamw1(g4[u].w, t4[u].w, m4[u].w, v4[u].w, s);
    }
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      __stcs(reinterpret_cast<float4*>(sg.theta + e0 + u * kStride), t4[u]);
      __stcs(reinterpret_cast<float4*>(sg.m + e0 + u * kStride), m4[u]);
      __stcs(reinterpret_cast<float4*>(sg.v + e0 + u * kStride), v4[u]);
    }
  }
  return acc;
}

// Ragged last tile: same element map and accumulation order, scalar and
// bounds-checked.
template <bool UPDATE>
__device__ __forceinline__ double tile_body_tail(const Seg& sg, int64_t base, const AdamScalars& s) {
  double acc = 0.0;
  for (int u = 0; u < kUnroll; ++u) {
    const int64_t e = base + ((int64_t)u * kThreads + threadIdx.x) * kVec;
#pragma unroll
    for (int j = 0; j < kVec; ++j) {
      const int64_t i = e + j;
      if (i < sg.n) {
        const float g = sg.g[i];
        acc = fma((double)g, (double)g, acc);
        if (UPDATE) {
          float th = sg.theta[i], m = sg.m[i], v = sg.v[i];
          adamw1(g, th, m, v, s);
          sg.theta[i] = th;
          sg.m[i] = m;
          sg.v[i] = v;
        }
      }
    }
  }
  return acc;
}

// K3: the last block to finish a layer sums its tile partials in a fixed order.
__device__ void finalize_layer(const Seg& sg, const DevState& st, int32_t mode, double* red) {
  __threadfence();
  const double* P = st.partials + sg.part_layer_base;
  double a = 0.0;
  for (int i = threadIdx.x; i < sg.layer_tiles; i += kThreads) a += __ldcg(P + i);
  __syncthreads();  // red[] reuse
  const double ss = block_sum(a, red);
  if (threadIdx.x == 0) {
    st.last_ss[sg.layer] = ss;
    if (mode == kFinalizeMgn) {
      if (isfinite(ss)) {
        st.S[sg.layer] += sqrt(ss / (double)sg.layer_numel);  // Eq. 2 inner term
        st.c[sg.layer] += 1;
      } else {
        atomicMin(st.flag, sg.layer);
      }
    } else {
      st.shard_ss[sg.out_slot] = ss;
    }
    st.counters[sg.layer] = 0u;  // ready for the next step
  }
}

template <bool UPDATE>
__global__ void __launch_bounds__(kThreads)
grass_fused_kernel(const __grid_constant__ Batch b, const DevState st) {
  __shared__ double red[kThreads / 32];
  __shared__ int last;
  const int total = b.tile_prefix[b.nseg];
  int s = 0;
  for (int t = blockIdx.x; t < total; t += gridDim.x) {
    while (t >= b.tile_prefix[s + 1]) ++s;
    const Seg& sg = b.seg[s];
    AdamScalars sc;
    sc.b1 = b.beta1; sc.omb1 = b.one_minus_beta1; sc.b2 = b.beta2; sc.omb2 = b.one_minus_beta2;
    sc.eps = b.eps; sc.decay = sg.decay; sc.step = sg.step_size; sc.inv_bc2s = sg.inv_bc2_sqrt;
    const int lt = t - b.tile_prefix[s];
    const int64_t base = (int64_t)lt * kTile;
    const double acc = (base + kTile <= sg.n) ? tile_body_full<UPDATE>(sg, base, sc)
                                              : tile_body_tail<UPDATE>(sg, base, sc);
    const double part = block_sum(acc, red);
    if (threadIdx.x == 0) {
      st.partials[sg.part_index + lt] = part;
      __threadfence();
      const unsigned prev = atomicAdd(st.counters + sg.layer, 1u);
      last = (prev == (unsigned)sg.layer_tiles - 1u);
    }
    __syncthreads();
    if (last) finalize_layer(sg, st, b.mode, red);
    __syncthreads();
  }
}

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
    atomicMin(st.flag, l);
  }
}

}  // namespace

cudaError_t launch_fused(bool update, const Batch& b, const DevState& st, int grid,
                         cudaStream_t s) {
  const int total = b.tile_prefix[b.nseg];
  if (total <= 0) return cudaSuccess;
  if (grid > total) grid = total;
  if (update)
    grass_fused_kernel<true><<<grid, kThreads, 0, s>>>(b, st);
  else
    grass_fused_kernel<false><<<grid, kThreads, 0, s>>>(b, st);
  return cudaGetLastError();
}

cudaError_t launch_rank_sum(const double* gathered, const RankSumArgs& a, const DevState& st,
                            cudaStream_t s) {
  if (a.n <= 0) return cudaSuccess;
  grass_rank_sum_kernel<<<1, 64, 0, s>>>(gathered, a, st);
  return cudaGetLastError();
}

// Persistent grid: every SM holds as many blocks as fit (results never depend
// on this number — see kTile in grass_internal.h).
int fused_grid(bool update, int device) {
  int sms = 0, per_sm = 0;
  if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device) != cudaSuccess) return 0;
  cudaError_t e = update ? cudaOccupancyMaxActiveBlocksPerMultiprocessor(
                               &per_sm, grass_fused_kernel<true>, kThreads, 0)
                         : cudaOccupancyMaxActiveBlocksPerMultiprocessor(
                               &per_sm, grass_fused_kernel<false>, kThreads, 0);
  if (e != cudaSuccess || per_sm < 1) per_sm = 1;
  return sms * per_sm;
}

}  // namespace grass
