// stream_kernel.cuh — K1 / K2: the persistent, warp-specialised streaming
// kernel (included by kernels.cu inside its anonymous namespace; uses the
// helpers defined there).
//
// Template parameters
//   UPDATE  false: K1, Eq. 2 squared norm only (probing)
//           true:  K2, fused Eq. 2 norm + AdamW (R1/R2)
//   TPS     tiles per ring stage ("unit")
//   STAGES  depth of the shared-memory ring
//   BF16    false: fp32 theta and g (28 B/param for K2, 4 B/param for K1)
//           true:  bf16 model parameters and gradients with an fp32 master
//                  copy and fp32 moments: K2 reads g
//                  (2 B), master (4 B; on a layer's first update the bf16
//                  parameter, 2 B, instead), m, v (4 B each) and writes master,
//                  m, v (4 B each) and the bf16 parameter RNE(master') (2 B):
//                  28 B/param; K1 reads 2 B/param.
//   P2P     true: data-parallel step with the gradient summed in the kernel
//           (R20): the producer bulk-copies every rank's gradient slice of the
//           unit into a gradient ring and the consumers add them in ascending
//           rank order in fp32.  GRASS_DP_P2P (Batch::ntpeer = W, SURVEY 8(f)
//           f2): the slices are read straight from the peers' HBM (NVLink) and
//           theta' is bulk-stored into every rank's parameter buffer — the
//           gradient reduction, the update and the all-gather in one kernel,
//           tile by tile.  GRASS_DP_NCCL (ntpeer = 0): the slices are the
//           local copies the NCCL exchange received; theta' goes to this
//           rank's buffer (then ncclAllGather).  Each rank updates only its
//           own element shard.
//
// Stage layout (bytes, every region 16-byte aligned):
//   [g: kUnit*GB][theta/master: kUnit*4][m: kUnit*4][v: kUnit*4][bf16 theta: kUnit*2 (BF16)]
// The bulk copies move the largest prefix of a unit whose narrowest array is a
// multiple of 16 bytes (4 elements fp32, 8 elements bf16); the 0-7 element
// tail of a segment is read and written directly in HBM by the consumers.

template <bool UPDATE, bool BF16, int TPS>
struct StageLayout {
  static constexpr int kUnit = TPS * (int)kTile;
  static constexpr int GB = BF16 ? 2 : 4;
  static constexpr int off_g = 0;
  static constexpr int off_t = kUnit * GB;
  static constexpr int off_m = off_t + kUnit * 4;
  static constexpr int off_v = off_m + kUnit * 4;
  static constexpr bool SEP = UPDATE && kSepOut;
  // in place: the bf16 parameters (read when the master is initialised, and
  // written) get their own slot; separate output: the bf16 input is read from
  // the (then unused) fp32 theta slot and the outputs follow the inputs
  static constexpr int off_tb = SEP ? off_t : off_v + kUnit * 4;  // bf16 theta input
  static constexpr int in_bytes = UPDATE ? off_v + kUnit * 4 + ((BF16 && !SEP) ? kUnit * 2 : 0) : kUnit * GB;
  static constexpr int o_t = SEP ? in_bytes : off_t;  // outputs theta', m', v', bf16 theta'
  static constexpr int o_m = SEP ? o_t + kUnit * 4 : off_m;
  static constexpr int o_v = SEP ? o_m + kUnit * 4 : off_v;
  static constexpr int o_tb = SEP ? o_v + kUnit * 4 : off_tb;
  static constexpr int bytes = SEP ? o_tb + (BF16 ? kUnit * 2 : 0) : in_bytes;
  static constexpr int vec = BF16 ? 8 : 4;
};

__device__ __forceinline__ float bf2f(uint32_t b) { return __uint_as_float(b << 16); }
__device__ __forceinline__ uint32_t f2bf(float f) {
  return (uint32_t)__bfloat16_as_ushort(__float2bfloat16_rn(f));
}
__device__ __forceinline__ float4 unpack_bf16x4(uint2 u) {
  return make_float4(bf2f(u.x & 0xffffu), bf2f(u.x >> 16), bf2f(u.y & 0xffffu), bf2f(u.y >> 16));
}
__device__ __forceinline__ uint2 pack_bf16x4(float4 f) {
  return make_uint2(f2bf(f.x) | (f2bf(f.y) << 16), f2bf(f.z) | (f2bf(f.w) << 16));
}
__device__ __forceinline__ float4 scale4(float4 v, float s) {
  return make_float4(v.x * s, v.y * s, v.z * s, v.w * s);
}
// 4 gradient values at (unit-relative) element e of a stage
template <bool BF16>
__device__ __forceinline__ float4 stage_g4(const char* stg, int e) {
  if (BF16) return unpack_bf16x4(*reinterpret_cast<const uint2*>(stg + 2 * e));
  return *reinterpret_cast<const float4*>(stg + 4 * e);
}
// Element (relative to the unit) of consumer thread `tid`'s vector q in tile
// k — the fixed map of the norm decomposition (grass_internal.h).
__device__ __forceinline__ int tile_elem(int k, int q, int tid) {
  return k * (int)kTile + (q * kThreads + tid) * kVec;
}
template <bool BF16>
__device__ __forceinline__ float seg_g(const Seg& sg, int64_t idx) {
  return BF16 ? bf2f(sg.g16[idx]) : sg.g[idx];
}

#ifndef GRASS_K1_DRAIN  // diagnostic only (wrong norms): K1 consumers hand every full unit back
#define GRASS_K1_DRAIN 0  // untouched — the ring's own speed (the K3 finding)
#endif

// Eq. 2: the value of one consumer thread in one tile — the sum of the squares
// of its kUnroll x 4 gradient values g[q].{x,y,z,w} (elements (q*kThreads +
// t)*4 + j; an element beyond a ragged end is 0 and adds nothing).
//  * fp32 gradients: every square is exact in fp64; acc_j = fma chains over q,
//    value (acc_0 + acc_1) + (acc_2 + acc_3).
//  * bf16 gradients: a bf16 value has 8 significant bits, so its square is
//    exact in fp32; the 8 squares are summed in fp32 in element order (one FMUL
//    + 7 FFMA: at most 7 roundings of a sum of non-negative terms, <= 7 * 2^-24
//    = 4.2e-7 relative, inside the 1e-6 bar) and widened ONCE — one conversion
//    per 8 elements instead of per element, which held the 2 B/param probe
//    above its no-math time (profiles/r01_variants_bf16_*).  Integer-valued
//    gradients stay exact while the sum is < 2^24.  The fp32 chain is only
//    used where it cannot underflow or overflow: a sum below 2^-100
//    (squares of magnitude < 2^-134 lose bits as fp32 subnormals, and < 2^-150
//    vanish) or above FLT_MAX (|g| > ~1.8e19) — and a NaN — takes the exact
//    fp64 squares instead, so the bound holds for every finite gradient and a
//    non-finite one still yields a non-finite norm.
#ifndef GRASS_BF16_GUARD  // A/B only: 0 = no exact fallback (wrong for tiny / huge gradients)
#define GRASS_BF16_GUARD 1
#endif
template <bool BF16>
__device__ __forceinline__ double tile_value_exact(const float4 (&g)[kUnroll]) {
  double a = 0.0;
#pragma unroll
  for (int q = 0; q < kUnroll; ++q) {
    a = fma((double)g[q].x, (double)g[q].x, a);
    a = fma((double)g[q].y, (double)g[q].y, a);
    a = fma((double)g[q].z, (double)g[q].z, a);
    a = fma((double)g[q].w, (double)g[q].w, a);
  }
  return a;
}
// A bf16 8-square fp32 sum is used where it is in [2^-100, FLT_MAX] (see
// above): one unsigned compare of the bits (false for 0, inf, NaN).
__device__ __forceinline__ bool sq_sum_in_range(float s) {
  return __float_as_uint(s) - 0x0D800000u <= 0x7F7FFFFFu - 0x0D800000u;
}
// The same fp32 chain straight from the packed bf16 words of a thread's two
// 4-element vectors (element order x.lo, x.hi, y.lo, y.hi): FHFMA.BF16 — the
// mixed-precision fma, bf16 operands taken as register halves, fp32
// accumulate — computes RN(x*x + s) with the exact product, i.e. the bits of
// __fmaf_rn on the widened values, with no unpack instructions.
__device__ __forceinline__ float bf16_sq_acc(uint32_t w, float s) {
  unsigned short lo, hi;
  asm("mov.b32 {%0, %1}, %2;" : "=h"(lo), "=h"(hi) : "r"(w));
  asm("fma.rn.f32.bf16 %0, %1, %1, %0;" : "+f"(s) : "h"(lo));
  asm("fma.rn.f32.bf16 %0, %1, %1, %0;" : "+f"(s) : "h"(hi));
  return s;
}
__device__ __forceinline__ float bf16_sq8(uint2 a, uint2 b) {
  float s = 0.f;
  s = bf16_sq_acc(a.x, s);
  s = bf16_sq_acc(a.y, s);
  s = bf16_sq_acc(b.x, s);
  return bf16_sq_acc(b.y, s);
}
template <bool BF16>
__device__ __forceinline__ double tile_value(const float4 (&g)[kUnroll]) {
  if (BF16) {
    float s = __fmul_rn(g[0].x, g[0].x);
    s = __fmaf_rn(g[0].y, g[0].y, s);
    s = __fmaf_rn(g[0].z, g[0].z, s);
    s = __fmaf_rn(g[0].w, g[0].w, s);
#pragma unroll
    for (int q = 1; q < kUnroll; ++q) {
      s = __fmaf_rn(g[q].x, g[q].x, s);
      s = __fmaf_rn(g[q].y, g[q].y, s);
      s = __fmaf_rn(g[q].z, g[q].z, s);
      const float w = g[q].w;
      s = __fmaf_rn(w, w, s);
    }
    if (!GRASS_BF16_GUARD || sq_sum_in_range(s)) return (double)s;
    return tile_value_exact<BF16>(g);
  }
  double acc[kVec] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
  for (int q = 0; q < kUnroll; ++q) {
    acc[0] = fma((double)g[q].x, (double)g[q].x, acc[0]);
    acc[1] = fma((double)g[q].y, (double)g[q].y, acc[1]);
    acc[2] = fma((double)g[q].z, (double)g[q].z, acc[2]);
    acc[3] = fma((double)g[q].w, (double)g[q].w, acc[3]);
  }
  return (acc[0] + acc[1]) + (acc[2] + acc[3]);
}

// P2P (Seg::gpeer): the gradient of a unit is the sum of the npeer ranks'
// slices in ascending rank order (fp32).  The producer bulk-copies each rank's
// slice (over NVLink for the peers) into a ring of P2PGSlots gradient slots;
// the consumers add the slices up in registers.  The 0-7 element tail of a
// segment is summed straight from the ranks' memory (peer_g1).
template <bool UPDATE, bool BF16>
struct P2PGSlots {
  // update (one-tile units): 64 KiB of slots next to the 2-stage theta/m/v
  // ring; norm only: the stage ring is unused (nothing but gradients is read)
  // and the slots take 192 KiB
  __host__ __device__ static constexpr int slots(int slot_bytes) { return UPDATE ? 65536 / slot_bytes : 196608 / slot_bytes; }
  static constexpr bool kNoStageRing = !UPDATE;  // (P2P) the stage ring holds no data
};
template <bool BF16>
__device__ __forceinline__ float peer_g1(const void* const* gp, int npeer, int64_t idx) {
  float a = 0.f;
#pragma unroll
  for (int q = 0; q < kMaxPeers; ++q) {
    if (q >= npeer) break;
    const float x = BF16 ? bf2f(static_cast<const uint16_t*>(gp[q])[idx]) : static_cast<const float*>(gp[q])[idx];
    a = q == 0 ? x : a + x;
  }
  return a;
}

// Bulk-stores the results of one unit from its stage: master/theta, m, v
// (and the bf16 parameter copy).  ntp > 0 (P2P): theta' (fp32) or the bf16
// copy goes to every rank's parameter buffer (this rank's included) over
// NVLink; ntp = 0: to this rank's buffers only.
template <bool BF16, class L>
__device__ __forceinline__ void store_unit_t(const Seg& sg, int ntp, int64_t e0, uint32_t nv, const char* stg) {
  if (nv) {
    if (BF16 || ntp == 0) bulk_store(sg.theta + e0, stg + L::o_t, nv * 4u);
    bulk_store(sg.m + e0, stg + L::o_m, nv * 4u);
    bulk_store(sg.v + e0, stg + L::o_v, nv * 4u);
    for (int q = 0; q < ntp; ++q) {
      char* dst = static_cast<char*>(sg.tpeer[q]) + (sg.poff + e0) * (BF16 ? 2 : 4);
      bulk_store(dst, stg + (BF16 ? L::o_tb : L::o_t), nv * (BF16 ? 2u : 4u));
    }
    if (BF16 && ntp == 0) bulk_store(sg.theta16 + e0, stg + L::o_tb, nv * 2u);
    bulk_commit();
  }
}

// Unit order of a CTA: rounds of kUB consecutive units per CTA (kUB = 1: unit
// b, b + grid, b + 2 grid, ...).  Any order gives the same results.
#ifndef GRASS_UNIT_BLOCK
#define GRASS_UNIT_BLOCK 1
#endif
constexpr int kUB = GRASS_UNIT_BLOCK;
__device__ __forceinline__ int unit_of(int i, int ub) {
  return (i / ub) * ((int)gridDim.x * ub) + (int)blockIdx.x * ub + (i % ub);
}

template <bool UPDATE, int TPS, int STAGES, bool BF16, bool P2P, bool DEVB = false>
__global__ void __launch_bounds__(kStreamThreads, 1)
grass_stream_kernel(const __grid_constant__ Batch b, const DevState st) {
  using L = StageLayout<UPDATE, BF16, TPS>;
  constexpr int kUnit = L::kUnit;
  extern __shared__ __align__(1024) char sbuf[];  // [STAGES][L::bytes]
  __shared__ __align__(8) uint64_t full_bar[STAGES];
  __shared__ __align__(8) uint64_t empty_bar[STAGES];
  __shared__ __align__(8) uint64_t outfree_bar[STAGES];  // L::SEP: output region writable
  constexpr int kGSlot = kUnit * L::GB;  // one rank's slice of a unit
  constexpr int NG = P2P ? P2PGSlots<UPDATE, BF16>::slots(kGSlot) : 1;  // P2P gradient ring
  static_assert(!P2P || !UPDATE || TPS == 1, "P2P update units are one tile");
  __shared__ __align__(8) uint64_t gfull_bar[NG];
  __shared__ __align__(8) uint64_t gempty_bar[NG];
  // P2P norm-only: the stage ring carries nothing, so it is not synchronised at
  // all and the producer runs ahead as far as the gradient ring allows
  constexpr bool kRing = !(P2P && P2PGSlots<UPDATE, BF16>::kNoStageRing);
  char* const gring = sbuf + (kRing ? (size_t)STAGES * L::bytes : 0);
  __shared__ int unit_prefix[kMaxSeg + 1];
  __shared__ double red[2][TPS][kConsumerWarps];
  // DEVB (device-resident schedule): this launch's segments, built from the
  // layer ids in device memory — the sampled set is never seen by the host
  __shared__ __align__(16) Seg dsegs[DEVB ? kMaxDevSeg : 1];
  __shared__ int dids[DEVB ? kMaxDevSeg : 1];
  __shared__ int dn;
  // ... and their AdamW scalars and bf16 master-initialisation flags (the
  // step prologue's arithmetic, per CTA; K3 advances t_l after this launch)
  __shared__ float dscal[DEVB ? kMaxDevSeg : 1][3];
  __shared__ int dinit[DEVB ? kMaxDevSeg : 1];

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (DEVB) {
    grid_dependency_wait();  // PDL: the previous step's K3 (ids, t_l, window) is complete and visible
    if (tid == 0) {  // ids ascending (R12), insertion sort of <= kMaxDevSeg entries
      const int n = b.dev_n < kMaxDevSeg ? b.dev_n : kMaxDevSeg;
      for (int j = 0; j < n; ++j) {
        const int x = b.dev_ids[j];
        int k = j;
        for (; k > 0 && dids[k - 1] > x; --k) dids[k] = dids[k - 1];
        dids[k] = x;
      }
      dn = n;
    }
    __syncthreads();
    constexpr int kWords = (int)(sizeof(Seg) / 8);
    static_assert(sizeof(Seg) % 8 == 0, "Seg copied in 8-byte words");
    for (int w = tid; w < dn * kWords; w += blockDim.x)
      reinterpret_cast<unsigned long long*>(dsegs)[w] =
          reinterpret_cast<const unsigned long long*>(b.dev_table + dids[w / kWords])[w % kWords];
    if (UPDATE && tid < dn) {  // as grass_step_prologue_kernel, for t = t_l + 1
      const int l = dids[tid];
      const long long t = st.t[l] + 1;
      const double lr = b.dev_lr_ptr ? (double)*b.dev_lr_ptr : (double)b.dev_lr;
      const double bc1 = 1.0 - pow(b.dev_beta1, (double)t);
      const double bc2 = 1.0 - pow(b.dev_beta2, (double)t);
      dscal[tid][0] = (float)(1.0 - lr * b.dev_wd);
      dscal[tid][1] = (float)(lr / bc1);
      dscal[tid][2] = (float)(1.0 / sqrt(bc2));
      dinit[tid] = BF16 && !st.mvalid[l] ? 1 : 0;
    }
    __syncthreads();
  }
  const Seg* const segs = DEVB ? dsegs : b.seg;
  const int nseg = DEVB ? dn : b.nseg;
  if (tid == 0) {
    unit_prefix[0] = 0;
    for (int s = 0; s < nseg; ++s) {
      unit_prefix[s + 1] = unit_prefix[s] + (segs[s].tiles + TPS - 1) / TPS;
    }
    for (int i = 0; i < STAGES; ++i) {
      mbar_init(&full_bar[i], 1);
      mbar_init(&empty_bar[i], kConsumerWarps);
      mbar_init(&outfree_bar[i], 1);
    }
    for (int i = 0; i < NG; ++i) {
      mbar_init(&gfull_bar[i], 1);
      mbar_init(&gempty_bar[i], kConsumerWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int total = unit_prefix[nseg];

  if (warp == kConsumerWarps) {
    // ------------------------------ producer ------------------------------
    if (lane == 0) {
      const uint64_t pol = l2_load_policy<UPDATE>();
      constexpr bool TS = UPDATE && kTmaStore;
      // TMA-store mode: the unit each stage last held (its results go out first)
      int pend_s[STAGES];
      int64_t pend_e0[STAGES];
      uint32_t pend_nv[STAGES];
      int s = 0, i = 0, gcount = 0;
      for (int u = unit_of(0, kUB); u < total; ++i, u = unit_of(i, kUB)) {
        const int stage = i % STAGES;
        char* stg = sbuf + (size_t)stage * L::bytes;
        if (kRing && i >= STAGES) {
          mbar_wait(&empty_bar[stage], ((i / STAGES) & 1) ^ 1);
          if (TS) {
            store_unit_t<BF16, L>(segs[pend_s[stage]], P2P ? b.ntpeer : 0, pend_e0[stage], pend_nv[stage], stg);
            if (!L::SEP) bulk_wait_read_all();  // stage reusable again
          }
        }
        while (u >= unit_prefix[s + 1]) ++s;
        const Seg& sg = segs[s];
        const int64_t e0 = (int64_t)(u - unit_prefix[s]) * kUnit;
        const int64_t ne = min((int64_t)kUnit, sg.n - e0);
        const uint32_t nv = (uint32_t)(ne & ~(int64_t)(L::vec - 1));
        if (TS) {
          pend_s[stage] = s;
          pend_e0[stage] = e0;
          pend_nv[stage] = nv;
        }
        if (nv && (UPDATE || !P2P)) {
          const bool init = BF16 && UPDATE && (DEVB ? dinit[s] : st.init_now[sg.layer]);
          // P2P: the gradient slices go to the gradient ring (below)
          const uint32_t tx = (P2P ? 0u : nv * (uint32_t)L::GB) + (UPDATE ? nv * (init ? 2u : 4u) + 8u * nv : 0u);
          mbar_arrive_expect_tx(&full_bar[stage], tx);
          if (!P2P)
            bulk_load(stg + L::off_g, BF16 ? (const void*)(sg.g16 + e0) : (const void*)(sg.g + e0),
                      nv * (uint32_t)L::GB, &full_bar[stage], pol);
          if (UPDATE) {
            if (init)
              bulk_load(stg + L::off_tb, sg.theta16 + e0, nv * 2u, &full_bar[stage], pol);
            else
              bulk_load(stg + L::off_t, sg.theta + e0, nv * 4u, &full_bar[stage], pol);
            bulk_load(stg + L::off_m, sg.m + e0, nv * 4u, &full_bar[stage], pol);
            bulk_load(stg + L::off_v, sg.v + e0, nv * 4u, &full_bar[stage], pol);
          }
        } else if (kRing) {
          mbar_arrive(&full_bar[stage]);
        }
        constexpr int kPf = P2P ? 0 : (UPDATE ? GRASS_L2_PREFETCH_UPD : GRASS_L2_PREFETCH_NORM);
        if (kPf > 0) {  // warm L2 with this CTA's unit kPf rounds ahead (same segment only)
          const int uf = u + kPf * (int)gridDim.x;
          if (uf < total && uf < unit_prefix[s + 1]) {
            const int64_t f0 = (int64_t)(uf - unit_prefix[s]) * kUnit;
            const uint32_t fn = (uint32_t)(min((int64_t)kUnit, sg.n - f0) & ~(int64_t)(L::vec - 1));
            if (fn) {
              bulk_prefetch_l2(BF16 ? (const void*)(sg.g16 + f0) : (const void*)(sg.g + f0), fn * (uint32_t)L::GB);
              if (UPDATE) {
                bulk_prefetch_l2(sg.theta + f0, fn * 4u);
                bulk_prefetch_l2(sg.m + f0, fn * 4u);
                bulk_prefetch_l2(sg.v + f0, fn * 4u);
              }
            }
          }
        }
        if (P2P && nv) {  // every rank's gradient slice of this unit, in rank order
          for (int r = 0; r < b.npeer; ++r, ++gcount) {
            const int gsl = gcount % NG;
            if (gcount >= NG) mbar_wait(&gempty_bar[gsl], ((gcount / NG) & 1) ^ 1);
            mbar_arrive_expect_tx(&gfull_bar[gsl], nv * (uint32_t)L::GB);
            bulk_load(gring + (size_t)gsl * kGSlot,
                      static_cast<const char*>(sg.gpeer[r]) + (sg.gpoff + e0) * L::GB, nv * (uint32_t)L::GB,
                      &gfull_bar[gsl], pol);
          }
        }
        if (L::SEP) {  // loads are in flight; now let the stores of unit i - STAGES finish reading
          if (i >= STAGES) bulk_wait_read_all();
          mbar_arrive(&outfree_bar[stage]);
        }
      }
      if (TS) {  // drain: results of the last (up to STAGES) units
        const int n_units = i;
        for (int j = (n_units > STAGES ? n_units - STAGES : 0); j < n_units; ++j) {
          const int stage = j % STAGES;
          mbar_wait(&empty_bar[stage], (j / STAGES) & 1);
          store_unit_t<BF16, L>(segs[pend_s[stage]], P2P ? b.ntpeer : 0, pend_e0[stage], pend_nv[stage],
                                sbuf + (size_t)stage * L::bytes);
        }
        bulk_wait_all();
      }
      if (P2P && b.ntpeer > 0) {  // the peer writes are complete; order them before the end barrier's signal
        asm volatile("fence.proxy.async.global;" ::: "memory");
        __threadfence_system();
      }
    }
    return;
  }

  // ------------------------------ consumers -------------------------------
  const float cf = (UPDATE && b.coef) ? *b.coef : 1.0f;
  const float gs = b.gscale;  // DP: 1/world turns the summed gradients into averages
  const int ntp = P2P ? b.ntpeer : 0;  // ranks whose parameter buffers receive theta' (P2P)
  int s = 0, i = 0, gcount = 0;
  for (int u = unit_of(0, kUB); u < total; ++i, u = unit_of(i, kUB)) {
    const int stage = i % STAGES;
    while (u >= unit_prefix[s + 1]) ++s;
    const Seg& sg = segs[s];
    AdamScalars sc;
    sc.b1 = b.beta1; sc.omb1 = b.one_minus_beta1; sc.b2 = b.beta2; sc.omb2 = b.one_minus_beta2;
    sc.eps = b.eps;
    if (UPDATE) {  // this step's AdamW scalars of the layer (step prologue)
      sc.decay = DEVB ? dscal[s][0] : st.scal[3 * sg.layer];
      sc.step = DEVB ? dscal[s][1] : st.scal[3 * sg.layer + 1];
      sc.inv_bc2s = DEVB ? dscal[s][2] : st.scal[3 * sg.layer + 2];
    }
    sc.cf = cf;
    const bool init = BF16 && UPDATE && (DEVB ? dinit[s] : st.init_now[sg.layer]);
    const int ui = u - unit_prefix[s];
    const int64_t e0 = (int64_t)ui * kUnit;
    const int ne = (int)min((int64_t)kUnit, sg.n - e0);
    const int nv = ne & ~(L::vec - 1);  // bulk-copied prefix; the tail is read from HBM
    const int ntiles = (ne + (int)kTile - 1) / (int)kTile;
    char* stg = sbuf + (size_t)stage * L::bytes;
    const int64_t pe0 = P2P ? sg.poff + e0 : 0;  // full-layer index of the unit's element 0
    if (kRing) mbar_wait(&full_bar[stage], (i / STAGES) & 1);
    if (L::SEP) mbar_wait(&outfree_bar[stage], (i / STAGES) & 1);
    // full norm-only units: the TPS tiles form groups of GS (a power of two);
    // slot t of this lane holds tile perm(t) = (t / GS) * GS + ((t % GS) ^ pm)
    // — the order in which warp_sum_perm keeps them (pm = the tile of each
    // group the lane ends with)
    constexpr int GS = kPermGroup<TPS>;
    using MS = MultiSlots<GS>;
    const int pm = (!UPDATE && ne == kUnit) ? (lane >> MS::SHIFT) & (GS - 1) : 0;
    auto perm = [&](int t) { return (t / GS) * GS + ((t % GS) ^ pm); };
    float4 gacc[P2P ? TPS : 1][kUnroll];  // P2P: this thread's summed gradient of the unit
    if (P2P && nv) {
      for (int r = 0; r < b.npeer; ++r, ++gcount) {
        const int gsl = gcount % NG;
        mbar_wait(&gfull_bar[gsl], (gcount / NG) & 1);
#pragma unroll
        for (int k0 = 0; k0 < (P2P ? TPS : 1); ++k0) {
          const int k = perm(k0);  // gacc[k0] holds tile k
#pragma unroll
          for (int q = 0; q < kUnroll; ++q) {
            const int e = tile_elem(k, q, tid);
            if (e < nv) {
              const float4 x = stage_g4<BF16>(gring + (size_t)gsl * kGSlot, e);
              if (r == 0) {
                gacc[k0][q] = x;
              } else {
                gacc[k0][q].x += x.x; gacc[k0][q].y += x.y; gacc[k0][q].z += x.z; gacc[k0][q].w += x.w;
              }
            }
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&gempty_bar[gsl]);
      }
    }
    bool released = false;  // this warp has handed the stage back already
    if (GRASS_K1_DRAIN && !UPDATE && !P2P && ne == kUnit) {  // A/B only: the ring without any consumer work
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty_bar[stage]);
      released = true;
      if (lane < TPS) red[i & 1][lane][warp] = 0.0;
    } else if (!UPDATE && ne == kUnit) {
      // Full unit of the norm-only stream: each lane reads (or, P2P, summed)
      // its tiles in the order warp_sum_perm keeps them (slot t = tile
      // perm(t)), so the all-tiles reduction needs no selects.  Same element
      // map and tile values as the guarded path below.
      double w[TPS];
      bool done = false;
      if constexpr (BF16 && !P2P) {
        if (gs == 1.f) {
          // bf16 fast path: the unit's data to registers, the 8-square fp32
          // sums with FHFMA.BF16 straight from the packed words; if every sum
          // of the warp is in fp32's normal range (it always is outside
          // pathological gradients), the stage is handed back at once — the
          // producer refills it while the widening and the reduction run —
          // else the generic path below (exact fallback) re-reads the stage.
          uint2 raw[TPS][kUnroll];
#pragma unroll
          for (int t = 0; t < TPS; ++t)
#pragma unroll
            for (int q = 0; q < kUnroll; ++q)
              raw[t][q] = *reinterpret_cast<const uint2*>(stg + L::off_g + 2 * tile_elem(perm(t), q, tid));
          float s8[TPS];
          uint32_t lo = 0xffffffffu, hi = 0u;
#pragma unroll
          for (int t = 0; t < TPS; ++t) {
            s8[t] = bf16_sq8(raw[t][0], raw[t][1]);
            lo = min(lo, __float_as_uint(s8[t]));
            hi = max(hi, __float_as_uint(s8[t]));
          }
          const bool ok = !GRASS_BF16_GUARD || (sq_sum_in_range(__uint_as_float(lo)) && sq_sum_in_range(__uint_as_float(hi)));
          if (__all_sync(0xffffffffu, ok)) {
            if (lane == 0) mbar_arrive(&empty_bar[stage]);
            released = true;
#pragma unroll
            for (int t = 0; t < TPS; ++t) w[t] = (double)s8[t];
            done = true;
          }
        }
      }
      if (!done) {
#pragma unroll
        for (int t = 0; t < TPS; ++t) {
          float4 g4[kUnroll];
#pragma unroll
          for (int q = 0; q < kUnroll; ++q) {
            if constexpr (P2P) g4[q] = gacc[t][q];
            else g4[q] = stage_g4<BF16>(stg + L::off_g, tile_elem(perm(t), q, tid));
          }
          if (gs != 1.f) {  // DP average (warp-uniform; x * 1 == x, so skipping it is exact)
#pragma unroll
            for (int q = 0; q < kUnroll; ++q) g4[q] = scale4(g4[q], gs);
          }
          w[t] = tile_value<BF16>(g4);
        }
      }
#pragma unroll
      for (int g = 0; g < TPS / GS; ++g) {  // all tiles of each group at once (bit-identical to warp_sum)
        double wg[GS];
#pragma unroll
        for (int j = 0; j < GS; ++j) wg[j] = w[g * GS + j];
        int slot;
        const double tsum = warp_sum_perm<GS>(wg, lane, &slot);
        if (slot >= 0) red[i & 1][g * GS + slot][warp] = tsum;
      }
    } else {
#pragma unroll
      for (int k = 0; k < TPS; ++k) {
        if (k < ntiles) {
          float4 gq[kUnroll];  // this thread's gradient values of the tile (0 beyond a ragged end)
#pragma unroll
          for (int q = 0; q < kUnroll; ++q) {
            gq[q] = make_float4(0.f, 0.f, 0.f, 0.f);
            const int e = tile_elem(k, q, tid);  // relative to e0
            if (e < nv) {
              const float4 g4 = scale4(P2P ? gacc[P2P ? k : 0][q] : stage_g4<BF16>(stg + L::off_g, e), gs);
              gq[q] = g4;
              if (UPDATE) {
                float4 t4 = init ? unpack_bf16x4(*reinterpret_cast<const uint2*>(stg + L::off_tb + 2 * e))
                                 : *reinterpret_cast<const float4*>(stg + L::off_t + 4 * e);
                float4 m4 = *reinterpret_cast<const float4*>(stg + L::off_m + 4 * e);
                float4 v4 = *reinterpret_cast<const float4*>(stg + L::off_v + 4 * e);
                adamw1(g4.x, t4.x, m4.x, v4.x, sc);
                adamw1(g4.y, t4.y, m4.y, v4.y, sc);
                adamw1(g4.z, t4.z, m4.z, v4.z, sc);
                adamw1(g4.w, t4.w, m4.w, v4.w, sc);
                if (kTmaStore) {  // results back into the stage; the producer bulk-stores them
                  *reinterpret_cast<float4*>(stg + L::o_t + 4 * e) = t4;
                  *reinterpret_cast<float4*>(stg + L::o_m + 4 * e) = m4;
                  *reinterpret_cast<float4*>(stg + L::o_v + 4 * e) = v4;
                  if (BF16) *reinterpret_cast<uint2*>(stg + L::o_tb + 2 * e) = pack_bf16x4(t4);
                } else {
                  if (BF16 || ntp == 0) st_stream(sg.theta + e0 + e, t4);
                  st_stream(sg.m + e0 + e, m4);
                  st_stream(sg.v + e0 + e, v4);
#pragma unroll
                  for (int q2 = 0; q2 < kMaxPeers; ++q2) {
                    if (q2 >= ntp) break;
                    if (BF16)
                      *reinterpret_cast<uint2*>(static_cast<uint16_t*>(sg.tpeer[q2]) + pe0 + e) = pack_bf16x4(t4);
                    else
                      st_stream(static_cast<float*>(sg.tpeer[q2]) + pe0 + e, t4);
                  }
                  if (BF16 && ntp == 0) *reinterpret_cast<uint2*>(sg.theta16 + e0 + e) = pack_bf16x4(t4);
                }
              }
            } else if (e < ne) {
              float gt[kVec] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
              for (int j = 0; j < kVec; ++j) {
                if (e + j < ne) {
                  const int64_t idx = e0 + e + j;
                  const float g = (P2P ? peer_g1<BF16>(sg.gpeer, b.npeer, sg.gpoff + e0 + e + j) : seg_g<BF16>(sg, idx)) * gs;
                  gt[j] = g;
                  if (UPDATE) {
                    float th = init ? bf2f(sg.theta16[idx]) : sg.theta[idx];
                    float m = sg.m[idx], v = sg.v[idx];
                    adamw1(g, th, m, v, sc);
                    if (BF16 || ntp == 0) sg.theta[idx] = th;
                    sg.m[idx] = m;
                    sg.v[idx] = v;
#pragma unroll
                    for (int q2 = 0; q2 < kMaxPeers; ++q2) {
                      if (q2 >= ntp) break;
                      if (BF16)
                        static_cast<uint16_t*>(sg.tpeer[q2])[pe0 + e + j] = (uint16_t)f2bf(th);
                      else
                        static_cast<float*>(sg.tpeer[q2])[pe0 + e + j] = th;
                    }
                    if (BF16 && ntp == 0) sg.theta16[idx] = (uint16_t)f2bf(th);
                  }
                }
              }
              gq[q] = make_float4(gt[0], gt[1], gt[2], gt[3]);
            }
          }
          const double t = warp_sum(tile_value<BF16>(gq));
          if (lane == 0) red[i & 1][k][warp] = t;
        }
      }
    }
    if (UPDATE && kTmaStore) fence_proxy_async_smem();  // results visible to the bulk store
    __syncwarp();
    if (kRing && !released && lane == 0) mbar_arrive(&empty_bar[stage]);  // this warp is done with the stage
    consumer_sync();
    if (tid < ntiles) {  // lane k of warp 0 finishes tile k (warp sums in ascending order)
      double p = 0.0;
#pragma unroll
      for (int w = 0; w < kConsumerWarps; ++w) p += red[i & 1][tid][w];
      st.partials[sg.part_index + (int64_t)ui * TPS + tid] = p;
    }
  }
  // (K3, the per-layer sum of the tile partials, is grass_finalize_kernel,
  // launched after this kernel for the layers it completed — in parallel over
  // the layers instead of in whichever CTA finished last)
}
