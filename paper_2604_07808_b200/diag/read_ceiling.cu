// read_ceiling.cu — measurement only (bench.py `probe` leg), not part of the
// hot path: the READ-ONLY HBM ceiling of this B200, the denominator of the
// probing kernel K1 (a pure read, 4 or 2 B/param), which the
// 1R1W copy peak of MEASURED_PEAKS.json does not bound.
//
// Two hand-written streaming reads of one buffer, each with a trivial
// accumulate that keeps every load alive:
//   mode 0  LDG.128: ld.global.nc.L1::no_allocate.v4, 8 independent loads in
//           flight per thread, grid-stride, `grid` CTAs x 512 threads;
//   mode 1  TMA bulk: one CTA per SM (`grid` CTAs), one producer thread
//           streams `unit`-byte pieces HBM -> shared memory with
//           cp.async.bulk into a ring of `stages` slots (mbarrier complete_tx),
//           one consumer warp reads one word per slot and hands it back —
//           K1's data movement with no arithmetic;
//   mode 2/3 K1's consumer protocol (16 warps, per-warp release, mode 3: a
//           named barrier per unit) on the same ring — diagnostics.
// C ABI: grass_diag_read(ptr, bytes, mode, grid, unit, stages, sink, stream);
// and the 4-read / 3-write mixes of K2: grass_diag_rw43 (LDG/STG) and
// grass_diag_rw43_tma (K2's TMA ring, no arithmetic).
#include <cuda_runtime.h>

#include <cstdint>

namespace {

__device__ __forceinline__ uint4 ld_stream(const uint4* p) {
  uint4 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p));
  return v;
}

__global__ void __launch_bounds__(512) read_ldg(const uint4* __restrict__ p, size_t n16,
                                                unsigned long long* sink) {
  uint32_t acc = 0;
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + 7 * stride < n16; i += 8 * stride) {
    uint4 v[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) v[j] = ld_stream(p + i + j * stride);
#pragma unroll
    for (int j = 0; j < 8; ++j) acc ^= v[j].x ^ v[j].y ^ v[j].z ^ v[j].w;
  }
  for (; i < n16; i += stride) {
    const uint4 v = ld_stream(p + i);
    acc ^= v.x ^ v.y ^ v.z ^ v.w;
  }
  if (acc == 0x9E3779B9u) atomicAdd(sink, 1ull);
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__global__ void __launch_bounds__(64, 1) read_tma(const char* __restrict__ p, size_t bytes, uint32_t unit,
                                                  int stages, unsigned long long* sink) {
  extern __shared__ __align__(1024) char ring[];
  __shared__ __align__(8) uint64_t full[16], empty[16];
  const int tid = threadIdx.x;
  if (tid == 0) {
    for (int s = 0; s < stages; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&full[s])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&empty[s])));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const size_t units = bytes / unit;  // (the caller passes a multiple of unit)
  if (tid == 0) {  // producer
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    int k = 0;
    for (size_t u = blockIdx.x; u < units; u += gridDim.x, ++k) {
      const int s = k % stages;
      if (k >= stages) {
        const uint32_t par = ((k / stages) & 1) ^ 1;
        asm volatile("{\n.reg .pred q;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 q, [%0], %1;\n@!q bra W_%=;\n}\n" ::"r"(
                         smem_u32(&empty[s])),
                     "r"(par)
                     : "memory");
      }
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&full[s])), "r"(unit)
                   : "memory");
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
              smem_u32(ring + (size_t)s * unit)),
          "l"(p + u * unit), "r"(unit), "r"(smem_u32(&full[s])), "l"(pol)
          : "memory");
    }
  } else if (tid == 32) {  // consumer: one word per slot, then hand it back
    uint32_t acc = 0;
    int k = 0;
    for (size_t u = blockIdx.x; u < units; u += gridDim.x, ++k) {
      const int s = k % stages;
      const uint32_t par = (k / stages) & 1;
      asm volatile("{\n.reg .pred q;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 q, [%0], %1;\n@!q bra W_%=;\n}\n" ::"r"(
                       smem_u32(&full[s])),
                   "r"(par)
                   : "memory");
      acc ^= *reinterpret_cast<const volatile uint32_t*>(ring + (size_t)s * unit + (k & 255) * 4);
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&empty[s])) : "memory");
    }
    if (acc == 0x9E3779B9u) atomicAdd(sink, 1ull);
  }
}

// mode 2 / 3: K1's protocol with no arithmetic — 16 consumer warps all wait
// on the full barrier, each warp hands the slot back (empty barrier count 16),
// and (mode 3) the consumers meet at a named barrier once per unit, as K1's
// per-unit tile-partial reduction does.
template <bool BAR>
__global__ void __launch_bounds__(544, 1) read_k1proto(const char* __restrict__ p, size_t bytes, uint32_t unit,
                                                       int stages, unsigned long long* sink) {
  extern __shared__ __align__(1024) char ring[];
  __shared__ __align__(8) uint64_t full[16], empty[16];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    for (int s = 0; s < stages; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&full[s])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 16;" ::"r"(smem_u32(&empty[s])));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const size_t units = bytes / unit;
  if (warp == 16) {
    if (lane == 0) {
      uint64_t pol;
      asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
      int k = 0;
      for (size_t u = blockIdx.x; u < units; u += gridDim.x, ++k) {
        const int s = k % stages;
        if (k >= stages) {
          const uint32_t par = ((k / stages) & 1) ^ 1;
          asm volatile("{\n.reg .pred q;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 q, [%0], %1;\n@!q bra W_%=;\n}\n" ::"r"(
                           smem_u32(&empty[s])),
                       "r"(par)
                       : "memory");
        }
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&full[s])), "r"(unit)
                     : "memory");
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
                smem_u32(ring + (size_t)s * unit)),
            "l"(p + u * unit), "r"(unit), "r"(smem_u32(&full[s])), "l"(pol)
            : "memory");
      }
    }
    return;
  }
  uint32_t acc = 0;
  int k = 0;
  for (size_t u = blockIdx.x; u < units; u += gridDim.x, ++k) {
    const int s = k % stages;
    const uint32_t par = (k / stages) & 1;
    asm volatile("{\n.reg .pred q;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 q, [%0], %1;\n@!q bra W_%=;\n}\n" ::"r"(
                     smem_u32(&full[s])),
                 "r"(par)
                 : "memory");
    acc ^= *reinterpret_cast<const volatile uint32_t*>(ring + (size_t)s * unit + tid * 4);
    __syncwarp();
    if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&empty[s])) : "memory");
    if (BAR) asm volatile("bar.sync 1, 512;" ::: "memory");
  }
  if (acc == 0x9E3779B9u) atomicAdd(sink, 1ull);
}

// 4-read / 3-write elementwise stream (K2's HBM mix: g, theta, m, v in;
// theta, m, v out) with plain per-thread 128-bit loads and streaming stores,
// U float4 of each array in flight per thread: the mixed read/write ceiling
// K2's TMA ring is compared with.
template <int U>
__global__ void __launch_bounds__(512) rw43(const float4* __restrict__ g, float4* __restrict__ th,
                                           float4* __restrict__ m, float4* __restrict__ v, size_t n4) {
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + (U - 1) * stride < n4; i += U * stride) {
    float4 a[U], b[U], c[U], d[U];
#pragma unroll
    for (int k = 0; k < U; ++k) {
      a[k] = __ldcs(g + i + k * stride);
      b[k] = __ldcs(th + i + k * stride);
      c[k] = __ldcs(m + i + k * stride);
      d[k] = __ldcs(v + i + k * stride);
    }
#pragma unroll
    for (int k = 0; k < U; ++k) {
      b[k].x += a[k].x; b[k].y += a[k].y; b[k].z += a[k].z; b[k].w += a[k].w;
      c[k].x += a[k].y; d[k].x += a[k].z;
      __stcs(th + i + k * stride, b[k]);
      __stcs(m + i + k * stride, c[k]);
      __stcs(v + i + k * stride, d[k]);
    }
  }
  for (; i < n4; i += stride) {
    float4 a = __ldcs(g + i), b = __ldcs(th + i);
    b.x += a.x;
    __stcs(th + i, b);
    __stcs(m + i, __ldcs(m + i));
    __stcs(v + i, __ldcs(v + i));
  }
}

// K2's data movement with no arithmetic: one CTA per SM, a ring of `stages`
// slots each holding one unit of `elems` fp32 of g, theta, m, v (16 B/elem in
// shared memory).  Thread 0 streams the four pieces HBM -> smem with
// cp.async.bulk (mbarrier complete_tx); thread 32 waits for the slot and
// bulk-stores theta, m, v back smem -> HBM (cp.async.bulk.global.shared::cta,
// one bulk group per unit) and hands the slot back once the stores of the
// PREVIOUS unit have finished reading shared memory.  The 4R3W TMA ceiling
// K2 (the same ring plus the Eq. 2 / AdamW arithmetic) is compared with.
// BF16 = true: K2's bf16 mode instead (R18: bf16 gradient and parameter,
// fp32 master + m + v): g is bf16 (2 B, read), th / m / v are the fp32
// master, m, v (read and written), and the bf16 parameter copy `p16` is
// written (2 B, from the gradient's slot) — 14 B read + 14 B written per
// element, the same 28 B as the fp32 mix in another read / write split.
template <bool BF16>
__global__ void __launch_bounds__(64, 1) rw43_tma(const float* __restrict__ g, float* __restrict__ th,
                                                  float* __restrict__ m, float* __restrict__ v,
                                                  uint16_t* __restrict__ p16, size_t n, uint32_t elems,
                                                  int stages) {
  extern __shared__ __align__(1024) char ring[];
  __shared__ __align__(8) uint64_t full[16], empty[16];
  const int tid = threadIdx.x;
  const uint32_t piece = elems * 4u;
  const uint32_t gpiece = BF16 ? elems * 2u : piece;
  if (tid == 0) {
    for (int s = 0; s < stages; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&full[s])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&empty[s])));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const size_t units = n / elems;
  if (tid == 0) {  // loads
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    int k = 0;
    for (size_t u = blockIdx.x; u < units; u += gridDim.x, ++k) {
      const int s = k % stages;
      if (k >= stages) {
        const uint32_t par = ((k / stages) & 1) ^ 1;
        asm volatile("{\n.reg .pred q;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 q, [%0], %1;\n@!q bra W_%=;\n}\n" ::"r"(
                         smem_u32(&empty[s])),
                     "r"(par)
                     : "memory");
      }
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&full[s])),
                   "r"(3 * piece + gpiece)
                   : "memory");
      const char* src[4] = {reinterpret_cast<const char*>(g) + u * gpiece, reinterpret_cast<const char*>(th + u * elems),
                            reinterpret_cast<const char*>(m + u * elems), reinterpret_cast<const char*>(v + u * elems)};
#pragma unroll
      for (int a = 0; a < 4; ++a)
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
                smem_u32(ring + ((size_t)s * 4 + a) * piece)),
            "l"(src[a]), "r"(a == 0 ? gpiece : piece), "r"(smem_u32(&full[s])), "l"(pol)
            : "memory");
    }
  } else if (tid == 32) {  // stores
    int k = 0;
    float* dst[3] = {th, m, v};
    for (size_t u = blockIdx.x; u < units; u += gridDim.x, ++k) {
      const int s = k % stages;
      const uint32_t par = (k / stages) & 1;
      asm volatile("{\n.reg .pred q;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 q, [%0], %1;\n@!q bra W_%=;\n}\n" ::"r"(
                       smem_u32(&full[s])),
                   "r"(par)
                   : "memory");
#pragma unroll
      for (int a = 0; a < 3; ++a)
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst[a] + u * elems),
                     "r"(smem_u32(ring + ((size_t)s * 4 + 1 + a) * piece)), "r"(piece)
                     : "memory");
      if (BF16)  // the bf16 parameter copy, from the gradient's slot
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(p16 + u * elems),
                     "r"(smem_u32(ring + (size_t)s * 4 * piece)), "r"(gpiece)
                     : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      if (k >= 1) {  // unit k-1's stores have read their slot
        asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&empty[(k - 1) % stages])) : "memory");
      }
    }
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
}

}  // namespace

extern "C" int grass_diag_rw43(void* const* bufs, unsigned long long n, int unroll, int grid, void* stream) {
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const float4* g = static_cast<const float4*>(bufs[0]);
  float4* th = static_cast<float4*>(bufs[1]);
  float4* m = static_cast<float4*>(bufs[2]);
  float4* v = static_cast<float4*>(bufs[3]);
  const size_t n4 = (size_t)n / 4;
  if (unroll == 1) rw43<1><<<grid, 512, 0, s>>>(g, th, m, v, n4);
  else if (unroll == 2) rw43<2><<<grid, 512, 0, s>>>(g, th, m, v, n4);
  else rw43<4><<<grid, 512, 0, s>>>(g, th, m, v, n4);
  return (int)cudaGetLastError();
}

// bufs: g, theta (master), m, v [, p16 when bf16]; bf16: g is bf16 (n x 2 B)
extern "C" int grass_diag_rw43_tma(void* const* bufs, unsigned long long n, unsigned int elems, int stages,
                                   int grid, int bf16, void* stream) {
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (!bufs || grid < 1 || elems == 0 || elems % 8 != 0 || n % elems != 0 || stages < 2 || stages > 16 ||
      (size_t)elems * 16 * stages > 227u * 1024u)
    return (int)cudaErrorInvalidValue;
  const size_t smem = (size_t)elems * 16 * stages;
  auto kern = bf16 ? rw43_tma<true> : rw43_tma<false>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return (int)e;
  kern<<<grid, 64, smem, s>>>(static_cast<const float*>(bufs[0]), static_cast<float*>(bufs[1]),
                              static_cast<float*>(bufs[2]), static_cast<float*>(bufs[3]),
                              bf16 ? static_cast<uint16_t*>(bufs[4]) : nullptr, (size_t)n, elems, stages);
  return (int)cudaGetLastError();
}

extern "C" int grass_diag_read(const void* ptr, unsigned long long bytes, int mode, int grid, unsigned int unit,
                               int stages, unsigned long long* sink, void* stream) {
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (!ptr || !sink || grid < 1 || reinterpret_cast<uintptr_t>(ptr) % 16 != 0) return (int)cudaErrorInvalidValue;
  if (mode == 0) {
    read_ldg<<<grid, 512, 0, s>>>(static_cast<const uint4*>(ptr), (size_t)bytes / 16, sink);
  } else if (mode >= 2) {
    if (unit % 16 != 0 || stages < 1 || stages > 16 || (size_t)unit * stages > 227u * 1024u || bytes % unit != 0)
      return (int)cudaErrorInvalidValue;
    const size_t smem = (size_t)unit * stages;
    auto kern = mode == 2 ? read_k1proto<false> : read_k1proto<true>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return (int)e;
    kern<<<grid, 544, smem, s>>>(static_cast<const char*>(ptr), (size_t)bytes, unit, stages, sink);
  } else {
    if (unit % 16 != 0 || stages < 1 || stages > 16 || (size_t)unit * stages > 227u * 1024u ||
        bytes % unit != 0)
      return (int)cudaErrorInvalidValue;
    const size_t smem = (size_t)unit * stages;
    cudaError_t e = cudaFuncSetAttribute(read_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return (int)e;
    read_tma<<<grid, 64, smem, s>>>(static_cast<const char*>(ptr), (size_t)bytes, unit, stages, sink);
  }
  return (int)cudaGetLastError();
}
