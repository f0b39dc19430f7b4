// zero_copy.cu — measurement only: SM-driven host-link traffic (zero copy
// over PCIe from / to pinned, device-mapped host memory) next to the copy
// engines, the question being whether the offload pipeline (row a6,
// PAPER.md:147-148) could move m / v faster from the SMs than through
// cudaMemcpyAsync on the two copy streams it uses now.
//
// grass_diag_zc(src, dst, bytes, grid, stream): `grid` CTAs x 512 threads
// copy `bytes` from src to dst with 128-bit loads / stores, 8 independent
// loads in flight per thread (grid-stride).  Either pointer may be a pinned
// host pointer (translated with cudaHostGetDevicePointer) or device memory.
#include <cuda_runtime.h>

#include <cstdint>

namespace {

__global__ void __launch_bounds__(512) zc_copy(const uint4* __restrict__ src, uint4* __restrict__ dst, size_t n16) {
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + 7 * stride < n16; i += 8 * stride) {
    uint4 v[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) v[j] = __ldcv(src + i + j * stride);
#pragma unroll
    for (int j = 0; j < 8; ++j) __stcs(dst + i + j * stride, v[j]);
  }
  for (; i < n16; i += stride) __stcs(dst + i, __ldcv(src + i));
}

void* device_view(void* p) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) return nullptr;
  if (a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged) return p;
  void* d = nullptr;
  if (cudaHostGetDevicePointer(&d, p, 0) != cudaSuccess) return nullptr;
  return d;
}

}  // namespace

extern "C" int grass_diag_zc(void* src, void* dst, unsigned long long bytes, int grid, void* stream) {
  if (!src || !dst || grid < 1 || bytes % 16 != 0) return (int)cudaErrorInvalidValue;
  void* s = device_view(src);
  void* d = device_view(dst);
  if (!s || !d) {
    cudaGetLastError();
    return (int)cudaErrorInvalidHostPointer;
  }
  zc_copy<<<grid, 512, 0, static_cast<cudaStream_t>(stream)>>>(static_cast<const uint4*>(s), static_cast<uint4*>(d),
                                                              (size_t)bytes / 16);
  return (int)cudaGetLastError();
}
