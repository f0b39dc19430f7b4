// comm.cpp — NCCL over NVLink/NVSwitch for the data-parallel (world > 1) path.
//
// NCCL is resolved at run time with dlopen: the process reuses the libnccl.so.2
// torch already loaded (one NCCL per process), and the library itself loads on
// machines without NCCL or a GPU (the CPU test suite only needs the host ABI).
#include "comm.h"

#include <dlfcn.h>

#include <cuda_runtime.h>

#include <cstdlib>
#include <mutex>
#include <string>

namespace grass {
namespace {

struct NcclApi {
  bool ok = false;
  std::string why;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

NcclApi& api() {
  static NcclApi a;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD | RTLD_GLOBAL);
    if (!h) {
      const char* p = std::getenv("GRASS_NCCL_LIB");
      h = dlopen(p ? p : "libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    }
    if (!h) {
      a.why = std::string("cannot load libnccl.so.2: ") + dlerror();
      return;
    }
#define GRASS_SYM(field, name)                                              \
  a.field = reinterpret_cast<decltype(a.field)>(dlsym(h, name));            \
  if (!a.field) {                                                           \
    a.why = std::string("libnccl.so.2 lacks ") + name;                      \
    return;                                                                 \
  }
    GRASS_SYM(GetUniqueId, "ncclGetUniqueId");
    GRASS_SYM(CommInitRank, "ncclCommInitRank");
    GRASS_SYM(CommDestroy, "ncclCommDestroy");
    GRASS_SYM(Send, "ncclSend");
    GRASS_SYM(Recv, "ncclRecv");
    GRASS_SYM(GroupStart, "ncclGroupStart");
    GRASS_SYM(GroupEnd, "ncclGroupEnd");
    GRASS_SYM(AllGather, "ncclAllGather");
    GRASS_SYM(GetErrorString, "ncclGetErrorString");
#undef GRASS_SYM
    a.ok = true;
  });
  return a;
}

std::string nccl_msg(const char* what, ncclResult_t r) {
  return std::string(what) + ": " + (api().GetErrorString ? api().GetErrorString(r) : "nccl error");
}

}  // namespace

bool nccl_available(std::string* why) {
  if (!api().ok && why) *why = api().why;
  return api().ok;
}

bool nccl_unique_id(void* out, std::string* err) {
  if (!nccl_available(err)) return false;
  ncclUniqueId id;
  ncclResult_t r = api().GetUniqueId(&id);
  if (r != ncclSuccess) {
    *err = nccl_msg("ncclGetUniqueId", r);
    return false;
  }
  static_assert(sizeof(id) == GRASS_NCCL_ID_BYTES, "ncclUniqueId size");
  memcpy(out, &id, sizeof(id));
  return true;
}

bool Comm::init(const void* unique_id, int rank, int world, std::string* err) {
  if (!nccl_available(err)) return false;
  ncclUniqueId id;
  memcpy(&id, unique_id, sizeof(id));
  ncclResult_t r = api().CommInitRank(&comm, world, id, rank);
  if (r != ncclSuccess) {
    *err = nccl_msg("ncclCommInitRank", r);
    comm = nullptr;
    return false;
  }
  this->rank = rank;
  this->world = world;
  return true;
}

void Comm::destroy() {
  if (comm && api().ok) api().CommDestroy(comm);
  comm = nullptr;
}

bool Comm::exchange_slices(const void* send, void* recv, size_t count, size_t stride, bool bf16, cudaStream_t s,
                           std::string* err) {
  const ncclDataType_t dt = bf16 ? ncclBfloat16 : ncclFloat32;
  const size_t esz = bf16 ? 2 : 4;
  // this rank's own slice: a device copy on the same stream (no NCCL
  // self-send: at world 1 the exchange issues no NCCL call at all)
  const cudaError_t ce = cudaMemcpyAsync(static_cast<char*>(recv) + (size_t)rank * stride * esz,
                                         static_cast<const char*>(send) + (size_t)rank * count * esz, count * esz,
                                         cudaMemcpyDeviceToDevice, s);
  if (ce != cudaSuccess) {
    *err = std::string("exchange: own slice copy: ") + cudaGetErrorString(ce);
    return false;
  }
  if (world == 1) return true;
  ncclResult_t r = api().GroupStart();
  if (r != ncclSuccess) {
    *err = nccl_msg("ncclGroupStart", r);
    return false;
  }
  ncclResult_t first = ncclSuccess;
  const char* what = "";
  for (int q = 0; q < world && first == ncclSuccess; ++q) {
    if (q == rank) continue;
    r = api().Send(static_cast<const char*>(send) + (size_t)q * count * esz, count, dt, q, comm, s);
    if (r != ncclSuccess) {
      first = r;
      what = "ncclSend";
      break;
    }
    r = api().Recv(static_cast<char*>(recv) + (size_t)q * stride * esz, count, dt, q, comm, s);
    if (r != ncclSuccess) {
      first = r;
      what = "ncclRecv";
    }
  }
  r = api().GroupEnd();  // always closes the group
  if (first == ncclSuccess && r != ncclSuccess) {
    first = r;
    what = "ncclGroupEnd";
  }
  if (first != ncclSuccess) {
    *err = nccl_msg(what, first);
    return false;
  }
  return true;
}

bool Comm::all_gather(const void* send, void* recv, size_t count, bool bf16, cudaStream_t s,
                      std::string* err) {
  ncclResult_t r = api().AllGather(send, recv, count, bf16 ? ncclBfloat16 : ncclFloat32, comm, s);
  if (r != ncclSuccess) {
    *err = nccl_msg("ncclAllGather", r);
    return false;
  }
  return true;
}

bool Comm::all_gather_f64(const double* send, double* recv, size_t count, cudaStream_t s,
                          std::string* err) {
  ncclResult_t r = api().AllGather(send, recv, count, ncclFloat64, comm, s);
  if (r != ncclSuccess) {
    *err = nccl_msg("ncclAllGather(f64)", r);
    return false;
  }
  return true;
}

}  // namespace grass
