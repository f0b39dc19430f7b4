"""Does this box support CUDA multicast (NVLS) objects, even with one GPU?"""
import json, os
import torch
out = {}
try:
    from cuda.bindings import driver as cu
except ImportError:
    from cuda import cuda as cu
torch.cuda.init()
err, dev = cu.cuDeviceGet(0)
for name in ("CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED", "CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_FABRIC_SUPPORTED"):
    attr = getattr(cu.CUdevice_attribute, name, None)
    if attr is not None:
        e, v = cu.cuDeviceGetAttribute(attr, dev)
        out[name] = (int(e), int(v))
try:
    prop = cu.CUmulticastObjectProp()
    prop.numDevices = 1
    prop.size = 2 << 20
    prop.handleTypes = cu.CUmemAllocationHandleType.CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR
    e, gran = cu.cuMulticastGetGranularity(prop, cu.CUmulticastGranularity_flags.CU_MULTICAST_GRANULARITY_RECOMMENDED)
    out["granularity"] = (int(e), int(gran) if e == 0 else None)
    e, mc = cu.cuMulticastCreate(prop)
    out["cuMulticastCreate"] = int(e)
    if e == 0:
        e = cu.cuMulticastAddDevice(mc, dev)
        out["cuMulticastAddDevice"] = int(e)
except Exception as ex:
    out["exception"] = repr(ex)
try:
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT="29533")
    dist.init_process_group("nccl", rank=0, world_size=1)
    import torch.distributed._symmetric_memory as symm
    t = symm.empty(1 << 20, device="cuda")
    h = symm.rendezvous(t, dist.group.WORLD)
    out["symm_multicast_ptr"] = int(getattr(h, "multicast_ptr", 0) or 0)
    out["symm_world"] = h.world_size
except Exception as ex:
    out["symm_exception"] = repr(ex)[:300]
print(json.dumps(out, indent=1))
