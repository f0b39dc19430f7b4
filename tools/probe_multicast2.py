"""Probe of CUDA multicast (NVLS) support on the GPU box through cuda-python:
cuMulticastCreate with each handle type (profiles/r01_multicast_probe*.json;
DESIGN §13 explains why the fused kernel uses plain peer memory instead)."""
import json
import torch
try:
    from cuda.bindings import driver as cu
except ImportError:
    from cuda import cuda as cu
torch.cuda.init()
torch.zeros(1, device="cuda")
err, dev = cu.cuDeviceGet(0)
out = {}
H = cu.CUmemAllocationHandleType
for name in ("CU_MEM_HANDLE_TYPE_NONE", "CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR", "CU_MEM_HANDLE_TYPE_FABRIC"):
    ht = getattr(H, name, None)
    if ht is None:
        out[name] = "n/a"
        continue
    prop = cu.CUmulticastObjectProp()
    prop.numDevices = 1
    prop.size = 32 << 20
    prop.handleTypes = ht
    e, mc = cu.cuMulticastCreate(prop)
    r = {"create": int(e)}
    if e == 0:
        r["add"] = int(cu.cuMulticastAddDevice(mc, dev)[0])
        # physical memory bound to the multicast object
        ap = cu.CUmemAllocationProp()
        ap.type = cu.CUmemAllocationType.CU_MEM_ALLOCATION_TYPE_PINNED
        ap.location.type = cu.CUmemLocationType.CU_MEM_LOCATION_TYPE_DEVICE
        ap.location.id = 0
        ap.requestedHandleTypes = ht
        e2, h = cu.cuMemCreate(32 << 20, ap, 0)
        r["memcreate"] = int(e2)
        if e2 == 0:
            r["bind"] = int(cu.cuMulticastBindMem(mc, 0, h, 0, 32 << 20, 0)[0])
            e3, va = cu.cuMemAddressReserve(32 << 20, 0, 0, 0)
            r["reserve"] = int(e3)
            r["map"] = int(cu.cuMemMap(va, 32 << 20, 0, mc, 0)[0])
            acc = cu.CUmemAccessDesc()
            acc.location.type = cu.CUmemLocationType.CU_MEM_LOCATION_TYPE_DEVICE
            acc.location.id = 0
            acc.flags = cu.CUmemAccess_flags.CU_MEM_ACCESS_FLAGS_PROT_READWRITE
            r["access"] = int(cu.cuMemSetAccess(va, 32 << 20, [acc], 1)[0])
    out[name] = r
print(json.dumps(out, indent=1))
