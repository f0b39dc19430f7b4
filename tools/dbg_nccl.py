"""Reproducer (raw NCCL through ctypes, no libgrass): on NCCL 2.28.9 a 1-rank
ncclReduceScatter(ncclAvg, fp32) drops the last 16 elements for counts = 16
(mod 64) from ~300 K elements up, while ncclSum is correct — why libgrass
reduce-scatters with ncclSum and scales by 1/W in the kernel."""
import ctypes as C, torch
nccl = C.CDLL("libnccl.so.2")
class UID(C.Structure):
    _fields_ = [("internal", C.c_char * 128)]
uid = UID()
print("getid", nccl.ncclGetUniqueId(C.byref(uid)))
comm = C.c_void_p()
print("init", nccl.ncclCommInitRank(C.byref(comm), 1, uid, 0))
nccl.ncclReduceScatter.argtypes = [C.c_void_p, C.c_void_p, C.c_size_t, C.c_int, C.c_int, C.c_void_p, C.c_void_p]
nccl.ncclAllGather.argtypes = [C.c_void_p, C.c_void_p, C.c_size_t, C.c_int, C.c_void_p, C.c_void_p]
s = torch.cuda.Stream()
for n in (304144, 304128, 304160, 4112, 1040, 16, 1 << 20 | 16, 202383360 // 8 + 16):
    for op, name in ((4, "avg"), (0, "sum")):
        x = torch.randn(n, device="cuda")
        y = torch.zeros(n, device="cuda")
        torch.cuda.synchronize()
        r = nccl.ncclReduceScatter(x.data_ptr(), y.data_ptr(), n, 7, op, comm, s.cuda_stream)
        torch.cuda.synchronize()
        bad = (x != y).nonzero()
        print(f"RS {name} n={n} rc={r} mismatches={bad.numel()} first={int(bad[0]) if bad.numel() else -1}")
    x = torch.randn(n, device="cuda"); y = torch.zeros(n, device="cuda")
    r = nccl.ncclAllGather(x.data_ptr(), y.data_ptr(), n, 7, comm, s.cuda_stream); torch.cuda.synchronize()
    print(f"AG n={n} rc={r} mismatches={(x != y).sum().item()}")
