"""Host-link traffic from the SMs (zero copy over PCIe, diag/zero_copy.cu)
next to the copy engines, one direction and duplex: is the copy-engine duplex
rate the offload pipeline is measured against (row a6) the link's ceiling?
CUDA events on the launching streams, 1 GiB per direction, best of 3.
-> stdout JSON"""
import ctypes as C
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2604_07808_b200 import build as B  # noqa: E402

B.build_diag()
lib = C.CDLL(B.DIAG_OUT)
zc = lib.grass_diag_zc
zc.restype = C.c_int
zc.argtypes = [C.c_void_p, C.c_void_p, C.c_ulonglong, C.c_int, C.c_void_p]
dev = torch.device("cuda", 0)
torch.cuda.set_device(dev)
n = 1 << 28                                           # fp32 elements: 1 GiB per buffer
nb = n * 4
h_src = torch.ones(n, dtype=torch.float32).pin_memory()
h_dst = torch.zeros(n, dtype=torch.float32).pin_memory()
d_src = torch.full((n,), 2.0, device=dev)
d_dst = torch.zeros(n, device=dev)
sa, sb = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
sms = torch.cuda.get_device_properties(dev).multi_processor_count
res = {}


def timed(key, legs):
    """legs: [(stream, fn)] launched together; GB/s per direction = nb / max time."""
    best = None
    for _ in range(3):
        torch.cuda.synchronize()
        ev = []
        for s, fn in legs:
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            fn(s)
            e1.record(s)
            ev.append((e0, e1))
        torch.cuda.synchronize()
        t = max(a.elapsed_time(b) for a, b in ev) / 1e3
        best = t if best is None else min(best, t)
    res[key] = {"ms": round(best * 1e3, 3), "GBps_per_dir": round(nb / best / 1e9, 2)}
    print(key, res[key], flush=True)


def ce(dst, src):
    def f(s):
        with torch.cuda.stream(s):
            dst.copy_(src, non_blocking=True)
    return f


def k(dst, src, grid):
    def f(s):
        assert zc(src.data_ptr(), dst.data_ptr(), nb, grid, s.cuda_stream) == 0
    return f


timed("ce h2d", [(sa, ce(d_dst, h_src))])
timed("ce d2h", [(sb, ce(h_dst, d_src))])
timed("ce duplex", [(sa, ce(d_dst, h_src)), (sb, ce(h_dst, d_src))])
for grid in (8, 16, 32, 74, 148, 296):
    timed(f"zc h2d grid={grid}", [(sa, k(d_dst, h_src, grid))])
    timed(f"zc d2h grid={grid}", [(sb, k(h_dst, d_src, grid))])
    timed(f"zc duplex grid={grid}+{grid}", [(sa, k(d_dst, h_src, grid)), (sb, k(h_dst, d_src, grid))])
for grid in (16, 74):
    timed(f"mixed: zc h2d grid={grid} + ce d2h", [(sa, k(d_dst, h_src, grid)), (sb, ce(h_dst, d_src))])
    timed(f"mixed: ce h2d + zc d2h grid={grid}", [(sa, ce(d_dst, h_src)), (sb, k(h_dst, d_src, grid))])
torch.cuda.synchronize()
assert torch.all(d_dst == 1.0) and torch.all(h_dst == 2.0)    # the copies moved the data
best = {d: max((v["GBps_per_dir"], kk) for kk, v in res.items() if d in kk) for d in ("h2d", "d2h", "duplex")}
res["best"] = {d: {"GBps_per_dir": v[0], "what": v[1]} for d, v in best.items()}
print(json.dumps(res))
