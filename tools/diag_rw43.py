"""K2's HBM mix (4 reads + 3 writes per element, 28 B) with plain per-thread
loads / streaming stores (paper_2604_07808_b200/diag, grass_diag_rw43) over
the bench's configs[1] element count, grid x unroll sweep: the mixed
read/write ceiling next to K2.  -> stdout JSON"""
import ctypes as C
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2604_07808_b200 import build as B  # noqa: E402

lib = C.CDLL(B.DIAG_OUT)
f = lib.grass_diag_rw43
f.restype = C.c_int
f.argtypes = [C.POINTER(C.c_void_p), C.c_ulonglong, C.c_int, C.c_int, C.c_void_p]
dev = torch.device("cuda", 0)
n = 2 * 202_383_360
bufs = [torch.randn(n, device=dev) * 1e-3 for _ in range(4)]
ptrs = (C.c_void_p * 4)(*[b.data_ptr() for b in bufs])
s = torch.cuda.Stream(device=dev)
sms = torch.cuda.get_device_properties(dev).multi_processor_count
res = {}
for u in (1, 2, 4):
    for k in (1, 2, 4, 8):
        ts = []
        for _ in range(5):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            assert f(ptrs, n, u, sms * k, s.cuda_stream) == 0
            e1.record(s)
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        ms = sorted(ts)[2]
        res[f"unroll={u} grid={sms * k}"] = {"ms": round(ms, 4), "GBps": round(28 * n / ms / 1e6, 1)}
        print(f"unroll={u} grid={sms*k}", res[f"unroll={u} grid={sms * k}"], flush=True)
print(json.dumps(res))
