"""Sweep of the read-ceiling diagnostics (paper_2604_07808_b200/diag): plain
TMA ring (mode 1) vs K1's consumer protocol (mode 2, + per-unit named
barrier: mode 3), per unit size / stage count.  -> gpurun_out/diag_read.json"""
import ctypes as C
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2604_07808_b200 import build as B  # noqa: E402

lib = C.CDLL(B.DIAG_OUT)
f = lib.grass_diag_read
f.restype = C.c_int
f.argtypes = [C.c_void_p, C.c_ulonglong, C.c_int, C.c_int, C.c_uint, C.c_int, C.c_void_p, C.c_void_p]
dev = torch.device("cuda", 0)
nbytes = 8 << 30
buf = torch.full((nbytes,), 7, dtype=torch.uint8, device=dev)
sink = torch.zeros(1, dtype=torch.int64, device=dev)
s = torch.cuda.Stream(device=dev)
res = {}
for mode in (1, 2, 3):
    for u, st in ((32, 6), (64, 3), (96, 2), (48, 4)):
        unit = u << 10
        nb = nbytes - nbytes % unit
        best = 0
        for _ in range(3):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            rc = f(buf.data_ptr(), nb, mode, 148, unit, st, sink.data_ptr(), s.cuda_stream)
            e1.record(s)
            torch.cuda.synchronize()
            assert rc == 0, rc
            best = max(best, nb / (e0.elapsed_time(e1) / 1e3) / 1e9)
        res[f"mode{mode} {u}KiBx{st}"] = round(best, 1)
        print(f"mode{mode} {u}KiBx{st}", round(best, 1), flush=True)
os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
json.dump(res, open(os.path.join(ROOT, "gpurun_out", "diag_read.json"), "w"), indent=1)
