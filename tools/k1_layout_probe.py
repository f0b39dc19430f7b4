"""Diagnostic: K1 (norm-only stream) vs the read-ceiling diag kernels on the
same bytes, one 8 GiB buffer vs 32 LLaMA-2-7B layer buffers — isolates the
kernel from the buffer layout.  GRASS_LIB_PATH selects a libgrass variant."""
import ctypes as C
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2604_07808_b200 as G  # noqa: E402
from paper_2604_07808_b200 import build as B  # noqa: E402

dev = torch.device("cuda", 0)
lib = C.CDLL(B.DIAG_OUT)
f = lib.grass_diag_read
f.restype = C.c_int
f.argtypes = [C.c_void_p, C.c_ulonglong, C.c_int, C.c_int, C.c_uint, C.c_int, C.c_void_p, C.c_void_p]
sink = torch.zeros(1, dtype=torch.int64, device=dev)
s = torch.cuda.Stream(device=dev)


def timed(fn, reps=5):
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        fn()
        e1.record(s)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return sorted(ts)[len(ts) // 2]


res = {}
n_big = 2 << 30      # 8 GiB of fp32 in ONE buffer
big = torch.full((n_big,), 1e-3, dtype=torch.float32, device=dev)
ctx = G.Grass([n_big], gamma=1)
ms = timed(lambda: ctx.mgn_accumulate([0], [big], stream=s))
res["K1 one 8GiB buffer"] = n_big * 4 / ms / 1e6
ms = timed(lambda: f(big.data_ptr(), n_big * 4 - (n_big * 4) % (96 << 10), 2, 148, 96 << 10, 2, sink.data_ptr(), s.cuda_stream))
res["diag proto 96KiBx2 one buffer"] = n_big * 4 / ms / 1e6
ctx.close()
del big
torch.cuda.empty_cache()
n, NL = 202_383_360, 32
bufs = [torch.full((n,), 1e-3, dtype=torch.float32, device=dev) for _ in range(NL)]
ctx = G.Grass([n] * NL, gamma=2)
ms = timed(lambda: ctx.mgn_accumulate(list(range(NL)), bufs, stream=s))
res["K1 32 layer buffers"] = n * NL * 4 / ms / 1e6
unit = 96 << 10
nb = n * 4 - (n * 4) % unit


def diag32():
    for b in bufs:
        f(b.data_ptr(), nb, 2, 148, unit, 2, sink.data_ptr(), s.cuda_stream)


ms = timed(diag32)
res["diag proto 96KiBx2 over the 32 layer buffers (32 launches)"] = nb * NL / ms / 1e6
ms = timed(lambda: ctx.mgn_accumulate([0], bufs[:1], stream=s))
res["K1 one layer buffer (810 MB)"] = n * 4 / ms / 1e6
print(json.dumps({k: round(v, 1) for k, v in res.items()}, indent=1))
