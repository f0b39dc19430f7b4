"""HBM speed-of-light for different read/write mixes on this B200, using torch
library kernels (plumbing, not the product): the ceiling a 4-read/3-write
stream can expect, and torch's own fused AdamW on the same 7B-layer shapes."""
import json
import torch

dev = "cuda:0"
N = 202_383_360 * 2
def t(fn, reps=10):
    s, e = torch.cuda.Event(True), torch.cuda.Event(True)
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(reps):
        s.record(); fn(); e.record(); torch.cuda.synchronize()
        best = min(best, s.elapsed_time(e) / 1e3)
    return best
a, b, c, d = (torch.randn(N, device=dev) for _ in range(4))
out = {}
out["copy_1R1W_GBs"] = 8 * N / t(lambda: b.copy_(a)) / 1e9
out["add_2R1W_GBs"] = 12 * N / t(lambda: torch.add(a, b, out=c)) / 1e9
out["addcmul_3R1W_GBs"] = 16 * N / t(lambda: a.addcmul_(b, c, value=1e-9)) / 1e9
out["sum_1R_GBs"] = 4 * N / t(lambda: a.sum()) / 1e9
ps = [a[:N // 2], a[N // 2:]]
gs = [b[:N // 2], b[N // 2:]]
ms = [c[:N // 2].zero_(), c[N // 2:].zero_()]
vs = [d[:N // 2].zero_(), d[N // 2:].zero_()]
steps = [torch.tensor(1.0, device=dev), torch.tensor(1.0, device=dev)]
def fused():
    torch._fused_adamw_(ps, gs, ms, vs, [], steps, lr=3e-5, beta1=0.9, beta2=0.999, weight_decay=0.0,
                        eps=1e-8, amsgrad=False, maximize=False)
tt = t(fused)
out["torch_fused_adamw_ms"] = tt * 1e3
out["torch_fused_adamw_GBs_28B"] = 28 * N / tt / 1e9
print(json.dumps(out, indent=1))
json.dump(out, open("gpurun_out/hbm_mix.json", "w"), indent=1)
