"""Timeline of one offloaded 7B step (gamma = 2), overlapped vs vanilla
(the paper's Fig. 4, measured), and of a period-residency swap, from the
library's own trace events.  Writes gpurun_out/offload_timeline.json."""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2604_07808_b200 as G  # noqa: E402
from synth import MODELS, layer_grad, layer_params  # noqa: E402

n = MODELS["llama2-7b"].layer_numel
dev = "cuda:0"
params = [layer_params(n, l, device=dev) for l in range(4)]
grads = [layer_grad(n, l, 1e-4, device=dev) for l in range(4)]
s = torch.cuda.Stream()


def lanes(tr):
    t0 = min(e["start_ms"] for e in tr)
    t1 = max(e["end_ms"] for e in tr)
    span = t1 - t0
    out = {"makespan_ms": span}
    for k in ("h2d", "update", "d2h"):
        iv = sorted((e["start_ms"], e["end_ms"]) for e in tr if e["kind"] == k)
        busy, cur = 0.0, None
        for a, b in iv:
            if cur is None or a > cur[1]:
                if cur:
                    busy += cur[1] - cur[0]
                cur = [a, b]
            else:
                cur[1] = max(cur[1], b)
        if cur:
            busy += cur[1] - cur[0]
        out[f"{k}_busy_frac"] = busy / span if span else 0.0
        out[f"{k}_ops"] = len(iv)
    return out


res = {}
for name, kw in (("overlapped", {"overlap": True}), ("vanilla", {"overlap": False}),
                 ("period", {"residency": G.RESIDENCY_PERIOD})):
    gr = G.Grass([n] * 4, gamma=2, offload=True, **kw)
    gr.step_layers([0, 1], params[:2], grads[:2], 3e-5, stream=s)
    torch.cuda.synchronize()
    gr.trace_enable(True)
    gr.step_layers([2, 3], params[2:], grads[2:], 3e-5, stream=s)   # period: swaps both
    tr = gr.trace_read()
    res[name] = {"summary": lanes(tr),
                 "events": [{k: (round(v, 4) if isinstance(v, float) else v) for k, v in e.items()} for e in tr]}
    print(name, res[name]["summary"], flush=True)
    gr.close()
os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
json.dump(res, open(os.path.join(ROOT, "gpurun_out", "offload_timeline.json"), "w"), indent=1)
