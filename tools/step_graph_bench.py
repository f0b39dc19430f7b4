"""Per-step time of the tiny decoder (examples/tiny_decoder_grass.py) trained
through GrassBlocks — eager, with the library update captured per period
(graphs=True), and with the whole step captured (step_graphs=True).  A small
model is launch-bound, so this is where capture pays.

    python tools/step_graph_bench.py      # on the GPU box; prints JSON
"""
import importlib.util
import json
import os
import sys

import torch
import torch.nn as nn

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2604_07808_b200 as G  # noqa: E402

spec = importlib.util.spec_from_file_location("tiny", os.path.join(ROOT, "examples", "tiny_decoder_grass.py"))
tiny = importlib.util.module_from_spec(spec)
spec.loader.exec_module(tiny)


def run(mode, dtype, steps=60, T_p=5, timed=40):
    torch.manual_seed(0)
    model = tiny.TinyDecoder().to(device="cuda", dtype=dtype)
    gb = G.GrassBlocks(model.blocks, always=[[model.emb.weight, model.pos, *model.head.parameters()]],
                       gamma=2, T_p=T_p, T_s=1000, T_u=1000, seed=0, graphs=mode == "update_graph",
                       step_graphs=mode == "step_graph")
    data = (torch.cumsum(torch.randint(-2, 3, (64, 65), generator=torch.Generator().manual_seed(0)), 1) % 256).cuda()

    def loss_fn():
        logits = model(data[:, :-1])
        return nn.functional.cross_entropy(logits.float().reshape(-1, 256), data[:, 1:].reshape(-1))

    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for step in range(steps):
        if step == steps - timed:
            torch.cuda.synchronize()
            e0.record()
        loss = gb.train_step(step, loss_fn, 1e-3)
    e1.record()
    torch.cuda.synchronize()
    return {"mode": mode, "dtype": str(dtype).split(".")[-1], "step_ms": e0.elapsed_time(e1) / timed,
            "final_loss": float(loss)}


def main():
    out = [run(m, d) for d in (torch.float32, torch.bfloat16) for m in ("eager", "update_graph", "step_graph")]
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
