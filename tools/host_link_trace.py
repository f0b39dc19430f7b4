"""Independent host-link evidence for row a6 (Fig. 4): the
configs[2] offloaded step (LLaMA-2-7B layers, gamma = 2, m/v in pinned host
memory, per-step round trip through the chunk ring) traced with CUPTI through
torch.profiler (Kineto) — nsys is not installed in this image.  The memcpy
and kernel rows come from CUPTI's activity records, not from the library's own
CUDA events (grass_trace_*).

Summarises per step: HtoD / DtoH bytes, each direction's busy time (union of
its copy intervals), their overlap with each other and with the update kernel,
achieved GB/s per direction over the step, against a measured duplex copy and
the 63 GB/s PCIe Gen5 x16 nominal.  Overlapped and Fig. 4 "vanilla"
(overlap = 0) pipelines.

    python tools/host_link_trace.py          # -> gpurun_out/host_link_cupti.{json,md}
"""
import json
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2604_07808_b200 as G  # noqa: E402
from synth import MODELS, grad_sigmas, layer_grad, layer_params  # noqa: E402


def union(iv):
    iv = sorted(iv)
    out = []
    for a, b in iv:
        if out and a <= out[-1][1]:
            out[-1][1] = max(out[-1][1], b)
        else:
            out.append([a, b])
    return out


def length(iv):
    return sum(b - a for a, b in iv)


def intersect(u, v):
    i = j = 0
    tot = 0.0
    while i < len(u) and j < len(v):
        a, b = max(u[i][0], v[j][0]), min(u[i][1], v[j][1])
        if a < b:
            tot += b - a
        if u[i][1] < v[j][1]:
            i += 1
        else:
            j += 1
    return tot


def duplex_gbs(dev):
    n = 1 << 28
    h1, h2 = (torch.empty(n, dtype=torch.float32, pin_memory=True) for _ in range(2))
    d1, d2 = (torch.empty(n, dtype=torch.float32, device=dev) for _ in range(2))
    a, b = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
    best = 1e9
    for _ in range(3):
        torch.cuda.synchronize()
        t = time.perf_counter()
        with torch.cuda.stream(a):
            d1.copy_(h1, non_blocking=True)
        with torch.cuda.stream(b):
            h2.copy_(d2, non_blocking=True)
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t)
    return n * 4 / best / 1e9


def trace(overlap: bool, steps: int, out_dir: str):
    dev = torch.device("cuda", 0)
    shape = MODELS["llama2-7b"]
    n, NL = shape.layer_numel, shape.n_layers
    ids = [5, 21]
    sig = grad_sigmas(NL, 0)
    params = {l: layer_params(n, l, device=dev, norm_numel=shape.norm_numel) for l in ids}
    grads = {l: layer_grad(n, l, sig[l], device=dev) for l in ids}
    ctx = G.Grass([n] * NL, gamma=2, offload=True, overlap=overlap)
    s = torch.cuda.Stream(device=dev)
    for _ in range(2):
        ctx.step_layers(ids, [params[l] for l in ids], [grads[l] for l in ids], 3e-5, stream=s)
    torch.cuda.synchronize()
    path = os.path.join(out_dir, f"host_link_cupti_{'overlap' if overlap else 'vanilla'}.trace.json")
    from torch.profiler import ProfilerActivity, profile
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(steps):
            ctx.step_layers(ids, [params[l] for l in ids], [grads[l] for l in ids], 3e-5, stream=s)
        torch.cuda.synchronize()
    prof.export_chrome_trace(path)
    ctx.close()
    with open(path) as f:
        ev = json.load(f)["traceEvents"]
    h2d, d2h, ker = [], [], []
    bh = bd = 0
    for e in ev:
        if e.get("ph") != "X":
            continue
        cat, name = e.get("cat", ""), e.get("name", "")
        iv = (float(e["ts"]), float(e["ts"]) + float(e["dur"]))
        if cat == "gpu_memcpy":
            nb = int(e.get("args", {}).get("bytes", 0))
            if "HtoD" in name:
                h2d.append(iv)
                bh += nb
            elif "DtoH" in name:
                d2h.append(iv)
                bd += nb
        elif cat == "kernel" and "grass_stream_kernel" in name:
            ker.append(iv)
    span = (min(a for a, _ in h2d + d2h + ker), max(b for _, b in h2d + d2h + ker))
    uh, ud, uk = union(h2d), union(d2h), union(ker)
    us = 1e-6
    res = {
        "mode": "overlapped (copy streams + events)" if overlap else "Fig. 4 vanilla (serial)",
        "steps": steps, "copies": {"HtoD": len(h2d), "DtoH": len(d2h)}, "update_kernels": len(ker),
        "HtoD_bytes_per_step": bh / steps, "DtoH_bytes_per_step": bd / steps,
        "step_ms": (span[1] - span[0]) / steps / 1e3,
        "HtoD_busy_ms_per_step": length(uh) / steps / 1e3, "DtoH_busy_ms_per_step": length(ud) / steps / 1e3,
        "kernel_busy_ms_per_step": length(uk) / steps / 1e3,
        "HtoD_GBps_while_busy": bh / (length(uh) * us) / 1e9 if uh else None,
        "DtoH_GBps_while_busy": bd / (length(ud) * us) / 1e9 if ud else None,
        "HtoD_GBps_over_step": bh / ((span[1] - span[0]) * us) / 1e9,
        "DtoH_GBps_over_step": bd / ((span[1] - span[0]) * us) / 1e9,
        "HtoD_DtoH_overlap_frac_of_step": intersect(uh, ud) / (span[1] - span[0]),
        "kernel_hidden_under_copies_frac": intersect(uk, union(h2d + d2h)) / max(length(uk), 1e-9),
        "trace": os.path.basename(path),
    }
    return res


def main():
    out_dir = os.path.join(ROOT, "gpurun_out")
    os.makedirs(out_dir, exist_ok=True)
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    dup = duplex_gbs(dev)
    res = {"tool": "CUPTI activity records via torch.profiler (Kineto); nsys is not in the image",
           "duplex_GBps_per_dir_measured": dup, "pcie5_x16_nominal_GBps_per_dir": 63.0,
           "runs": [trace(True, 3, out_dir), trace(False, 2, out_dir)]}
    for r in res["runs"]:
        floor = max(r["HtoD_bytes_per_step"], r["DtoH_bytes_per_step"]) / (dup * 1e9) * 1e3
        r["duplex_floor_ms"] = floor
        r["frac_of_duplex_floor"] = floor / r["step_ms"]
        r["HtoD_frac_of_nominal"] = r["HtoD_GBps_over_step"] / 63.0
    with open(os.path.join(out_dir, "host_link_cupti.json"), "w") as f:
        json.dump(res, f, indent=1)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
