"""Measure the GPU box facts the roofline needs: host cores/RAM, PCIe link,
pinned H2D / D2H / duplex bandwidth, HBM copy. Plumbing only (torch copies)."""
import json, os, subprocess, time
import torch

out = {}
out["nproc"] = os.cpu_count()
out["sched_affinity"] = len(os.sched_getaffinity(0))
with open("/proc/meminfo") as f:
    out["meminfo"] = {l.split(":")[0]: l.split(":")[1].strip() for l in f if l.split(":")[0] in ("MemTotal", "MemAvailable", "Hugepagesize")}
def sh(c):
    try:
        return subprocess.run(c, shell=True, capture_output=True, text=True, timeout=60).stdout
    except Exception as e:
        return str(e)
out["smi"] = sh("nvidia-smi --query-gpu=name,pci.bus_id,pcie.link.gen.current,pcie.link.gen.max,pcie.link.width.current,clocks.sm,clocks.max.sm,memory.total --format=csv")
out["topo"] = sh("nvidia-smi topo -m")
out["numa"] = sh("lscpu | grep -i -E 'numa|model name|socket'")
dev = torch.device("cuda:0")
n = 1 << 28  # 1 GiB fp32
h = torch.empty(n, dtype=torch.float32, pin_memory=True)
h2 = torch.empty(n, dtype=torch.float32, pin_memory=True)
d = torch.empty(n, dtype=torch.float32, device=dev)
d2 = torch.empty(n, dtype=torch.float32, device=dev)
s1 = torch.cuda.Stream(); s2 = torch.cuda.Stream()
def timeit(fn, reps=5):
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize(); t = time.perf_counter(); fn(); torch.cuda.synchronize(); best = min(best, time.perf_counter() - t)
    return best
b = n * 4
out["h2d_GBs"] = b / timeit(lambda: d.copy_(h, non_blocking=True)) / 1e9
out["d2h_GBs"] = b / timeit(lambda: h.copy_(d, non_blocking=True)) / 1e9
def duplex():
    with torch.cuda.stream(s1):
        d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2):
        h2.copy_(d2, non_blocking=True)
out["duplex_GBs_each_dir"] = b / timeit(duplex) / 1e9
out["hbm_copy_GBs"] = 2 * b / timeit(lambda: d2.copy_(d)) / 1e9
t = time.perf_counter(); big = torch.empty(8 << 30 >> 2, dtype=torch.float32, pin_memory=True); out["pin_8GiB_s"] = time.perf_counter() - t
print(json.dumps(out, indent=1))
os.makedirs("gpurun_out", exist_ok=True)
json.dump(out, open("gpurun_out/box_probe.json", "w"), indent=1)
