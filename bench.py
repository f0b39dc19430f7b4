#!/usr/bin/env python
"""bench.py — GRASS layer-wise update hot path on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl grass|reference]

One STEP = one pass of the whole hot path on the
BASELINE.json configs[1] workload: LLaMA-2-7B-shaped stack (32 decoder layers
of N_p = 202,383,360 fp32 parameters), gamma = 2 active layers, optimizer
states resident (no offload), 1 B200:
    fused Eq. 2 norm + AdamW of the 2 active layers        (a1 + a5, one kernel)
    MGN window accumulation                                (a2, in the kernel)
    window commit + Eq. 4 EMA + Eq. 3 softmax              (a2 + a3, host fp64)
    gamma-of-N_L resampling                                (a4, host)
i.e. the bench resamples EVERY step (T_s = T_u = 1), the most expensive legal
schedule.  Further legs in the same JSON line (--legs): "probe" (a1 alone over
all 32 layers, against the measured read-only HBM ceiling), "offload" (row
a6, configs[2], + Fig. 4 vanilla), "period" (f1, T_s = 25), "p2p" (f2, the
fused peer-memory data-parallel kernel), "bf16" (f3), "e2e" (gradients from
pinned host memory through the public call), "cpu" (the oracle on one core
and on all host cores); opt-in: "train" (synthetic 7B fwd+bwd with resident /
period+prefetch / per-step offload after and during the backward, ~10 s of
GEMMs).

Timing: CUDA events on the stream the library launches on, W untimed warm-up
steps, K timed steps bracketed by barrier + synchronize, max over ranks.  Every
step streams 11.3 GB through HBM (>> 126 MB L2), so no L2 flush is needed.
For N > 1 (torchrun) the same total work is element-sharded over the ranks
(gradients reduce-scattered and parameters all-gathered over NCCL): strong
scaling.  `--impl reference` times the fp64 CPU oracle on the host cores.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "active-layer params updated/s and offloaded step ms; % of HBM / host-link roofline"
UNIT = "params/s"
BYTES_PER_PARAM_UPDATE = 28      # read g, theta, m, v + write theta, m, v (fp32)
BYTES_PER_PARAM_PROBE = 4        # read g
DEFAULT_LEGS = "main,probe,p2p,offload,period,bf16,e2e,cpu"   # "train" (R4, ~10 s of GEMMs) is opt-in
FALLBACK_HBM_GBS = 6650.0        # B200_PROFILING.md fallback, used only if MEASURED_PEAKS.json is absent


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="grass", choices=["grass", "reference"])
    ap.add_argument("--model", default="llama2-7b")
    ap.add_argument("--gamma", type=int, default=2)
    ap.add_argument("--legs", default=DEFAULT_LEGS,
                    help="comma list of legs to run (main is always run)")
    ap.add_argument("--offload-steps", type=int, default=10)
    ap.add_argument("--lr", type=float, default=3e-5)
    return ap.parse_args()


# --------------------------------------------------------------------- utils
def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    return FALLBACK_HBM_GBS, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled DURING the timed region."""
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index, self.rows, self.proc = index, [], None
        self.stop = threading.Event()
        self.thread = None

    def _nvml_poll(self, h, nv, ready):
        """Poll NVML every 2 ms: the timed region is ~0.1 s, far below nvidia-smi's start-up."""
        bits = [nv.nvmlClocksThrottleReasonHwSlowdown, nv.nvmlClocksThrottleReasonHwThermalSlowdown,
                nv.nvmlClocksThrottleReasonSwThermalSlowdown, nv.nvmlClocksThrottleReasonSwPowerCap]
        try:
            mx = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
        except Exception:
            return               # no sample: __enter__ falls back to nvidia-smi
        while True:
            try:
                sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
                r = nv.nvmlDeviceGetCurrentClocksThrottleReasons(h)
                self.rows.append([str(sm), str(mx)] + ["Active" if r & b else "Not Active" for b in bits])
            except Exception:
                pass
            ready.set()
            if self.stop.wait(0.002):
                return

    def _nvml_handle(self, nv):
        """The NVML handle of THIS process's CUDA device: NVML enumerates every
        GPU of the box and ignores CUDA_VISIBLE_DEVICES, so resolve it by PCI
        bus id (then UUID); the bare index only if neither is available."""
        import torch
        prop = torch.cuda.get_device_properties(self.index)
        dom, bus, dv = (getattr(prop, k, None) for k in ("pci_domain_id", "pci_bus_id", "pci_device_id"))
        if bus is not None and dv is not None:
            try:
                return nv.nvmlDeviceGetHandleByPciBusId(f"{dom or 0:08X}:{bus:02X}:{dv:02X}.0".encode())
            except Exception:
                pass
        uuid = getattr(prop, "uuid", None)
        if uuid is not None:
            try:
                return nv.nvmlDeviceGetHandleByUUID(f"GPU-{uuid}".encode())
            except Exception:
                pass
        return nv.nvmlDeviceGetHandleByIndex(self.index)

    def __enter__(self):
        self.nv = None
        try:
            import pynvml as nv
            nv.nvmlInit()
            self.nv = nv
            h = self._nvml_handle(nv)
            self.bus_id = nv.nvmlDeviceGetPciInfo(h).busId
            ready = threading.Event()
            self.thread = threading.Thread(target=self._nvml_poll, args=(h, nv, ready), daemon=True)
            self.thread.start()
            if ready.wait(2.0):  # first sample taken before the timed region starts
                return self
            self.stop.set()      # the poll never sampled: fall back to nvidia-smi
            self.thread.join(timeout=1.0)
            self.stop.clear()
        except Exception:
            pass
        self.thread = None
        try:
            sel = getattr(self, "bus_id", None)
            sel = sel.decode() if isinstance(sel, bytes) else (sel or str(self.index))
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", sel, f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "20"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            threading.Thread(target=self._read, daemon=True).start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) == 6:
                self.rows.append(parts)

    def __exit__(self, *a):
        if self.thread:
            self.stop.set()
            self.thread.join(timeout=1.0)
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
        if self.nv is not None:
            try:
                self.nv.nvmlShutdown()
            except Exception:
                pass

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({n for r in self.rows for n, v in zip(names, r[2:]) if v.lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def dist_setup(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist
        backend = "nccl" if args.impl == "grass" else "gloo"
        if backend == "nccl":
            import torch
            torch.cuda.set_device(local)
        dist.init_process_group(backend, init_method="env://")
    return rank, world, local


def max_over_ranks(x: float, world: int, device=None) -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


# ------------------------------------------------------------ oracle (CPU)
def oracle_sample_time(n_p: int, gamma: int, sample_per_layer: int, lr: float, reps: int = 1):
    """Times the fp64 oracle (oracle/, as it stands) on a bounded sample of one
    step: Eq. 2 norms + AdamW over `sample_per_layer` elements of each of the
    gamma active layers, then commit/EMA/softmax/sampling over N_L = 32."""
    import numpy as np
    from threadpoolctl import threadpool_limits

    from oracle import grass_oracle as O
    from synth import grad_sigmas, layer_grad, layer_params
    sig = grad_sigmas(32, 0)
    th = [layer_params(sample_per_layer, l).numpy() for l in range(gamma)]
    g = [layer_grad(sample_per_layer, l, sig[l]).numpy() for l in range(gamma)]
    m = [np.zeros(sample_per_layer, np.float32) for _ in range(gamma)]
    v = [np.zeros(sample_per_layer, np.float32) for _ in range(gamma)]
    st = O.MgnState(32)
    for l in range(32):
        st.record(l, 1e-4 * (l + 1))
    st.commit(0.5)
    times = []
    with threadpool_limits(limits=1):
        for r in range(reps):
            t0 = time.perf_counter()
            for l in range(gamma):
                ss = O.sq_norm(g[l])
                st.record(l, O.rms_norm(ss, n_p))
                O.adamw_step(th[l], m[l], v[l], g[l], r + 1, lr, weight_decay=0.0)
            mm = st.commit(0.5)
            p = O.softmax_probs(mm, 1.0, True)
            O.sample_layers(p, gamma, 1234, r)
            times.append(time.perf_counter() - t0)
    return times


def _oracle_chunk(args):
    """One worker of the all-core oracle timing: Eq. 2 norm + AdamW over its
    element chunk of the step's sample (single-threaded numpy)."""
    n, layer, lr, reps = args
    import numpy as np
    from threadpoolctl import threadpool_limits

    from oracle import grass_oracle as O
    from synth import grad_sigmas, layer_grad, layer_params
    sig = grad_sigmas(32, 0)
    th = layer_params(n, layer).numpy()
    g = layer_grad(n, layer, sig[layer]).numpy()
    m = np.zeros(n, np.float32)
    v = np.zeros(n, np.float32)
    with threadpool_limits(limits=1):
        t0 = time.perf_counter()
        for r in range(reps):
            O.sq_norm(g)
            O.adamw_step(th, m, v, g, r + 1, lr, weight_decay=0.0)
        return time.perf_counter() - t0


def oracle_all_cores(gamma: int, sample_per_layer: int, lr: float):
    """The same bounded sample split into element chunks over every host core
    (multiprocessing, one numpy thread per worker): params/s of the slowest
    worker's wall time (the per-layer commit / softmax / sampling over 32
    layers is microseconds and omitted)."""
    import multiprocessing as mp
    cores = os.cpu_count() or 1
    per = max(1, gamma * sample_per_layer // cores)
    jobs = [(per, k % gamma, lr, 2) for k in range(cores)]
    with mp.get_context("spawn").Pool(cores) as pool:
        pool.map(_oracle_chunk, [(1024, 0, lr, 1)] * cores)          # workers imported and warm
        t0 = time.perf_counter()
        times = pool.map(_oracle_chunk, jobs)
        wall = time.perf_counter() - t0
    return {"value": 2 * per * cores / wall, "unit": UNIT, "cores": cores, "kind": "oracle",
            "sample": f"{cores} workers x {per} elements x 2 steps (fp64 norm + AdamW), spawn pool, "
                      f"threadpoolctl 1 thread each; slowest worker {max(times):.2f} s, wall {wall:.2f} s"}


def measure_read_ceiling(dev, gib: int = 8) -> dict:
    """Read-only HBM ceiling: hand-written streaming reads
    of an 8 GiB buffer (>> 126 MB L2) — LDG.128 (no-allocate, 8 loads in flight
    per thread) over a grid sweep and TMA bulk copies into a shared-memory ring
    (K1's data movement, no arithmetic) over a unit / stage sweep
    (paper_2604_07808_b200/diag/read_ceiling.cu); best of 3 per config, CUDA
    events on the launching stream.  The probe's denominator."""
    import ctypes as C

    import torch
    from paper_2604_07808_b200 import build as B
    lib = C.CDLL(B.build_diag())                 # built in-tree by __graft_entry__.build()
    f = lib.grass_diag_read
    f.restype = C.c_int
    f.argtypes = [C.c_void_p, C.c_ulonglong, C.c_int, C.c_int, C.c_uint, C.c_int, C.c_void_p, C.c_void_p]
    nbytes = gib << 30
    buf = torch.empty(nbytes, dtype=torch.uint8, device=dev)
    buf.fill_(7)
    sink = torch.zeros(1, dtype=torch.int64, device=dev)
    s = torch.cuda.Stream(device=dev)
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    cfgs = [("ldg", 0, sms * k, 0, 0) for k in (2, 4, 8)] + \
           [("tma", 1, sms, u << 10, st) for u, st in ((16, 12), (32, 6), (64, 3), (96, 2))]
    sweep, errors = {}, {}
    for name, mode, grid, unit, st in cfgs:
        nb = nbytes - nbytes % unit if unit else nbytes      # whole units
        key = f"{name} grid={grid}" + (f" unit={unit >> 10}KiB x{st}" if mode else "")
        best = 0.0
        for _ in range(3):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            rc = f(buf.data_ptr(), nb, mode, grid, unit, st, sink.data_ptr(), s.cuda_stream)
            e1.record(s)
            torch.cuda.synchronize()
            if rc != 0:
                errors[key] = f"cuda error {rc}"
                break
            best = max(best, nb / (e0.elapsed_time(e1) / 1e3) / 1e9)
        if best:
            sweep[key] = round(best, 1)
    del buf
    torch.cuda.empty_cache()
    k = max(sweep, key=sweep.get)
    return {"GBps": sweep[k], "best": k, "sweep": sweep, "bytes": nbytes, **({"errors": errors} if errors else {})}


def measure_mix_ceiling(dev, n: int = 2 * 202_383_360, bf16: bool = False) -> dict:
    """K2's own traffic-mix ceiling: 4 reads + 3 writes per element (g, theta,
    m, v in; theta, m, v out — 28 B) with NO arithmetic, over 4 fp32 arrays of
    n elements (configs[1]'s gamma x N_p: 11.3 GB moved per launch, >> L2; not
    a power of two — four 2^k-byte arrays would start on the same HBM channels
    and measure channel conflicts, not the mix): K2's TMA ring (bulk loads into
    a shared-memory ring, bulk stores back; diag `rw43_tma`) over a small
    unit / stage / grid set, and plain LDG/STG (`rw43`); best of 3 each, CUDA
    events on the launching stream.  K2 at this number is at the ceiling of the
    data movement it must do."""
    import ctypes as C

    import torch
    from paper_2604_07808_b200 import build as B
    lib = C.CDLL(B.build_diag())                 # built in-tree by __graft_entry__.build()
    ft, fl = lib.grass_diag_rw43_tma, lib.grass_diag_rw43
    ft.restype = fl.restype = C.c_int
    ft.argtypes = [C.POINTER(C.c_void_p), C.c_ulonglong, C.c_uint, C.c_int, C.c_int, C.c_int, C.c_void_p]
    fl.argtypes = [C.POINTER(C.c_void_p), C.c_ulonglong, C.c_int, C.c_int, C.c_void_p]
    # bf16 (K2's R18 mode): bf16 gradient read, fp32 master / m / v read and
    # written, bf16 parameter copy written — 14 + 14 B per element
    n -= n % 4096                                # whole units of every swept size
    bufs = [torch.full((n,), 1e-3, device=dev, dtype=torch.bfloat16 if bf16 else torch.float32)]
    bufs += [torch.full((n,), 1e-3, device=dev) for _ in range(3)]
    if bf16:
        bufs.append(torch.empty(n, device=dev, dtype=torch.bfloat16))
    ptrs = (C.c_void_p * len(bufs))(*[b.data_ptr() for b in bufs])
    s = torch.cuda.Stream(device=dev)
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    cfgs = [(f"tma unit={e} x{st} grid={g}", lambda e=e, st=st, g=g: ft(ptrs, n, e, st, g, int(bf16), s.cuda_stream))
            for e, st, g in ((4096, 3, 128), (2048, 3, sms), (2048, 6, 128), (1024, 4, sms), (2048, 2, 2 * sms))]
    if not bf16:
        cfgs += [(f"ldg unroll={u} grid={g}", lambda u=u, g=g: fl(ptrs, n, u, g, s.cuda_stream))
                 for u, g in ((2, sms), (4, 8 * sms))]
    sweep, errors = {}, {}
    for key, call in cfgs:
        best = 0.0
        for _ in range(3):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            rc = call()
            e1.record(s)
            torch.cuda.synchronize()
            if rc != 0:
                errors[key] = f"cuda error {rc}"
                break
            best = max(best, 28 * n / (e0.elapsed_time(e1) / 1e3) / 1e9)
        if best:
            sweep[key] = round(best, 1)
    del bufs
    torch.cuda.empty_cache()
    k = max(sweep, key=sweep.get)
    return {"GBps": sweep[k], "best": k, "sweep": sweep, "bytes_per_launch": 28 * n,
            **({"errors": errors} if errors else {})}


def workload_config(model: str, gamma: int, world: int) -> dict:
    """The `config` of the JSON line, identical for the GRASS and reference arms."""
    from synth import MODELS
    shape = MODELS[model]
    active = gamma * shape.layer_numel
    return {"workload": f"{model}-stack gamma={gamma} no-offload" +
                        (" (configs[1])" if (model, gamma) == ("llama2-7b", 2) else ""),
            "n_layers": shape.n_layers, "layer_numel": shape.layer_numel, "gamma": gamma,
            "active_params_per_step": active, "schedule": "resample every step (T_s=T_u=1)",
            "l2": (f"no flush: {BYTES_PER_PARAM_UPDATE * active / 1e9:.1f} GB streamed per step >> 126 MB L2"
                   if BYTES_PER_PARAM_UPDATE * active > 4 * 126e6 else
                   "L2-resident: a small test stack, not a measurement configuration"),
            "parallelism": f"dp{world} element-sharded" if world > 1 else "single GPU"}


# ------------------------------------------------------------ reference arm
def run_reference(args, rank, world):
    if rank != 0:
        return
    from synth import MODELS
    n_p = MODELS[args.model].layer_numel
    sample = 1 << 22                   # 4 Mi elements per active layer per step
    times = oracle_sample_time(n_p, args.gamma, sample, args.lr, reps=args.warmup + args.steps)
    timed = times[args.warmup:]
    per_step = sum(timed) / len(timed)
    value = args.gamma * sample / per_step
    desc = (f"{args.gamma} x {sample} elements (of N_p = {n_p}) per step: fp64 Eq. 2 norm + AdamW, "
            "MGN commit/EMA/softmax/sampling over 32 layers; single thread (threadpoolctl)")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": per_step * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": workload_config(args.model, args.gamma, args.gpus),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": "oracle", "sample": desc},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------ GRASS arm
def run_grass(args, rank, world, local):
    import torch

    import paper_2604_07808_b200 as G
    from synth import MODELS, grad_sigmas, layer_grad, layer_params

    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    legs = set(args.legs.split(","))
    if world > 1 and args.legs == DEFAULT_LEGS:
        # the north star's per-N numbers: resident step, e2e, and the offloaded
        # step (per-step round trip and period residency) on element shards
        legs = {"main", "e2e", "p2p", "offload", "period"}
    shape = MODELS[args.model]
    NL, n_p, gamma = shape.n_layers, shape.layer_numel, args.gamma
    sig = grad_sigmas(NL, 0)
    params = [layer_params(n_p, l, device=dev, norm_numel=shape.norm_numel) for l in range(NL)]
    grads = [layer_grad(n_p, l, sig[l], step=0, device=dev, rank=rank) for l in range(NL)]
    torch.cuda.synchronize()
    s = torch.cuda.Stream(device=dev)
    ctx = G.Grass([n_p] * NL, gamma=gamma, T_p=1, T_s=1, T_u=1, seed=1234, device=local,
                  rank=rank, world=world)
    hbm_peak, peak_kind = peaks()
    out = {}

    # ---- probing pass (a1 alone over every layer) -> MGN initialisation
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    probe_ms = []
    for it in range(6 if "probe" in legs else 1):
        ev[0].record(s)
        ctx.mgn_accumulate(list(range(NL)), grads, stream=s)
        ev[1].record(s)
        torch.cuda.synchronize()
        probe_ms.append(ev[0].elapsed_time(ev[1]))
    probs = ctx.update_probs()
    ids = ctx.sample_layers(0)
    read_ceiling = None
    if "probe" in legs:
        t = statistics.median(probe_ms[1:]) / 1e3
        gbs = BYTES_PER_PARAM_PROBE * NL * n_p / world / t / 1e9
        try:
            read_ceiling = measure_read_ceiling(dev)
        except Exception as ex:  # recorded, never fatal to the line
            read_ceiling = {"error": f"{type(ex).__name__}: {ex}"[:300]}
        rc = read_ceiling.get("GBps")
        out["probe"] = {"ms": t * 1e3, "layers": NL, "GBps": gbs, "frac_hbm": gbs / hbm_peak,
                        "read_ceiling_GBps": rc, "frac_read_peak": gbs / rc if rc else None,
                        "read_ceiling": read_ceiling,
                        "bytes": BYTES_PER_PARAM_PROBE * NL * n_p // world}

    # ---- main leg: configs[1].  World 1: the device-resident schedule — each
    # step is grass_device_step (update of the layers sampled on the device,
    # commit, resample of the next period), no host round trip between steps.
    # World > 1: the host-driven loop (step_layers, update_probs, sample_layers).
    use_dev = world == 1

    def host_step(step, timing):
        nonlocal ids
        if timing is not None:
            timing[0].record(s)
        ctx.step_layers(ids, [params[l] for l in ids], [grads[l] for l in ids], args.lr, stream=s)
        if timing is not None:
            timing[1].record(s)
        ctx.update_probs()
        ids = ctx.sample_layers(step + 1)

    def dev_step(step, timing):
        # no per-step events here: an event between two steps would stand
        # between K3 and the next K2, which are launched as programmatic
        # dependents of each other (their launches overlap the previous
        # kernel's drain); kernel_ms is then the timed region's mean step
        ctx.device_step(args.lr, stream=s)

    one_step = dev_step if use_dev else host_step
    if use_dev:
        ctx.register_layers(params, grads)
        ctx.device_schedule_begin(0, stream=s)

    for w in range(args.warmup):
        one_step(w, None)
    torch.cuda.synchronize()
    barrier(world)
    kev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(args.steps)]
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    launches0 = ctx.launch_count
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        t0.record(s)
        for k in range(args.steps):
            one_step(args.warmup + k, kev[k])
        t1.record(s)
        torch.cuda.synchronize()
    launches = ctx.launch_count - launches0
    if use_dev:
        ids = ctx.device_schedule_end()
    barrier(world)
    elapsed = max_over_ranks(t0.elapsed_time(t1) / 1e3, world, dev)
    kernel_ms = (statistics.mean(a.elapsed_time(b) for a, b in kev) if not use_dev
                 else t0.elapsed_time(t1) / args.steps)
    active = gamma * n_p
    host_schedule = None
    if use_dev and "main" in legs:
        # the same step driven from the host (grass_step_layers + grass_update_probs
        # + grass_sample_layers): the host round trip per step, for comparison
        for w in range(3):
            host_step(10_000 + w, None)
        torch.cuda.synchronize()
        hev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
               for _ in range(args.steps)]
        h0, h1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        h0.record(s)
        for k in range(args.steps):
            host_step(10_100 + k, hev[k])
        h1.record(s)
        torch.cuda.synchronize()
        hms = h0.elapsed_time(h1) / args.steps
        gaps = [hev[i][1].elapsed_time(hev[i + 1][0]) for i in range(args.steps - 1)]
        host_schedule = {"step_ms": hms, "params_per_s": active / (hms / 1e3),
                         "gpu_idle_between_steps_us": statistics.median(gaps) * 1e3 if gaps else None,
                         "what": "the same step through grass_step_layers + grass_update_probs + "
                                 "grass_sample_layers (host commit and sampler, one host round trip per step)"}
    value = args.steps * active / elapsed
    achieved = BYTES_PER_PARAM_UPDATE * active / world / (kernel_ms / 1e3) / 1e9
    traffic = None
    tp = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tp):
        with open(tp) as f:
            traffic = json.load(f).get(f"fused_update/{args.model}/g{gamma}/w{world}")

    # Optional legs.  At world == 1 a failing optional leg is recorded under
    # "leg_errors" instead of costing the main line; at world > 1 an exception is
    # not caught (a rank-local failure inside a collective leg would hang).
    leg_errors = {}

    def guarded(name, fn):
        if name not in legs:
            return None
        if world > 1:
            return fn()
        try:
            return fn()
        except Exception as ex:
            leg_errors[name] = f"{type(ex).__name__}: {ex}"[:400]
            try:
                torch.cuda.synchronize()
            except Exception:
                pass
            return None

    # ---- e2e: same step through the C ABI from pinned HOST gradients
    def leg_e2e():
        host_g = [grads[l].to("cpu").pin_memory() for l in range(gamma)]
        h2d = sum(h.numel() * 4 for h in host_g)
        d2h = NL * 16 + 4
        for w in range(2):
            host_step(w, None)                  # the device schedule has ended: the host API
        torch.cuda.synchronize()
        barrier(world)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ksteps = max(3, min(args.steps, 10))
        def e2e_step(step):
            nonlocal ids
            if world == 1:
                # the public call with the step's gradients in pinned HOST memory: the
                # library streams them chunk-wise into HBM, overlapped with the update
                ctx.step_layers(ids, [params[l] for l in ids], host_g[:len(ids)], args.lr, stream=s)
            else:
                # the DP path reduce-scatters device buffers: stage the host gradients first
                with torch.cuda.stream(s):
                    for j, l in enumerate(ids):
                        grads[l].copy_(host_g[j], non_blocking=True)
                ctx.step_layers(ids, [params[l] for l in ids], [grads[l] for l in ids], args.lr, stream=s)
            ctx.update_probs()                  # reads S, c back (d2h)
            ids = ctx.sample_layers(step + 1)
        e0.record(s)
        for k in range(ksteps):
            e2e_step(1000 + k)
        e1.record(s)
        torch.cuda.synchronize()
        et = max_over_ranks(e0.elapsed_time(e1) / 1e3, world, dev)
        return {"value": ksteps * active / et, "unit": UNIT, "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h, "ms_per_step": et / ksteps * 1e3, "steps": ksteps,
                "note": "the step's gradients enter from pinned host memory (the same gamma host buffers "
                        "stand for whichever layers were sampled: their values do not change the timing); "
                        "the result read back is the committed MGN window (S, c, flag); theta' and m/v "
                        "stay in HBM"}

    e2e = guarded("e2e", leg_e2e)

    # ---- the same resident step on the paper's schedule (T_s = T_u = 25:
    # commit + resample once per 25 steps) — what a training run
    # sees per step, next to the every-step-resample `value`
    def leg_paper_schedule():
        nonlocal ids
        T = 25
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        barrier(world)
        if use_dev:                               # the device-resident schedule, as the main leg
            ctx.device_schedule_begin(10_000, stream=s)
            torch.cuda.synchronize()
        e0.record(s)
        for k in range(2 * T):
            if use_dev:                           # commit + resample after the period's last step
                last = (k + 1) % T == 0
                ctx.device_step(args.lr, commit=last, resample=last, stream=s)
                continue
            if k and k % T == 0:                  # period boundary (the window holds T steps)
                ctx.update_probs()
                ids = ctx.sample_layers(10_000 + k // T)
            ctx.step_layers(ids, [params[l] for l in ids], [grads[l] for l in ids], args.lr, stream=s)
        e1.record(s)
        torch.cuda.synchronize()
        if use_dev:
            ids = ctx.device_schedule_end()
        t = max_over_ranks(e0.elapsed_time(e1) / 1e3, world, dev) / (2 * T)
        return {"schedule": f"T_s=T_u={T} (2 periods)", "step_ms": t * 1e3, "params_per_s": active / t,
                "driver": "grass_device_step" if use_dev else "grass_step_layers + host commit / sampler"}

    paper_schedule = guarded("main", leg_paper_schedule)
    ctx.close()                                 # frees its 51.8 GB of HBM state
    try:
        mix_ceiling = measure_mix_ceiling(dev)
    except Exception as ex:  # recorded, never fatal to the line
        mix_ceiling = {"error": f"{type(ex).__name__}: {ex}"[:300]}
    torch.cuda.empty_cache()

    # ---- P2P data parallelism: the same step with ONE fused
    # kernel per call reading every rank's gradient over peer memory and storing
    # theta' into every rank (no NCCL on the data path).  At N > 1 the ranks'
    # buffers are mapped through CUDA IPC.  Every rank takes the same branches:
    # a failure on any rank is agreed on (all_reduce) before the next collective.
    def all_ok(flag: bool) -> bool:
        if world == 1:
            return flag
        t = torch.tensor([1 if flag else 0], device=dev)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MIN)
        return bool(t.item())

    def leg_p2p():
        err = None
        pctx = None
        try:
            pctx = G.Grass([n_p] * NL, gamma=gamma, T_p=1, T_s=1, T_u=1, seed=1234, device=local,
                           rank=rank, world=world, dp_mode=G.DP_P2P)
            pctx.p2p_setup({l: (params[l], grads[l]) for l in range(NL)}) if world > 1 else None
            if world == 1:
                pctx.p2p_attach([pctx.p2p_exchange_block()[0]])
                for l in range(NL):
                    pctx.p2p_register_layer(l, [params[l]], [grads[l]])
        except Exception as ex:
            err = f"setup: {type(ex).__name__}: {ex}"[:300]
        if not all_ok(err is None):
            if pctx is not None:
                pctx.close()
            return {"error": err or "setup failed on another rank"}
        pev = []
        probe_ms = 0.0
        try:
            pe = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
            pe[0].record(s)
            pctx.mgn_accumulate(list(range(NL)), grads, stream=s)     # probing pass (K1 over peers)
            pe[1].record(s)
            pctx.mgn_accumulate(list(range(NL)), grads, stream=s)
            pe[2].record(s)
            torch.cuda.synchronize()
            probe_ms = pe[1].elapsed_time(pe[2])
            pctx.update_probs()
            pids = pctx.sample_layers(0)
            for k in range(args.warmup + args.steps):
                timed = k >= args.warmup
                if timed:
                    e = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                    e[0].record(s)
                pctx.step_layers(pids, [params[l] for l in pids], [grads[l] for l in pids], args.lr, stream=s)
                if timed:
                    e[1].record(s)
                    pev.append(e)
                pctx.update_probs()
                pids = pctx.sample_layers(k + 1)
            torch.cuda.synchronize()
            call_ms = statistics.mean(a.elapsed_time(b) for a, b in pev)
        except Exception as ex:
            err = f"run: {type(ex).__name__}: {ex}"[:300]
            call_ms = 0.0
        ok = all_ok(err is None)
        call_ms = max_over_ranks(call_ms, world, dev)
        pctx.close()
        if not ok:
            return {"error": err or "failed on another rank"}
        hbm = BYTES_PER_PARAM_UPDATE * active / world          # per rank: local shard traffic
        link = 8 * active * (world - 1) / world                 # per rank: peer grad reads + theta' stores
        probe_ms = max_over_ranks(probe_ms, world, dev)
        return {"workload": f"{args.model}-stack gamma={gamma}, P2P fused RS+update+AG kernel, dp{world}",
                "call_ms": call_ms, "params_per_s": active / (call_ms / 1e3),
                "probe_call_ms": probe_ms,
                "probe_hbm_GBps_per_rank": BYTES_PER_PARAM_PROBE * NL * n_p / world / (probe_ms / 1e3) / 1e9,
                "hbm_GBps_per_rank": hbm / (call_ms / 1e3) / 1e9,
                "nvlink_bytes_per_rank": link, "calls": len(pev),
                "nvlink_GBps_per_rank": link / (call_ms / 1e3) / 1e9 if world > 1 else None}


    def agreed_ctx(**kw):
        """A context every rank created (pinned-host allocations can fail on one
        rank only): None on every rank if any rank failed, so no rank is left
        waiting in a later collective."""
        c_, err_ = None, None
        try:
            c_ = G.Grass([n_p] * NL, device=local, rank=rank, world=world, **kw)
        except Exception as ex:
            err_ = f"{type(ex).__name__}: {ex}"[:300]
        if all_ok(c_ is not None):
            return c_, None
        if c_ is not None:
            c_.close()
        return None, err_ or "context creation failed on another rank"

    # ---- offload leg: configs[2] (row a6)
    def leg_offload():
        t_pin = time.perf_counter()
        octx, err = agreed_ctx(gamma=gamma, T_p=1, T_s=1, T_u=1, seed=1234, offload=True)
        if octx is None:
            return {"error": err}
        t_pin = time.perf_counter() - t_pin
        duplex = measure_duplex(dev)
        octx.mgn_accumulate(list(range(NL)), grads, stream=s)
        octx.update_probs()
        oids = octx.sample_layers(0)

        def ostep(step):
            nonlocal oids
            octx.step_layers(oids, [params[l] for l in oids], [grads[l] for l in oids], args.lr, stream=s)
            octx.update_probs()
            oids = octx.sample_layers(step + 1)
        for w in range(2):
            ostep(w)
        torch.cuda.synchronize()
        barrier(world)
        o0, o1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ok = args.offload_steps
        o0.record(s)
        for k in range(ok):
            ostep(10 + k)
        o1.record(s)
        torch.cuda.synchronize()
        ot = max_over_ranks(o0.elapsed_time(o1) / 1e3, world, dev) / ok
        link_bytes = 8 * active // world                       # per direction per rank
        floor = link_bytes / (duplex * 1e9)
        res = {"workload": f"{args.model}-stack gamma={gamma} offload, per-step round trip (row a6)",
               "step_ms": ot * 1e3, "params_per_s": active / ot,
               "h2d_bytes": link_bytes, "d2h_bytes": link_bytes,
               "link_GBps_per_dir": link_bytes / ot / 1e9,
               "duplex_GBps_per_dir_measured": duplex,
               "frac_of_pcie5_x16_nominal": link_bytes / ot / 1e9 / 63.0,  # 64 GT/s x16, 128b/130b
               "floor_ms": floor * 1e3, "frac_of_link_floor": floor / ot,
               "R1_within_10pct_of_link_floor": ot <= 1.10 * floor,
               "R2_offload_over_resident": ot / (elapsed / args.steps),
               "pinned_host_GB": octx.host_bytes / 1e9, "create_s": t_pin,
               "device_state_bytes": octx.device_bytes}
        octx.close()
        # Fig. 4 "vanilla" (HtoD -> update -> DtoH serially, overlap = 0) on the
        # same workload: the overlap speedup the paper quotes as 1.08x on a full
        # training step
        vctx, err = agreed_ctx(gamma=gamma, T_p=1, T_s=1, T_u=1, seed=1234, offload=True, overlap=False)
        if vctx is None:
            res["vanilla_error"] = err
            return res
        vctx.mgn_accumulate(list(range(NL)), grads, stream=s)
        vctx.update_probs()
        vids = vctx.sample_layers(0)
        v0, v1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        nv = 3
        for k in range(nv + 1):
            if k == 1:
                torch.cuda.synchronize()
                barrier(world)
                v0.record(s)
            vctx.step_layers(vids, [params[l] for l in vids], [grads[l] for l in vids], args.lr, stream=s)
            vctx.update_probs()
            vids = vctx.sample_layers(k + 1)
        v1.record(s)
        torch.cuda.synchronize()
        vt = max_over_ranks(v0.elapsed_time(v1) / 1e3, world, dev) / nv
        res["vanilla_step_ms"] = vt * 1e3
        res["overlap_speedup"] = vt / ot
        vctx.close()
        # optimizer-state HBM with offload as gamma grows (paper: LISA +1.63 GB vs
        # GRASS +0.14 GB from gamma 2 to 4): the ring does not grow
        g4, err = agreed_ctx(gamma=min(2 * gamma, NL), T_p=1, T_s=1, T_u=1, offload=True)
        if g4 is None:
            res["device_state_bytes_2x_gamma_error"] = err
            return res
        res["device_state_bytes_2x_gamma"] = g4.device_bytes
        g4.close()
        return res

    offload = guarded("offload", leg_offload)

    # ---- period residency: paper schedule T_s = T_u = 25
    def leg_period():
        torch.cuda.empty_cache()
        T_s = 25
        pctx, err = agreed_ctx(gamma=gamma, T_p=1, T_s=T_s, T_u=T_s, seed=1234, offload=True,
                               residency=G.RESIDENCY_PERIOD)
        if pctx is None:
            return {"error": err}
        pctx.mgn_accumulate(list(range(NL)), grads, stream=s)
        pctx.update_probs()
        pids = pctx.sample_layers(0)
        swaps = 0

        def pstep(step):
            nonlocal pids, swaps
            if step > 0 and step % T_s == 0:          # period boundary: commit, probs, resample
                pctx.update_probs()
                new = pctx.sample_layers(step // T_s)
                swaps += len(set(new) - set(pids))
                pids = new
            pctx.step_layers(pids, [params[l] for l in pids], [grads[l] for l in pids], args.lr,
                             stream=s)
        for w in range(T_s):                          # warm: one full period (cache filled)
            pstep(w)
        torch.cuda.synchronize()
        barrier(world)
        swaps = 0
        nper = 2 * T_s
        p0, p1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        p0.record(s)
        for k in range(nper):
            pstep(T_s + k)                            # starts at a period boundary
        p1.record(s)
        torch.cuda.synchronize()
        pt = max_over_ranks(p0.elapsed_time(p1) / 1e3, world, dev) / nper
        res = {"workload": f"{args.model}-stack gamma={gamma} offload, period residency "
                           f"(SURVEY 8(f) f1), T_s=T_u={T_s}",
               "steps": nper, "layer_swaps": swaps, "step_ms_amortized": pt * 1e3,
               "params_per_s": active / pt,
               "link_bytes_per_dir": swaps * 8 * n_p // world,
               "over_resident": pt / (elapsed / args.steps),
               "device_cache_bytes": pctx.device_bytes}
        pctx.close()
        return res

    offload_period = guarded("period", leg_period)

    # ---- full training step: the north star's "offloaded step
    # within 10% of the no-offload step" in the paper's own framing (PAPER.md:355,
    # b4 s1024).  The caller's forward+backward is a SYNTHETIC stand-in: bf16
    # GEMMs with the FLOPs of a LLaMA-2-7B fwd+bwd on 4 x 1024 tokens.
    def leg_train():
        T_s, nsteps = 25, 50
        flops = 6 * 6.74e9 * 4 * 1024
        a = torch.randn(8192, 8192, device=dev, dtype=torch.bfloat16)
        bm = torch.randn(8192, 8192, device=dev, dtype=torch.bfloat16)
        cm = torch.empty_like(a)
        n_mm = max(1, round(flops / (2 * 8192 ** 3)))

        def fwd_bwd():
            with torch.cuda.stream(s):
                for _ in range(n_mm):
                    torch.matmul(a, bm, out=cm)

        # the same GEMMs split as a forward (1/3) and a per-layer backward (2/3,
        # layer NL-1 first), so an update can be issued as soon as its layer's
        # gradient is ready (offload "layer by layer")
        n_f = n_mm // 3
        cuts = [n_f + round((n_mm - n_f) * (NL - l) / NL) for l in range(NL + 1)]  # cuts[l] .. cuts[l+1]
        side = torch.cuda.Stream(device=dev)

        def fwd_bwd_layerwise(on_grad_ready):
            with torch.cuda.stream(s):
                for _ in range(n_f):
                    torch.matmul(a, bm, out=cm)
                for l in reversed(range(NL)):
                    for _ in range(cuts[l] - cuts[l + 1]):
                        torch.matmul(a, bm, out=cm)
                    on_grad_ready(l)

        def run(mode):
            kw = dict(T_p=1, T_s=T_s, T_u=T_s, seed=1234, device=local, rank=rank, world=world)
            if mode == "prefetch":
                kw.update(offload=True, residency=G.RESIDENCY_PERIOD)
            elif mode in ("offload", "offload_bwd"):
                kw.update(offload=True)
            elif mode == "step_prefetch":
                kw.update(offload=True, residency=G.RESIDENCY_STEP_PREFETCH)
            key = tuple(sorted(kw.items()))
            if key not in ctx_cache:          # pinned-host contexts take ~20 s to create: reuse
                ctx_cache[key] = G.Grass([n_p] * NL, gamma=gamma, **kw)
            tc = ctx_cache[key]
            tc.mgn_accumulate(list(range(NL)), grads, stream=s)
            tc.update_probs()
            cur = tc.sample_layers(0)

            def tstep(k):
                nonlocal cur
                if k % T_s == 0:                       # period boundary
                    tc.update_probs()
                    cur = tc.sample_layers(k // T_s + 1)
                    if mode == "prefetch":
                        tc.prefetch_layers(cur, stream=s)   # moves during fwd/bwd
                if mode == "step_prefetch":
                    # the paper's per-step round trip with its prefetch: fetch the
                    # trainable layers' m/v during the forward, update each as soon
                    # as the backward has produced its gradient, write back at once
                    tc.prefetch_layers(cur, stream=s)
                if mode in ("offload_bwd", "step_prefetch"):
                    # per-step round trip of each trainable layer's m/v, issued on a
                    # side stream the moment backward has produced its gradient:
                    # fetch / update / write-back overlap the rest of the backward
                    def ready(l):
                        if l in cur:
                            e = torch.cuda.Event()
                            e.record(s)
                            side.wait_event(e)
                            tc.step_layers([l], [params[l]], [grads[l]], args.lr, stream=side)
                    fwd_bwd_layerwise(ready)
                    s.wait_stream(side)
                    return
                fwd_bwd()
                tc.step_layers(cur, [params[l] for l in cur], [grads[l] for l in cur], args.lr, stream=s)
            for k in range(1, 4):                     # warm (no boundary: the window was just committed)
                tstep(k)
            torch.cuda.synchronize()
            barrier(world)
            t0_, t1_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            t0_.record(s)
            for k in range(nsteps):
                tstep(T_s + k)                        # two period boundaries in the window
            tc.sync()                                 # + background write-backs (STEP_PREFETCH) of the last step
            t1_.record(s)
            torch.cuda.synchronize()
            return max_over_ranks(t0_.elapsed_time(t1_) / 1e3, world, dev) / nsteps * 1e3

        e0_, e1_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        fwd_bwd()
        e0_.record(s)
        fwd_bwd()
        e1_.record(s)
        torch.cuda.synchronize()
        res = {"standin": f"{n_mm} bf16 GEMMs 8192^3 = {n_mm * 2 * 8192 ** 3:.3g} FLOP "
                          "(LLaMA-2-7B fwd+bwd, 4 x 1024 tokens; SYNTHETIC)",
               "standin_ms": e0_.elapsed_time(e1_), "schedule": f"T_s=T_u={T_s}, {nsteps} steps"}
        ctx_cache = {}
        for mode in ("resident", "prefetch", "offload", "offload_bwd", "step_prefetch"):
            res[f"{mode}_step_ms"] = run(mode)
        for c_ in ctx_cache.values():
            c_.close()
        torch.cuda.empty_cache()
        res["period_prefetch_over_resident"] = res["prefetch_step_ms"] / res["resident_step_ms"]
        res["per_step_offload_over_resident"] = res["offload_step_ms"] / res["resident_step_ms"]
        res["per_step_offload_during_backward_over_resident"] = res["offload_bwd_step_ms"] / res["resident_step_ms"]
        res["per_step_round_trip_with_prefetch_over_resident"] = res["step_prefetch_step_ms"] / res["resident_step_ms"]
        res["offloaded_within_10pct_of_resident"] = res["period_prefetch_over_resident"] <= 1.10
        return res

    train = guarded("train", leg_train)

    # ---- bf16 params/grads with fp32 master + moments
    def leg_bf16():
        params.clear()                            # the fp32 buffers are not needed any more
        grads.clear()
        torch.cuda.empty_cache()
        p16 = [layer_params(n_p, l, device=dev, norm_numel=shape.norm_numel).to(torch.bfloat16)
               for l in range(NL)]
        g16 = [layer_grad(n_p, l, sig[l], step=0, device=dev, rank=rank).to(torch.bfloat16)
               for l in range(NL)]
        bctx = G.Grass([n_p] * NL, gamma=gamma, T_p=1, T_s=1, T_u=1, seed=1234, device=local,
                       rank=rank, world=world, param_dtype=G.DTYPE_BF16)
        bp = []
        for _ in range(6):                       # bf16 probing pass (K1, 2 B/param)
            e = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
            e[0].record(s)
            bctx.mgn_accumulate(list(range(NL)), g16, stream=s)
            e[1].record(s)
            bp.append(e)
        torch.cuda.synchronize()
        bprobe_ms = statistics.median(a.elapsed_time(b) for a, b in bp[1:])
        bctx.update_probs()
        bids = bctx.sample_layers(0)
        bev = []

        def bstep(step, timing):
            nonlocal bids
            if timing:
                e = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                e[0].record(s)
            bctx.step_layers(bids, [p16[l] for l in bids], [g16[l] for l in bids], args.lr, stream=s)
            if timing:
                e[1].record(s)
                bev.append(e)
            bctx.update_probs()
            bids = bctx.sample_layers(step + 1)
        for w in range(args.warmup):
            bstep(w, False)
        torch.cuda.synchronize()
        barrier(world)
        b0, b1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        b0.record(s)
        for k in range(args.steps):
            bstep(args.warmup + k, True)
        b1.record(s)
        torch.cuda.synchronize()
        bt = max_over_ranks(b0.elapsed_time(b1) / 1e3, world, dev)
        bk = statistics.mean(a.elapsed_time(b) for a, b in bev)
        bgbs = BYTES_PER_PARAM_UPDATE * active / world / (bk / 1e3) / 1e9
        bctx.close()
        try:
            bmix = measure_mix_ceiling(dev, n=gamma * n_p // world, bf16=True)
        except Exception as ex:  # recorded, never fatal to the leg
            bmix = {"error": f"{type(ex).__name__}: {ex}"[:300]}
        return {"workload": f"{args.model}-stack gamma={gamma} bf16 params/grads, fp32 master+m+v, resident",
                "mix_ceiling": bmix,
                "frac_mix_ceiling": bgbs / bmix["GBps"] if bmix.get("GBps") else None,
                "params_per_s": args.steps * active / bt, "step_ms": bt / args.steps * 1e3,
                "kernel_ms": bk, "GBps": bgbs, "frac_hbm": bgbs / hbm_peak,
                "bytes_per_param": BYTES_PER_PARAM_UPDATE,
                "probe_ms": bprobe_ms, "probe_GBps": 2 * NL * n_p / world / (bprobe_ms / 1e3) / 1e9,
                "probe_frac_read_peak": (2 * NL * n_p / world / (bprobe_ms / 1e3) / 1e9 / read_ceiling["GBps"]
                                         if read_ceiling and read_ceiling.get("GBps") else None),
                "probe_frac_nominal_8TBps": 2 * NL * n_p / world / (bprobe_ms / 1e3) / 1e9 / 8000.0}

    # P2P runs after the other multi-GPU legs: at N > 1 it is the one leg whose
    # data path (peer memory over CUDA IPC) could not be run on the 1-GPU pool,
    # so an exception in it is recorded instead of costing the line
    try:
        p2p = guarded("p2p", leg_p2p)
    except Exception as ex:
        p2p = {"error": f"{type(ex).__name__}: {ex}"[:300]}
    bf16 = guarded("bf16", leg_bf16)

    # ---- CPU oracle baseline (rank 0, N = 1 only)
    def leg_cpu():
        sample = 1 << 23
        times = oracle_sample_time(n_p, gamma, sample, args.lr, reps=2)
        v = gamma * sample / min(times)
        res = {"value": v, "unit": UNIT, "cores": 1, "kind": "oracle", "host_cores": os.cpu_count(),
               "sample": f"{gamma} x {sample} elements of one step (fp64 norm + AdamW) + commit/"
                         f"softmax/sampling over {NL} layers, best of 2, single thread"}
        try:
            res["all_cores"] = oracle_all_cores(gamma, sample, args.lr)
        except Exception as ex:
            res["all_cores"] = {"error": f"{type(ex).__name__}: {ex}"[:300]}
        return res

    cpu = guarded("cpu", leg_cpu) if (rank == 0 and world == 1) else None

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": elapsed / args.steps * 1e3,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic",
            "config": workload_config(args.model, gamma, world),
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm_peak, "unit": "GB/s",
                         "frac": achieved / hbm_peak, "traffic": traffic,
                         "kernel": "grass_stream_kernel<true,1,2> (fused Eq.2 norm + AdamW, TMA bulk-copy ring); "
                                   + ("kernel_ms = the timed region's mean device step (K2 + K3 with the fused "
                                      "commit + resample)" if use_dev else
                                      "kernel_ms = events around one step's launches (prologue, K2, K3)"),
                         "kernel_ms": kernel_ms, "peak_kind": peak_kind,
                         "traffic_source": "ncu --set full dram__bytes_read.sum + dram__bytes_write.sum of this "
                                           "kernel at this config (profiles/ncu_traffic.json, from "
                                           "profiles/r02_ncu_full.md)" if traffic else None,
                         "algorithmic_bytes_per_launch": BYTES_PER_PARAM_UPDATE * active // world,
                         "mix_ceiling": mix_ceiling,
                         "frac_mix_ceiling": achieved / mix_ceiling["GBps"] if mix_ceiling.get("GBps") else None},
            "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches,
            "step_driver": ("grass_device_step: update of the layers sampled on the device, then the commit "
                            "(Eq. 2/4/3) and resample kernel — no host round trip between steps"
                            if use_dev else "host: grass_step_layers + grass_update_probs + grass_sample_layers"),
            # world > 1: the NCCL gradient exchange (grouped send/recv of the
            # slices, summed in rank order by the update kernel) + all-gather of
            # the parameters, (W-1)/W of 4 B per active parameter each, per rank
            "dp_comm": ({"bytes_per_rank_per_step": 8 * active * (world - 1) // world,
                         "GBps_per_rank": 8 * active * (world - 1) / world / (elapsed / args.steps) / 1e9}
                        if world > 1 else None),
            "clocks": clk.summary(), "probe": out.get("probe"), "offload": offload,
            "offload_period": offload_period, "bf16": bf16, "train_step": train, "p2p": p2p,
            "paper_schedule": paper_schedule, "host_schedule": host_schedule,
            "paper_context": {
                "hardware": "2 x H100 80GB, precision not stated (PAPER.md:410)",
                "overlap_speedup": {"paper": 1.08, "what": "training throughput, overlapped vs "
                                    "non-overlapped offload, LLaMA2-7B b4 s1024 (PAPER.md:355)",
                                    "this_run": (offload or {}).get("overlap_speedup"),
                                    "this_run_what": "optimizer step alone (configs[2]), vanilla / overlapped"},
                "optimizer_state_hbm_growth_gamma_2_to_4_GB": {
                    "paper_LISA": 1.63, "paper_GRASS": 0.14, "source": "PAPER.md:261,270 (Table 4)",
                    "this_run": (((offload or {}).get("device_state_bytes_2x_gamma", 0) -
                                  (offload or {}).get("device_state_bytes", 0)) / 1e9) if offload else None},
                "grass_overhead_pct_of_training": {"paper": 2.01, "what": "probing + MGN update, "
                                                   "LLaMA2-7B (PAPER.md:367, Table 5)"},
            },
        }
        if leg_errors:
            line["leg_errors"] = leg_errors
        print(json.dumps(line), flush=True)


def measure_duplex(dev) -> float:
    """Pinned H2D || D2H copy bandwidth per direction (GB/s), plumbing only."""
    import torch
    n = 1 << 28
    h1 = torch.empty(n, dtype=torch.float32, pin_memory=True)
    h2 = torch.empty(n, dtype=torch.float32, pin_memory=True)
    d1 = torch.empty(n, dtype=torch.float32, device=dev)
    d2 = torch.empty(n, dtype=torch.float32, device=dev)
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


def main():
    args = parse()
    rank, world, local = dist_setup(args)
    if args.impl == "reference":
        run_reference(args, rank, world)
    else:
        run_grass(args, rank, world, local)
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
