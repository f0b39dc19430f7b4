"""Developer A/B: build variants of libgrass.so with compile-time knobs, then
time each with bench.py on the GPU (GRASS_LIB_PATH selects the variant).
    python tools/variants.py build
    python tools/variants.py run        # on the GPU box
"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
VARIANTS = {   # edit per experiment; the knobs are listed at the top of csrc/kernels.cu
    "base": [],
    "k3_nosampler": ["GRASS_K3_DIAG=3"],
}
OUTDIR = os.path.join(ROOT, "build", "variants")


def build():
    from paper_2604_07808_b200 import build as b
    os.makedirs(OUTDIR, exist_ok=True)
    for name, d in VARIANTS.items():
        b.build(force=True, defines=d, out=os.path.join(OUTDIR, f"libgrass_{name}.so"))
        print("built", name)


def run(legs="main,p2p", extra=()):
    res = {}
    for name in VARIANTS:
        env = dict(os.environ, GRASS_LIB_PATH=os.path.join(OUTDIR, f"libgrass_{name}.so"))
        r = subprocess.run([sys.executable, "bench.py", "--legs", legs, *extra], cwd=ROOT, env=env,
                           capture_output=True, text=True, timeout=600)
        try:
            d = json.loads(r.stdout.strip().splitlines()[-1])
            res[name] = {"kernel_ms": d["roofline"]["kernel_ms"], "frac": d["roofline"]["frac"],
                         "step_ms": d["ms_per_step"],
                         "probe_GBps": (d.get("probe") or {}).get("GBps"),
                         "bf16_kernel_ms": (d.get("bf16") or {}).get("kernel_ms"),
                         "p2p_probe_ms": (d.get("p2p") or {}).get("probe_call_ms"),
                         "bf16_probe_ms": (d.get("bf16") or {}).get("probe_ms"),
                         "p2p_call_ms": (d.get("p2p") or {}).get("call_ms")}
        except Exception:
            res[name] = {"error": r.stderr[-2000:]}
        print(name, res[name], flush=True)
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", "variants.json"), "w") as f:
        json.dump(res, f, indent=1)


if __name__ == "__main__":
    build() if sys.argv[1] == "build" else run()
