"""Mutation check of the GPU parity tests: libgrass variants built with
-DGRASS_MUTANT=k each plant one plausible kernel mistake (kernels.cu /
stream_kernel.cuh, `kMutant`); a fast subset of tests/test_gpu_parity.py and
tests/test_gpu_p2p.py must FAIL for every one of them.

    python tools/kernel_mutation.py build      # here (nvcc cross-compiles)
    python tools/kernel_mutation.py run        # on the GPU box
"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
OUTDIR = os.path.join(ROOT, "build", "mutants")
MUTANTS = {
    1: "AdamW: weight decay dropped",
    2: "AdamW: bias correction 1/sqrt(1-b2^t) dropped",
    3: "norm: one warp's partial left out of each tile sum",
    4: "ragged tail: last element of a segment skipped",
    5: "DP: gradient not scaled by 1/W",
    6: "P2P: last rank's gradient slice not summed",
    7: "bf16: parameter copy truncated instead of RNE",
    8: "step prologue: t_l not advanced (bias corrections of step 1 forever)",
    9: "P2P: theta' not stored into the last rank's parameters",
    10: "bf16: master never initialised from the bf16 parameter",
    11: "non-finite norm not flagged",
    12: "norm: all-tiles warp reduction (warp_sum_multi) pairs the wrong halves",
    13: "bf16 norm: the 4th square of each fp32 quad sum dropped",
}
TESTS = ("test_step_layers_vs_oracle_multi_step or test_norms_ragged_sizes_vs_oracle or "
         "test_bf16_mixed_precision_vs_oracle or test_p2p_virtual_ranks_vs_oracle or "
         "test_zero_grad_zero_state_is_identity_on_theta or test_nonfinite_gradient_reported_and_not_recorded or "
         "test_norms_probe_equals_update_bitwise or test_norms_integer_grads_exact_bf16")


def build():
    from paper_2604_07808_b200 import build as b
    os.makedirs(OUTDIR, exist_ok=True)
    for k in MUTANTS:
        b.build(force=True, defines=[f"GRASS_MUTANT={k}"], out=os.path.join(OUTDIR, f"libgrass_m{k}.so"))
        print("built mutant", k, flush=True)


def run():
    res = {}
    for k, what in MUTANTS.items():
        env = dict(os.environ, GRASS_LIB_PATH=os.path.join(OUTDIR, f"libgrass_m{k}.so"))
        r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-p", "no:cacheprovider",
                            "tests/test_gpu_parity.py", "tests/test_gpu_p2p.py", "-k", TESTS],
                           cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
        failed = [l for l in r.stdout.splitlines() if l.startswith("FAILED")]
        res[k] = {"mutation": what, "killed": r.returncode != 0, "by": failed[:1]}
        print(k, res[k], flush=True)
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", "kernel_mutation.json"), "w") as f:
        json.dump(res, f, indent=1)
    killed = sum(v["killed"] for v in res.values())
    print(f"{killed}/{len(res)} kernel mutations killed by the GPU parity tests")
    return 0 if killed == len(res) else 1


if __name__ == "__main__":
    sys.exit(build() if sys.argv[1:] == ["build"] else run())
