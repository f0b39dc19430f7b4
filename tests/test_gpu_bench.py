"""bench.py end to end on a small stack with the same block layout
(`--model tiny-bench`): every default leg runs without a recorded error and
the JSON line carries the contract's keys (roofline, cpu_baseline, e2e with
host<->device bytes, gpu_launches, clocks); the reference arm prints its line.
Catches a broken leg before the driver's full-size run does."""
import json
import os
import subprocess
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(*extra):
    r = subprocess.run([sys.executable, "bench.py", "--model", "tiny-bench", "--steps", "3", "--warmup", "3", *extra],
                       cwd=ROOT, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    return json.loads(lines[0])


@pytest.fixture(autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def test_bench_all_default_legs_run():
    d = _run()
    assert not d.get("leg_errors"), d.get("leg_errors")
    assert d["value"] > 0 and d["ms_per_step"] > 0 and d["n_gpus"] == 1
    r = d["roofline"]
    for k in ("bound", "achieved", "peak", "unit", "frac", "traffic", "mix_ceiling"):
        assert k in r, k
    assert r["frac"] == pytest.approx(r["achieved"] / r["peak"])
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    e = d["e2e"]
    assert e and e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    assert d["gpu_launches"] > 0
    assert d["clocks"]["samples"] > 0
    for leg in ("probe", "offload", "offload_period", "bf16", "p2p", "host_schedule", "paper_schedule"):
        assert d.get(leg), leg


def test_bench_reference_arm_prints_its_line():
    d = _run("--impl", "reference")
    assert d["impl"] == "reference" and d["value"] > 0
    assert d["cpu_baseline"]["kind"] == "oracle"
    assert d["e2e"]["h2d_bytes_per_step"] == 0
