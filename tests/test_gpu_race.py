"""Race check of the offload pipeline on the GPU timeline (SURVEY §5 race
detection; "no update before its shard arrives"; VERDICT r1 item
6).  compute-sanitizer is not run on this pool (runs under it left GPUs
needing a reset — a dead GPU would close the round's GPU tests), so the
hazards are checked from the library's own trace instead: every traced
operation carries the state range it touches — the device copy (ring slot,
cache slot or resident state) and the pinned host copy — and its [start, end)
on the GPU.  For every pair of operations on overlapping state with at least
one writer (fetch: host read, device write; update: device read + write;
write-back: device read, host write), the one issued first must END before the
later one STARTS.  Under stress — 2-slot rings, chunks of 2 tiles, layers
revisited in consecutive steps (a single-chunk layer among them), prefetches that evict, background write-backs, random
busy work injected on the caller stream — across per-step offload, period
residency and the per-step round trip with prefetch, fp32 and bf16; the final
states must also equal the resident run bit for bit."""
import numpy as np
import pytest
import torch

import paper_2604_07808_b200 as G
from race_check import happens_before_violations
from synth import layer_grad, layer_params

pytestmark = pytest.mark.gpu
DEV = "cuda:0"


@pytest.fixture(autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    torch.cuda.set_device(0)


def _busy(ms_scale):
    a = torch.randn(2048, 2048, device=DEV)
    for _ in range(ms_scale):
        a = a @ a.T * 1e-3


@pytest.mark.parametrize("dtype", [G.DTYPE_FP32, G.DTYPE_BF16])
@pytest.mark.parametrize("residency", [G.RESIDENCY_STEP, G.RESIDENCY_PERIOD, G.RESIDENCY_STEP_PREFETCH])
def test_offload_pipeline_happens_before_under_stress(dtype, residency):
    rng = np.random.default_rng(7 + residency + 10 * dtype)
    tdt = torch.bfloat16 if dtype == G.DTYPE_BF16 else torch.float32
    numel = [4096 * 9 + 8, 4096 * 5, 4096 * 12, 4096 * 7 + 24, 4096 * 2]   # layer 4: a single chunk
    kw = dict(gamma=2, weight_decay=0.01, param_dtype=dtype, offload=True, chunk_elems=8192, ring_slots=2,
              residency=residency)
    if residency != G.RESIDENCY_STEP:
        kw["cache_layers"] = 2
    gr = G.Grass(numel, **kw)
    ref = G.Grass(numel, gamma=2, weight_decay=0.01, param_dtype=dtype)
    pr = [layer_params(n, l, device=DEV).to(tdt) for l, n in enumerate(numel)]
    pg = [p.clone() for p in pr]
    gr.trace_enable(True)
    total_checked, all_bad = 0, []
    for step in range(16):
        ids = [int(x) for x in rng.choice(len(numel), size=2, replace=False)]
        if step % 4 in (1, 2):   # the single-chunk layer alone in consecutive steps: its next fetch
            ids = [4]              # lands in another ring slot than its last write-back
        if residency != G.RESIDENCY_STEP and rng.random() < 0.5:   # a prefetch that may evict
            gr.prefetch_layers([int(x) for x in rng.choice(len(numel), size=2, replace=False)])
        if residency == G.RESIDENCY_STEP_PREFETCH and rng.random() < 0.7:
            gr.prefetch_layers(ids)
        if rng.random() < 0.5:
            _busy(int(rng.integers(1, 4)))                            # jitter on the caller stream
        grads = [layer_grad(numel[l], l, 1e-3, step=step, device=DEV).to(tdt) for l in ids]
        gr.step_layers(ids, [pg[l] for l in ids], grads, 1e-3)
        ref.step_layers(ids, [pr[l] for l in ids], grads, 1e-3)
        if step % 4 == 3:
            tr = gr.trace_read()
            bad, checked = happens_before_violations(tr)
            all_bad += bad
            total_checked += checked
    tr = gr.trace_read()
    bad, checked = happens_before_violations(tr)
    all_bad += bad
    total_checked += checked
    gr.trace_enable(False)
    assert not all_bad, all_bad[:5]
    assert total_checked > 20                      # the hazards were there to check
    torch.cuda.synchronize()
    for l in range(len(numel)):                    # and the result is the resident one
        assert torch.equal(pr[l], pg[l]), l
        a, b = ref.read_state(l), gr.read_state(l)
        assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
