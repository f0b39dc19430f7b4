"""The schedule driver (paper_2604_07808_b200/schedule.py) on CPU with a
recording stand-in for the context: the call sequence must follow
PAPER.md:111-121 (probe T_p steps, commit + resample at T_p, resample every
T_s, commit every T_u), the sampled periods must be consecutive, and prefetch
is issued at each resample under period residency."""
import types

import pytest

from paper_2604_07808_b200 import GrassSchedule


class FakeGrass:
    def __init__(self, n_layers, T_p, T_s, T_u, offload=0, residency=0):
        self.n_layers = n_layers
        self.cfg = types.SimpleNamespace(T_p=T_p, T_s=T_s, T_u=T_u, offload=offload, residency=residency)
        self.calls = []

    def update_probs(self):
        self.calls.append(("commit",))
        return [1.0 / self.n_layers] * self.n_layers

    def sample_layers(self, period):
        self.calls.append(("sample", period))
        return [period % self.n_layers, (period + 1) % self.n_layers]

    def prefetch_layers(self, ids, stream=None):
        self.calls.append(("prefetch", tuple(ids)))

    def mgn_accumulate(self, ids, grads, stream=None):
        self.calls.append(("probe", len(ids)))

    def step_layers(self, ids, params, grads, lr, stream=None):
        self.calls.append(("update", tuple(ids)))


@pytest.mark.parametrize("period_res", [False, True])
def test_schedule_call_sequence(period_res):
    g = FakeGrass(4, T_p=3, T_s=2, T_u=4, offload=int(period_res), residency=int(period_res))
    s = GrassSchedule(g)
    for step in range(11):
        layers = s.begin_step(step)
        s.end_step(step, [None] * len(layers), [None] * len(layers), 1e-3)
    kinds = [c[0] for c in g.calls]
    assert kinds[:3] == ["probe"] * 3                                  # T_p probing steps
    commits = [i for i, c in enumerate(g.calls) if c[0] == "commit"]
    samples = [c[1] for c in g.calls if c[0] == "sample"]
    assert samples == [0, 1, 2, 3]                                     # resamples at steps 3, 5, 7, 9
    assert len(commits) == 2                                           # commits at 3 and 7 (T_u = 4)
    from oracle import grass_oracle as O                               # same decisions as the oracle
    want = [O.schedule_decision(t, 3, 2, 4) for t in range(11)]
    assert want.count("commit+resample") == 2 and want.count("resample") == 2
    assert ("prefetch" in kinds) == period_res
    assert kinds.count("update") == 8


def test_schedule_paper_values():
    g = FakeGrass(32, T_p=150, T_s=25, T_u=25)
    s = GrassSchedule(g)
    for step in range(0, 226):
        layers = s.begin_step(step)
        s.end_step(step, [None] * len(layers), [None] * len(layers), 3e-5)
    samples = [c[1] for c in g.calls if c[0] == "sample"]
    assert samples == [0, 1, 2, 3]                                     # steps 150, 175, 200, 225
    assert sum(1 for c in g.calls if c[0] == "probe") == 150


def test_schedule_always_groups_join_every_update_and_skip_probing():
    # R19: always-active groups (embedding / head) are not probed or sampled;
    # every adaptive step's update lists them after the sampled set.
    g = FakeGrass(4, T_p=2, T_s=2, T_u=2)
    g.n_layers = 6
    g.always_ids = [4, 5]
    s = GrassSchedule(g)
    seen = []
    for step in range(6):
        layers = s.begin_step(step)
        seen.append(layers)
        s.end_step(step, [None] * len(layers), [None] * len(layers), 1e-3)
    assert seen[0] == seen[1] == [0, 1, 2, 3]                      # probing: sampled layers only
    for layers in seen[2:]:
        assert layers[-2:] == [4, 5] and len(layers) == 4
    updates = [c[1] for c in g.calls if c[0] == "update"]
    assert all(u[-2:] == (4, 5) for u in updates) and len(updates) == 4
    assert [c for c in g.calls if c[0] == "probe"] == [("probe", 4), ("probe", 4)]


def test_schedule_prob_trace_jsonl(tmp_path):
    # SPEC.md:313 prob-trace: one JSON line per commit (m, p) and per resample (sampled ids)
    import json
    g = FakeGrass(4, T_p=2, T_s=2, T_u=4)
    path = tmp_path / "probs.jsonl"
    s = GrassSchedule(g, trace_path=str(path))
    for step in range(9):
        layers = s.begin_step(step)
        s.end_step(step, [None] * len(layers), [None] * len(layers), 1e-3)
    recs = [json.loads(line) for line in path.read_text().splitlines()]
    assert [r["event"] for r in recs] == ["commit", "resample", "resample", "commit", "resample",
                                         "resample"]
    assert [r["step"] for r in recs] == [2, 2, 4, 6, 6, 8]
    assert recs[0]["p"] == [0.25] * 4 and recs[1]["sampled"] == [0, 1] and recs[2]["period"] == 1
