"""The race checker of the GPU offload test (tests/race_check.py) on
hand-written traces: ordered pairs pass, an overlapping pair on the same state
is reported, disjoint state is not compared (CPU only)."""
from race_check import happens_before_violations


def test_race_checker_detects_an_unordered_pair():
    """The checker itself: two operations on one state range whose GPU
    intervals overlap are reported; ordered ones are not."""
    e = lambda k, t0, t1, dev, host: {"kind": k, "layer": 0, "offset": 0, "count": 16, "start_ms": t0,
                                      "end_ms": t1, "state_dev": dev, "state_host": host}
    ok = [e("h2d", 0.0, 1.0, 4096, 65536), e("update", 1.0, 2.0, 4096, 0), e("d2h", 2.0, 3.0, 4096, 65536)]
    bad, checked = happens_before_violations(ok)
    assert not bad and checked == 4          # 3 on the device copy, 1 on the host copy
    racy = [e("h2d", 0.0, 1.0, 4096, 65536), e("update", 0.5, 2.0, 4096, 0)]
    assert happens_before_violations(racy)[0]
    disjoint = [e("h2d", 0.0, 1.0, 4096, 65536), e("update", 0.5, 2.0, 4096 + 64, 0)]
    assert not happens_before_violations(disjoint)[0] and happens_before_violations(disjoint)[1] == 0
