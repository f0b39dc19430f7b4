"""Happens-before check of the offload pipeline's trace (test infrastructure;
used by tests/test_gpu_race.py, pinned on CPU by tests/test_race_check_host.py).

Every traced operation carries the optimizer-state range it touches: the
device copy (ring slot, cache slot or resident state, `state_dev`) and the
pinned host copy (`state_host`), as addresses of its m array (v / master
follow the same layout).  Accesses: fetch (h2d) reads the host copy and writes
the device copy; the update reads and writes the device copy; the write-back
(d2h) reads the device copy and writes the host copy.  For every pair of
operations on overlapping state with at least one writer, the one issued first
must END before the later one STARTS on the GPU timeline.
"""
ACCESS = {"h2d": (("host", "r"), ("dev", "w")), "update": (("dev", "rw"),), "d2h": (("dev", "r"), ("host", "w"))}


def happens_before_violations(tr, esz=4, eps_ms=2e-3):
    """(violations, pairs checked) of the rule above on one trace."""
    ops = []
    for i, e in enumerate(tr):
        if e["kind"] not in ACCESS:
            continue
        for space, mode in ACCESS[e["kind"]]:
            base = e["state_dev"] if space == "dev" else e["state_host"]
            if base:
                ops.append((i, space, base, base + esz * e["count"], mode, e))
    bad, checked = [], 0
    for a in range(len(ops)):
        ia, sa, lo_a, hi_a, ma, ea = ops[a]
        for b in range(a + 1, len(ops)):
            ib, sb, lo_b, hi_b, mb, eb = ops[b]
            if ib == ia or sa != sb or hi_a <= lo_b or hi_b <= lo_a or ("w" not in ma and "w" not in mb):
                continue
            checked += 1
            if ea["end_ms"] > eb["start_ms"] + eps_ms:
                bad.append((ea["kind"], ea["layer"], ea["offset"], eb["kind"], eb["layer"], eb["offset"],
                            ea["end_ms"], eb["start_ms"]))
    return bad, checked
