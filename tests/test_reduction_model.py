"""Host model of the two warp reductions in csrc/kernels.cu (no GPU):
`warp_sum` (shfl_down tree, lane 0's result) and `warp_sum_multi` (the
transposed butterfly that reduces the sums of all tiles of a unit at once).
DESIGN §8 claims every tile sum of the latter is bit-identical to the former —
the same pairs of lane groups are added at every level, and IEEE addition is
commutative.  This checks the pairing argument on the algorithm itself with
fp64 values spanning many magnitudes (cancellation included), for every
N = 1..16; the kernels are checked against each other on the GPU by
tests/test_gpu_parity.py::test_norms_probe_equals_update_bitwise."""
import numpy as np
import pytest


def warp_sum_down(x):
    """lane 0 of: for o in 16, 8, 4, 2, 1: x[i] += x[i + o] (shfl_down; lanes
    i + o >= 32 read their own value, which never reaches lane 0)."""
    x = list(x)
    for o in (16, 8, 4, 2, 1):
        x = [x[i] + (x[i + o] if i + o < 32 else x[i]) for i in range(32)]
    return x[0]


def slots(n):
    """C = next power of two >= n (the kernel's MultiSlots<N>::C), its log2."""
    c = 1
    while c < n:
        c *= 2
    return c, c.bit_length() - 1


def warp_sum_multi(vals, n):
    """vals[lane][t], t < n.  Returns out[lane] as the kernel's lanes hold it:
    split levels at o = 16, 8, ... (log2 C of them), then a plain butterfly."""
    C, LOG = slots(n)
    v = [[vals[l][t] if t < n else 0.0 for t in range(C)] for l in range(32)]
    c, o = C, 16
    while c > 1:
        new = [row[:] for row in v]
        for lane in range(32):
            up = (lane & o) != 0
            partner = lane ^ o
            pup = (partner & o) != 0
            for j in range(c // 2):
                send_p = v[partner][j] if pup else v[partner][j + c // 2]   # what the partner sends
                keep = v[lane][j + c // 2] if up else v[lane][j]
                new[lane][j] = keep + send_p
        v = new
        c //= 2
        o //= 2
    x = [v[lane][0] for lane in range(32)]
    o = 16 >> LOG
    while o > 0:
        x = [x[lane] + x[lane ^ o] for lane in range(32)]
        o //= 2
    return x


def holder(lane, n):
    """(tile index, writes?) of a lane after warp_sum_multi: the kernel's *slot."""
    C, LOG = slots(n)
    sh = 5 - LOG
    idx = (lane >> sh) & (C - 1)
    return idx, (lane & ((1 << sh) - 1)) == 0 and idx < n


@pytest.mark.parametrize("n", list(range(1, 17)))
def test_multi_equals_per_tile_tree_bitwise(n):
    rng = np.random.default_rng(n)
    for trial in range(20):
        mag = 10.0 ** rng.integers(-30, 30, size=(32, n))
        sign = rng.choice([-1.0, 1.0], size=(32, n)) if trial % 2 else 1.0
        vals = (rng.random((32, n)) * mag * sign).tolist()
        out = warp_sum_multi(vals, n)
        for t in range(n):
            want = warp_sum_down([vals[l][t] for l in range(32)])
            lanes = [l for l in range(32) if holder(l, n)[0] == t]     # the lanes that hold tile t
            assert sum(holder(l, n)[1] for l in lanes) == 1            # exactly one writes it
            for l in lanes:
                assert out[l] == want, (n, t, l)


def test_multi_result_lane_map():
    """N = 16: tile t's sum lands in lanes 2t and 2t + 1 (the kernel writes from the even one)."""
    vals = [[float(1 << l) * (t + 1) for t in range(16)] for l in range(32)]
    out = warp_sum_multi(vals, 16)
    for l in range(32):
        t = l >> 1
        assert out[l] == float((1 << 32) - 1) * (t + 1)
