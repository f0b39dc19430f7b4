"""World-size-2 CPU test (gloo) of the host side of P2P data parallelism
(Grass.p2p_setup): every rank exports its exchange block and its
layer buffers, the handles are all-gathered over the process group, and each
rank attaches / registers the [world] address tables with its OWN addresses at
index `rank` and the imported peer addresses elsewhere, in rank order.

CUDA IPC itself needs a GPU (tests/test_gpu_p2p.py::test_p2p_two_processes_ipc);
here ipc_export / ipc_import are replaced by a deterministic stand-in so that
the exchange logic runs on CPU.
"""
import os
import socket
import sys
import types

import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


class _Buf:
    def __init__(self, addr):
        self.addr = addr

    def data_ptr(self):
        return self.addr


def _addr(rank, kind, layer=0):
    return (rank + 1) * 1_000_000 + kind * 10_000 + layer * 16


def _worker(rank, world, port, q):
    try:
        sys.path.insert(0, ROOT)
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        import paper_2604_07808_b200.binding as B

        # stand-in IPC: the "handle" names the exporting address; importing it
        # in this process maps it to a recognisable peer address
        B.ipc_export = lambda ptr: (f"h{ptr}".encode().ljust(64, b"\0"), 0)
        B.ipc_import = lambda dev, h, off: 7_000_000_000 + int(h.rstrip(b"\0")[1:]) + off
        calls = {"attach": None, "reg": {}}
        fake = types.SimpleNamespace(world=world, rank=rank, cfg=types.SimpleNamespace(device=0))
        fake.p2p_exchange_block = lambda: (_addr(rank, 0), 4096)
        fake.p2p_attach = lambda blocks: calls.__setitem__("attach", list(blocks))
        fake.p2p_register_layer = lambda l, ps, gs: calls["reg"].__setitem__(l, (list(ps), list(gs)))
        bufs = {l: (_Buf(_addr(rank, 1, l)), _Buf(_addr(rank, 2, l))) for l in (0, 3, 5)}
        B.Grass.p2p_setup(fake, bufs)
        q.put((rank, calls))
        dist.destroy_process_group()
    except Exception as ex:  # surfaced by the parent
        q.put((rank, repr(ex)))


def test_p2p_setup_exchanges_address_tables_world2():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    imp = 7_000_000_000
    for r in range(world):
        calls = res[r]
        assert isinstance(calls, dict), calls
        # blocks: own address at index r, the peer's (imported) elsewhere
        want = [_addr(q_, 0) if q_ == r else imp + _addr(q_, 0) for q_ in range(world)]
        assert calls["attach"] == want
        assert sorted(calls["reg"]) == [0, 3, 5]
        for l, (ps, gs) in calls["reg"].items():
            assert ps == [_addr(q_, 1, l) if q_ == r else imp + _addr(q_, 1, l) for q_ in range(world)]
            assert gs == [_addr(q_, 2, l) if q_ == r else imp + _addr(q_, 2, l) for q_ in range(world)]
