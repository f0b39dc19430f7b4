"""Debug: NCCL grouped send/recv to self on a 1-rank communicator (the NCCL
data path's gradient exchange at world 1), raw and through the library, eager
and captured.  Each stage runs in its own process under a timeout.
    python tools/dbg_nccl_a2a.py [stage]
"""
import ctypes as C
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def raw():
    import torch
    torch.cuda.init()
    nccl = C.CDLL("libnccl.so.2", mode=C.RTLD_GLOBAL)

    class Uid(C.Structure):
        _fields_ = [("internal", C.c_char * 128)]
    uid = Uid()
    assert nccl.ncclGetUniqueId(C.byref(uid)) == 0
    comm = C.c_void_p()
    nccl.ncclCommInitRank.argtypes = [C.POINTER(C.c_void_p), C.c_int, Uid, C.c_int]
    r = nccl.ncclCommInitRank(C.byref(comm), 1, uid, 0)
    print("init", r, flush=True)
    a = torch.arange(1 << 20, dtype=torch.float32, device="cuda")
    b = torch.zeros_like(a)
    s = torch.cuda.current_stream().cuda_stream
    print("groupstart", nccl.ncclGroupStart(), flush=True)
    print("send", nccl.ncclSend(C.c_void_p(a.data_ptr()), C.c_size_t(a.numel()), 7, 0, comm, C.c_void_p(s)), flush=True)
    print("recv", nccl.ncclRecv(C.c_void_p(b.data_ptr()), C.c_size_t(b.numel()), 7, 0, comm, C.c_void_p(s)), flush=True)
    print("groupend", nccl.ncclGroupEnd(), flush=True)
    torch.cuda.synchronize()
    print("raw self send/recv equal:", bool(torch.equal(a, b)), flush=True)


def lib(capture, order="graph_first"):
    import torch
    import paper_2604_07808_b200 as G
    from synth import layer_grad, layer_params
    numel = [4096 * 4, 8192 + 64]
    gr = G.Grass(numel, gamma=2, force_nccl=True)
    ref = G.Grass(numel, gamma=2)
    p = [layer_params(n, l, device="cuda") for l, n in enumerate(numel)]
    q = [x.clone() for x in p]
    g = [layer_grad(n, l, 1e-3, device="cuda") for l, n in enumerate(numel)]
    print("ctx ok", flush=True)
    gr.mgn_accumulate([0, 1], g)
    gr.sync()
    print("probe ok", flush=True)
    gr.step_layers([0, 1], p, g, 1e-3)
    ref.step_layers([0, 1], q, g, 1e-3)
    gr.sync()
    print("eager step ok, equal:", all(torch.equal(a, b) for a, b in zip(p, q)), flush=True)
    if capture:
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph):
            gr.step_layers([0, 1], p, g, 1e-3, stream=torch.cuda.current_stream())
        print("captured", flush=True)
        graph.replay()
        torch.cuda.synchronize()
        print("replay ok", flush=True)
        if order == "graph_first":
            del graph
            torch.cuda.synchronize()
            gr.close()
        else:
            gr.close()
            del graph
        print("closed", order, flush=True)


if __name__ == "__main__":
    if len(sys.argv) > 1:
        {"raw": raw, "lib": lambda: lib(False), "cap": lambda: lib(True),
         "cap_ctx_first": lambda: lib(True, "ctx_first")}[sys.argv[1]]()
        sys.exit(0)
    for st in ("raw", "lib", "cap", "cap_ctx_first"):
        env = dict(os.environ, NCCL_DEBUG="WARN")
        try:
            r = subprocess.run([sys.executable, __file__, st], capture_output=True, text=True, timeout=90, env=env)
            print(f"== {st}: rc={r.returncode}\n{r.stdout[-2000:]}\n{r.stderr[-2000:]}", flush=True)
        except subprocess.TimeoutExpired as e:
            print(f"== {st}: TIMEOUT\n{(e.stdout or b'')[-2000:]}\n{(e.stderr or b'')[-2000:]}", flush=True)
