"""Thin ctypes binding of libgrass.so (include/grass.h).

Argument marshalling only: every step of the hot path runs in the library's
CUDA kernels / NCCL calls.  torch supplies device memory, streams and process
groups.  There is NO fallback: if libgrass.so is missing or fails to load,
every entry point raises.
"""
from __future__ import annotations

import ctypes as C
import os
from typing import Sequence

_PKG = os.path.dirname(os.path.abspath(__file__))
# GRASS_LIB_PATH: developer override to load an A/B build variant of the same
# library (tools/variants.py); the default is the in-tree product build.
LIB_PATH = os.environ.get("GRASS_LIB_PATH") or os.path.join(_PKG, "libgrass.so")

OK, E_INVALID, E_STATE, E_CUDA, E_NCCL, E_OOM, E_NONFINITE, E_IO = range(8)
POLICY_ADAPTIVE, POLICY_STATIC, POLICY_UNIFORM = range(3)
DECIDE_PROBE, DECIDE_COMMIT_RESAMPLE, DECIDE_RESAMPLE, DECIDE_CONTINUE = range(4)
RESIDENCY_STEP, RESIDENCY_PERIOD, RESIDENCY_STEP_PREFETCH = range(3)
DTYPE_FP32, DTYPE_BF16 = range(2)
DP_NCCL, DP_P2P = range(2)
IPC_HANDLE_BYTES = 64
NCCL_ID_BYTES = 128

_STATUS = {0: "GRASS_OK", 1: "GRASS_E_INVALID", 2: "GRASS_E_STATE", 3: "GRASS_E_CUDA",
           4: "GRASS_E_NCCL", 5: "GRASS_E_OOM", 6: "GRASS_E_NONFINITE", 7: "GRASS_E_IO"}


class GrassError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{_STATUS.get(status, status)}: {msg}")
        self.status = status


class TraceEvent(C.Structure):
    _fields_ = [("kind", C.c_int32), ("layer", C.c_int32), ("offset", C.c_int64),
                ("count", C.c_int64), ("start_ms", C.c_float), ("end_ms", C.c_float),
                ("state_dev", C.c_uint64), ("state_host", C.c_uint64)]


TRACE_KINDS = {0: "h2d", 1: "update", 2: "d2h", 3: "norm", 4: "rs", 5: "ag", 6: "p2p"}


class GrassConfig(C.Structure):
    _fields_ = [
        ("n_layers", C.c_int32), ("layer_numel", C.POINTER(C.c_int64)), ("gamma", C.c_int32),
        ("T_p", C.c_int32), ("T_s", C.c_int32), ("T_u", C.c_int32),
        ("tau", C.c_double), ("alpha", C.c_double), ("normalize_mgn", C.c_int32),
        ("policy", C.c_int32),
        ("beta1", C.c_double), ("beta2", C.c_double), ("eps", C.c_double),
        ("weight_decay", C.c_double), ("seed", C.c_uint64), ("device", C.c_int32),
        ("offload", C.c_int32), ("overlap", C.c_int32), ("chunk_elems", C.c_int64),
        ("ring_slots", C.c_int32), ("rank", C.c_int32), ("world", C.c_int32),
        ("nccl_unique_id", C.c_void_p), ("residency", C.c_int32), ("cache_layers", C.c_int32),
        ("max_grad_norm", C.c_double), ("param_dtype", C.c_int32), ("n_always", C.c_int32),
        ("dp_mode", C.c_int32), ("p2p_sync", C.c_int32), ("debug_check", C.c_int32),
    ]


_lib = None

# name -> (restype, argtypes)
_SIGS = {
    "grass_config_init": (C.c_int, [C.POINTER(GrassConfig)]),
    "grass_create": (C.c_int, [C.POINTER(GrassConfig), C.POINTER(C.c_void_p)]),
    "grass_destroy": (None, [C.c_void_p]),
    "grass_last_error": (C.c_char_p, [C.c_void_p]),
    "grass_sync": (C.c_int, [C.c_void_p]),
    "grass_mgn_accumulate": (C.c_int, [C.c_void_p, C.POINTER(C.c_int32), C.c_int32,
                                       C.POINTER(C.c_void_p), C.c_void_p]),
    "grass_update_probs": (C.c_int, [C.c_void_p, C.POINTER(C.c_double)]),
    "grass_sample_layers": (C.c_int, [C.c_void_p, C.POINTER(C.c_double), C.c_uint64,
                                      C.POINTER(C.c_int32)]),
    "grass_step_layers": (C.c_int, [C.c_void_p, C.POINTER(C.c_int32), C.c_int32,
                                    C.POINTER(C.c_void_p), C.POINTER(C.c_void_p), C.c_float,
                                    C.c_void_p]),
    "grass_read_state": (C.c_int, [C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p,
                                   C.POINTER(C.c_int64)]),
    "grass_write_state": (C.c_int, [C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p, C.c_int64]),
    "grass_flush_states": (C.c_int, [C.c_void_p]),
    "grass_prefetch_layers": (C.c_int, [C.c_void_p, C.POINTER(C.c_int32), C.c_int32, C.c_void_p]),
    "grass_mgn_accumulate_bf16": (C.c_int, [C.c_void_p, C.POINTER(C.c_int32), C.c_int32,
                                            C.POINTER(C.c_void_p), C.c_void_p]),
    "grass_step_layers_bf16": (C.c_int, [C.c_void_p, C.POINTER(C.c_int32), C.c_int32,
                                         C.POINTER(C.c_void_p), C.POINTER(C.c_void_p), C.c_float,
                                         C.c_void_p]),
    "grass_read_master": (C.c_int, [C.c_void_p, C.c_int32, C.c_void_p]),
    "grass_trace_enable": (C.c_int, [C.c_void_p, C.c_int32]),
    "grass_trace_read": (C.c_int, [C.c_void_p, C.POINTER(TraceEvent), C.c_int32,
                                   C.POINTER(C.c_int32)]),
    "grass_write_master": (C.c_int, [C.c_void_p, C.c_int32, C.c_void_p]),
    "grass_save_state": (C.c_int, [C.c_void_p, C.c_char_p]),
    "grass_load_state": (C.c_int, [C.c_void_p, C.c_char_p]),
    "grass_get_mgn": (C.c_int, [C.c_void_p, C.POINTER(C.c_double), C.POINTER(C.c_double),
                                C.POINTER(C.c_int64), C.POINTER(C.c_double),
                                C.POINTER(C.c_double)]),
    "grass_device_bytes": (C.c_int64, [C.c_void_p]),
    "grass_host_bytes": (C.c_int64, [C.c_void_p]),
    "grass_launch_count": (C.c_int64, [C.c_void_p]),
    "grass_tile_elems": (C.c_int64, []),
    "grass_version": (C.c_char_p, []),
    "grass_splitmix64": (C.c_uint64, [C.c_uint64]),
    "grass_uniform": (C.c_double, [C.c_uint64, C.c_uint64, C.c_uint32]),
    "grass_softmax_probs": (C.c_int, [C.POINTER(C.c_double), C.c_int32, C.c_double, C.c_int32,
                                      C.POINTER(C.c_double)]),
    "grass_sample_from_probs": (C.c_int, [C.POINTER(C.c_double), C.c_int32, C.c_int32,
                                          C.c_uint64, C.c_uint64, C.POINTER(C.c_int32)]),
    "grass_shard_range": (C.c_int, [C.c_int64, C.c_int32, C.c_int32, C.POINTER(C.c_int64),
                                    C.POINTER(C.c_int64)]),
    "grass_schedule_decision": (C.c_int32, [C.c_int64, C.c_int32, C.c_int32, C.c_int32]),
    "grass_nccl_get_unique_id": (C.c_int, [C.c_void_p]),
    "grass_p2p_exchange_block": (C.c_int, [C.c_void_p, C.POINTER(C.c_void_p), C.POINTER(C.c_int64)]),
    "grass_p2p_attach": (C.c_int, [C.c_void_p, C.POINTER(C.c_void_p)]),
    "grass_p2p_register_layer": (C.c_int, [C.c_void_p, C.c_int32, C.POINTER(C.c_void_p),
                                           C.POINTER(C.c_void_p)]),
    "grass_p2p_finish": (C.c_int, [C.c_void_p, C.c_void_p]),
    "grass_ipc_export": (C.c_int, [C.c_void_p, C.c_void_p, C.POINTER(C.c_int64)]),
    "grass_set_lr_device": (C.c_int, [C.c_void_p, C.c_void_p]),
    "grass_selftest_p2p": (C.c_int, [C.c_int32, C.c_int32, C.c_int32, C.POINTER(C.c_int64),
                                     C.POINTER(C.c_int32)]),
    "grass_ipc_import": (C.c_int, [C.c_int32, C.c_void_p, C.c_int64, C.POINTER(C.c_void_p)]),
    "grass_enable_peer_access": (C.c_int, [C.c_int32, C.c_int32]),
    "grass_register_layers": (C.c_int, [C.c_void_p, C.c_int32, C.POINTER(C.c_void_p), C.POINTER(C.c_void_p)]),
    "grass_device_schedule_begin": (C.c_int, [C.c_void_p, C.c_uint64, C.c_void_p]),
    "grass_device_step": (C.c_int, [C.c_void_p, C.c_float, C.c_int32, C.c_int32, C.c_uint64, C.c_void_p]),
    "grass_device_schedule_end": (C.c_int, [C.c_void_p, C.POINTER(C.c_int32)]),
}


def lib() -> C.CDLL:
    """Loads libgrass.so (raises if it was not built — there is no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} missing: run __graft_entry__.build() "
                              "(python -m paper_2604_07808_b200.build)")
        h = C.CDLL(LIB_PATH, mode=C.RTLD_GLOBAL)
        for name, (res, args) in _SIGS.items():
            f = getattr(h, name)
            f.restype = res
            f.argtypes = args
        _lib = h
    return _lib


def exported_symbols():
    return sorted(_SIGS)


def _check(status: int, ctx=None):
    if status != OK:
        msg = lib().grass_last_error(ctx)
        raise GrassError(status, msg.decode() if msg else "")


def _dbl(xs):
    return (C.c_double * len(xs))(*[float(x) for x in xs])


# ----------------------------------------------------------- context-free helpers
def tile_elems() -> int:
    return int(lib().grass_tile_elems())


def splitmix64(x: int) -> int:
    return int(lib().grass_splitmix64(x & ((1 << 64) - 1)))


def uniform(seed: int, period: int, k: int) -> float:
    return float(lib().grass_uniform(seed, period, k))


def softmax_probs(m: Sequence[float], tau: float, normalize: bool = True):
    out = (C.c_double * len(m))()
    _check(lib().grass_softmax_probs(_dbl(m), len(m), tau, int(normalize), out))
    return list(out)


def sample_from_probs(p: Sequence[float], gamma: int, seed: int, period: int):
    out = (C.c_int32 * gamma)()
    _check(lib().grass_sample_from_probs(_dbl(p), len(p), gamma, seed, period, out))
    return list(out)


def shard_range(numel: int, world: int, rank: int):
    off, cnt = C.c_int64(), C.c_int64()
    _check(lib().grass_shard_range(numel, world, rank, C.byref(off), C.byref(cnt)))
    return off.value, cnt.value


def schedule_decision(step: int, T_p: int, T_s: int, T_u: int | None = None) -> int:
    return int(lib().grass_schedule_decision(step, T_p, T_s, T_s if T_u is None else T_u))


def nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(NCCL_ID_BYTES)
    _check(lib().grass_nccl_get_unique_id(buf))
    return buf.raw


# ------------------------------------------------------------------ context
def _stream_ptr(stream) -> int:
    import torch
    if stream is None:
        stream = torch.cuda.current_stream()
    return int(stream.cuda_stream) if hasattr(stream, "cuda_stream") else int(stream)


def _ptrs(tensors, itemsize: int = 4, host_ok: bool = False):
    arr = (C.c_void_p * len(tensors))()
    for i, t in enumerate(tensors):
        on_dev = t.is_cuda or (host_ok and t.is_pinned())
        if not on_dev or not t.is_contiguous() or t.dtype.itemsize != itemsize:
            raise ValueError(f"layer buffers must be contiguous CUDA tensors of {itemsize}-byte "
                             "elements (fp32, or bf16 for a bf16 context)")
        arr[i] = t.data_ptr()
    return arr


def selftest_p2p(world: int, rounds: int = 100, device: int = 0):
    """(mismatched rows, timed out) of the P2P barrier protocol, emulated on one GPU."""
    mm, to = C.c_int64(), C.c_int32()
    _check(lib().grass_selftest_p2p(device, world, rounds, C.byref(mm), C.byref(to)))
    return mm.value, bool(to.value)


def ipc_export(ptr: int):
    """(64-byte CUDA IPC handle of the allocation containing ptr, byte offset)."""
    h = C.create_string_buffer(IPC_HANDLE_BYTES)
    off = C.c_int64()
    _check(lib().grass_ipc_export(C.c_void_p(ptr), h, C.byref(off)))
    return h.raw, off.value


def ipc_import(device: int, handle: bytes, offset: int) -> int:
    """Address (in this process) of an allocation exported by another process."""
    out = C.c_void_p()
    _check(lib().grass_ipc_import(device, handle, offset, C.byref(out)))
    return out.value


def enable_peer_access(device: int, peer: int):
    """Several ranks in one process (one thread per GPU): device may read /
    write peer's memory through plain pointers (P2P data path)."""
    _check(lib().grass_enable_peer_access(device, peer))


class Grass:
    """One GRASS hot-path context (one per process / GPU).

    Parameters mirror ``grass_config`` (include/grass.h).  For world > 1 pass a
    torch.distributed process group (any backend): rank 0 creates the NCCL id
    and it is broadcast through the group.
    """

    def __init__(self, layer_numel: Sequence[int], gamma: int, *, T_p: int = 150, T_s: int = 25,
                 T_u: int | None = None, tau: float = 1.0, alpha: float = 0.5,
                 normalize_mgn: bool = True, policy: int = POLICY_ADAPTIVE, beta1: float = 0.9,
                 beta2: float = 0.999, eps: float = 1e-8, weight_decay: float = 0.0,
                 seed: int = 1234, device: int = 0, offload: bool = False, overlap: bool = True,
                 chunk_elems: int = 0, ring_slots: int = 0, rank: int = 0, world: int = 1,
                 process_group=None, force_nccl: bool = False, residency: int = RESIDENCY_STEP,
                 cache_layers: int = 0, max_grad_norm: float = 0.0, param_dtype: int = DTYPE_FP32,
                 n_always: int = 0, dp_mode: int = DP_NCCL, p2p_sync: bool = True,
                 debug_check: bool = False, nccl_id: bytes | None = None):
        L = lib()
        self.layer_numel = [int(x) for x in layer_numel]
        self.n_layers = len(self.layer_numel)
        self.gamma = gamma
        # the last n_always entries are always-active groups (embedding, head; R19)
        self.n_always = int(n_always)
        self.n_sampled = self.n_layers - self.n_always
        self.always_ids = list(range(self.n_sampled, self.n_layers))
        self._numel = (C.c_int64 * self.n_layers)(*self.layer_numel)
        cfg = GrassConfig()
        _check(L.grass_config_init(C.byref(cfg)))
        cfg.n_layers = self.n_layers
        cfg.layer_numel = self._numel
        cfg.gamma = gamma
        cfg.T_p, cfg.T_s, cfg.T_u = T_p, T_s, (T_s if T_u is None else T_u)
        cfg.tau, cfg.alpha, cfg.normalize_mgn, cfg.policy = tau, alpha, int(normalize_mgn), policy
        cfg.beta1, cfg.beta2, cfg.eps, cfg.weight_decay = beta1, beta2, eps, weight_decay
        cfg.seed = seed & ((1 << 64) - 1)
        cfg.device = device
        cfg.offload, cfg.overlap = int(offload), int(overlap)
        cfg.chunk_elems, cfg.ring_slots = chunk_elems, ring_slots
        cfg.rank, cfg.world = rank, world
        cfg.residency, cfg.cache_layers = residency, cache_layers
        cfg.max_grad_norm = max_grad_norm
        cfg.param_dtype = param_dtype
        cfg.n_always = self.n_always
        cfg.dp_mode, cfg.p2p_sync = dp_mode, int(p2p_sync)
        cfg.debug_check = int(debug_check)
        self.dp_mode = dp_mode
        self.bf16 = param_dtype == DTYPE_BF16
        self._uid = None
        if nccl_id is not None and dp_mode == DP_NCCL:
            # the caller distributed the id (e.g. several ranks as threads of one process)
            self._uid = C.create_string_buffer(bytes(nccl_id), NCCL_ID_BYTES)
            cfg.nccl_unique_id = C.cast(self._uid, C.c_void_p)
        elif world == 1 and force_nccl:
            self._uid = C.create_string_buffer(nccl_unique_id(), NCCL_ID_BYTES)
            cfg.nccl_unique_id = C.cast(self._uid, C.c_void_p)
        elif world > 1 and dp_mode == DP_NCCL:
            import torch.distributed as dist
            obj = [nccl_unique_id() if rank == 0 else None]
            dist.broadcast_object_list(obj, src=0, group=process_group)
            self._uid = C.create_string_buffer(obj[0], NCCL_ID_BYTES)
            cfg.nccl_unique_id = C.cast(self._uid, C.c_void_p)
        self.cfg = cfg
        self.rank, self.world = rank, world
        h = C.c_void_p()
        _check(L.grass_create(C.byref(cfg), C.byref(h)))
        self._h = h

    # lifetime ---------------------------------------------------------------
    def close(self):
        if getattr(self, "_h", None):
            lib().grass_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    # hot path ---------------------------------------------------------------
    def mgn_accumulate(self, layer_ids: Sequence[int], grads, stream=None):
        ids = (C.c_int32 * len(layer_ids))(*layer_ids)
        f = lib().grass_mgn_accumulate_bf16 if self.bf16 else lib().grass_mgn_accumulate
        _check(f(self._h, ids, len(layer_ids), _ptrs(grads, 2 if self.bf16 else 4),
                 _stream_ptr(stream)), self._h)

    def update_probs(self):
        out = (C.c_double * self.n_layers)()
        _check(lib().grass_update_probs(self._h, out), self._h)
        return list(out)

    def sample_layers(self, period: int, probs: Sequence[float] | None = None):
        out = (C.c_int32 * self.gamma)()
        p = _dbl(probs) if probs is not None else None
        if probs is not None and len(probs) == self.n_sampled and self.n_always:
            p = _dbl(list(probs) + [0.0] * self.n_always)
        elif probs is not None and len(probs) != self.n_layers:
            raise ValueError("probs must have n_layers (or N_L sampled) entries")
        _check(lib().grass_sample_layers(self._h, p, period, out), self._h)
        return list(out)

    def step_layers(self, layer_ids: Sequence[int], params, grads, lr: float, stream=None):
        ids = (C.c_int32 * len(layer_ids))(*layer_ids)
        f = lib().grass_step_layers_bf16 if self.bf16 else lib().grass_step_layers
        isz = 2 if self.bf16 else 4
        _check(f(self._h, ids, len(layer_ids), _ptrs(params, isz), _ptrs(grads, isz, host_ok=True),
                 float(lr), _stream_ptr(stream)), self._h)

    # device-resident schedule ------------------------------------------------
    PERIOD_NEXT = (1 << 64) - 1

    def register_layers(self, params, grads):
        """The buffers of every layer (the device schedule reads them by id)."""
        isz = 2 if self.bf16 else 4
        if len(params) != self.n_layers or len(grads) != self.n_layers:
            raise ValueError("one parameter and one gradient buffer per layer")
        self._registered = (list(params), list(grads))      # keep them alive
        _check(lib().grass_register_layers(self._h, self.n_layers, _ptrs(params, isz), _ptrs(grads, isz)), self._h)

    def device_schedule_begin(self, period: int, stream=None):
        _check(lib().grass_device_schedule_begin(self._h, period, _stream_ptr(stream)), self._h)

    def device_step(self, lr: float, commit: bool = True, resample: bool = True,
                    next_period: int | None = None, stream=None):
        """Update the device-sampled layers, then (optionally) commit and
        resample — no host synchronisation; next_period None = the next one."""
        per = self.PERIOD_NEXT if next_period is None else int(next_period)
        _check(lib().grass_device_step(self._h, float(lr), int(commit), int(resample), per,
                                       _stream_ptr(stream)), self._h)

    def device_schedule_end(self):
        """Synchronises; the current sampled ids (host state updated)."""
        out = (C.c_int32 * self.gamma)()
        _check(lib().grass_device_schedule_end(self._h, out), self._h)
        return list(out)

    def sync(self):
        _check(lib().grass_sync(self._h), self._h)

    def set_lr_device(self, lr_tensor=None):
        """Read eta from a device float32 scalar (e.g. a torch tensor a captured
        graph's schedule updates); None restores the step_layers argument."""
        self._lr_tensor = lr_tensor          # keep it alive
        ptr = None if lr_tensor is None else lr_tensor.data_ptr()
        _check(lib().grass_set_lr_device(self._h, ptr), self._h)

    # state ------------------------------------------------------------------
    def shard(self, layer: int):
        return shard_range(self.layer_numel[layer], self.world, self.rank)

    def read_state(self, layer: int):
        import numpy as np
        n = self.shard(layer)[1]
        m = np.empty(n, np.float32)
        v = np.empty(n, np.float32)
        t = C.c_int64()
        _check(lib().grass_read_state(self._h, layer, m.ctypes.data, v.ctypes.data, C.byref(t)), self._h)
        return m, v, t.value

    def write_state(self, layer: int, m, v, t: int):
        import numpy as np
        m = np.ascontiguousarray(m, np.float32)
        v = np.ascontiguousarray(v, np.float32)
        n = self.shard(layer)[1]
        if m.size != n or v.size != n:
            raise ValueError("state size must equal the shard length")
        _check(lib().grass_write_state(self._h, layer, m.ctypes.data, v.ctypes.data, t), self._h)

    # P2P data parallelism (dp_mode=DP_P2P) --------------------------------
    def p2p_exchange_block(self):
        ptr, n = C.c_void_p(), C.c_int64()
        _check(lib().grass_p2p_exchange_block(self._h, C.byref(ptr), C.byref(n)), self._h)
        return ptr.value, n.value

    def p2p_attach(self, blocks: Sequence[int]):
        arr = (C.c_void_p * len(blocks))(*blocks)
        _check(lib().grass_p2p_attach(self._h, arr), self._h)

    def p2p_register_layer(self, layer: int, params: Sequence, grads: Sequence):
        """params / grads: [world] full-layer buffers (tensors or raw addresses), index = rank."""
        def addr(x):
            return x if isinstance(x, int) else x.data_ptr()
        pa = (C.c_void_p * len(params))(*[addr(x) for x in params])
        ga = (C.c_void_p * len(grads))(*[addr(x) for x in grads])
        _check(lib().grass_p2p_register_layer(self._h, layer, pa, ga), self._h)

    def p2p_finish(self, stream=None):
        _check(lib().grass_p2p_finish(self._h, _stream_ptr(stream)), self._h)

    def p2p_setup(self, layer_buffers: dict, process_group=None):
        """Collective over the process group (any backend): exports this rank's
        exchange block and every {layer: (param, grad)} buffer through CUDA IPC,
        gathers every rank's handles, imports the peers' and registers them."""
        import torch.distributed as dist
        mine = {"exch": ipc_export(self.p2p_exchange_block()[0]),
                "layers": {int(l): (ipc_export(p.data_ptr()), ipc_export(g.data_ptr()))
                           for l, (p, g) in layer_buffers.items()}}
        allr = [None] * self.world
        dist.all_gather_object(allr, mine, group=process_group)
        dev = self.cfg.device

        def addr(q, h, own):
            return own if q == self.rank else ipc_import(dev, *h)
        blocks = [addr(q, allr[q]["exch"], self.p2p_exchange_block()[0]) for q in range(self.world)]
        self.p2p_attach(blocks)
        for l, (p, g) in layer_buffers.items():
            ps = [addr(q, allr[q]["layers"][int(l)][0], p.data_ptr()) for q in range(self.world)]
            gs = [addr(q, allr[q]["layers"][int(l)][1], g.data_ptr()) for q in range(self.world)]
            self.p2p_register_layer(int(l), ps, gs)

    def save_state(self, path: str):
        _check(lib().grass_save_state(self._h, os.fsencode(path)), self._h)

    def load_state(self, path: str):
        _check(lib().grass_load_state(self._h, os.fsencode(path)), self._h)

    def read_master(self, layer: int):
        import numpy as np
        out = np.empty(self.shard(layer)[1], np.float32)
        _check(lib().grass_read_master(self._h, layer, out.ctypes.data), self._h)
        return out

    def write_master(self, layer: int, master):
        import numpy as np
        a = np.ascontiguousarray(master, np.float32)
        if a.size != self.shard(layer)[1]:
            raise ValueError("master size must equal the shard length")
        _check(lib().grass_write_master(self._h, layer, a.ctypes.data), self._h)

    def trace_enable(self, on: bool = True):
        _check(lib().grass_trace_enable(self._h, int(on)), self._h)

    def trace_read(self, capacity: int = 1 << 16):
        """Trace events since the last enable/read: list of dicts (ms)."""
        buf = (TraceEvent * capacity)()
        n = C.c_int32()
        _check(lib().grass_trace_read(self._h, buf, capacity, C.byref(n)), self._h)
        return [{"kind": TRACE_KINDS[e.kind], "layer": e.layer, "offset": e.offset,
                 "count": e.count, "start_ms": e.start_ms, "end_ms": e.end_ms,
                 "state_dev": e.state_dev, "state_host": e.state_host}
                for e in buf[:min(n.value, capacity)]]

    def prefetch_layers(self, layer_ids: Sequence[int], stream=None):
        ids = (C.c_int32 * len(layer_ids))(*layer_ids)
        _check(lib().grass_prefetch_layers(self._h, ids, len(layer_ids), _stream_ptr(stream)), self._h)

    def flush_states(self):
        _check(lib().grass_flush_states(self._h), self._h)

    def get_mgn(self):
        n = self.n_layers
        m, S, ss, p = ((C.c_double * n)() for _ in range(4))
        c = (C.c_int64 * n)()
        _check(lib().grass_get_mgn(self._h, m, S, c, ss, p), self._h)
        return {"m": list(m), "S": list(S), "c": list(c), "last_ss": list(ss), "probs": list(p)}

    @property
    def device_bytes(self) -> int:
        return int(lib().grass_device_bytes(self._h))

    @property
    def host_bytes(self) -> int:
        return int(lib().grass_host_bytes(self._h))

    @property
    def launch_count(self) -> int:
        return int(lib().grass_launch_count(self._h))
