"""GRASS (arxiv 2604.07808) layer-wise update hot path, B200-native.

The product is libgrass.so (C ABI, include/grass.h) built from csrc/; this
package is its thin ctypes binding.  It never imports oracle/.
"""
from .binding import (DECIDE_COMMIT_RESAMPLE, DECIDE_CONTINUE, DECIDE_PROBE, DECIDE_RESAMPLE,
                      RESIDENCY_PERIOD, RESIDENCY_STEP, RESIDENCY_STEP_PREFETCH, DTYPE_BF16, DTYPE_FP32, DP_NCCL, DP_P2P,
                      POLICY_ADAPTIVE, POLICY_STATIC, POLICY_UNIFORM, Grass, GrassError,
                      exported_symbols, lib, nccl_unique_id, sample_from_probs,
                      schedule_decision, shard_range, softmax_probs, splitmix64, tile_elems,
                      uniform, ipc_export, ipc_import, selftest_p2p, enable_peer_access)

from .schedule import GrassSchedule  # noqa: E402
from .torch_blocks import GrassBlocks, flatten_params  # noqa: E402

__all__ = ["Grass", "GrassSchedule", "GrassBlocks", "flatten_params", "GrassError", "lib", "exported_symbols", "nccl_unique_id",
           "sample_from_probs", "schedule_decision", "shard_range", "softmax_probs",
           "splitmix64", "tile_elems", "uniform", "POLICY_ADAPTIVE", "POLICY_STATIC",
           "POLICY_UNIFORM", "DECIDE_PROBE", "DECIDE_COMMIT_RESAMPLE", "DECIDE_RESAMPLE",
           "DECIDE_CONTINUE", "RESIDENCY_STEP", "RESIDENCY_PERIOD", "RESIDENCY_STEP_PREFETCH", "DTYPE_FP32", "DTYPE_BF16",
           "DP_NCCL", "DP_P2P", "ipc_export", "ipc_import", "selftest_p2p",
           "enable_peer_access"]
