"""B200-native DELTA decode-step attention stack (arXiv 2510.09883).

The product is ``libdelta.so`` (C ABI in ``include/delta.h``; sm_100a kernels in
``csrc/``); :mod:`.binding` is a thin ctypes layer over it.
"""
from .binding import (DELTA_BF16, DELTA_FP32, POLICY_DELTA, POLICY_QUEST, POLICY_RAAS, ROLE_FULL, ROLE_QUEST,
                      ROLE_RAAS, ROLE_SELECT, ROLE_SPARSE, DeltaConfig, DeltaError,
                      DeltaStack, declared_functions, load_library, nccl_unique_id, query_sizes, read_bandwidth_probe,
                      shard_range)

__all__ = ["DELTA_BF16", "DELTA_FP32", "POLICY_DELTA", "POLICY_QUEST", "POLICY_RAAS", "ROLE_FULL", "ROLE_QUEST",
           "ROLE_RAAS", "ROLE_SELECT",
           "ROLE_SPARSE", "DeltaConfig", "DeltaError",
           "DeltaStack", "declared_functions", "load_library", "nccl_unique_id", "query_sizes",
           "read_bandwidth_probe", "shard_range"]
