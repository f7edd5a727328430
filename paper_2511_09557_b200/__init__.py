"""B200-native NVRAR: hierarchical recursive-doubling all-reduce (arXiv 2511.09557).

The product is libnvrar_b200.so (CUDA, sm_100a) behind the C ABI in
include/nvrar.h; this package is the host-side mirror of the reference's
C++ API (``NvrarAllreduce``, ``NvrarConfig``, ``ClusterTopology``, errors).
"""
from .comm import (BlockedRank, ClusterTopology, Communicator, CudaError, DeadlockError,
                   InvalidArgumentError, InvalidTopologyError, LocalGroup, NvrarAllreduce,
                   NvrarConfig, ProtocolFaultError, RankId, dtype_code, is_power_of_two,
                   log2_exact)

__all__ = [
    "BlockedRank", "ClusterTopology", "Communicator", "CudaError", "DeadlockError",
    "InvalidArgumentError", "InvalidTopologyError", "LocalGroup", "NvrarAllreduce",
    "NvrarConfig", "ProtocolFaultError", "RankId", "dtype_code", "is_power_of_two",
    "log2_exact",
]
