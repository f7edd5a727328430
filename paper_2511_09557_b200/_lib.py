"""ctypes binding of libnvrar_b200.so (the C ABI in include/nvrar.h).

There is no fallback: if the CUDA library is missing the import of any
collective fails loudly (build it with ``python -m paper_2511_09557_b200.build``
or ``__graft_entry__.build()``).
"""
from __future__ import annotations

import ctypes
import os

from . import build as _build

LIB_PATH = os.environ.get("NVRAR_LIB") or _build.LIB  # override: experiment builds

SUCCESS = 0
ERR_INTERNAL = 1
ERR_INVALID_ARGUMENT = 2
ERR_INVALID_TOPOLOGY = 3
ERR_PROTOCOL_FAULT = 4
ERR_DEADLOCK = 5
ERR_CUDA = 6
ERR_NOT_CONNECTED = 7

INT32, FLOAT32, BF16 = 0, 1, 2
SUM = 0
ALGO_AUTO, ALGO_HIER, ALGO_TWOSHOT, ALGO_ONESHOT, ALGO_DIRECT, ALGO_MCAST = 0, 1, 2, 3, 4, 5
ALGO_NAMES = {ALGO_AUTO: "auto", ALGO_HIER: "hier", ALGO_TWOSHOT: "twoshot",
              ALGO_ONESHOT: "oneshot", ALGO_DIRECT: "direct", ALGO_MCAST: "mcast"}

PROTO_AUTO, PROTO_LL, PROTO_LAMPORT = 0, 1, 2
PROTO_CODES = {"auto": PROTO_AUTO, "ll": PROTO_LL, "lamport": PROTO_LAMPORT}

HANDLE_BYTES = 256
MAX_LOCAL = 32

ALLGATHER_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p,
                                ctypes.c_void_p, ctypes.c_size_t)


class InitArgs(ctypes.Structure):
    _fields_ = [
        ("world_size", ctypes.c_int),
        ("rank", ctypes.c_int),
        ("nodes", ctypes.c_int),
        ("gpus_per_node", ctypes.c_int),
        ("device", ctypes.c_int),
        ("max_bytes", ctypes.c_size_t),
        ("blocks", ctypes.c_int),
        ("chunk_bytes", ctypes.c_uint64),
        ("timeout_s", ctypes.c_double),
        ("allgather", ALLGATHER_FN),
        ("allgather_ctx", ctypes.c_void_p),
    ]


class Handle(ctypes.Structure):
    _fields_ = [("bytes", ctypes.c_ubyte * HANDLE_BYTES)]


class PlanEntry(ctypes.Structure):
    _fields_ = [("max_bytes", ctypes.c_uint64), ("algo", ctypes.c_int), ("blocks", ctypes.c_int)]


class Blocked(ctypes.Structure):
    _fields_ = [
        ("global_rank", ctypes.c_int),
        ("kind", ctypes.c_int),
        ("peer_rank", ctypes.c_int),
        ("expected", ctypes.c_uint32),
        ("word_index", ctypes.c_uint64),
        ("observed", ctypes.c_uint64),
        ("status", ctypes.c_int),
        ("phase", ctypes.c_int),
        ("cta", ctypes.c_int),
    ]


# Every symbol include/nvrar.h declares, with its ctypes signature.
_c = ctypes
_vp = _c.c_void_p
SIGNATURES = {
    "nvrar_init": (_c.c_int, [_c.POINTER(InitArgs), _c.POINTER(_vp)]),
    "nvrar_comm_create": (_c.c_int, [_c.POINTER(InitArgs), _c.POINTER(_vp)]),
    "nvrar_comm_export": (_c.c_int, [_vp, _c.POINTER(Handle)]),
    "nvrar_comm_connect": (_c.c_int, [_vp, _c.POINTER(Handle), _c.c_int]),
    "nvrar_finalize": (_c.c_int, [_vp]),
    "nvrar_alloc_symmetric": (_c.c_int, [_vp, _c.c_size_t, _c.POINTER(_vp)]),
    "nvrar_register_buffer": (_c.c_int, [_vp, _vp, _c.c_size_t, _c.POINTER(Handle),
                                         _c.POINTER(_c.c_int)]),
    "nvrar_connect_buffer": (_c.c_int, [_vp, _c.c_int, _c.POINTER(Handle), _c.c_int]),
    "nvrar_deregister_buffer": (_c.c_int, [_vp, _c.c_int]),
    "nvrar_buffer_peer_ptr": (_c.c_int, [_vp, _c.c_int, _c.c_int, _c.POINTER(_vp)]),
    "nvrar_allreduce_registered": (_c.c_int, [_vp, _vp, _vp, _c.c_size_t, _c.c_int, _c.c_int,
                                              _vp]),
    "nvrar_allreduce": (_c.c_int, [_vp, _vp, _vp, _c.c_size_t, _c.c_int, _c.c_int, _vp]),
    "nvrar_allreduce_local": (_c.c_int, [_c.POINTER(_vp), _c.c_int, _c.POINTER(_vp),
                                         _c.POINTER(_vp), _c.c_size_t, _c.c_int, _c.c_int, _vp,
                                         _c.c_uint64]),
    "nvrar_set_config": (_c.c_int, [_vp, _c.c_int, _c.c_uint64]),
    "nvrar_set_algo": (_c.c_int, [_vp, _c.c_int]),
    "nvrar_set_timeout": (_c.c_int, [_vp, _c.c_double]),
    "nvrar_set_protocol": (_c.c_int, [_vp, _c.c_int]),
    "nvrar_set_plan_table": (_c.c_int, [_vp, _c.POINTER(PlanEntry), _c.c_int]),
    "nvrar_plan": (_c.c_int, [_vp, _c.c_size_t, _c.c_int, _c.POINTER(_c.c_int),
                              _c.POINTER(_c.c_int)]),
    "nvrar_allreduce_host": (_c.c_int, [_vp, _vp, _vp, _c.c_size_t, _c.c_int, _c.c_int, _vp]),
    "nvrar_set_host_chunk": (_c.c_int, [_vp, _c.c_size_t]),
    "nvrar_allreduce_local_host": (_c.c_int, [_c.POINTER(_vp), _c.c_int, _c.POINTER(_vp),
                                              _c.POINTER(_vp), _c.c_size_t, _c.c_int, _c.c_int,
                                              _vp]),
    "nvrar_allreduce_residual": (_c.c_int, [_vp, _vp, _vp, _vp, _c.c_size_t, _c.c_int, _c.c_int,
                                            _vp]),
    "nvrar_allreduce_local_residual": (_c.c_int, [_c.POINTER(_vp), _c.c_int, _c.POINTER(_vp),
                                                  _c.POINTER(_vp), _c.POINTER(_vp), _c.c_size_t,
                                                  _c.c_int, _c.c_int, _vp, _c.c_uint64]),
    "nvrar_ring_allreduce": (_c.c_int, [_vp, _vp, _vp, _c.c_size_t, _c.c_int, _c.c_int, _vp]),
    "nvrar_tree_allreduce": (_c.c_int, [_vp, _vp, _vp, _c.c_size_t, _c.c_int, _c.c_int, _vp]),
    "nvrar_allreduce_local_order": (_c.c_int, [_c.POINTER(_vp), _c.c_int, _c.c_int,
                                               _c.POINTER(_vp), _c.POINTER(_vp), _c.c_size_t,
                                               _c.c_int, _c.c_int, _vp, _c.c_uint64]),
    "nvrar_reduce_scatter": (_c.c_int, [_vp, _vp, _vp, _c.c_size_t, _c.c_int, _c.c_int, _vp]),
    "nvrar_all_gather": (_c.c_int, [_vp, _vp, _vp, _c.c_size_t, _c.c_int, _vp]),
    "nvrar_rd_inter": (_c.c_int, [_vp, _vp, _vp, _c.c_size_t, _c.c_int, _vp]),
    "nvrar_phase_local": (_c.c_int, [_c.POINTER(_vp), _c.c_int, _c.c_int, _c.POINTER(_vp),
                                     _c.POINTER(_vp), _c.c_size_t, _c.c_int, _vp, _c.c_uint64]),
    "nvrar_mc_bytes": (_c.c_int, [_vp, _c.POINTER(_c.c_size_t)]),
    "nvrar_mc_attach": (_c.c_int, [_vp, _vp, _vp, _c.c_size_t]),
    "nvrar_mc_ready": (_c.c_int, [_vp, _c.POINTER(_c.c_int)]),
    "nvrar_plan_local": (_c.c_int, [_c.POINTER(_vp), _c.c_int, _c.c_size_t, _c.c_int,
                                    _c.c_uint64, _c.POINTER(_c.c_int), _c.POINTER(_c.c_int)]),
    "nvrar_plan_for": (_c.c_int, [_c.c_int, _c.c_int, _c.c_int, _c.c_size_t, _c.c_int, _c.c_int,
                                  _c.c_int, _c.c_int, _c.POINTER(_c.c_int), _c.POINTER(_c.c_int)]),
    "nvrar_get_sequence": (_c.c_int, [_vp, _c.POINTER(_c.c_uint32)]),
    "nvrar_get_peers": (_c.c_int, [_vp, _c.POINTER(_c.c_int), _c.c_int, _c.POINTER(_c.c_int)]),
    "nvrar_set_profile": (_c.c_int, [_vp, _c.c_int]),
    "nvrar_get_phase_times": (_c.c_int, [_vp, _c.POINTER(_c.c_uint64), _c.c_int]),
    "nvrar_pingpong": (_c.c_int, [_vp, _c.c_int, _c.c_int, _c.c_int, _vp,
                                  _c.POINTER(_c.c_uint64)]),
    "nvrar_pingpong_clock": (_c.c_int, [_vp, _c.POINTER(_c.c_uint64)]),
    "nvrar_debug_dirty_cells": (_c.c_int, [_vp, _c.POINTER(_c.c_uint64),
                                           _c.POINTER(_c.c_uint64)]),
    "nvrar_debug_read_region": (_c.c_int, [_vp, _c.c_uint64, _c.c_uint64, _vp,
                                           _c.POINTER(_c.c_uint64)]),
    "nvrar_debug_seq_slots": (_c.c_int, [_vp, _c.POINTER(_c.c_uint32), _c.c_int]),
    "nvrar_set_jitter": (_c.c_int, [_vp, _c.c_uint32, _c.c_uint32]),
    "nvrar_debug_canary": (_c.c_int, [_vp, _c.c_int, _c.c_int, _c.c_int, _c.c_uint32,
                                      _c.c_uint32, _vp]),
    "nvrar_debug_canary_result": (_c.c_int, [_vp, _c.POINTER(_c.c_uint32)]),
    "nvrar_check":(_c.c_int, [_vp]),
    "nvrar_get_blocked": (_c.c_int, [_vp, _c.POINTER(Blocked)]),
    "nvrar_last_error": (_c.c_char_p, [_vp]),
    "nvrar_status_string": (_c.c_char_p, [_c.c_int]),
    "nvrar_abi_version": (_c.c_int, []),
    "nvrar_symmetric_bytes": (_c.c_size_t, [_vp]),
}

_lib = None


def load():
    """Load the in-tree CUDA library; raise if it has not been built."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: the NVRAR CUDA library must be built "
                "(python -m paper_2511_09557_b200.build); there is no CPU fallback")
        lib = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib
