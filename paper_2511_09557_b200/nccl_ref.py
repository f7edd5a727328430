"""The NCCL baseline, called directly through its C API (ctypes) — the paper's
comparison point (ncclAllReduce, graph-captured) rather than
torch.distributed's wrapper around it. Any libnccl.so.2 can be loaded: the
system one (2.27.3, the version the paper used) or the one torch bundles
(2.28.9). NCCL_ALGO / NCCL_PROTO are read by NCCL at communicator creation,
so a (algorithm, protocol) pair is a property of the process that creates
the communicator (rankbench launches one set of processes per pair).

This is measurement plumbing only: nothing on the NVRAR path uses NCCL.
"""
from __future__ import annotations

import ctypes
import glob
import os
from typing import Optional

import torch

NCCL_SUM = 0
NCCL_DTYPES = {torch.int32: 2, torch.float32: 7, torch.bfloat16: 9}
SYSTEM_LIB = "/usr/lib/x86_64-linux-gnu/libnccl.so.2"


def torch_lib() -> Optional[str]:
    """The libnccl.so.2 torch's CUDA library links against."""
    base = os.path.dirname(os.path.dirname(torch.__file__))
    for p in glob.glob(os.path.join(base, "nvidia", "nccl", "lib", "libnccl.so*")):
        return p
    return None


def lib_path(which: str) -> str:
    if which == "system":
        return SYSTEM_LIB
    if which == "torch":
        p = torch_lib()
        if p is None:
            raise FileNotFoundError("torch's bundled libnccl.so.2 not found")
        return p
    return which


class UniqueId(ctypes.Structure):
    _fields_ = [("internal", ctypes.c_char * 128)]


class Nccl:
    """One rank's NCCL communicator over a chosen libnccl."""

    def __init__(self, path: str):
        # RTLD_LOCAL: a second libnccl in the process (torch's) stays separate
        self.path = path
        self.lib = ctypes.CDLL(path, mode=ctypes.RTLD_LOCAL)
        L = self.lib
        L.ncclGetVersion.argtypes = [ctypes.POINTER(ctypes.c_int)]
        L.ncclGetUniqueId.argtypes = [ctypes.POINTER(UniqueId)]
        L.ncclCommInitRank.argtypes = [ctypes.POINTER(ctypes.c_void_p), ctypes.c_int, UniqueId,
                                       ctypes.c_int]
        L.ncclAllReduce.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int,
                                    ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p]
        L.ncclCommDestroy.argtypes = [ctypes.c_void_p]
        L.ncclGetErrorString.restype = ctypes.c_char_p
        L.ncclGetErrorString.argtypes = [ctypes.c_int]
        self.comm = ctypes.c_void_p()

    def _ck(self, rc: int, what: str) -> None:
        if rc != 0:
            raise RuntimeError(f"{what}: {self.lib.ncclGetErrorString(rc).decode()} ({rc})")

    def version(self) -> str:
        v = ctypes.c_int()
        self._ck(self.lib.ncclGetVersion(ctypes.byref(v)), "ncclGetVersion")
        code = v.value  # MAJOR*10000 + MINOR*100 + PATCH for >= 2.9
        return f"{code // 10000}.{(code // 100) % 100}.{code % 100}"

    def unique_id(self) -> bytes:
        u = UniqueId()
        self._ck(self.lib.ncclGetUniqueId(ctypes.byref(u)), "ncclGetUniqueId")
        # not u.internal: a c_char array reads back as NUL-terminated bytes
        return ctypes.string_at(ctypes.addressof(u), 128)

    def init_rank(self, nranks: int, uid: bytes, rank: int) -> None:
        u = UniqueId()
        ctypes.memmove(ctypes.addressof(u), uid, 128)
        self._ck(self.lib.ncclCommInitRank(ctypes.byref(self.comm), nranks, u, rank),
                 "ncclCommInitRank")

    def all_reduce(self, send: torch.Tensor, recv: torch.Tensor,
                   stream: Optional[torch.cuda.Stream] = None) -> None:
        s = stream if stream is not None else torch.cuda.current_stream()
        self._ck(self.lib.ncclAllReduce(send.data_ptr(), recv.data_ptr(), send.numel(),
                                        NCCL_DTYPES[send.dtype], NCCL_SUM, self.comm,
                                        s.cuda_stream), "ncclAllReduce")

    def close(self) -> None:
        if self.comm:
            self.lib.ncclCommDestroy(self.comm)
            self.comm = ctypes.c_void_p()
