"""Bootstrap of the symmetric-region handles without torch.distributed: every
rank writes its opaque nvrar handle into a shared directory and reads the
others' (the allgather callback of nvrar_init, include/nvrar.h, over a file
system). Used where a process group is unwanted — smoke(), time-sliced
multi-process tests — and by hosts that already have a shared directory.
"""
from __future__ import annotations

import os
import time
from typing import List

from .comm import ClusterTopology, Communicator, InvalidArgumentError


def file_allgather(path: str, rank: int, world: int, mine: bytes, tag: str = "h",
                   timeout_s: float = 120.0) -> List[bytes]:
    """All-gather one blob per rank through files `<path>/<tag><rank>`; the
    write is atomic (rename), so a reader never sees a partial handle."""
    os.makedirs(path, exist_ok=True)
    tmp = os.path.join(path, f".{tag}{rank}.{os.getpid()}")
    with open(tmp, "wb") as fh:
        fh.write(mine)
    os.replace(tmp, os.path.join(path, f"{tag}{rank}"))
    out: List[bytes] = []
    deadline = time.monotonic() + timeout_s
    for r in range(world):
        f = os.path.join(path, f"{tag}{r}")
        while not os.path.exists(f):
            if time.monotonic() > deadline:
                raise TimeoutError(f"bootstrap: rank {r} did not publish {f}")
            time.sleep(0.01)
        with open(f, "rb") as fh:
            out.append(fh.read())
    return out


def file_barrier(path: str, rank: int, world: int, tag: str, timeout_s: float = 120.0) -> None:
    file_allgather(path, rank, world, b"1", tag=tag, timeout_s=timeout_s)


def communicator_from_dir(path: str, topo: ClusterTopology, rank: int, max_bytes: int,
                          device: int = 0, **kw) -> Communicator:
    """One rank's communicator, peers mapped through CUDA IPC after a file
    exchange of the handles (collective over the `topo.world_size()` ranks)."""
    if not 0 <= rank < topo.world_size():
        raise InvalidArgumentError(f"rank {rank} out of range")
    comm = Communicator(topo, rank, device, max_bytes, **kw)
    world = topo.world_size()
    comm.exchange = lambda blob, tag: file_allgather(path, rank, world, blob, tag=tag)
    comm.connect(comm.exchange(comm.export(), "h"))
    return comm
