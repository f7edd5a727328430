"""Process-group plumbing around the communicator: bootstrap exchange of the
symmetric-region handles, the selector consensus check, and max-over-ranks
reduction of device timings (the reference's makespan, bench.hpp:116-118).

torch.distributed is only the control plane here (gloo on CPU, nccl on GPU);
no collective on the data path goes through it.
"""
from __future__ import annotations

from typing import List, Optional, Sequence, Tuple

import torch
import torch.distributed as dist


def exchange_handles(mine: bytes, group=None) -> List[bytes]:
    """All-gather one opaque handle per rank (rank-major), like nvrar_init's
    allgather callback."""
    out: List[Optional[bytes]] = [None] * dist.get_world_size(group)
    dist.all_gather_object(out, bytes(mine), group=group)
    for i, h in enumerate(out):
        if not isinstance(h, (bytes, bytearray)):
            raise RuntimeError(f"rank {i} sent no handle")
    return [bytes(h) for h in out]  # type: ignore[arg-type]


def plan_consensus(plan: Tuple[str, int], group=None) -> Tuple[str, int]:
    """Every rank must run the same schedule and CTA count; a disagreement would
    deadlock the kernel, so fail loudly on the host instead."""
    plans: List[Optional[Tuple[str, int]]] = [None] * dist.get_world_size(group)
    dist.all_gather_object(plans, tuple(plan), group=group)
    if any(p != plans[0] for p in plans):
        raise RuntimeError(f"ranks disagree on the schedule: {plans}")
    return plans[0]  # type: ignore[return-value]


def max_over_ranks(values: Sequence[float], group=None, device: Optional[torch.device] = None
                   ) -> List[float]:
    """Elementwise max over ranks of per-sample times (µs or ms)."""
    backend = dist.get_backend(group)
    if backend == "nccl":
        dev = device if device is not None else torch.device("cuda", torch.cuda.current_device())
    else:
        dev = torch.device("cpu")
    t = torch.tensor(list(values), dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return t.cpu().tolist()
