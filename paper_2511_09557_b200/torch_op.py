"""NVRAR as a CUDA-graph-capturable torch custom op.

    comm = Communicator.from_process_group(topo, max_bytes)
    cid = torch_op.register(comm)
    y = torch.ops.nvrar.all_reduce(x, cid)      # out of place
    torch.ops.nvrar.all_reduce_(x, cid)         # in place

The op enqueues one nvrar_allreduce on the current stream (no host sync), so
a model step that calls it can be captured in a CUDA graph and replayed; the
call counter lives on the device and advances on every replay. The fake
(meta) implementation lets torch.compile trace through it as an opaque op.
"""
from __future__ import annotations

import itertools
from typing import Dict

import torch

from .comm import Communicator

_COMMS: Dict[int, Communicator] = {}
_IDS = itertools.count(1)  # never reused: an unregistered id stays dead


def register(comm: Communicator) -> int:
    """Make `comm` addressable from the op; returns its id."""
    cid = next(_IDS)
    _COMMS[cid] = comm
    return cid


def unregister(cid: int) -> None:
    _COMMS.pop(cid, None)


def _comm(cid: int) -> Communicator:
    try:
        return _COMMS[cid]
    except KeyError:
        raise ValueError(f"nvrar: no communicator registered under id {cid}") from None


@torch.library.custom_op("nvrar::all_reduce", mutates_args=())
def all_reduce(x: torch.Tensor, comm_id: int) -> torch.Tensor:
    """Sum of `x` over every rank of the communicator (out of place)."""
    src = x.contiguous()
    out = torch.empty_like(src)
    _comm(comm_id).allreduce(src, out)
    return out


@all_reduce.register_fake
def _all_reduce_fake(x: torch.Tensor, comm_id: int) -> torch.Tensor:
    return torch.empty_like(x, memory_format=torch.contiguous_format)


@torch.library.custom_op("nvrar::all_reduce_", mutates_args=("x",))
def all_reduce_(x: torch.Tensor, comm_id: int) -> None:
    """In-place sum (send == recv is allowed)."""
    if not x.is_contiguous():
        raise ValueError("nvrar::all_reduce_: x must be contiguous")
    _comm(comm_id).allreduce(x, x)


@all_reduce_.register_fake
def _all_reduce__fake(x: torch.Tensor, comm_id: int) -> None:
    return None


@torch.library.custom_op("nvrar::all_reduce_residual_", mutates_args=("residual",))
def all_reduce_residual_(x: torch.Tensor, residual: torch.Tensor, comm_id: int) -> None:
    """residual += all_reduce(x), fused into the all-reduce's final store (one
    kernel; bit-identical to all_reduce followed by the add)."""
    if not (x.is_contiguous() and residual.is_contiguous()):
        raise ValueError("nvrar::all_reduce_residual_: tensors must be contiguous")
    _comm(comm_id).allreduce_residual(x, residual)


@all_reduce_residual_.register_fake
def _all_reduce_residual__fake(x: torch.Tensor, residual: torch.Tensor, comm_id: int) -> None:
    return None
