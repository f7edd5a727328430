"""Host-side mirror of the reference's all-reduce API over the CUDA C ABI.

Names, argument meaning and error behaviour follow the reference
(/root/reference/proj/include/ccsim):

* ``ClusterTopology`` / ``RankId``           topology.hpp:24-67
* ``NvrarConfig``                            collectives/fused.hpp:106-116
* ``InvalidArgumentError`` ... ``DeadlockError`` (+ ``BlockedRank``)  errors.hpp:15-85
* ``NvrarAllreduce(comm, max_elems)`` with ``run(in, out, cfg)``,
  ``sequence()`` and ``peers()``             collectives/nvrar.hpp:41-250
* ``LocalGroup.run_all`` — every rank of a topology in one process (one GPU),
  the shape of the reference's ``run_ranks`` (run.hpp:15-24); used by the
  parity tests, as the reference's own tests drive all ranks in one process.

Device tensors are torch tensors (torch is the memory/stream plumbing); all
collective work happens in libnvrar_b200.so.
"""
from __future__ import annotations

import ctypes
import struct
import enum
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import torch

from . import _lib as L


# ---- errors (errors.hpp) ------------------------------------------------------

class InvalidArgumentError(ValueError):
    """errors.hpp:15-18"""


class InvalidTopologyError(ValueError):
    """errors.hpp:22-25"""


class ProtocolFaultError(RuntimeError):
    """errors.hpp:29-43"""

    def __init__(self, global_rank: int, what: str):
        super().__init__(what if global_rank < 0 else f"rank {global_rank}: {what}")
        self._global_rank = global_rank

    def global_rank(self) -> int:
        return self._global_rank


@dataclass
class BlockedRank:
    """errors.hpp:46-57 (word_index / region describe a FlagWait)."""

    class Kind(enum.IntEnum):
        FlagWait = 0
        SeqWait = 1

    global_rank: int = -1
    kind: "BlockedRank.Kind" = Kind.FlagWait
    region: int = -1
    word_index: int = 0
    peer_rank: int = -1
    expected: int = 0
    phase: int = -1  # GPU diagnosis: kernel phase (2 push, 3 sync, 4 reduce/RD, 5 all-gather)
    cta: int = -1


class DeadlockError(RuntimeError):
    """errors.hpp:61-85 — carries the blocked set."""

    def __init__(self, blocked: List[BlockedRank]):
        self._blocked = list(blocked)
        parts = []
        for b in self._blocked:
            if b.kind == BlockedRank.Kind.FlagWait:
                parts.append(f"[rank {b.global_rank} awaits flag {b.expected} from rank "
                             f"{b.peer_rank} word {b.word_index} (phase {b.phase}, cta {b.cta})]")
            else:
                parts.append(f"[rank {b.global_rank} awaits seq {b.expected} from rank "
                             f"{b.peer_rank}]")
        super().__init__(f"deadlock: {len(self._blocked)} rank(s) blocked: " + " ".join(parts))

    def blocked(self) -> List[BlockedRank]:
        return self._blocked


class CudaError(RuntimeError):
    pass


def _raise(code: int, msg: str, rank: int = -1):
    if code == L.ERR_INVALID_ARGUMENT:
        raise InvalidArgumentError(msg)
    if code == L.ERR_INVALID_TOPOLOGY:
        raise InvalidTopologyError(msg)
    if code == L.ERR_PROTOCOL_FAULT:
        raise ProtocolFaultError(rank, msg)
    if code == L.ERR_DEADLOCK:
        raise DeadlockError([])
    raise CudaError(f"nvrar error {code}: {msg}")


# ---- topology (topology.hpp) ------------------------------------------------

def is_power_of_two(v: int) -> bool:
    return v > 0 and (v & (v - 1)) == 0


def log2_exact(v: int) -> int:
    lv = 0
    while (1 << lv) < v:
        lv += 1
    return lv


@dataclass(frozen=True)
class ClusterTopology:
    nodes: int = 1
    gpus_per_node: int = 1

    def world_size(self) -> int:
        return self.nodes * self.gpus_per_node

    def validate(self) -> None:
        if self.nodes < 1 or self.gpus_per_node < 1:
            raise InvalidArgumentError("topology: nodes and gpus_per_node must be >= 1")

    def require_power_of_two_nodes(self, who: str) -> None:
        self.validate()
        if not is_power_of_two(self.nodes):
            raise InvalidTopologyError(
                f"{who}: node count must be a power of two, got {self.nodes}")


@dataclass(frozen=True)
class RankId:
    node_rank: int = 0
    local_rank: int = 0

    def global_(self, topo: ClusterTopology) -> int:
        return self.node_rank * topo.gpus_per_node + self.local_rank

    @staticmethod
    def from_global(g: int, topo: ClusterTopology) -> "RankId":
        return RankId(g // topo.gpus_per_node, g % topo.gpus_per_node)

    def same_node(self, other: "RankId") -> bool:
        return self.node_rank == other.node_rank


# ---- config (fused.hpp:106-116) ------------------------------------------------

@dataclass
class NvrarConfig:
    """``blocks`` = CTAs per rank (the reference's independent block ranges);
    ``chunk_bytes`` is validated like the reference's. On the GPU every thread
    forwards its own 4-element unit as soon as it is reduced, so the chunk
    pipeline of rd_block (nvrar.hpp:193-220) runs at unit granularity and the
    result is, as in the reference, invariant to (blocks, chunk_bytes).
    ``blocks = 0`` lets the selector choose."""

    blocks: int = 0
    chunk_bytes: int = 65536

    def validate(self) -> None:
        if self.blocks < 0:
            raise InvalidArgumentError("nvrar config: blocks must be >= 1")
        if self.chunk_bytes < 8 or self.chunk_bytes % 8 != 0:
            raise InvalidArgumentError("nvrar config: chunk_bytes must be a multiple of 8, >= 8")


_DTYPES = {torch.float32: L.FLOAT32, torch.bfloat16: L.BF16, torch.int32: L.INT32}
_ALGOS = {"auto": L.ALGO_AUTO, "hier": L.ALGO_HIER, "twoshot": L.ALGO_TWOSHOT,
          "oneshot": L.ALGO_ONESHOT, "direct": L.ALGO_DIRECT, "mcast": L.ALGO_MCAST}


def dtype_code(t: torch.dtype) -> int:
    try:
        return _DTYPES[t]
    except KeyError:
        raise InvalidArgumentError(f"unsupported dtype {t} (int32, float32, bfloat16)") from None


def _stream_ptr(stream: Optional[torch.cuda.Stream]) -> int:
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


# ---- communicator --------------------------------------------------------------

class Communicator:
    """One rank's NVRAR communicator (nvrar_comm_t)."""

    def __init__(self, topo: ClusterTopology, rank: int, device: int, max_bytes: int,
                 timeout_s: float = 10.0, blocks: int = 0, chunk_bytes: int = 65536):
        topo.require_power_of_two_nodes("nvrar")
        self.topo = topo
        self.rank = rank
        self.device = device
        self.max_bytes = max_bytes
        self._lib = L.load()
        args = L.InitArgs(world_size=topo.world_size(), rank=rank, nodes=topo.nodes,
                          gpus_per_node=topo.gpus_per_node, device=device,
                          max_bytes=max_bytes, blocks=blocks, chunk_bytes=chunk_bytes,
                          timeout_s=timeout_s)
        h = ctypes.c_void_p()
        rc = self._lib.nvrar_comm_create(ctypes.byref(args), ctypes.byref(h))
        if rc != 0:
            _raise(rc, self._lib.nvrar_last_error(None).decode(), rank)
        self._h = h
        self.connected = False

    # -- bootstrap --------------------------------------------------------------
    def export(self) -> bytes:
        hd = L.Handle()
        self._check(self._lib.nvrar_comm_export(self._h, ctypes.byref(hd)))
        return bytes(hd.bytes)

    def connect(self, handles: Sequence[bytes]) -> None:
        arr = (L.Handle * len(handles))()
        for i, b in enumerate(handles):
            ctypes.memmove(arr[i].bytes, b, L.HANDLE_BYTES)
        self._check(self._lib.nvrar_comm_connect(self._h, arr, len(handles)))
        self.connected = True

    @classmethod
    def from_process_group(cls, topo: ClusterTopology, max_bytes: int, device: Optional[int] = None,
                           group=None, **kw) -> "Communicator":
        """One process per GPU: exchange IPC handles over torch.distributed."""
        import torch.distributed as dist
        rank = dist.get_rank(group)
        if device is None:
            device = torch.cuda.current_device()
        comm = cls(topo, rank, device, max_bytes, **kw)
        comm.exchange = lambda blob, tag: _dist_allgather(blob, group)
        comm.connect(comm.exchange(comm.export(), "comm"))
        return comm

    def enable_multicast(self, group=None) -> bool:
        """Attach an NVLS multicast area from torch symmetric memory (the
        plumbing: allocation + multicast rendezvous) so NVRAR_ALGO_MCAST can
        run. Collective. Returns whether every rank has it; on any failure no
        rank uses it."""
        import torch.distributed as dist
        ok = False
        buf = None
        nbytes = ctypes.c_size_t()
        try:
            import torch.distributed._symmetric_memory as symm
            self._check(self._lib.nvrar_mc_bytes(self._h, ctypes.byref(nbytes)))
            buf = symm.empty(nbytes.value, dtype=torch.uint8, device=f"cuda:{self.device}")
        except Exception as e:  # noqa: BLE001 — no multicast: the unicast schedules remain
            self.mc_error = f"{type(e).__name__}: {e}"
        # every rank enters the (collective) rendezvous, or none does
        if not self._all_ok(buf is not None, group):
            return False
        try:
            grp = group if group is not None else dist.group.WORLD
            hdl = symm.rendezvous(buf, grp.group_name)
            mc = int(getattr(hdl, "multicast_ptr", 0) or 0)
            if mc:
                ok = self._lib.nvrar_mc_attach(self._h, mc, buf.data_ptr(), nbytes.value) == 0
            self._mc_keep = (buf, hdl)  # the memory must outlive the communicator's use
        except Exception as e:  # noqa: BLE001
            self.mc_error = f"{type(e).__name__}: {e}"
        ok = self._all_ok(ok, group)
        if not ok and self.multicast_ready():
            self._check(self._lib.nvrar_mc_attach(self._h, None, None, 0))  # detach
        return ok

    def multicast_ready(self) -> bool:
        r = ctypes.c_int()
        self._check(self._lib.nvrar_mc_ready(self._h, ctypes.byref(r)))
        return bool(r.value)

    @staticmethod
    def _all_ok(ok: bool, group) -> bool:
        import torch.distributed as dist
        dev = "cuda" if dist.get_backend(group) == "nccl" else "cpu"
        t = torch.tensor([1 if ok else 0], dtype=torch.int32, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MIN, group=group)
        return bool(t.item())

    # -- registered buffers (nvrar_register_buffer, include/nvrar.h) ------------
    # `exchange(blob, tag) -> [blob per rank]` is the bootstrap all-gather the
    # comm was connected with (torch.distributed, or a shared directory)
    exchange = None

    def register_buffer(self, t: torch.Tensor) -> int:
        """Register `t` (a CUDA tensor, same size on every rank, registered in
        the same order) and map every peer's; collective. Returns the id."""
        if not (t.is_cuda and t.is_contiguous()):
            raise InvalidArgumentError("nvrar: registered buffers are contiguous CUDA tensors")
        if self.exchange is None:
            raise InvalidArgumentError("nvrar: this communicator has no bootstrap exchange")
        hd = L.Handle()
        buf = ctypes.c_int()
        self._check(self._lib.nvrar_register_buffer(self._h, t.data_ptr(),
                                                    t.numel() * t.element_size(),
                                                    ctypes.byref(hd), ctypes.byref(buf)))
        allh = self.exchange(bytes(hd.bytes), f"reg{buf.value}")
        arr = (L.Handle * len(allh))()
        for i, b in enumerate(allh):
            ctypes.memmove(arr[i].bytes, b, L.HANDLE_BYTES)
        self._check(self._lib.nvrar_connect_buffer(self._h, buf.value, arr, len(allh)))
        self._registered = getattr(self, "_registered", {})
        self._registered[buf.value] = t  # keep the memory alive while registered
        return buf.value

    def alloc_symmetric(self, numel: int, dtype: torch.dtype = torch.bfloat16) -> torch.Tensor:
        """A zeroed tensor registered with the comm (Ctx::alloc_region for caller
        data, transport.hpp:146-148); collective."""
        t = torch.zeros(numel, dtype=dtype, device=f"cuda:{self.device}")
        self.register_buffer(t)
        return t

    def deregister_buffer(self, buf: int) -> None:
        self._check(self._lib.nvrar_deregister_buffer(self._h, buf))
        getattr(self, "_registered", {}).pop(buf, None)

    def buffer_peer_ptr(self, buf: int, peer: int) -> int:
        p = ctypes.c_void_p()
        self._check(self._lib.nvrar_buffer_peer_ptr(self._h, buf, peer, ctypes.byref(p)))
        return int(p.value or 0)

    def allreduce_registered(self, send: torch.Tensor, recv: torch.Tensor,
                             stream: Optional[torch.cuda.Stream] = None) -> None:
        """nvrar_allreduce_registered: `send` inside a registered buffer (same
        offset on every rank); peers' inputs are read in place."""
        _check_pair(send, recv)
        self._check(self._lib.nvrar_allreduce_registered(
            self._h, send.data_ptr(), recv.data_ptr(), send.numel(), dtype_code(send.dtype),
            L.SUM, _stream_ptr(stream)))

    # -- knobs / introspection --------------------------------------------------
    def set_config(self, cfg: NvrarConfig) -> None:
        cfg.validate()
        self._check(self._lib.nvrar_set_config(self._h, cfg.blocks, cfg.chunk_bytes))

    def set_algo(self, algo: str) -> None:
        self._check(self._lib.nvrar_set_algo(self._h, _ALGOS[algo]))

    def set_timeout(self, seconds: float) -> None:
        self._check(self._lib.nvrar_set_timeout(self._h, seconds))

    def set_protocol(self, proto: str) -> None:
        """'auto' | 'll' (fused seq words, as the reference) | 'lamport' (raw payload)."""
        self._check(self._lib.nvrar_set_protocol(self._h, L.PROTO_CODES[proto]))

    def set_jitter(self, max_ns: int, seed: int = 0) -> None:
        """Delay injection (RunOptions::delay_max_us analogue): seeded random
        sleeps of up to max_ns before remote stores and between polls; 0 = off."""
        self._check(self._lib.nvrar_set_jitter(self._h, max_ns, seed & 0xFFFFFFFF))

    def canary(self, peer: int, iters: int, writer: bool, jitter_ns: int = 0, seed: int = 0,
               stream: Optional[torch.cuda.Stream] = None) -> None:
        """Launch one side of the word-atomicity canary (nvrar_debug_canary)."""
        self._check(self._lib.nvrar_debug_canary(self._h, peer, iters, int(writer), jitter_ns,
                                                 seed & 0xFFFFFFFF, _stream_ptr(stream)))

    def canary_result(self) -> int:
        t = ctypes.c_uint32()
        self._check(self._lib.nvrar_debug_canary_result(self._h, ctypes.byref(t)))
        return t.value

    def plan(self, count: int, dtype: torch.dtype):
        a, b = ctypes.c_int(), ctypes.c_int()
        self._check(self._lib.nvrar_plan(self._h, count, dtype_code(dtype), ctypes.byref(a),
                                         ctypes.byref(b)))
        return L.ALGO_NAMES[a.value], b.value

    def sequence(self) -> int:
        s = ctypes.c_uint32()
        self._check(self._lib.nvrar_get_sequence(self._h, ctypes.byref(s)))
        return s.value

    def peers(self) -> List[RankId]:
        arr = (ctypes.c_int * 8)()
        steps = ctypes.c_int()
        self._check(self._lib.nvrar_get_peers(self._h, arr, 8, ctypes.byref(steps)))
        return [RankId.from_global(arr[i], self.topo) for i in range(steps.value)]

    def blocked(self) -> L.Blocked:
        b = L.Blocked()
        self._check(self._lib.nvrar_get_blocked(self._h, ctypes.byref(b)))
        return b

    def check_status(self) -> int:
        """Synchronise and return the sticky device status (0 = ok)."""
        return self._lib.nvrar_check(self._h)

    def check(self) -> None:
        rc = self.check_status()
        if rc == L.ERR_DEADLOCK:
            raise DeadlockError([_blocked_rank(self.blocked())])
        if rc:
            _raise(rc, self.last_error(), self.rank)

    def last_error(self) -> str:
        return self._lib.nvrar_last_error(self._h).decode()

    def dirty_cells(self):
        """(count, first byte offset) of non-empty slot words — must be (0, -1) between calls."""
        cnt, first = ctypes.c_uint64(), ctypes.c_uint64()
        self._check(self._lib.nvrar_debug_dirty_cells(self._h, ctypes.byref(cnt), ctypes.byref(first)))
        return cnt.value, (-1 if first.value == (1 << 64) - 1 else first.value)

    def symmetric_bytes(self) -> int:
        return int(self._lib.nvrar_symmetric_bytes(self._h))

    # -- the collective -------------------------------------------------------------
    def allreduce(self, send: torch.Tensor, recv: torch.Tensor,
                  stream: Optional[torch.cuda.Stream] = None) -> None:
        """nvrar_allreduce(send, recv, count, dtype, SUM, stream) — asynchronous."""
        _check_pair(send, recv)
        rc = self._lib.nvrar_allreduce(self._h, send.data_ptr(), recv.data_ptr(), send.numel(),
                                       dtype_code(send.dtype), L.SUM, _stream_ptr(stream))
        if rc:
            _raise(rc, self.last_error(), self.rank)

    def set_host_chunk(self, nbytes: int) -> None:
        """Chunk of the host-buffer pipeline (0 = automatic); same on every rank."""
        self._check(self._lib.nvrar_set_host_chunk(self._h, nbytes))

    def allreduce_host(self, send: torch.Tensor, recv: torch.Tensor,
                       stream: Optional[torch.cuda.Stream] = None) -> None:
        """nvrar_allreduce_host: CPU tensors in and out (pin them for overlap);
        stream-ordered — synchronise `stream` before reading `recv`."""
        _check_host_pair(send, recv)
        self._check(self._lib.nvrar_allreduce_host(self._h, send.data_ptr(), recv.data_ptr(),
                                                   send.numel(), dtype_code(send.dtype), L.SUM,
                                                   _stream_ptr(stream)))

    def allreduce_residual(self, send: torch.Tensor, residual: torch.Tensor,
                           out: Optional[torch.Tensor] = None,
                           stream: Optional[torch.cuda.Stream] = None) -> torch.Tensor:
        """out = residual + all_reduce(send) in one kernel (out defaults to residual,
        i.e. in place) — the TP-decode `x = x + all_reduce(a)`."""
        _check_pair(send, residual)
        out = residual if out is None else out
        _check_pair(send, out)
        self._check(self._lib.nvrar_allreduce_residual(
            self._h, send.data_ptr(), out.data_ptr(), residual.data_ptr(), send.numel(),
            dtype_code(send.dtype), L.SUM, _stream_ptr(stream)))
        return out

    # ---- the reference's baseline collectives (ring.hpp / tree.hpp orders) ----
    def ring_allreduce(self, send: torch.Tensor, recv: torch.Tensor,
                       stream: Optional[torch.cuda.Stream] = None) -> None:
        """RingAllreduce<T>::run's result bits (ring_order_sum)."""
        _check_pair(send, recv)
        self._check(self._lib.nvrar_ring_allreduce(self._h, send.data_ptr(), recv.data_ptr(),
                                                   send.numel(), dtype_code(send.dtype), L.SUM,
                                                   _stream_ptr(stream)))

    def tree_allreduce(self, send: torch.Tensor, recv: torch.Tensor,
                       stream: Optional[torch.cuda.Stream] = None) -> None:
        """TreeAllreduce<T>::run's result bits (tree_order_sum)."""
        _check_pair(send, recv)
        self._check(self._lib.nvrar_tree_allreduce(self._h, send.data_ptr(), recv.data_ptr(),
                                                   send.numel(), dtype_code(send.dtype), L.SUM,
                                                   _stream_ptr(stream)))

    # ---- phase-only entry points (nvrar.h "phase-only entry points") ----------
    def reduce_scatter(self, send: torch.Tensor, shard: torch.Tensor,
                       stream: Optional[torch.cuda.Stream] = None) -> None:
        """IntraReduceScatter<T>::run (nvrar.hpp:280-299): `shard` gets this rank's
        ceil(n/G) elements of the node-local sum."""
        _check_phase_io(PHASE_REDUCE_SCATTER, send, shard, self.topo.gpus_per_node)
        self._check(self._lib.nvrar_reduce_scatter(self._h, send.data_ptr(), shard.data_ptr(),
                                                   send.numel(), dtype_code(send.dtype), L.SUM,
                                                   _stream_ptr(stream)))

    def all_gather(self, shard: torch.Tensor, recv: torch.Tensor,
                   stream: Optional[torch.cuda.Stream] = None) -> None:
        """IntraAllGather<T>::run (nvrar.hpp:348-364): recv = the node members'
        shards concatenated in local-rank order."""
        _check_phase_io(PHASE_ALL_GATHER, shard, recv, self.topo.gpus_per_node)
        self._check(self._lib.nvrar_all_gather(self._h, shard.data_ptr(), recv.data_ptr(),
                                               shard.numel(), dtype_code(shard.dtype),
                                               _stream_ptr(stream)))

    def rd_inter(self, packed: torch.Tensor, out: torch.Tensor, dtype: torch.dtype = torch.int32,
                 stream: Optional[torch.cuda.Stream] = None) -> None:
        """NvrarAllreduce<T>::rd_inter (nvrar.hpp:132-155) on LL-packed int64 words."""
        _check_phase_io(PHASE_RD_INTER, packed, out, self.topo.gpus_per_node)
        self._check(self._lib.nvrar_rd_inter(self._h, packed.data_ptr(), out.data_ptr(),
                                             packed.numel(), dtype_code(dtype),
                                             _stream_ptr(stream)))

    def allreduce_raw(self, send_ptr: int, recv_ptr: int, count: int, dtype: int,
                      stream_ptr: int) -> None:
        rc = self._lib.nvrar_allreduce(self._h, send_ptr, recv_ptr, count, dtype, L.SUM,
                                       stream_ptr)
        if rc:
            _raise(rc, self.last_error(), self.rank)

    def close(self) -> None:
        if getattr(self, "_h", None):
            self._lib.nvrar_finalize(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _check(self, rc: int) -> None:
        if rc:
            _raise(rc, self.last_error(), self.rank)


def _dist_allgather(blob: bytes, group=None) -> List[bytes]:
    import torch.distributed as dist
    out: List[Optional[bytes]] = [None] * dist.get_world_size(group)
    dist.all_gather_object(out, bytes(blob), group=group)
    return [bytes(b) for b in out]  # type: ignore[arg-type]


def _blocked_rank(b: L.Blocked) -> BlockedRank:
    return BlockedRank(global_rank=b.global_rank,
                       kind=BlockedRank.Kind.SeqWait if b.kind == 1 else BlockedRank.Kind.FlagWait,
                       word_index=b.word_index, peer_rank=b.peer_rank, expected=b.expected,
                       phase=b.phase, cta=b.cta)


def _check_host_pair(send: torch.Tensor, recv: torch.Tensor) -> None:
    if send.numel() != recv.numel() or send.dtype != recv.dtype:
        raise InvalidArgumentError("nvrar: input and output differ in length or dtype")
    if send.is_cuda or recv.is_cuda:
        raise InvalidArgumentError("nvrar: host path takes CPU tensors")
    if not (send.is_contiguous() and recv.is_contiguous()):
        raise InvalidArgumentError("nvrar: buffers must be contiguous")


def _check_uniform(inputs: Sequence[torch.Tensor], outputs: Sequence[torch.Tensor],
                   device: Optional[int] = None) -> None:
    """One launch covers every virtual rank with inputs[0]'s length and dtype,
    so every buffer must have them (a shorter one would be read or written past
    its end) and, for device buffers, live on the group's device."""
    n, dt = inputs[0].numel(), inputs[0].dtype
    for t in list(inputs) + list(outputs):
        if t.numel() != n or t.dtype != dt:
            raise InvalidArgumentError("nvrar: every rank's buffers must have the same length "
                                       "and dtype")
        if device is not None and t.is_cuda and t.device.index != device:
            raise InvalidArgumentError(f"nvrar: buffer on {t.device}, group is on cuda:{device}")


def _check_pair(send: torch.Tensor, recv: torch.Tensor) -> None:
    if send.numel() != recv.numel():
        raise InvalidArgumentError("nvrar: input and output lengths differ")
    if send.dtype != recv.dtype:
        raise InvalidArgumentError("nvrar: input and output dtypes differ")
    if not (send.is_cuda and recv.is_cuda):
        raise InvalidArgumentError("nvrar: buffers must be CUDA tensors")
    if not (send.is_contiguous() and recv.is_contiguous()):
        raise InvalidArgumentError("nvrar: buffers must be contiguous")


PHASE_REDUCE_SCATTER, PHASE_RD_INTER, PHASE_ALL_GATHER = 1, 2, 3
# reduction orders of the reference's three all-reduces (nvrar.h nvrar_order_t)
_ORDERS = {"nvrar": 0, "ring": 1, "tree": 2}
_PHASES = {"reduce_scatter": PHASE_REDUCE_SCATTER, "rd_inter": PHASE_RD_INTER,
           "all_gather": PHASE_ALL_GATHER}


def _check_phase_io(phase: int, src: torch.Tensor, dst: torch.Tensor, gpus: int) -> None:
    if not (src.is_cuda and dst.is_cuda):
        raise InvalidArgumentError("nvrar: buffers must be CUDA tensors")
    if not (src.is_contiguous() and dst.is_contiguous()):
        raise InvalidArgumentError("nvrar: buffers must be contiguous")
    if src.dtype != dst.dtype:
        raise InvalidArgumentError("nvrar: input and output dtypes differ")
    n = src.numel()
    if phase == PHASE_REDUCE_SCATTER and dst.numel() != -(-n // gpus):
        raise InvalidArgumentError("intra reduce-scatter: shard output must be ceil(n/G)")
    if phase == PHASE_ALL_GATHER and dst.numel() != n * gpus:
        raise InvalidArgumentError("intra all-gather: output must be G * shard")
    if phase == PHASE_RD_INTER:
        if src.dtype != torch.int64:
            raise InvalidArgumentError("rd_inter: packed words are int64 tensors")
        if dst.numel() != n:
            raise InvalidArgumentError("rd_inter: bad shard length")


# ---- the reference-shaped collective ------------------------------------------------

class NvrarAllreduce:
    """Per-rank NVRAR state, as ``ccsim::NvrarAllreduce<T>`` (nvrar.hpp:41-250).

    ``comm`` owns the symmetric staging sized for ``max_elems`` elements of the
    widest use; ``run`` launches the persistent kernel on the current stream.
    """

    def __init__(self, comm: Communicator, max_elems: int):
        self.comm = comm
        self.max_elems = max_elems

    def sequence(self) -> int:
        return self.comm.sequence()

    def peers(self) -> List[RankId]:
        return self.comm.peers()

    def run(self, inp: torch.Tensor, out: torch.Tensor, cfg: NvrarConfig = NvrarConfig(),
            stream: Optional[torch.cuda.Stream] = None, sync: bool = False) -> None:
        cfg.validate()
        if inp.numel() != out.numel():
            raise InvalidArgumentError("nvrar: input and output lengths differ")
        if inp.numel() > self.max_elems:
            raise InvalidArgumentError("nvrar: vector longer than the preallocated maximum")
        self.comm.set_config(cfg)
        self.comm.allreduce(inp, out, stream)
        if sync:
            self.comm.check()


class LocalGroup:
    """Every rank of ``topo`` as a virtual rank on ONE device, each with its own
    communicator and symmetric region; one cooperative launch runs them all.
    This is the all-ranks-in-one-process shape of the reference's run_ranks
    (run.hpp:15-24), on a GPU."""

    def __init__(self, topo: ClusterTopology, max_bytes: int, device: int = 0,
                 timeout_s: float = 10.0):
        topo.require_power_of_two_nodes("nvrar")
        p = topo.world_size()
        if p > L.MAX_LOCAL:
            raise InvalidArgumentError(f"at most {L.MAX_LOCAL} virtual ranks per device")
        self.topo = topo
        self.device = device
        self.comms = [Communicator(topo, r, device, max_bytes, timeout_s=timeout_s)
                      for r in range(p)]
        handles = [c.export() for c in self.comms]
        for c in self.comms:
            c.connect(handles)
        self._lib = L.load()
        self._arr = (ctypes.c_void_p * p)(*[c._h.value for c in self.comms])
        # pointer arrays built from packed bytes (half the cost of the ctor)
        self._ptrs, self._ptr_fmt = ctypes.c_void_p * p, f"{p}Q"

    def set_config(self, cfg: NvrarConfig) -> None:
        for c in self.comms:
            c.set_config(cfg)

    def set_algo(self, algo: str) -> None:
        for c in self.comms:
            c.set_algo(algo)

    def set_timeout(self, s: float) -> None:
        for c in self.comms:
            c.set_timeout(s)

    def set_protocol(self, proto: str) -> None:
        for c in self.comms:
            c.set_protocol(proto)

    def set_jitter(self, max_ns: int, seed: int = 0) -> None:
        for r, c in enumerate(self.comms):
            c.set_jitter(max_ns, seed * 131 + r)

    def set_host_chunk(self, nbytes: int) -> None:
        for c in self.comms:
            c.set_host_chunk(nbytes)

    def launch_host(self, inputs: Sequence[torch.Tensor], outputs: Sequence[torch.Tensor],
                    stream: Optional[torch.cuda.Stream] = None) -> None:
        """nvrar_allreduce_local_host: every virtual rank's CPU tensors in and out."""
        p = len(self.comms)
        if len(inputs) != p or len(outputs) != p:
            raise InvalidArgumentError("one input and one output per rank")
        # one pass over the buffers (this call's own cost is part of the e2e step)
        n, dt = inputs[0].numel(), inputs[0].dtype
        send, recv = [], []
        for a, b in zip(inputs, outputs):
            if a.numel() != n or b.numel() != n or a.dtype != dt or b.dtype != dt:
                _check_host_pair(a, b)
                _check_uniform(inputs, outputs)
            if a.is_cuda or b.is_cuda or not (a.is_contiguous() and b.is_contiguous()):
                _check_host_pair(a, b)
            send.append(a.data_ptr())
            recv.append(b.data_ptr())
        pack, arr = struct.pack, self._ptrs.from_buffer_copy
        rc = self._lib.nvrar_allreduce_local_host(self._arr, p, arr(pack(self._ptr_fmt, *send)),
                                                  arr(pack(self._ptr_fmt, *recv)), n,
                                                  dtype_code(dt), L.SUM, _stream_ptr(stream))
        if rc:
            _raise(rc, self.comms[0].last_error())

    def plan(self, count: int, dtype: torch.dtype, active: Optional[Sequence[int]] = None):
        """(schedule, CTAs per rank) a launch of this group runs for `count` elements."""
        a, b = ctypes.c_int(), ctypes.c_int()
        mask = (1 << 64) - 1 if active is None else sum(1 << r for r in active)
        rc = self._lib.nvrar_plan_local(self._arr, self.topo.world_size(), count,
                                        dtype_code(dtype), mask, ctypes.byref(a), ctypes.byref(b))
        if rc:
            _raise(rc, self.comms[0].last_error())
        return L.ALGO_NAMES[a.value], b.value

    def launch(self, inputs: Sequence[torch.Tensor], outputs: Sequence[torch.Tensor],
               active: Optional[Sequence[int]] = None,
               stream: Optional[torch.cuda.Stream] = None, order: str = "nvrar",
               residuals: Optional[Sequence[torch.Tensor]] = None) -> None:
        p = self.topo.world_size()
        if len(inputs) != p or len(outputs) != p:
            raise InvalidArgumentError("one input and one output per rank")
        for a, b in zip(inputs, outputs):
            _check_pair(a, b)
        _check_uniform(inputs, outputs, self.device)
        n = inputs[0].numel()
        dt = dtype_code(inputs[0].dtype)
        send = (ctypes.c_void_p * p)(*[t.data_ptr() for t in inputs])
        recv = (ctypes.c_void_p * p)(*[t.data_ptr() for t in outputs])
        mask = (1 << 64) - 1 if active is None else sum(1 << r for r in active)
        if residuals is not None:
            if len(residuals) != p:
                raise InvalidArgumentError("one residual per rank")
            for x in residuals:
                _check_pair(inputs[0], x)
            _check_uniform(inputs, residuals, self.device)
            res = (ctypes.c_void_p * p)(*[t.data_ptr() for t in residuals])
            rc = self._lib.nvrar_allreduce_local_residual(self._arr, p, send, recv, res, n, dt,
                                                          L.SUM, _stream_ptr(stream), mask)
        elif order == "nvrar":
            rc = self._lib.nvrar_allreduce_local(self._arr, p, send, recv, n, dt, L.SUM,
                                                 _stream_ptr(stream), mask)
        else:
            rc = self._lib.nvrar_allreduce_local_order(self._arr, p, _ORDERS[order], send, recv,
                                                       n, dt, L.SUM, _stream_ptr(stream), mask)
        if rc:
            _raise(rc, self.comms[0].last_error())

    def check(self) -> None:
        """Synchronise; raise the reference's exception for the first fault.
        A deadlock reports the blocked set over all ranks (errors.hpp:61-85)."""
        torch.cuda.synchronize(self.device)
        codes = [c.check_status() for c in self.comms]
        if any(code == L.ERR_DEADLOCK for code in codes) and not any(
                code == L.ERR_PROTOCOL_FAULT for code in codes):
            blocked = [_blocked_rank(c.blocked()) for c, code in zip(self.comms, codes)
                       if code == L.ERR_DEADLOCK]
            raise DeadlockError(sorted(blocked, key=lambda b: b.global_rank))
        for c, code in zip(self.comms, codes):
            if code:
                _raise(code, c.last_error(), c.rank)

    def launch_phase(self, phase: str, inputs: Sequence[torch.Tensor],
                     outputs: Sequence[torch.Tensor], dtype: Optional[torch.dtype] = None,
                     active: Optional[Sequence[int]] = None,
                     stream: Optional[torch.cuda.Stream] = None) -> None:
        """One phase-only launch for every virtual rank (nvrar_phase_local).
        phase: 'reduce_scatter' | 'all_gather' | 'rd_inter' (dtype = the packed
        words' element type, int32 or float32)."""
        code = _PHASES[phase]
        p = self.topo.world_size()
        if len(inputs) != p or len(outputs) != p:
            raise InvalidArgumentError("one input and one output per rank")
        for a, b in zip(inputs, outputs):
            _check_phase_io(code, a, b, self.topo.gpus_per_node)
        _check_uniform(inputs, [], self.device)
        _check_uniform(outputs, [], self.device)
        dt = dtype_code(dtype if code == PHASE_RD_INTER else inputs[0].dtype)
        send = (ctypes.c_void_p * p)(*[t.data_ptr() for t in inputs])
        recv = (ctypes.c_void_p * p)(*[t.data_ptr() for t in outputs])
        mask = (1 << 64) - 1 if active is None else sum(1 << r for r in active)
        rc = self._lib.nvrar_phase_local(self._arr, p, code, send, recv, inputs[0].numel(), dt,
                                         _stream_ptr(stream), mask)
        if rc:
            _raise(rc, self.comms[0].last_error())

    def run_phase(self, phase: str, inputs: Sequence[torch.Tensor],
                  outputs: Sequence[torch.Tensor], dtype: Optional[torch.dtype] = None,
                  active: Optional[Sequence[int]] = None) -> None:
        self.launch_phase(phase, inputs, outputs, dtype, active)
        self.check()

    def run_all(self, inputs: Sequence[torch.Tensor], outputs: Sequence[torch.Tensor],
                cfg: Optional[NvrarConfig] = None, active: Optional[Sequence[int]] = None,
                check: bool = True, order: str = "nvrar") -> None:
        if cfg is not None:
            self.set_config(cfg)
        self.launch(inputs, outputs, active, order=order)
        if check:
            self.check()

    def sequences(self) -> List[int]:
        return [c.sequence() for c in self.comms]

    def close(self) -> None:
        for c in self.comms:
            c.close()
