"""The C-ABI library loads and exports every symbol include/nvrar.h declares;
host-side validation mirrors the reference's errors (no GPU needed)."""
import ctypes
import os
import re

import pytest

from paper_2511_09557_b200 import _lib as L
from paper_2511_09557_b200 import comm as C

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    src = open(os.path.join(ROOT, "include", "nvrar.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(nvrar_[a-z_]+)\s*\(", src)) - {"nvrar_allgather_fn"})


def test_library_exports_every_declared_symbol():
    lib = L.load()
    syms = header_symbols()
    assert len(syms) >= 20
    for s in syms:
        assert hasattr(lib, s), s
    assert set(syms) == set(L.SIGNATURES), set(syms) ^ set(L.SIGNATURES)


def test_abi_version_and_status_strings():
    lib = L.load()
    assert lib.nvrar_abi_version() == 1
    assert lib.nvrar_status_string(L.ERR_DEADLOCK) == b"deadlock"
    assert lib.nvrar_status_string(L.ERR_PROTOCOL_FAULT) == b"protocol fault"


def _args(**kw):
    d = dict(world_size=8, rank=0, nodes=2, gpus_per_node=4, device=0, max_bytes=1 << 20,
             blocks=0, chunk_bytes=65536, timeout_s=1.0)
    d.update(kw)
    return L.InitArgs(**d)


def test_create_validates_before_touching_the_device():
    lib = L.load()
    h = ctypes.c_void_p()
    # InvalidTopologyError: non power-of-two node count (nvrar.hpp:46)
    assert lib.nvrar_comm_create(ctypes.byref(_args(nodes=3, world_size=12)), ctypes.byref(h)) \
        == L.ERR_INVALID_TOPOLOGY
    assert b"power of two" in lib.nvrar_last_error(None)
    assert lib.nvrar_comm_create(ctypes.byref(_args(world_size=7)), ctypes.byref(h)) \
        == L.ERR_INVALID_ARGUMENT
    assert lib.nvrar_comm_create(ctypes.byref(_args(chunk_bytes=12)), ctypes.byref(h)) \
        == L.ERR_INVALID_ARGUMENT
    assert lib.nvrar_comm_create(ctypes.byref(_args(rank=8)), ctypes.byref(h)) \
        == L.ERR_INVALID_ARGUMENT
    assert lib.nvrar_init(ctypes.byref(_args()), ctypes.byref(h)) == L.ERR_INVALID_ARGUMENT


def plan_for(world, nodes, gpus, count, dtype, algo=0, blocks=0, max_ctas=148):
    lib = L.load()
    a, b = ctypes.c_int(), ctypes.c_int()
    rc = lib.nvrar_plan_for(world, nodes, gpus, count, dtype, algo, blocks, max_ctas,
                            ctypes.byref(a), ctypes.byref(b))
    assert rc == 0
    return L.ALGO_NAMES[a.value], b.value


def test_selector_is_a_pure_function():
    assert plan_for(8, 2, 4, 65536, L.BF16) == plan_for(8, 2, 4, 65536, L.BF16)
    algo, blocks = plan_for(8, 2, 4, 1 << 20, L.BF16)
    assert algo in ("twoshot", "hier", "oneshot") and 1 <= blocks <= 148
    # flat schedules are capped at 16 ranks / MAXG gpus per node -> hier
    assert plan_for(16, 8, 2, 1 << 16, L.FLOAT32)[0] in ("oneshot", "twoshot")
    assert plan_for(32, 8, 4, 1 << 16, L.FLOAT32)[0] == "hier"
    # forced schedule and CTA count win
    assert plan_for(8, 2, 4, 1 << 20, L.BF16, algo=L.ALGO_HIER, blocks=7) == ("hier", 7)
    # one-shot is bounded by its staging size
    assert plan_for(8, 2, 4, 4 << 20, L.BF16, algo=L.ALGO_ONESHOT)[0] == "twoshot"


def test_python_mirror_errors():
    with pytest.raises(C.InvalidTopologyError):
        C.ClusterTopology(3, 1).require_power_of_two_nodes("nvrar")
    with pytest.raises(C.InvalidArgumentError):
        C.ClusterTopology(0, 1).validate()
    with pytest.raises(C.InvalidArgumentError):
        C.NvrarConfig(blocks=-1).validate()
    with pytest.raises(C.InvalidArgumentError):
        C.NvrarConfig(chunk_bytes=12).validate()
    C.NvrarConfig(blocks=1, chunk_bytes=8).validate()
    with pytest.raises(C.InvalidTopologyError):
        C.Communicator(C.ClusterTopology(3, 1), 0, 0, 1 << 20)
    topo = C.ClusterTopology(2, 4)
    assert C.RankId(1, 2).global_(topo) == 6
    assert C.RankId.from_global(6, topo) == C.RankId(1, 2)
    assert C.log2_exact(8) == 3 and C.is_power_of_two(4) and not C.is_power_of_two(6)


def test_deadlock_error_formats_blocked_set():
    e = C.DeadlockError([C.BlockedRank(0, C.BlockedRank.Kind.FlagWait, peer_rank=1, expected=2),
                         C.BlockedRank(1, C.BlockedRank.Kind.SeqWait, peer_rank=3, expected=2)])
    assert "2 rank(s) blocked" in str(e)
    assert e.blocked()[1].peer_rank == 3


def test_selector_default_policy_and_fallbacks():
    """The built-in policy (nvrar_comm.cu default_plan) and the schedule fallbacks."""
    # one-shot while (P-1)M inbound stays small; two-shot above it at P <= 4
    assert plan_for(4, 2, 2, (256 << 10) // 2, L.BF16)[0] == "oneshot"
    assert plan_for(4, 2, 2, (2 << 20) // 2, L.BF16)[0] == "twoshot"
    # the paper's hierarchy in the middle at P = 8
    assert plan_for(8, 2, 4, (1 << 20) // 2, L.BF16)[0] == "hier"
    assert plan_for(8, 2, 4, (8 << 20) // 2, L.BF16)[0] == "twoshot"
    assert plan_for(8, 2, 4, (2 << 20) // 2, L.BF16)[0] == "twoshot"
    # single rank: a copy through the one-shot
    assert plan_for(1, 1, 1, 1000, L.FLOAT32)[0] == "oneshot"
    # multicast one-shot: bounded like the one-shot; hierarchy where flat is not allowed
    assert plan_for(4, 2, 2, 1000, L.BF16, algo=L.ALGO_MCAST)[0] == "mcast"
    assert plan_for(4, 2, 2, (4 << 20) // 2, L.BF16, algo=L.ALGO_MCAST)[0] == "twoshot"
    assert plan_for(32, 8, 4, 1000, L.BF16, algo=L.ALGO_MCAST)[0] == "hier"
    # the direct schedule exists only for a local group of virtual ranks
    assert plan_for(8, 2, 4, 1000, L.FLOAT32, algo=L.ALGO_DIRECT)[0] == "hier"


def test_host_buffer_argument_checks():
    """The host-buffer path's Python checks (no device needed)."""
    import torch
    from paper_2511_09557_b200.comm import InvalidArgumentError, _check_host_pair
    a = torch.zeros(16, dtype=torch.float32)
    _check_host_pair(a, torch.zeros(16, dtype=torch.float32))
    with pytest.raises(InvalidArgumentError):
        _check_host_pair(a, torch.zeros(8, dtype=torch.float32))
    with pytest.raises(InvalidArgumentError):
        _check_host_pair(a, torch.zeros(16, dtype=torch.bfloat16))
    with pytest.raises(InvalidArgumentError):
        _check_host_pair(torch.zeros(32)[::2], torch.zeros(16))


def test_flat_fallback_applies_after_the_oneshot_size_rewrite():
    """a >1 MB multicast / one-shot request on a topology the flat
    kernels cannot hold (32 ranks) must run the hierarchy, not a two-shot that
    has no kernel."""
    big = (2 << 20) // 2
    for algo in (L.ALGO_MCAST, L.ALGO_ONESHOT, L.ALGO_TWOSHOT):
        assert plan_for(32, 4, 8, big, L.BF16, algo=algo)[0] == "hier"


def test_local_group_buffers_must_be_uniform():
    """one launch covers every virtual rank with inputs[0]'s length
    and dtype, so a shorter or differently typed buffer is rejected."""
    import torch
    from paper_2511_09557_b200.comm import InvalidArgumentError, _check_uniform
    a = [torch.zeros(16) for _ in range(4)]
    _check_uniform(a, [torch.zeros(16) for _ in range(4)])
    with pytest.raises(InvalidArgumentError):
        _check_uniform(a, [torch.zeros(16)] * 3 + [torch.zeros(15)])
    with pytest.raises(InvalidArgumentError):
        _check_uniform(a[:3] + [torch.zeros(16, dtype=torch.bfloat16)], a)


def test_local_group_launch_host_checks_every_buffer():
    """LocalGroup.launch_host's one-pass checks (no device: the C call is a
    stub that records its arguments): every rank's pair is checked for length,
    dtype, device and layout, and the pointers reach the C ABI in rank order."""
    import ctypes

    import torch
    from paper_2511_09557_b200.comm import InvalidArgumentError, LocalGroup

    p = 4
    seen = {}

    class Lib:
        def nvrar_allreduce_local_host(self, arr, np_, send, recv, n, dt, op, stream):
            seen.update(p=np_, send=[send[i] for i in range(np_)],
                        recv=[recv[i] for i in range(np_)], n=n, dt=dt)
            return 0

    g = LocalGroup.__new__(LocalGroup)
    g.comms = [None] * p
    g._lib = Lib()
    g._arr = (ctypes.c_void_p * p)()
    g._ptrs, g._ptr_fmt = ctypes.c_void_p * p, f"{p}Q"
    ins = [torch.zeros(16) for _ in range(p)]
    outs = [torch.zeros(16) for _ in range(p)]

    class S:
        cuda_stream = 0

    g.launch_host(ins, outs, stream=S())
    assert seen["send"] == [t.data_ptr() for t in ins]
    assert seen["recv"] == [t.data_ptr() for t in outs]
    assert seen["n"] == 16 and seen["p"] == p
    bad = [
        (ins, outs[:3] + [torch.zeros(15)]),                      # a short output
        (ins[:2] + [torch.zeros(15), ins[3]], outs),               # a short input
        (ins, outs[:3] + [torch.zeros(16, dtype=torch.bfloat16)]),  # another dtype
        (ins[:3] + [torch.zeros(32)[::2]], outs),                  # not contiguous
        (ins[:3], outs[:3]),                                       # a rank missing
    ]
    for a, b in bad:
        with pytest.raises(InvalidArgumentError):
            g.launch_host(a, b, stream=S())


def test_torch_op_ids_are_never_reused():
    """unregister + register must not hand out a live id again."""
    from paper_2511_09557_b200 import torch_op
    a = torch_op.register(object())
    b = torch_op.register(object())
    torch_op.unregister(a)
    c = torch_op.register(object())
    assert len({a, b, c}) == 3
    torch_op.unregister(b)
    torch_op.unregister(c)
