"""GPU parity: the CUDA path (libnvrar_b200.so through the C ABI) against the
oracle on the same inputs, every rank of a hierarchy as a virtual rank on one
B200 (nvrar_allreduce_local: one cooperative launch, ranks co-resident).

Bar: fp32 and int32 bit-exact; bf16 bit-exact to the bf16 rule (fp32
reference on the up-cast inputs, one RNE rounding) — i.e. a stated tolerance
of 0 bf16 ulp against that oracle and <= 1/2 bf16 ulp against the exact fp32
reference result.
"""
import hashlib

import numpy as np
import pytest
import torch

from oracle import oracle as O

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2511_09557_b200 import (BlockedRank, ClusterTopology, DeadlockError,  # noqa: E402
                                   InvalidArgumentError, LocalGroup, NvrarConfig)

DEV = 0
ALGOS = ["hier", "twoshot", "oneshot", "direct"]
FLAT_MAXG = {1: 8, 2: 8, 4: 4, 8: 2}

_groups = {}


def group(nodes, gpus, max_bytes=4 << 20):
    key = (nodes, gpus, max_bytes)
    if key not in _groups:
        # keep at most a few groups alive (each owns P symmetric regions)
        if len(_groups) > 3:
            k0 = next(iter(_groups))
            _groups.pop(k0).close()
        _groups[key] = LocalGroup(ClusterTopology(nodes, gpus), max_bytes, device=DEV,
                                  timeout_s=20.0)
    return _groups[key]


def flat_ok(nodes, gpus):
    return gpus <= FLAT_MAXG[nodes] and nodes * gpus <= 16


def inputs_for(dtype, p, n, seed, dist="uniform"):
    if dtype == "i32":
        return O.random_inputs(p, n, seed, "i32")
    x = O.random_inputs(p, n, seed, "f32")
    if dist == "normal":
        rng = np.random.default_rng(seed)
        x = rng.standard_normal((p, n)).astype(np.float32)
    if dtype == "bf16":
        return O.bf16_bits_from_f32(x)
    return x


def to_dev(a, dtype):
    t = torch.from_numpy(np.ascontiguousarray(a))
    if dtype == "bf16":
        t = t.view(torch.int16).view(torch.bfloat16)
    return t.to(f"cuda:{DEV}")


def from_dev(t, dtype):
    if dtype == "bf16":
        return t.view(torch.int16).cpu().numpy().view(np.uint16)
    return t.cpu().numpy()


def run(g, x, dtype, algo="auto", cfg=None, active=None, proto="auto"):
    g.set_algo(algo)
    g.set_protocol(proto)
    ins = [to_dev(x[r], dtype) for r in range(x.shape[0])]
    outs = [torch.empty_like(t) for t in ins]
    g.run_all(ins, outs, cfg=cfg or NvrarConfig(), active=active)
    return np.stack([from_dev(o, dtype) for o in outs])


def assert_parity(out, x, nodes, gpus, dtype):
    want = O.nvrar_order_sum(x, nodes, gpus, {"f32": "f32", "i32": "i32", "bf16": "bf16"}[dtype])
    if dtype == "f32":
        out, want = out.view(np.uint32), want.view(np.uint32)
    for r in range(out.shape[0]):
        bad = np.flatnonzero(out[r] != want)
        assert bad.size == 0, f"rank {r}: {bad.size} mismatches, first at {bad[:5]}"


HIERS = [(1, 1), (1, 2), (2, 1), (1, 4), (2, 2), (4, 1), (1, 8), (2, 4), (4, 2), (8, 1),
         (2, 3), (8, 2)]


@pytest.mark.parametrize("nodes,gpus", HIERS)
@pytest.mark.parametrize("algo", ALGOS)
@pytest.mark.parametrize("dtype,proto", [("f32", "lamport"), ("f32", "ll"), ("bf16", "lamport"),
                                         ("bf16", "ll"), ("i32", "auto")])
def test_parity_hierarchies(nodes, gpus, algo, dtype, proto):
    if algo in ("twoshot", "oneshot") and not flat_ok(nodes, gpus):
        pytest.skip("flat schedules cover P <= 16 within MAXG")
    g = group(nodes, gpus)
    for n in (1, 7, 1031, 65539):
        x = inputs_for(dtype, nodes * gpus, n, 19 + n)
        assert_parity(run(g, x, dtype, algo, proto=proto), x, nodes, gpus, dtype)
    g.set_protocol("auto")


@pytest.mark.parametrize("algo", ALGOS)
@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_lamport_sentinel_pattern_is_data_not_a_hang(algo, dtype):
    """An all-ones input (the Lamport 'empty' pattern, a NaN) must travel as a NaN
    and never stall the receiver; every other element stays bit-exact."""
    g = group(2, 4)
    x = inputs_for(dtype, 8, 4099, 3)
    if dtype == "f32":
        xv = x.view(np.uint32)
        xv[3, 10] = 0xFFFFFFFF
        xv[0, 4000] = 0xFFFFFFFF
    else:
        x[3, 10] = 0xFFFF
        x[0, 4000] = 0xFFFF
    out = run(g, x, dtype, algo, proto="lamport")
    want = O.nvrar_order_sum(x, 2, 4, dtype)
    f = (lambda a: a.view(np.float32)) if dtype == "f32" else O.f32_from_bf16_bits
    for r in range(8):
        got = f(out[r])
        assert np.isnan(got[10]) and np.isnan(got[4000])
        keep = np.ones(4099, bool)
        keep[[10, 4000]] = False
        assert np.array_equal(out[r][keep], want[keep])


@pytest.mark.parametrize("algo", ALGOS)
def test_c1_golden_2x4_1MB_fp32(golden, algo):
    """BASELINE configs[0]: 2x4, 1 MB fp32, seed 1234 — reference's bits (sha256)."""
    _, meta = golden
    x = O.random_inputs(8, 262144, 1234, "f32")
    out = run(group(2, 4), x, "f32", algo)
    for r in range(8):
        assert hashlib.sha256(out[r].tobytes()).hexdigest() == meta["c1_2x4_1MB_f32_s1234_sha256"]


@pytest.mark.parametrize("algo", ALGOS)
def test_c2_golden_2x4_1MB_bf16(golden, algo):
    _, meta = golden
    xb = O.bf16_bits_from_f32(O.random_inputs(8, 262144, 1234, "f32"))
    out = run(group(2, 4), xb, "bf16", algo)
    for r in range(8):
        assert hashlib.sha256(out[r].tobytes()).hexdigest() == meta["c2_2x4_1MB_bf16_s1234_sha256"]


@pytest.mark.parametrize("algo", ALGOS)
def test_bf16_tolerance_signed_inputs(algo):
    """N(0,1) bf16 inputs (cancellation): exact vs the bf16 rule, and within half a
    bf16 ulp of the fp32 reference result."""
    g = group(2, 4)
    xb = inputs_for("bf16", 8, 100003, 5, dist="normal")
    out = run(g, xb, "bf16", algo)
    assert_parity(out, xb, 2, 4, "bf16")
    ref32 = O.nvrar_order_sum(O.f32_from_bf16_bits(xb).reshape(8, -1), 2, 4)
    got = O.f32_from_bf16_bits(out[0])
    # half a bf16 ulp: ulp(x) = 2^(e-7) for x in [2^e, 2^(e+1)) -> |err| <= 2^-8 |x|
    assert np.all(np.abs(got - ref32) <= np.ldexp(np.abs(ref32), -8) + 1e-45)


def test_ct_fixtures(golden):
    g_, _ = golden
    x = O.random_inputs(8, 129, 19, "f32")
    for algo in ALGOS:
        out = run(group(4, 2), x, "f32", algo)
        assert np.array_equal(out[0].view(np.uint32), g_["ct_float_4x2_n129_s19"].view(np.uint32))
    out = run(group(2, 2), np.arange(4, dtype=np.int32).reshape(4, 1), "i32", "hier")
    assert out[:, 0].tolist() == [6, 6, 6, 6]


def test_acceptance_grid_int32(golden):
    """acceptance_test.cpp:85-112 grid against the reference's hashes (hier schedule)."""
    _, meta = golden
    seed = 100
    for n in (1, 2, 4, 8):
        for gp in (1, 2, 4):
            g = group(n, gp, max_bytes=1 << 20)
            for nbytes in (8, 1024, 65536, 131072, 1048576):
                seed += 1
                x = O.random_inputs(n * gp, nbytes // 4, seed, "i32")
                out = run(g, x, "i32", "hier")
                h = meta["acceptance1_sha256"][f"{n}x{gp}_{nbytes}_s{seed}"]
                for r in range(n * gp):
                    assert hashlib.sha256(out[r].tobytes()).hexdigest() == h, (n, gp, nbytes, r)


@pytest.mark.parametrize("algo", ALGOS)
def test_block_chunk_invariance(algo):
    """acceptance criterion 4: results invariant to (blocks, chunk_bytes)."""
    g = group(2, 4)
    x = inputs_for("f32", 8, 262147, 4242)
    first = None
    for cfg in (NvrarConfig(1, 8), NvrarConfig(3, 64), NvrarConfig(8, 16384),
                NvrarConfig(32, 32768), NvrarConfig(0, 131072)):
        out = run(g, x, "f32", algo, cfg)
        assert_parity(out, x, 2, 4, "f32")
        if first is None:
            first = out
        assert np.array_equal(out.view(np.uint32), first.view(np.uint32))
    g.set_config(NvrarConfig())


@pytest.mark.parametrize("algo", ALGOS)
def test_back_to_back_100_calls(algo):
    """acceptance criterion 5 / collectives_test.cpp:397-423: fresh inputs each call,
    parity slots reused, sequence advances by exactly 100."""
    g = group(4, 2)
    g.set_algo(algo)
    n = 32768
    before = g.sequences()
    xs = [O.random_inputs(8, n, 5000 + c, "i32") for c in range(100)]
    ins = [[to_dev(x[r], "i32") for r in range(8)] for x in xs]
    outs = [[torch.empty_like(t) for t in row] for row in ins]
    g.set_config(NvrarConfig(8, 4096))
    for c in range(100):
        g.launch(ins[c], outs[c])
    g.check()
    for c in range(100):
        want = O.serial_sum(xs[c])
        for r in range(8):
            assert np.array_equal(outs[c][r].cpu().numpy(), want), (c, r)
    after = g.sequences()
    assert [a - b for a, b in zip(after, before)] == [100] * 8
    g.set_config(NvrarConfig())


def test_count_zero_bumps_sequence_and_in_place():
    g = group(2, 2)
    before = g.sequences()
    z = [torch.empty(0, device=f"cuda:{DEV}") for _ in range(4)]
    g.run_all(z, z)
    assert [a - b for a, b in zip(g.sequences(), before)] == [1] * 4
    x = inputs_for("f32", 4, 4099, 77)
    bufs = [to_dev(x[r], "f32") for r in range(4)]
    g.set_algo("hier")
    g.run_all(bufs, bufs)  # send == recv
    out = np.stack([b.cpu().numpy() for b in bufs])
    assert_parity(out, x, 2, 2, "f32")


def test_too_long_is_invalid_argument():
    g = group(2, 2, max_bytes=1 << 16)
    t = [torch.zeros(1 << 15, device=f"cuda:{DEV}") for _ in range(4)]
    with pytest.raises(InvalidArgumentError):
        g.run_all(t, t)
    with pytest.raises(InvalidArgumentError):
        g.run_all(t, [torch.zeros(5, device=f"cuda:{DEV}")] * 4)


def test_stalled_rank_blocks_exactly_its_step_peers(golden):
    """collectives_test.cpp:462-497 / acceptance criterion 6: 4x1, rank 3 stalls
    before call 2. The watchdog's blocked set must equal the reference's:
    rank 0 FlagWait; ranks 1 and 2 SeqWait on rank 3."""
    g_, _ = golden
    grp = LocalGroup(ClusterTopology(4, 1), 1 << 16, device=DEV, timeout_s=0.5)
    try:
        grp.set_algo("hier")
        x1 = O.random_inputs(4, 32, 31, "i32")
        x2 = O.random_inputs(4, 32, 32, "i32")
        out = run(grp, x1, "i32", "hier")
        for r in range(4):
            assert np.array_equal(out[r], O.serial_sum(x1))
        ins = [to_dev(x2[r], "i32") for r in range(4)]
        outs = [torch.empty_like(t) for t in ins]
        with pytest.raises(DeadlockError) as ei:
            grp.run_all(ins, outs, active=[0, 1, 2])
        b = ei.value.blocked()
        ref_rows = g_["stalled_4x1_rows"]
        assert [x.global_rank for x in b] == ref_rows[:, 0].tolist() == [0, 1, 2]
        assert [int(x.kind) for x in b] == ref_rows[:, 1].tolist()
        assert b[0].kind == BlockedRank.Kind.FlagWait
        assert b[1].kind == BlockedRank.Kind.SeqWait and b[1].peer_rank == 3
        assert b[2].kind == BlockedRank.Kind.SeqWait and b[2].peer_rank == 3
        assert all(x.expected == 2 for x in b)
    finally:
        grp.close()


def test_peers_and_sequence_api():
    g = group(4, 2)
    # nvrar.hpp:72-75: step-l peer = (node ^ 2^l, local)
    peers = g.comms[5].peers()
    assert [(p.node_rank, p.local_rank) for p in peers] == [(3, 1), (0, 1)]
    algo, blocks = g.comms[0].plan(1 << 20, torch.bfloat16)
    assert algo in ALGOS and blocks >= 1
    # a full local group of virtual ranks may take the direct schedule
    la, lb = g.plan(1 << 20, torch.bfloat16)
    assert la in ALGOS and lb >= 1
    assert g.plan(1 << 20, torch.bfloat16, active=[0, 1])[0] != "direct"


@pytest.mark.parametrize("nodes,gpus", HIERS)
@pytest.mark.parametrize("order", ["ring", "tree"])
@pytest.mark.parametrize("algo", ["auto", "oneshot", "twoshot"])
@pytest.mark.parametrize("dtype", ["f32", "bf16", "i32"])
def test_baseline_orders(nodes, gpus, order, algo, dtype):
    """nvrar_allreduce_local_order: the result bits of the reference's
    RingAllreduce / TreeAllreduce (ring_order_sum / tree_order_sum, pinned by
    tests/test_oracle.py against the reference's own runs)."""
    g = group(nodes, gpus)
    p = nodes * gpus
    ring_ok = p <= 8
    tree_ok = flat_ok(nodes, gpus)
    g.set_algo(algo)
    try:
        for n in (1, 7, 1031, 65539):
            x = inputs_for(dtype, p, n, 23 + n)
            ins = [to_dev(x[r], dtype) for r in range(p)]
            outs = [torch.empty_like(t) for t in ins]
            if (order == "ring" and not ring_ok) or (order == "tree" and not tree_ok):
                with pytest.raises(InvalidArgumentError):
                    g.run_all(ins, outs, order=order)
                return
            g.run_all(ins, outs, order=order)
            want = O.order_sum(x, nodes, gpus, order, dtype)
            got = np.stack([from_dev(o, dtype) for o in outs])
            if dtype == "f32":
                got, want = got.view(np.uint32), want.view(np.uint32)
            for r in range(p):
                assert np.array_equal(got[r], want), f"rank {r} differs"
    finally:
        g.set_algo("auto")


def test_baseline_orders_golden(golden):
    g_, meta = golden
    x = O.random_inputs(8, 1031, 19, "f32")
    grp = group(2, 4)
    for order in ("ring", "tree"):
        ins = [to_dev(x[r], "f32") for r in range(8)]
        outs = [torch.empty_like(t) for t in ins]
        grp.run_all(ins, outs, order=order)
        for o in outs:
            got = from_dev(o, "f32")
            assert hashlib.sha256(got.tobytes()).hexdigest() == \
                meta["baseline_orders_n1031_s19_sha256"][f"{order}_2x4"]


def _add_like(want, resid, dtype):
    """The element type's own add (what `residual + all_reduce(x)` gives)."""
    if dtype == "f32":
        return (want.view(np.float32) + resid.view(np.float32)).view(np.uint32)
    if dtype == "bf16":
        return O.bf16_bits_from_f32(O.f32_from_bf16_bits(want) + O.f32_from_bf16_bits(resid))
    with np.errstate(over="ignore"):
        return (want.astype(np.int64) + resid.astype(np.int64)).astype(np.int32)


@pytest.mark.parametrize("nodes,gpus", [(1, 2), (2, 2), (2, 4), (4, 2), (8, 1), (2, 3)])
@pytest.mark.parametrize("algo", ALGOS)
@pytest.mark.parametrize("dtype", ["f32", "bf16", "i32"])
@pytest.mark.parametrize("inplace", [False, True])
def test_allreduce_residual_fused(nodes, gpus, algo, dtype, inplace):
    """nvrar_allreduce_local_residual: out = residual + all_reduce(x), bit-identical
    to the all-reduce followed by the element type's add."""
    if algo in ("twoshot", "oneshot") and not flat_ok(nodes, gpus):
        pytest.skip("flat schedules")
    g = group(nodes, gpus)
    p = nodes * gpus
    g.set_algo(algo)
    try:
        for n in (7, 1031, 65539):
            x = inputs_for(dtype, p, n, 61 + n)
            res = inputs_for(dtype, p, n, 62 + n)
            ins = [to_dev(x[r], dtype) for r in range(p)]
            rs = [to_dev(res[r], dtype) for r in range(p)]
            outs = rs if inplace else [torch.empty_like(t) for t in ins]
            g.launch(ins, outs, residuals=rs)
            g.check()
            want = O.nvrar_order_sum(x, nodes, gpus, dtype)
            if dtype == "f32":
                want = want.view(np.uint32)
            for r in range(p):
                got = from_dev(outs[r], dtype)
                exp = _add_like(want, res[r].view(np.uint32) if dtype == "f32" else res[r], dtype)
                assert np.array_equal(got.view(exp.dtype), exp), f"rank {r}"
    finally:
        g.set_algo("auto")


@pytest.mark.parametrize("nodes,gpus", [(1, 2), (2, 2), (2, 4), (2, 3), (1, 3), (8, 1)])
@pytest.mark.parametrize("dtype", ["f32", "bf16", "i32"])
@pytest.mark.parametrize("chunk", [0, 256 << 10])
def test_host_buffer_pipeline_matches_whole_vector(nodes, gpus, dtype, chunk):
    """nvrar_allreduce_local_host: pinned host buffers used in place (zero-copy)
    or staged in chunks (256 KB windows of the whole vector) give the bits of ONE
    all-reduce of the whole vector — the windows keep the whole vector's
    reduction order (G = 3 makes the fold order depend on the element's shard,
    so a plain per-chunk all-reduce would differ)."""
    g = group(nodes, gpus, max_bytes=8 << 20)
    p = nodes * gpus
    # 0: pinned buffers are read / written in place by the kernels (zero-copy);
    # 256 KB: staged in several windows per vector
    g.set_host_chunk(chunk)
    for n in (5, 65536 + 3, 3 * 65536 + 1001):
        x = inputs_for(dtype, p, n, 71 + n)
        if dtype == "bf16":
            ins = [torch.from_numpy(x[r]).view(torch.int16).view(torch.bfloat16).pin_memory()
                   for r in range(p)]
        else:
            ins = [torch.from_numpy(np.ascontiguousarray(x[r])).pin_memory() for r in range(p)]
        outs = [torch.empty_like(t).pin_memory() for t in ins]
        g.launch_host(ins, outs)
        torch.cuda.synchronize()
        g.check()
        want = O.nvrar_order_sum(x, nodes, gpus, dtype)
        for r in range(p):
            got = outs[r].view(torch.int16).numpy().view(np.uint16) if dtype == "bf16" \
                else outs[r].numpy()
            if dtype == "f32":
                assert np.array_equal(got.view(np.uint32), want.view(np.uint32)), f"rank {r}"
            else:
                assert np.array_equal(got, want), f"rank {r}"
    g.set_host_chunk(0)


def test_host_buffer_pageable_memory():
    """Pageable (unpinned) host buffers take the staged path — same bits."""
    g = group(2, 2)
    x = inputs_for("f32", 4, 70001, 91)
    ins = [torch.from_numpy(np.ascontiguousarray(x[r])) for r in range(4)]  # not pinned
    outs = [torch.empty_like(t) for t in ins]
    g.launch_host(ins, outs)
    torch.cuda.synchronize()
    g.check()
    want = O.nvrar_order_sum(x, 2, 2).view(np.uint32)
    for r in range(4):
        assert np.array_equal(outs[r].numpy().view(np.uint32), want)


@pytest.mark.parametrize("chunk", [0, 64 << 10])
def test_host_buffer_longer_than_max_bytes(chunk):
    """A host vector longer than the comm's max_bytes runs as windows of the
    whole vector (zero-copy or staged) — still the bits of one all-reduce."""
    g = LocalGroup(ClusterTopology(2, 3), 256 << 10, device=DEV, timeout_s=20.0)
    try:
        g.set_host_chunk(chunk)
        x = inputs_for("f32", 6, 300001, 93)
        ins = [torch.from_numpy(np.ascontiguousarray(x[r])).pin_memory() for r in range(6)]
        outs = [torch.empty_like(t).pin_memory() for t in ins]
        g.launch_host(ins, outs)
        torch.cuda.synchronize()
        g.check()
        want = O.nvrar_order_sum(x, 2, 3).view(np.uint32)
        for r in range(6):
            assert np.array_equal(outs[r].numpy().view(np.uint32), want), f"rank {r}"
    finally:
        g.close()
