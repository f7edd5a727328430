"""GPU parity of the phase-only entry points (nvrar_reduce_scatter,
nvrar_all_gather, nvrar_rd_inter through nvrar_phase_local) against the
reference's own standalone phases — golden vectors produced by
ccsim::IntraReduceScatter / IntraAllGather / NvrarAllreduce::rd_inter
(tests/golden/make_golden.py) — and the oracle restatements. Mirrors
collectives_test.cpp:179-354. Bar: bit-exact (int32, fp32); bf16 = the bf16
rule (fp32 fold of the up-cast inputs, one RNE rounding), 0 ulp.
"""
import hashlib

import numpy as np
import pytest
import torch

from oracle import oracle as O

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2511_09557_b200 import (ClusterTopology, InvalidArgumentError,  # noqa: E402
                                   LocalGroup, NvrarConfig, ProtocolFaultError)

TORCH = {"f32": torch.float32, "i32": torch.int32}


def grp(nodes, gpus, max_bytes=1 << 20):
    return LocalGroup(ClusterTopology(nodes, gpus), max_bytes, device=0, timeout_s=10.0)


def run_rs(g, x, dt):
    p, n = x.shape
    G = g.topo.gpus_per_node
    ins = [torch.from_numpy(np.ascontiguousarray(x[r])).cuda() for r in range(p)]
    outs = [torch.empty(-(-n // G), dtype=ins[0].dtype, device="cuda") for _ in range(p)]
    g.run_phase("reduce_scatter", ins, outs)
    return np.stack([o.cpu().numpy() for o in outs])


def run_ag(g, shards):
    p, ce = shards.shape
    G = g.topo.gpus_per_node
    ins = [torch.from_numpy(np.ascontiguousarray(shards[r])).cuda() for r in range(p)]
    outs = [torch.empty(ce * G, dtype=ins[0].dtype, device="cuda") for _ in range(p)]
    g.run_phase("all_gather", ins, outs)
    return np.stack([o.cpu().numpy() for o in outs])


def run_rd(g, shards, dt, seq=None, cfg=None):
    """The collectives_test.cpp:286-302 driver: pack with sequence()+1, run
    rd_inter, unpack with the new sequence()."""
    if cfg is not None:
        g.set_config(cfg)
    call = (g.sequences()[0] + 1) if seq is None else seq
    packed = O.pack_fused(shards, call)
    ins = [torch.from_numpy(packed[r].view(np.int64)).cuda() for r in range(shards.shape[0])]
    outs = [torch.empty_like(t) for t in ins]
    g.run_phase("rd_inter", ins, outs, dtype=TORCH[dt])
    seqs = g.sequences()
    assert all(s == call for s in seqs) or seq is not None
    return np.stack([O.unpack_fused(o.cpu().numpy().view(np.uint64), call,
                                    np.float32 if dt == "f32" else np.int32) for o in outs])


def test_rs_hand_checked_two_ranks():
    """collectives_test.cpp:180-195: [1,2] and [3,4] -> rank 0 owns {4}, rank 1 {6}."""
    g = grp(1, 2)
    try:
        out = run_rs(g, np.array([[1, 2], [3, 4]], np.int32), "i32")
        assert out.tolist() == [[4], [6]]
    finally:
        g.close()


@pytest.mark.parametrize("nodes,gpus,n,dt,seed", [(1, 4, 64, "i32", 17), (2, 4, 1031, "f32", 19),
                                                  (1, 3, 1000, "f32", 21), (2, 3, 4099, "f32", 23)])
def test_rs_then_ag_match_reference(golden, nodes, gpus, n, dt, seed):
    """collectives_test.cpp:196-216: shards concatenate to the node sum (the
    reference's bits) and the all-gather restores them on every member."""
    g_, meta = golden
    key = f"rs_{dt}_{nodes}x{gpus}_n{n}_s{seed}"
    x = O.random_inputs(nodes * gpus, n, seed, dt)
    g = grp(nodes, gpus)
    try:
        rs = run_rs(g, x, dt)
        assert np.array_equal(rs.view(np.uint32), g_[key].view(np.uint32))
        ag = run_ag(g, rs)
        assert hashlib.sha256(ag.tobytes()).hexdigest() == meta[f"ag_{key[3:]}_sha256"]
        # the phases consumed one sequence number each, on every rank
        assert g.sequences() == [2] * (nodes * gpus)
    finally:
        g.close()


@pytest.mark.parametrize("nodes,gpus,n", [(1, 4, 4099), (2, 4, 65539), (1, 8, 1000), (1, 2, 7)])
@pytest.mark.parametrize("dt", ["f32", "bf16", "i32"])
def test_rs_ag_random_vs_oracle(nodes, gpus, n, dt):
    x = O.random_inputs(nodes * gpus, n, 101 + n, "i32" if dt == "i32" else "f32")
    g = grp(nodes, gpus)
    try:
        if dt == "bf16":
            xb = O.bf16_bits_from_f32(x)
            ins = [torch.from_numpy(xb[r]).view(torch.int16).view(torch.bfloat16).cuda()
                   for r in range(nodes * gpus)]
            G = gpus
            outs = [torch.empty(-(-n // G), dtype=torch.bfloat16, device="cuda")
                    for _ in ins]
            g.run_phase("reduce_scatter", ins, outs)
            got = np.stack([o.view(torch.int16).cpu().numpy().view(np.uint16) for o in outs])
            up = O.f32_from_bf16_bits(xb)
            for node in range(nodes):
                want = O.bf16_bits_from_f32(O.intra_rs_sum(up[node * gpus:(node + 1) * gpus]))
                assert np.array_equal(got[node * gpus:(node + 1) * gpus].reshape(-1), want)
            full = [torch.empty(-(-n // G) * G, dtype=torch.bfloat16, device="cuda") for _ in ins]
            g.run_phase("all_gather", outs, full)
            for r in range(nodes * gpus):
                node = r // gpus
                assert np.array_equal(full[r].view(torch.int16).cpu().numpy().view(np.uint16),
                                      got[node * gpus:(node + 1) * gpus].reshape(-1))
            return
        rs = run_rs(g, x, dt)
        for node in range(nodes):
            want = O.intra_rs_sum(x[node * gpus:(node + 1) * gpus])
            assert np.array_equal(rs[node * gpus:(node + 1) * gpus].reshape(-1).view(np.uint32),
                                  want.view(np.uint32))
        ag = run_ag(g, rs)
        for r in range(nodes * gpus):
            node = r // gpus
            assert np.array_equal(ag[r], rs[node * gpus:(node + 1) * gpus].reshape(-1))
    finally:
        g.close()


def test_rs_single_participant_passthrough():
    """collectives_test.cpp:217-227."""
    g = grp(1, 1)
    try:
        assert run_rs(g, np.array([[9, 8, 7]], np.int32), "i32").tolist() == [[9, 8, 7]]
    finally:
        g.close()


def test_rd_inter_hand_cases():
    """collectives_test.cpp:304-316: one node = identity, two nodes exchange once."""
    g = grp(1, 1)
    try:
        assert run_rd(g, np.array([[5, -6, 7]], np.int32), "i32").tolist() == [[5, -6, 7]]
    finally:
        g.close()
    g = grp(2, 1)
    try:
        out = run_rd(g, np.array([[1, 2], [10, 20]], np.int32), "i32")
        assert out.tolist() == [[11, 22], [11, 22]]
    finally:
        g.close()


@pytest.mark.parametrize("nodes,gpus,w,dt,seed", [(8, 2, 96, "i32", 5), (4, 2, 777, "f32", 29),
                                                  (8, 1, 1000, "f32", 31), (2, 4, 100, "f32", 37)])
def test_rd_inter_matches_reference(golden, nodes, gpus, w, dt, seed):
    g_, _ = golden
    x = O.random_inputs(nodes * gpus, w, seed, dt)
    want = g_[f"rd_{dt}_{nodes}x{gpus}_w{w}_s{seed}"]
    g = grp(nodes, gpus)
    try:
        # collectives_test.cpp:317-341: every (blocks, chunk) agrees bit for bit
        for blocks in (1, 2, 4):
            for chunk in (8, 64, 512):
                out = run_rd(g, x, dt, cfg=NvrarConfig(blocks, chunk))
                assert np.array_equal(out.view(np.uint32), want.view(np.uint32))
        assert np.array_equal(want.view(np.uint32), O.rd_inter(x, nodes, gpus).view(np.uint32))
    finally:
        g.close()


def test_rd_inter_stale_flag_is_a_protocol_fault():
    """A shard packed with the wrong sequence number (nvrar.hpp:145-150)."""
    g = grp(2, 1)
    try:
        x = O.random_inputs(2, 64, 3, "i32")
        with pytest.raises(ProtocolFaultError):
            run_rd(g, x, "i32", seq=7)
    finally:
        g.close()


def test_phase_argument_checks():
    g = grp(1, 2)
    try:
        a = [torch.zeros(8, dtype=torch.int32, device="cuda") for _ in range(2)]
        with pytest.raises(InvalidArgumentError):  # shard must be ceil(n/G)
            g.launch_phase("reduce_scatter", a, [torch.zeros(3, dtype=torch.int32,
                                                             device="cuda")] * 2)
        with pytest.raises(InvalidArgumentError):  # empty vector (nvrar.hpp:282-284)
            e = [torch.zeros(0, dtype=torch.int32, device="cuda") for _ in range(2)]
            g.launch_phase("reduce_scatter", e, e)
        with pytest.raises(InvalidArgumentError):  # all-gather output must be G * shard
            g.launch_phase("all_gather", a, a)
        p = [torch.zeros(4, dtype=torch.int64, device="cuda") for _ in range(2)]
        with pytest.raises(InvalidArgumentError):  # packed words carry int32/fp32
            g.launch_phase("rd_inter", p, p, dtype=torch.bfloat16)
        with pytest.raises(InvalidArgumentError):  # longer than max_bytes allows
            big = [torch.zeros(1 << 20, dtype=torch.int32, device="cuda") for _ in range(2)]
            g.launch_phase("reduce_scatter", big, [torch.zeros(1 << 19, dtype=torch.int32,
                                                               device="cuda")] * 2)
    finally:
        g.close()


def test_phases_interleave_with_allreduce():
    """Phase calls share the comm's call counter with the all-reduce: a mixed
    sequence stays in step and every result stays exact."""
    nodes, gpus = 2, 4
    g = grp(nodes, gpus)
    try:
        for it in range(3):
            x = O.random_inputs(8, 5000 + it, 40 + it, "f32")
            rs = run_rs(g, x, "f32")
            ag = run_ag(g, rs)
            assert ag.shape == (8, rs.shape[1] * gpus)
            sh = O.random_inputs(8, 300, 50 + it, "f32")
            assert np.array_equal(run_rd(g, sh, "f32").view(np.uint32),
                                  O.rd_inter(sh, nodes, gpus).view(np.uint32))
            for algo in ("hier", "twoshot", "oneshot", "direct"):
                g.set_algo(algo)
                ins = [torch.from_numpy(x[r]).cuda() for r in range(8)]
                outs = [torch.empty_like(t) for t in ins]
                g.run_all(ins, outs)
                want = O.nvrar_order_sum(x, nodes, gpus).view(np.uint32)
                for o in outs:
                    assert np.array_equal(o.cpu().numpy().view(np.uint32), want)
        assert g.sequences() == [3 * 7] * 8
    finally:
        g.close()
