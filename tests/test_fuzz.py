"""GPU counterpart of the reference's concurrency fuzzing (acceptance
criterion 7, acceptance_test.cpp:314-367): seeded delay injection before
remote stores and between polls (nvrar_set_jitter, the analogue of
RunOptions::delay_max_us, concurrent_transport.hpp:393-419) must not change a
single output bit, and the 16-byte fused cells the transport moves must never
be observed torn (the word-atomicity canary)."""
import numpy as np
import pytest
import torch

from oracle import oracle as O

pytestmark = pytest.mark.gpu


def _group(nodes, gpus):
    from paper_2511_09557_b200 import ClusterTopology, LocalGroup
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    return LocalGroup(ClusterTopology(nodes, gpus), 1 << 20, device=0, timeout_s=30.0)


@pytest.mark.parametrize("seed", list(range(20)))
def test_delay_injection_keeps_results(seed):
    """Criterion 7's case — 4x2, 128 KiB int32, NvrarConfig{2, 8192} — on every
    message-passing schedule (virtual ranks, one cooperative launch), plus fp32
    and bf16 through the Lamport cells, under seeded delays of up to 2 us."""
    from paper_2511_09557_b200 import NvrarConfig
    g = _group(4, 2)
    try:
        g.set_jitter(2000, seed)
        g.set_config(NvrarConfig(2, 8192))
        cases = [("i32", 32768, 90), ("f32", 4099 + seed, 91), ("bf16", 65536 + 3 * seed, 92)]
        for algo in ("hier", "twoshot", "oneshot"):
            g.set_algo(algo)
            for dtype, n, s in cases:
                x = O.random_inputs(8, n, s, "i32" if dtype == "i32" else "f32")
                if dtype == "bf16":
                    x = O.bf16_bits_from_f32(x)
                want = O.nvrar_order_sum(x, 4, 2, dtype)
                ins = [torch.from_numpy(np.ascontiguousarray(x[r])) for r in range(8)]
                if dtype == "bf16":
                    ins = [t.view(torch.int16).view(torch.bfloat16) for t in ins]
                ins = [t.cuda() for t in ins]
                outs = [torch.empty_like(t) for t in ins]
                g.run_all(ins, outs)
                for r in range(8):
                    got = outs[r].cpu()
                    got = got.view(torch.int16).numpy().view(np.uint16) if dtype == "bf16" \
                        else got.numpy().view(np.uint32)
                    exp = want if dtype == "bf16" else want.view(np.uint32)
                    assert np.array_equal(got, exp), f"seed {seed} {algo} {dtype}: rank {r}"
        g.set_jitter(0)
    finally:
        g.close()


def test_word_atomicity_canary():
    """acceptance_test.cpp:338-364 on the device transport: 100 seeds, a
    writer streaming 64 fused 16-byte cells with random gaps and a reader
    polling with random gaps, concurrently (two comms, two streams)."""
    g = _group(2, 1)
    try:
        w, r = g.comms
        s_w, s_r = torch.cuda.Stream(), torch.cuda.Stream()
        for seed in range(100):
            r.canary(0, 64, writer=False, jitter_ns=300, seed=seed, stream=s_r)
            w.canary(1, 64, writer=True, jitter_ns=1000, seed=seed, stream=s_w)
            assert r.canary_result() == 0, f"seed {seed}: torn cell observed"
            assert w.canary_result() == 0
    finally:
        g.close()
