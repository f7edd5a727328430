"""The torch custom op and the TP-decode workload shapes."""
import pytest
import torch

from paper_2511_09557_b200 import torch_op  # noqa: F401  (registers torch.ops.nvrar.*)
from paper_2511_09557_b200.tp_decode import LLAMA, DecodeWorkload


def test_decode_message_sizes():
    """workload_test.cpp:11-26 (decode_msg_bytes, workload.hpp:67-72)."""
    assert DecodeWorkload(8, 8192, 2, 80).msg_bytes() == 128 * 1024
    assert DecodeWorkload(8, 16384, 2, 126).msg_bytes() == 256 * 1024
    assert DecodeWorkload(32, 8192, 2, 80).msg_bytes() == 512 * 1024
    assert DecodeWorkload(32, 16384, 2, 126).msg_bytes() == 1024 * 1024
    base = DecodeWorkload(4, 1024, 2, 1).msg_bytes()
    assert DecodeWorkload(8, 1024, 2, 1).msg_bytes() == 2 * base
    assert DecodeWorkload(4, 2048, 2, 1).msg_bytes() == 2 * base
    assert DecodeWorkload(4, 1024, 4, 1).msg_bytes() == 2 * base
    with pytest.raises(ValueError):
        DecodeWorkload(0, 8192, 2, 1).msg_bytes()
    with pytest.raises(ValueError):
        DecodeWorkload(8, 8192, 3, 1).msg_bytes()
    # C4/C5: 160 and 252 all-reduces per decode step
    assert DecodeWorkload(8, LLAMA["70b"]["hidden"], 2, LLAMA["70b"]["layers"]).allreduces_per_step() == 160
    assert DecodeWorkload(8, LLAMA["405b"]["hidden"], 2, LLAMA["405b"]["layers"]).allreduces_per_step() == 252


def test_op_registered_with_fake_impl():
    x = torch.empty(4096, dtype=torch.bfloat16, device="meta")
    y = torch.ops.nvrar.all_reduce(x, 1)
    assert y.shape == x.shape and y.dtype == x.dtype
    torch.ops.nvrar.all_reduce_(x, 1)


@pytest.mark.gpu
def test_op_single_rank_and_graph_capture():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from paper_2511_09557_b200 import ClusterTopology, Communicator
    c = Communicator(ClusterTopology(1, 1), 0, 0, 1 << 20)
    c.connect([c.export()])
    cid = torch_op.register(c)
    try:
        x = torch.randn(70000, device="cuda").to(torch.bfloat16)
        assert torch.equal(torch.ops.nvrar.all_reduce(x, cid), x)
        buf = x.clone()
        s0 = c.sequence()
        g = torch.cuda.CUDAGraph()
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            torch.ops.nvrar.all_reduce_(buf, cid)
        torch.cuda.current_stream().wait_stream(s)
        with torch.cuda.graph(g):
            torch.ops.nvrar.all_reduce_(buf, cid)
            torch.ops.nvrar.all_reduce_(buf, cid)
        for _ in range(5):
            g.replay()
        torch.cuda.synchronize()
        c.check()
        assert torch.equal(buf, x)
        assert c.sequence() - s0 == 1 + 2 * 5  # one eager call + 5 replays of 2 captured calls
    finally:
        torch_op.unregister(cid)
        c.close()
