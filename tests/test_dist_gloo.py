"""Host logic of the N>1 path on CPU: world_size-2 gloo process group driving
the bootstrap handle exchange, the selector consensus and the max-over-ranks
timing reduction (no GPU)."""
import os
import socket

import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2511_09557_b200 import _lib as L
        from paper_2511_09557_b200 import dist as D
        import ctypes
        hs = D.exchange_handles(bytes([rank]) * L.HANDLE_BYTES)
        assert [h[0] for h in hs] == list(range(world))
        lib = L.load()
        a, b = ctypes.c_int(), ctypes.c_int()
        assert lib.nvrar_plan_for(world, world, 1, 1 << 19, L.BF16, 0, 0, 148,
                                  ctypes.byref(a), ctypes.byref(b)) == 0
        plan = D.plan_consensus((L.ALGO_NAMES[a.value], b.value))
        assert plan[0] in ("oneshot", "twoshot", "hier")
        bad = None
        try:
            D.plan_consensus(("twoshot", 4 + rank))
        except RuntimeError as e:
            bad = str(e)
        assert bad is not None and "disagree" in bad
        m = D.max_over_ranks([1.0 + rank, 5.0 - rank])
        assert m == [2.0, 5.0]
        q.put((rank, "ok"))
    except Exception as e:  # pragma: no cover
        q.put((rank, repr(e)))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_host_logic():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=120) for _ in ps)
    for p in ps:
        p.join(timeout=60)
    assert res == {0: "ok", 1: "ok"}, res


def test_alpha_beta_fit():
    """selector.fit_alpha_beta recovers t = alpha + M / beta exactly."""
    from paper_2511_09557_b200.selector import fit_alpha_beta, fit_schedules
    pts = {m: 5.0 + m / (400.0 * 1e3) for m in (65536, 262144, 1 << 20, 4 << 20)}
    a, b = fit_alpha_beta(pts)
    assert abs(a - 5.0) < 1e-9 and abs(b - 400.0) < 1e-6
    fs = fit_schedules({65536: {"oneshot/32": 5.2, "oneshot/64": 5.1, "hier/32": 7.0},
                        1 << 20: {"oneshot/32": 9.0, "hier/32": 9.5}})
    assert set(fs) == {"oneshot", "hier"} and fs["oneshot"]["beta_GBs"] > 0
