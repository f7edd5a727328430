"""The directory bootstrap (paper_2511_09557_b200/bootstrap.py) that lets rank
processes exchange their nvrar handles without a process group — the
allgather of nvrar_init over a shared directory. CPU only: P processes
all-gather blobs, repeatedly, with distinct tags, and every rank sees every
blob in rank order."""
import multiprocessing as mp
import os

from paper_2511_09557_b200 import bootstrap as B


def _rank(path, rank, world, q):
    try:
        got = []
        for tag in ("h", "reg1", "reg2", "done"):
            got.append(B.file_allgather(path, rank, world, f"{tag}:{rank}".encode() * (rank + 1),
                                        tag=tag, timeout_s=60))
        q.put((rank, got))
    except Exception as e:  # noqa: BLE001
        q.put((rank, repr(e)))


def test_file_allgather_many_rounds(tmp_path):
    world = 4
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_rank, args=(str(tmp_path), r, world, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(60)
    for r in range(world):
        assert not isinstance(res[r], str), res[r]
        for i, tag in enumerate(("h", "reg1", "reg2", "done")):
            assert res[r][i] == [f"{tag}:{q}".encode() * (q + 1) for q in range(world)]
    # writes are atomic renames: no temporary file is left behind
    assert not [f for f in os.listdir(tmp_path) if f.startswith(".")]


def test_file_allgather_times_out_on_a_missing_rank(tmp_path):
    import pytest
    with pytest.raises(TimeoutError):
        B.file_allgather(str(tmp_path), 0, 2, b"x", timeout_s=0.2)
