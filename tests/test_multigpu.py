"""Real multi-process, multi-GPU runs (one rank per B200, IPC-mapped peers over
NVLink/NVSwitch). Skipped unless at least 2 devices are visible."""
import os
import socket
import subprocess
import sys

import pytest
import torch

pytestmark = [pytest.mark.gpu, pytest.mark.multigpu]

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
NDEV = torch.cuda.device_count() if torch.cuda.is_available() else 0

TOPOS = {2: [(2, 1), (1, 2)], 4: [(2, 2), (4, 1), (1, 4)],
         8: [(2, 4), (4, 2), (8, 1), (1, 8)]}


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _run(world, nodes, gpus, extra=()):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={world}", "--master-addr", "127.0.0.1",
           "--master-port", str(_port()), os.path.join(ROOT, "tests", "mp_worker.py"),
           "--nodes", str(nodes), "--gpus", str(gpus), *extra]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    return r.returncode, r.stdout + r.stderr


CASES = [(w, n, g) for w in (2, 4, 8) for (n, g) in TOPOS[w]]


@pytest.mark.parametrize("world,nodes,gpus", CASES)
def test_multiprocess_parity(world, nodes, gpus):
    if NDEV < world:
        pytest.skip(f"needs {world} GPUs, have {NDEV}")
    rc, out = _run(world, nodes, gpus)
    assert rc == 0, out[-4000:]
    assert out.count(": OK") == world, out[-4000:]


@pytest.mark.parametrize("nodes,gpus", [(2, 1), (1, 2)])
def test_length_mismatch_is_protocol_fault(nodes, gpus):
    if NDEV < 2:
        pytest.skip("needs 2 GPUs")
    rc, out = _run(2, nodes, gpus, ("--mismatch",))
    assert rc == 0, out[-4000:]
    assert "status 4" in out, out[-4000:]


def test_all_gather_length_mismatch_is_protocol_fault():
    """collectives_test.cpp:226-237 across processes: shard 4 vs 3 elements."""
    if NDEV < 2:
        pytest.skip("needs 2 GPUs")
    rc, out = _run(2, 1, 2, ("--ag-mismatch",))
    assert rc == 0, out[-4000:]
    assert out.count("ag mismatch status 4") == 2, out[-4000:]


@pytest.mark.parametrize("world,nodes,gpus", [(2, 2, 1), (4, 2, 2), (4, 1, 4), (8, 2, 4)])
def test_multicast_oneshot_parity(world, nodes, gpus):
    """NVLS multicast one-shot (NVRAR_ALGO_MCAST) is bit-exact like every schedule."""
    if NDEV < world:
        pytest.skip(f"needs {world} GPUs, have {NDEV}")
    rc, out = _run(world, nodes, gpus, ("--multicast",))
    assert rc == 0, out[-4000:]
    assert out.count(": OK") == world, out[-4000:]


@pytest.mark.parametrize("world", [2, 4])
def test_mixed_call_stress(world):
    """Hundreds of back-to-back calls switching schedule (incl. the multicast
    one-shot), CTA count, dtype, size and call kind (all-reduce, fused
    residual, ring / tree orders) — every result checked (tests/mp_stress.py)."""
    if NDEV < world:
        pytest.skip(f"needs {world} GPUs, have {NDEV}")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={world}", "--master-addr", "127.0.0.1",
           "--master-port", str(_port()), os.path.join(ROOT, "tests", "mp_stress.py"),
           "--calls", "600", "--multicast", "--sync-every", "7"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    out = r.stdout + r.stderr
    assert r.returncode == 0, out[-4000:]
    assert out.count(": OK after 600 calls") == world, out[-4000:]


@pytest.mark.parametrize("nodes,gpus", [(2, 4), (4, 2), (8, 1)])
def test_eight_rank_layout_on_fewer_gpus(nodes, gpus):
    """The P=8 layouts (2x4 configs[1]; 4x2, 8x1 configs[2]) with 8 processes on 4 GPUs: two ranks
    share a device and progress by time-slicing, so every non-virtual P=8 kernel
    instantiation (flat N=2 x MAXG=4, hierarchical N=2 x MG=4) and the 8-rank
    bootstrap run against the oracle (timing meaningless)."""
    if NDEV < 4:
        pytest.skip("needs 4 GPUs")
    if NDEV >= 8:
        pytest.skip("8 GPUs present: test_multiprocess_parity covers P=8 directly")
    rc, out = _run(8, nodes, gpus, ("--dev-mod", "4", "--quick"))
    assert rc == 0, out[-4000:]
    assert out.count(": OK") == 8, out[-4000:]


@pytest.mark.parametrize("world,nodes,gpus", [(2, 2, 1), (4, 2, 2), (4, 4, 1)])
def test_multigpu_registered_fuzz_ops(world, nodes, gpus):
    """One rank per GPU over NVLink (tests/ipc_worker.py, directory bootstrap):
    registered buffers read in place, torch.ops.nvrar across ranks, mixed
    pinned/pageable host paths, delay injection and the word-atomicity canary
    — every result bit-exact against the oracle."""
    if NDEV < world:
        pytest.skip(f"needs {world} GPUs, have {NDEV}")
    import tempfile
    with tempfile.TemporaryDirectory(prefix="nvrar_mg_") as d:
        procs = [subprocess.Popen([sys.executable, os.path.join(ROOT, "tests", "ipc_worker.py"),
                                   "--dir", d, "--rank", str(r), "--nodes", str(nodes),
                                   "--gpus", str(gpus), "--device", str(r), "--quick",
                                   "--registered", "--ops", "--host", "--jitter-seeds", "4",
                                   "--canary", "20"],
                                  stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True,
                                  cwd=ROOT) for r in range(world)]
        outs = [p.communicate(timeout=600)[0] for p in procs]
    text = "".join(outs)
    assert all(p.returncode == 0 for p in procs), text[-4000:]
    assert text.count(": OK") == world, text[-4000:]
