"""Measured message-size x schedule selector (north star subsystem 3).

`autotune(comm, ...)` times every (schedule, CTA count) candidate for each
message size on the running system — CUDA graphs of back-to-back calls, CUDA
events, max over ranks — and installs the winners in the communicator with
`nvrar_set_plan_table`. Every rank derives the table from the same
max-over-ranks numbers, so all ranks agree (a disagreement would deadlock the
kernel). Without a table the built-in policy (csrc/nvrar_comm.cu
`default_plan`, fitted to the B200 sweeps in DESIGN.md) applies.
"""
from __future__ import annotations

import ctypes
import json
import math
import statistics
from typing import Dict, List, Sequence, Tuple

import torch
import torch.distributed as dist

from . import _lib as L
from . import dist as D
from .comm import Communicator, NvrarConfig

DEFAULT_SIZES = (64 << 10, 128 << 10, 256 << 10, 512 << 10, 1 << 20, 2 << 20, 4 << 20, 8 << 20)
ALGO_CODE = {"hier": L.ALGO_HIER, "twoshot": L.ALGO_TWOSHOT, "oneshot": L.ALGO_ONESHOT,
             "mcast": L.ALGO_MCAST}


def _graph(fn, calls, stream):
    stream.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(stream):
        for i in range(min(calls, 3)):
            fn(i)
    torch.cuda.current_stream().wait_stream(stream)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=stream):
        for i in range(calls):
            fn(i)
    torch.cuda.synchronize()
    return g


def measure(comm: Communicator, size: int, dtype: torch.dtype, algo: str, blocks: int,
            calls: int = 30, reps: int = 5, group=None) -> float:
    """p50 per-call µs (max over ranks) of `calls` back-to-back all-reduces."""
    esz = torch.finfo(dtype).bits // 8 if dtype.is_floating_point else 4
    n = size // esz
    nbuf = max(2, min(calls, (160 << 20) // (2 * size)))
    bufs = [(torch.randn(n, device="cuda").to(dtype), torch.empty(n, device="cuda", dtype=dtype))
            for _ in range(nbuf)]
    comm.set_algo(algo)
    comm.set_config(NvrarConfig(blocks, 65536))
    stream = torch.cuda.Stream()
    g = _graph(lambda i: comm.allreduce(*bufs[i % nbuf]), calls, stream)
    for _ in range(2):
        g.replay()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        dist.barrier(group)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(stream):
            a.record(stream)
            g.replay()
            b.record(stream)
        b.synchronize()
        ts.append(a.elapsed_time(b))
    ts = D.max_over_ranks(ts, group)
    comm.set_algo("auto")
    comm.set_config(NvrarConfig())
    return statistics.median(ts) * 1e3 / calls


def table_from(best: Dict[int, Tuple[str, int, float]]) -> List[Tuple[int, str, int]]:
    """Rows (max_bytes, algo, blocks): each measured size owns the range up to the
    geometric midpoint with the next one; the last row covers everything above."""
    sizes = sorted(best)
    rows = []
    for i, s in enumerate(sizes):
        hi = int(math.sqrt(s * sizes[i + 1])) if i + 1 < len(sizes) else (1 << 62)
        rows.append((hi, best[s][0], best[s][1]))
    return rows


def install(comm: Communicator, rows: Sequence[Tuple[int, str, int]]) -> None:
    arr = (L.PlanEntry * len(rows))()
    for i, (mx, algo, blocks) in enumerate(rows):
        arr[i].max_bytes = mx
        arr[i].algo = ALGO_CODE[algo]
        arr[i].blocks = blocks
    rc = comm._lib.nvrar_set_plan_table(comm._h, arr, len(rows))
    if rc:
        raise RuntimeError(comm.last_error())


def autotune(comm: Communicator, sizes: Sequence[int] = DEFAULT_SIZES,
             dtype: torch.dtype = torch.bfloat16, blocks: Sequence[int] = (16, 32, 64, 128),
             calls: int = 30, reps: int = 5, group=None) -> dict:
    """Measure, agree, install. Returns {"rows": [...], "measured": {size: {cand: µs}}}."""
    measured: Dict[int, Dict[str, float]] = {}
    best: Dict[int, Tuple[str, int, float]] = {}
    flat_ok = comm.topo.world_size() <= 16
    # the multicast one-shot is a candidate only where every rank set it up
    mcast = comm.multicast_ready() and dtype != torch.int32
    for size in sizes:
        row: Dict[str, float] = {}
        for algo in ("oneshot", "mcast", "hier", "twoshot"):
            if algo != "hier" and not flat_ok:
                continue
            if algo in ("oneshot", "mcast") and size > (1 << 20):
                continue
            if algo == "mcast" and not mcast:
                continue
            for b in blocks:
                row[f"{algo}/{b}"] = measure(comm, size, dtype, algo, b, calls, reps, group)
        k = min(row, key=row.get)  # identical on every rank: row holds max-over-ranks values
        best[size] = (k.split("/")[0], int(k.split("/")[1]), row[k])
        measured[size] = {kk: round(v, 3) for kk, v in row.items()}
    rows = table_from(best)
    install(comm, rows)
    return {"rows": rows, "measured": measured}


def fit_alpha_beta(points: Dict[int, float]) -> Tuple[float, float]:
    """Least-squares fit of the alpha-beta cost model t(M) = alpha + M / beta
    (cost_model.hpp's per-algorithm form, ModelPrediction::of) to measured
    (bytes, µs) points. Returns (alpha_us, beta_GBs); beta is inf when the
    points show no size dependence."""
    xs = [float(m) for m in points]
    ys = [float(points[m]) for m in points]
    n = len(xs)
    if n == 0:
        raise ValueError("no points")
    if n == 1:
        return ys[0], math.inf
    mx, my = sum(xs) / n, sum(ys) / n
    sxx = sum((x - mx) ** 2 for x in xs)
    slope = sum((x - mx) * (y - my) for x, y in zip(xs, ys)) / sxx if sxx else 0.0
    alpha = my - slope * mx
    beta = math.inf if slope <= 0 else 1.0 / slope / 1e3  # bytes/µs -> GB/s
    return alpha, beta


def fit_schedules(measured: Dict[int, Dict[str, float]]) -> Dict[str, dict]:
    """alpha/beta per schedule from autotune()'s measurements (best CTA count
    per size)."""
    per: Dict[str, Dict[int, float]] = {}
    for size, cands in measured.items():
        for k, t in cands.items():
            algo = k.split("/")[0]
            per.setdefault(algo, {})
            per[algo][size] = min(t, per[algo].get(size, math.inf))
    out = {}
    for algo, pts in per.items():
        a, b = fit_alpha_beta(pts)
        out[algo] = {"alpha_us": round(a, 3), "beta_GBs": None if math.isinf(b) else round(b, 1),
                     "sizes": sorted(pts)}
    return out


def save(path: str, result: dict) -> None:
    with open(path, "w") as fh:
        json.dump({"rows": result["rows"]}, fh)


def load(comm: Communicator, path: str) -> None:
    with open(path) as fh:
        install(comm, [tuple(r) for r in json.load(fh)["rows"]])
