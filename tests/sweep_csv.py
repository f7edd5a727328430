"""GPU sweep in the reference's CSV schema (bench.hpp:185-320).

Runs, on the GPUs of one node (one process per GPU), the reference's sweep
order — algorithm (ring, tree, nvrar), then nodes, message size, blocks, chunk
bytes — and writes `sweep_csv` rows with the reference's header:

    algorithm,nodes,gpus_per_node,msg_bytes,blocks,chunk_bytes,iters,mean_us,
    model_us,speedup_vs_ring,correct,best,error

* ring / tree: the GPU collectives with the reduction order of RingAllreduce /
  TreeAllreduce (nvrar_ring_allreduce / nvrar_tree_allreduce); nvrar: the
  NVRAR all-reduce with `blocks` CTAs per rank (the tuning cells; chunk_bytes is
  validated and recorded — results are invariant to it, as in the reference).
* mean_us: mean per-call time of `iters` back-to-back calls in a CUDA graph,
  CUDA events, max over ranks (the reference reports the mean too).
* model_us: the B200 roofline of §8(d): max(2(P-1)/P·M / BW_link, log2(P)·α)
  with α measured by the device ping-pong in the same run.
* correct: the last call's output equals the oracle's bits for that order.
* best / speedup_vs_ring: as bench.hpp:258-283 (fastest cell per (algorithm,
  nodes, msg); ring time / this time).
* Extra rows with algorithm "nccl" time torch.distributed.all_reduce the same
  way (the real-world baseline; not part of the reference's enum).

    torchrun --nproc-per-node 4 tests/sweep_csv.py --out sweep.csv

(Lives under tests/: the `correct` column uses the oracle as the checker.)
"""
from __future__ import annotations

import argparse
import math
import os
import statistics

import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import oracle as O  # noqa: E402  (the checker of the `correct` column)
from paper_2511_09557_b200 import dist as D  # noqa: E402
from paper_2511_09557_b200.comm import ClusterTopology, Communicator, NvrarConfig  # noqa: E402
from paper_2511_09557_b200.harness import alpha_signal_us  # noqa: E402
from paper_2511_09557_b200.selector import _graph  # noqa: E402

HEADER = ("algorithm,nodes,gpus_per_node,msg_bytes,blocks,chunk_bytes,iters,mean_us,"
          "model_us,speedup_vs_ring,correct,best,error\n")
LINK_GBS = 770.0  # measured peer bandwidth per direction


def _fmt(v: float) -> str:
    return f"{v:.3f}"


def time_calls(fn, calls: int, reps: int) -> float:
    stream = torch.cuda.Stream()
    g = _graph(fn, calls, stream)
    for _ in range(2):
        g.replay()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        dist.barrier()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(stream):
            a.record(stream)
            g.replay()
            b.record(stream)
        b.synchronize()
        ts.append(a.elapsed_time(b))
    ts = D.max_over_ranks(ts)
    return statistics.mean(ts) * 1e3 / calls


def csv_row(r: dict) -> str:
    tuned = r["algorithm"] == "nvrar"
    ok = not r.get("error")
    return ",".join([
        r["algorithm"], str(r["nodes"]), str(r["gpus"]), str(r["msg"]),
        str(r["blocks"]) if tuned else "", str(r["chunk"]) if tuned else "", str(r["iters"]),
        _fmt(r["mean_us"]) if ok else "", _fmt(r["model_us"]) if ok else "",
        _fmt(r["speedup"]) if r.get("speedup", 0.0) > 0 else "",
        ("1" if r["correct"] else "0") if ok else "", "1" if r.get("best") else "",
        (r.get("error") or "").replace(",", ";").replace("\n", ";"),
    ]) + "\n"


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--nodes", default="1,2", help="virtual node counts (gpus = world / nodes)")
    ap.add_argument("--msg-bytes", default="65536,131072,262144,524288,1048576,2097152")
    ap.add_argument("--blocks", default="16,32,64,128")
    ap.add_argument("--chunk-bytes", default="65536")
    ap.add_argument("--algorithms", default="ring,tree,nvrar,nccl")
    ap.add_argument("--dtype", default="f32", choices=["f32", "bf16"])
    ap.add_argument("--iters", type=int, default=50)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--out", default="")
    args = ap.parse_args()

    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    os.environ.setdefault("NCCL_DEBUG", "WARN")
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    rank, world = dist.get_rank(), dist.get_world_size()
    tdt = torch.float32 if args.dtype == "f32" else torch.bfloat16
    esz = 4 if args.dtype == "f32" else 2
    msgs = sorted(int(m) for m in args.msg_bytes.split(","))
    nodes_list = sorted(int(n) for n in args.nodes.split(",") if world % int(n) == 0)
    algos = [a for a in ("ring", "tree", "nvrar", "nccl") if a in args.algorithms.split(",")]
    rows = []
    for algo in algos:
        for nodes in nodes_list:
            gpus = world // nodes
            topo = ClusterTopology(nodes, gpus)
            comm = Communicator.from_process_group(topo, max(msgs), device=local)
            alpha = alpha_signal_us(comm, rank, world) or 0.0
            for msg in msgs:
                n = msg // esz
                nbuf = max(2, min(args.iters, (160 << 20) // (2 * msg)))
                xs = O.random_inputs(world, n, 7 + msg, "f32")
                if args.dtype == "bf16":
                    xs = O.bf16_bits_from_f32(xs)
                    base = torch.from_numpy(xs[rank]).view(torch.int16).view(torch.bfloat16)
                else:
                    base = torch.from_numpy(xs[rank])
                bufs = [(base.cuda(), torch.empty(n, dtype=tdt, device="cuda"))
                        for _ in range(nbuf)]
                model = max(2 * (world - 1) / world * msg / (LINK_GBS * 1e3),
                            math.log2(world) * alpha if world > 1 else 0.0)
                cells = [int(b) for b in args.blocks.split(",")] if algo == "nvrar" else [0]
                chunks = [int(c) for c in args.chunk_bytes.split(",")] if algo == "nvrar" else [65536]
                for b in cells:
                    for ch in chunks:
                        r = {"algorithm": algo, "nodes": nodes, "gpus": gpus, "msg": msg,
                             "blocks": b, "chunk": ch, "iters": args.iters, "model_us": model}
                        try:
                            if algo == "nccl":
                                # in place on the outputs (no copy kernel in the timed
                                # calls); correctness from one separate call below
                                fn = lambda i: dist.all_reduce(bufs[i % nbuf][1])  # noqa: E731
                            elif algo == "nvrar":
                                comm.set_config(NvrarConfig(b, ch))
                                fn = lambda i: comm.allreduce(*bufs[i % nbuf])  # noqa: E731
                            else:
                                fn = (lambda op: lambda i: op(*bufs[i % nbuf]))(  # noqa: E731
                                    getattr(comm, f"{algo}_allreduce"))
                            r["mean_us"] = time_calls(fn, args.iters, args.reps)
                            comm.check()
                            got = bufs[(args.iters - 1) % nbuf][1]
                            if algo == "nccl":
                                got.copy_(bufs[0][0])
                                dist.all_reduce(got)
                                torch.cuda.synchronize()
                            order = "nvrar" if algo == "nccl" else algo
                            want = O.order_sum(xs, nodes, gpus, order, args.dtype)
                            g = got.view(torch.int16).cpu().numpy().view(np.uint16) \
                                if args.dtype == "bf16" else got.cpu().numpy().view(np.uint32)
                            w = want if args.dtype == "bf16" else want.view(np.uint32)
                            # NCCL's order is its own: "correct" = within rounding
                            if algo == "nccl":
                                ref = O.serial_sum(O.f32_from_bf16_bits(xs).astype(np.float32)
                                                   if args.dtype == "bf16" else xs)
                                r["correct"] = bool(np.allclose(got.float().cpu().numpy(), ref,
                                                                rtol=1e-2 if args.dtype == "bf16"
                                                                else 1e-5))
                            else:
                                r["correct"] = bool(np.array_equal(g, w))
                        except Exception as e:  # noqa: BLE001 — the sweep records and continues
                            r["error"] = f"{type(e).__name__}: {e}"
                        rows.append(r)
                comm.set_config(NvrarConfig())
                del bufs
            comm.close()
    # best per (algorithm, nodes, msg); speedup vs the ring row (bench.hpp:258-283)
    for r in rows:
        grp = [q for q in rows if (q["algorithm"], q["nodes"], q["msg"]) ==
               (r["algorithm"], r["nodes"], r["msg"]) and not q.get("error")]
        if grp and not r.get("error"):
            r["best"] = r is min(grp, key=lambda q: q["mean_us"])
        ring = [q for q in rows if q["algorithm"] == "ring" and q["nodes"] == r["nodes"]
                and q["msg"] == r["msg"] and not q.get("error")]
        if r["algorithm"] != "ring" and ring and not r.get("error"):
            r["speedup"] = ring[0]["mean_us"] / r["mean_us"]
    if rank == 0:
        text = HEADER + "".join(csv_row(r) for r in rows)
        if args.out:
            with open(args.out, "w") as fh:
                fh.write(text)
        print(text, end="", flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
