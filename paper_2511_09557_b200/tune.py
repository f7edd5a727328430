"""Measured sweep behind the selector (run under torch.distributed.run, one rank per GPU).

For each message size and each (schedule, CTA count) it times a CUDA graph of
`calls` back-to-back all-reduces (max over ranks, p50 over replays) and prints
one JSON object on rank 0:

    {"world": P, "nodes": N, "dtype": "bf16", "table": {"131072": {"hier/16": 6.1, ...}},
     "best": {"131072": ["oneshot", 16, 6.0], ...}, "phases": {...}}

`phases` are steady-state CTA-0 timestamps of the LAST call of a replay
(entry, pdl wait done, RS pushed, peers synced, reduced + AG pushed, AG
received, exit), relative to entry, max over ranks.

    python -m torch.distributed.run --nproc-per-node 4 --master-addr 127.0.0.1 \
        -m paper_2511_09557_b200.tune --sizes 131072,1048576
"""
from __future__ import annotations

import argparse
import ctypes
import json
import os
import statistics

import torch
import torch.distributed as dist

from . import dist as D
from .comm import ClusterTopology, Communicator, NvrarConfig

ALGOS = ("hier", "twoshot", "oneshot")


def graph_of(fn, calls, stream):
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


def time_graph(g, reps, stream, local):
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
    return D.max_over_ranks(ts)


def tune_emulated(args):
    """Virtual ranks on one GPU (the N=1 bench workload): same sweep, no process group."""
    from .comm import LocalGroup
    nodes, gpus = args.emu_topo
    p = nodes * gpus
    g = LocalGroup(ClusterTopology(nodes, gpus), 8 << 20, device=0, timeout_s=30.0)
    g.set_protocol(args.proto)
    dt = torch.bfloat16 if args.dtype == "bf16" else torch.float32
    esz = 2 if dt == torch.bfloat16 else 4
    stream = torch.cuda.Stream()
    table, best = {}, {}
    for size in [int(s) for s in args.sizes.split(",")]:
        n = size // esz
        nbuf = max(2, min(args.calls, (160 << 20) // (2 * size * p)))
        bufs = [([torch.randn(n, device="cuda").to(dt) for _ in range(p)],
                 [torch.empty(n, device="cuda", dtype=dt) for _ in range(p)]) for _ in range(nbuf)]
        row = {}
        for algo in ALGOS:
            if algo == "oneshot" and size > (1 << 20):
                continue
            g.set_algo(algo)
            for blocks in [int(b) for b in args.blocks.split(",")]:
                if blocks * p > 148:
                    continue
                g.set_config(NvrarConfig(blocks, 65536))
                gr = graph_of(lambda i: g.launch(*bufs[i % nbuf], stream=torch.cuda.current_stream()),
                              args.calls, stream)
                for _ in range(2):
                    gr.replay()
                torch.cuda.synchronize()
                ts = []
                for _ in range(args.reps):
                    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    with torch.cuda.stream(stream):
                        a.record(stream)
                        gr.replay()
                        b.record(stream)
                    b.synchronize()
                    ts.append(a.elapsed_time(b))
                row[f"{algo}/{blocks}"] = round(statistics.median(ts) * 1e3 / args.calls, 3)
                del gr
        g.check()
        k = min(row, key=row.get)
        table[str(size)] = row
        best[str(size)] = [k.split("/")[0], int(k.split("/")[1]), row[k]]
    res = {"world": 1, "emulated": f"{nodes}x{gpus}", "dtype": args.dtype, "proto": args.proto,
           "table": table, "best": best}
    line = json.dumps(res)
    print(line, flush=True)
    if args.out:
        with open(args.out, "w") as fh:
            fh.write(line + "\n")
    g.close()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--emu", default="", help="NxG: virtual ranks on one GPU instead of a process group")
    ap.add_argument("--sizes", default="65536,131072,262144,524288,1048576,2097152,4194304")
    ap.add_argument("--blocks", default="4,8,16,32,64,128")
    ap.add_argument("--nodes", type=int, default=0)
    ap.add_argument("--dtype", default="bf16")
    ap.add_argument("--calls", type=int, default=40)
    ap.add_argument("--reps", type=int, default=7)
    ap.add_argument("--proto", default="auto")
    ap.add_argument("--out", default="")
    args = ap.parse_args()
    if args.emu:
        args.emu_topo = tuple(int(v) for v in args.emu.split("x"))
        tune_emulated(args)
        return
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    nodes = args.nodes or (2 if world > 1 else 1)
    comm = Communicator.from_process_group(ClusterTopology(nodes, world // nodes), 8 << 20,
                                           device=local, timeout_s=30.0)
    comm.set_protocol(args.proto)
    dt = torch.bfloat16 if args.dtype == "bf16" else torch.float32
    esz = 2 if dt == torch.bfloat16 else 4
    stream = torch.cuda.Stream()
    table, best, phases = {}, {}, {}
    for size in [int(s) for s in args.sizes.split(",")]:
        n = size // esz
        nbuf = max(2, min(args.calls, (160 << 20) // (2 * size)))
        bufs = [(torch.randn(n, device="cuda").to(dt), torch.empty(n, device="cuda", dtype=dt))
                for _ in range(nbuf)]
        row = {}
        for algo in ALGOS:
            if algo == "oneshot" and size > (2 << 20):
                continue
            comm.set_algo(algo)
            for blocks in [int(b) for b in args.blocks.split(",")]:
                comm.set_config(NvrarConfig(blocks, 65536))
                g = graph_of(lambda i: comm.allreduce(*bufs[i % nbuf]), args.calls, stream)
                ts = time_graph(g, args.reps, stream, local)
                row[f"{algo}/{blocks}"] = round(statistics.median(ts) * 1e3 / args.calls, 3)
                del g
        comm.check()
        k = min(row, key=row.get)
        table[str(size)] = row
        best[str(size)] = [k.split("/")[0], int(k.split("/")[1]), row[k]]
        # steady-state phases of the best configuration
        comm.set_algo(best[str(size)][0])
        comm.set_config(NvrarConfig(best[str(size)][1], 65536))
        comm._lib.nvrar_set_profile(comm._h, 1)
        g = graph_of(lambda i: comm.allreduce(*bufs[i % nbuf]), 20, stream)
        g.replay()
        torch.cuda.synchronize()
        tsb = (ctypes.c_uint64 * (512 * 8))()
        comm._lib.nvrar_get_phase_times(comm._h, tsb, 512 * 8)
        nb = best[str(size)][1]
        cta = [[tsb[b * 8 + i] for i in range(8)] for b in range(nb)]  # [7] = released
        t0 = min(c[7] for c in cta)  # earliest release of the last call
        rel = [(cta[0][i] - cta[0][0]) / 1e3 for i in range(8)]
        summary = [
            (max(c[7] for c in cta) - t0) / 1e3,                        # release spread
            statistics.median((c[6] - c[7]) / 1e3 for c in cta),         # median CTA work
            (max(c[6] for c in cta) - t0) / 1e3,                        # last exit
            statistics.median((c[7] - c[0]) / 1e3 for c in cta),         # median entry->release
            statistics.median((c[2] - c[7]) / 1e3 for c in cta),         # release->pushed
            statistics.median((c[3] - c[2]) / 1e3 for c in cta),         # pushed->synced
            statistics.median((c[4] - c[3]) / 1e3 for c in cta),         # synced->reduced
            statistics.median((c[5] - c[4]) / 1e3 for c in cta),         # reduced->ag recv
        ]
        phases[str(size)] = {"cta0": [round(v, 3) for v in D.max_over_ranks(rel)],
                             "summary": [round(v, 3) for v in D.max_over_ranks(summary)]}
        comm._lib.nvrar_set_profile(comm._h, 0)
        del g
    comm.check()
    if rank == 0:
        res = {"world": world, "nodes": nodes, "dtype": args.dtype, "proto": args.proto,
               "calls": args.calls, "table": table, "best": best, "phases": phases,
               "phase_names": ["entry", "pdl_wait", "rs_pushed", "synced", "reduced+ag_pushed",
                               "ag_received", "exit"],
               "summary_names": ["release_spread", "median_cta_work", "last_exit",
                                 "entry_to_release", "release_to_pushed", "pushed_to_synced",
                                 "synced_to_reduced", "reduced_to_ag_received"]}
        line = json.dumps(res)
        print(line, flush=True)
        if args.out:
            with open(args.out, "w") as fh:
                fh.write(line + "\n")
    dist.barrier()
    comm.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
