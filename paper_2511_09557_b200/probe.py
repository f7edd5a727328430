"""Latency probes for the roofline and for tuning (run under torch.distributed.run).

    python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 \
        -m paper_2511_09557_b200.probe [--sizes 65536,1048576]

Prints, on rank 0, one JSON object:
  alpha_signal_us  one-way NVLink flag latency (p50 of device ping-pong, rank 0 <-> each peer)
  launch_floor_us  per-call time of a count==0 call (the sequence bump kernel) in a graph
  phases           per size and schedule: CTA 0 phase timestamps of one call
                   (entry, after pdl wait, RS pushed, peers synced, reduced, AG received, exit)
"""
from __future__ import annotations

import argparse
import ctypes
import json
import os
import statistics

import torch
import torch.distributed as dist

from . import _lib as L
from .comm import ClusterTopology, Communicator
from . import dist as D


def pingpong_us(comm: Communicator, rank: int, world: int, iters: int = 200, reps: int = 5):
    out = {}
    lib = comm._lib
    for peer in range(1, world):
        vals = []
        for _ in range(reps):
            dist.barrier()
            ns = ctypes.c_uint64()
            if rank == 0:
                rc = lib.nvrar_pingpong(comm._h, peer, iters, 1, None, ctypes.byref(ns))
            elif rank == peer:
                rc = lib.nvrar_pingpong(comm._h, 0, iters, 0, None, ctypes.byref(ns))
            else:
                rc = 0
            if rc:
                raise RuntimeError(comm.last_error())
            if rank == 0:
                vals.append(ns.value / iters / 2 / 1e3)
        if rank == 0:
            out[peer] = statistics.median(vals)
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sizes", default="65536,262144,1048576,2097152")
    ap.add_argument("--nodes", type=int, default=0)
    args = ap.parse_args()
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    nodes = args.nodes or (2 if world > 1 else 1)
    comm = Communicator.from_process_group(ClusterTopology(nodes, world // nodes), 8 << 20,
                                           device=local)
    res = {"world": world, "nodes": nodes}
    pp = pingpong_us(comm, rank, world)
    if rank == 0:
        res["alpha_signal_us_by_peer"] = pp
        res["alpha_signal_us"] = statistics.median(list(pp.values()))

    # launch floor: count == 0 calls (one tiny kernel each) in a graph
    z = torch.empty(0, device="cuda")
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        comm.allreduce(z, z)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(100):
            comm.allreduce(z, z)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    g.replay()
    torch.cuda.synchronize()
    a.record()
    g.replay()
    b.record()
    torch.cuda.synchronize()
    res["launch_floor_us"] = a.elapsed_time(b) * 1e3 / 100

    # copy floor: a 1x1 communicator (the same kernel, no peers) in a graph —
    # launch + input load + output store + grid completion, per call
    solo = Communicator(ClusterTopology(1, 1), 0, local, 8 << 20)
    solo.connect([solo.export()])
    floors = {}
    from .comm import NvrarConfig
    for size, blocks, prof in ((128 << 10, 32, 1), (128 << 10, 32, 0), (128 << 10, 4, 0),
                               (128 << 10, 128, 0), (1 << 20, 32, 1), (1 << 20, 128, 0)):
        solo.set_config(NvrarConfig(blocks, 65536))
        xs = [(torch.randn(size // 2, device="cuda").to(torch.bfloat16),
               torch.empty(size // 2, device="cuda", dtype=torch.bfloat16)) for _ in range(80)]
        solo._lib.nvrar_set_profile(solo._h, prof)
        s2 = torch.cuda.Stream()
        s2.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s2):
            solo.allreduce(*xs[0])
        torch.cuda.current_stream().wait_stream(s2)
        torch.cuda.synchronize()
        g2 = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g2, stream=s2):
            for i in range(80):
                solo.allreduce(*xs[i])
        g2.replay()
        torch.cuda.synchronize()
        a.record()
        g2.replay()
        b.record()
        torch.cuda.synchronize()
        ts = (ctypes.c_uint64 * 8)()
        solo._lib.nvrar_get_phase_times(solo._h, ts, 8)
        floors[f"{size >> 10}KB_b{blocks}_prof{prof}"] = {
            "per_call_us": round(a.elapsed_time(b) * 1e3 / 80, 3),
            "cta0_release_to_exit_us": round((ts[6] - ts[7]) / 1e3, 3),
            "cta0_release_to_loaded_us": round((ts[2] - ts[7]) / 1e3, 3),
            "entry_to_release_us": round((ts[7] - ts[0]) / 1e3, 3)}
        del g2
    solo.close()
    res["copy_floor_p1"] = floors

    # phase breakdown of single calls
    comm._lib.nvrar_set_profile(comm._h, 1)
    phases = {}
    for size in [int(x) for x in args.sizes.split(",")]:
        for algo in ("hier", "twoshot", "oneshot"):
            if algo == "oneshot" and size > (1 << 20):
                continue
            comm.set_algo(algo)
            x = torch.randn(size // 2, device="cuda").to(torch.bfloat16)
            y = torch.empty_like(x)
            rows = []
            for _ in range(5):
                dist.barrier()
                comm.allreduce(x, y)
                torch.cuda.synchronize()
                ts = (ctypes.c_uint64 * 8)()
                comm._lib.nvrar_get_phase_times(comm._h, ts, 8)
                t = [ts[i] for i in range(7)]
                rows.append([round((t[i] - t[0]) / 1e3, 3) for i in range(7)])
            rows = D.max_over_ranks([v for r in rows for v in r])
            last = rows[-7:]
            phases[f"{size >> 10}KB_{algo}"] = last
    comm._lib.nvrar_set_profile(comm._h, 0)
    comm.check()
    if rank == 0:
        res["phases_us"] = phases
        res["phase_names"] = ["entry", "pdl_wait", "rs_pushed", "synced", "reduced+ag_pushed",
                              "ag_received", "exit"]
        print(json.dumps(res), flush=True)
    dist.barrier()
    comm.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
