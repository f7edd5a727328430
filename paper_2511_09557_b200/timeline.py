"""Cross-GPU timeline of one steady-state call (diagnostics; run under torch.distributed.run).

Estimates each GPU's %globaltimer offset to rank 0 with a device ping-pong,
then replays a graph of back-to-back calls with per-CTA phase stamps and
prints, for the last call, every rank's phase times (min / median / max over
CTAs) on rank 0's clock, relative to rank 0's median release.

    python -m torch.distributed.run --nproc-per-node 4 --master-addr 127.0.0.1 \
        -m paper_2511_09557_b200.timeline --bytes 131072 --algo oneshot --blocks 32
"""
from __future__ import annotations

import argparse
import ctypes
import json
import os
import statistics

import torch
import torch.distributed as dist

from .comm import ClusterTopology, Communicator, NvrarConfig
from .harness import graph_of

NAMES = ["entry", "release", "seq", "pushed", "synced", "reduced", "ag_recv", "exit"]
ORDER = [0, 7, 1, 2, 3, 4, 5, 6]  # stamp slots in phase order


def clock_offsets(comm, rank, world, iters=50):
    """offset[p] = clock_p - clock_0 (ns), from the last ping-pong round."""
    offs = [0.0] * world
    for peer in range(1, world):
        vals = []
        for _ in range(5):
            dist.barrier()
            ns = ctypes.c_uint64()
            st = (ctypes.c_uint64 * 2)()
            if rank == 0:
                comm._lib.nvrar_pingpong(comm._h, peer, iters, 1, None, ctypes.byref(ns))
                comm._lib.nvrar_pingpong_clock(comm._h, st)
            elif rank == peer:
                comm._lib.nvrar_pingpong(comm._h, 0, iters, 0, None, ctypes.byref(ns))
                comm._lib.nvrar_pingpong_clock(comm._h, st)
            mine = [int(st[0]), int(st[1])]
            allv = [None] * world
            dist.all_gather_object(allv, mine)
            s, r = allv[0]
            q = allv[peer][0]
            vals.append(q - (s + r) / 2.0)
        offs[peer] = statistics.median(vals)
    return offs


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--bytes", type=int, default=128 << 10)
    ap.add_argument("--algo", default="oneshot")
    ap.add_argument("--blocks", type=int, default=32)
    ap.add_argument("--nodes", type=int, default=2)
    ap.add_argument("--calls", type=int, default=20)
    args = ap.parse_args()
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    nodes = min(args.nodes, world)
    comm = Communicator.from_process_group(ClusterTopology(nodes, world // nodes), 8 << 20,
                                           device=local)
    offs = clock_offsets(comm, rank, world)
    comm.set_algo(args.algo)
    comm.set_config(NvrarConfig(args.blocks, 65536))
    n = args.bytes // 2
    bufs = [(torch.randn(n, device="cuda").to(torch.bfloat16),
             torch.empty(n, device="cuda", dtype=torch.bfloat16)) for _ in range(args.calls)]
    comm._lib.nvrar_set_profile(comm._h, 1)
    stream = torch.cuda.Stream()
    g = graph_of(lambda i: comm.allreduce(*bufs[i]), args.calls, stream)
    dist.barrier()
    g.replay()
    torch.cuda.synchronize()
    ts = (ctypes.c_uint64 * (512 * 8))()
    comm._lib.nvrar_get_phase_times(comm._h, ts, 512 * 8)
    mine = [[int(ts[b * 8 + k]) for k in ORDER] for b in range(args.blocks)]
    allv = [None] * world
    dist.all_gather_object(allv, mine)
    comm.check()
    if rank == 0:
        ref = statistics.median(c[1] for c in allv[0])
        out = {"bytes": args.bytes, "algo": args.algo, "blocks": args.blocks, "world": world,
               "clock_offset_ns": offs, "phases": NAMES, "ranks": {}}
        for r in range(world):
            rows = [[(t - offs[r] - ref) / 1e3 for t in c] for c in allv[r]]
            out["ranks"][r] = {NAMES[k]: [round(min(x[k] for x in rows), 3),
                                          round(statistics.median(x[k] for x in rows), 3),
                                          round(max(x[k] for x in rows), 3)]
                               for k in range(len(NAMES))}
        print(json.dumps(out), flush=True)
    comm._lib.nvrar_set_profile(comm._h, 0)
    dist.barrier()
    comm.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
