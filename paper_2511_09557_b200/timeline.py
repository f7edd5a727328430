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


REGION = {"A": 0, "B": 1, "C": 2}  # slot areas: RS / one-shot inputs, all-gather, RD steps


def trace_csv(args, world, nodes, offs, ref, allv) -> str:
    """The reference's trace schema `time_us,src,dst,region,offset,bytes`
    (bench.hpp:322-334; a row per put there) at the GPU's granularity: one row
    per (rank, CTA, destination) push batch of the last call, timed by the
    CTA's phase stamps on rank 0's clock (µs from rank 0's median release).
    Regions: 0 = A slots (reduce-scatter / one-shot inputs), 1 = B (all-gather),
    2 = C (recursive-doubling steps); offset = the batch's first byte in the
    destination's slot."""
    gpus = world // nodes
    n = args.bytes // 2
    ue_elems = 8  # bf16 Lamport: 16-byte units of 8 elements
    rows = ["time_us,src,dst,region,offset,bytes\n"]

    def units(elems):
        return -(-elems // ue_elems)

    def cta_range(u_total, b):
        return u_total * b // args.blocks, u_total * (b + 1) // args.blocks

    for r in range(world):
        node, local = divmod(r, gpus)
        for b, stamps in enumerate(allv[r]):
            t_push = (stamps[3] - offs[r] - ref) / 1e3   # "pushed"
            t_red = (stamps[5] - offs[r] - ref) / 1e3    # "reduced" (RD + all-gather pushes done)
            batches = []
            if args.algo in ("oneshot", "twoshot", "mcast"):
                sp = n if args.algo != "twoshot" else -(-n // world)
                u0, u1 = cta_range(units(sp), b)
                for q in range(world):
                    if q != r:
                        batches.append((t_push, q, "A", u0, u1))
                        if args.algo == "twoshot":
                            batches.append((t_red, q, "B", u0, u1))
            else:  # hier
                u0, u1 = cta_range(units(-(-n // gpus)), b)
                for j in range(1, gpus):
                    batches.append((t_push, node * gpus + (local + j) % gpus, "A", u0, u1))
                    batches.append((t_red, node * gpus + (local + j) % gpus, "B", u0, u1))
                step = 1
                while step < nodes:
                    batches.append((t_red, (node ^ step) * gpus + local, "C", u0, u1))
                    step <<= 1
            for t, q, reg, a, z in batches:
                if z > a:
                    ub = 32 if reg == "C" else 16  # RD partials travel as fp32 (2x bf16)
                    rows.append(f"{t:.3f},{r},{q},{REGION[reg]},{a * ub},{(z - a) * ub}\n")
    return "".join(rows)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--bytes", type=int, default=128 << 10)
    ap.add_argument("--algo", default="oneshot")
    ap.add_argument("--blocks", type=int, default=32)
    ap.add_argument("--nodes", type=int, default=2)
    ap.add_argument("--calls", type=int, default=20)
    ap.add_argument("--trace-csv", default="",
                    help="write the reference's trace CSV (bench.hpp:322-334) for the last call")
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
        if args.trace_csv:
            with open(args.trace_csv, "w") as fh:
                fh.write(trace_csv(args, world, nodes, offs, ref, allv))
    comm._lib.nvrar_set_profile(comm._h, 0)
    dist.barrier()
    comm.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
