"""Per-rank all-reduce measurement, NVRAR against NCCL called directly.

One process per GPU (`launch` spawns them; no torchrun), gloo for the control
plane (barriers, max over ranks), the collective under test on the data path:

    python -m paper_2511_09557_b200.rankbench launch --world 2 --impl nvrar
    python -m paper_2511_09557_b200.rankbench launch --world 2 --impl nccl \
        --nccl-lib system --nccl-algo Ring --nccl-proto LL   (NCCL_ALGO / NCCL_PROTO)
    python -m paper_2511_09557_b200.rankbench nccl-best --world 2      # every algo x proto x lib

Timing (bench.py's rules): a step is one CUDA-graph replay of `calls`
back-to-back all-reduces over rotating buffers larger than the L2, CUDA
events on the launching stream, max over ranks per step, p50 over steps.
`--producer gemm` puts a cuBLAS GEMM that WRITES the all-reduce's input in
front of every call (the decode layer's row-parallel projection): no PDL
overlap with the previous all-reduce, an L2-hot input, and the per-call
all-reduce cost is (step - GEMM-only step) / calls — the same for both arms.

`--profile`: a few eager calls per size instead (for a kernel profiler on
rank 0 only: `launch --ncu-rank0 "ncu --metrics ..."` — the other ranks run
unprofiled, so a profiler that serialises one process's kernels does not
serialise the ranks against each other; only single-pass metric sets work,
a replayed kernel would wait for peers that have moved on).
"""
from __future__ import annotations

import argparse
import json
import os
import shlex
import socket
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SIZES = [64 << 10, 128 << 10, 256 << 10, 512 << 10, 1 << 20, 2 << 20, 4 << 20, 8 << 20]
NCCL_ALGOS = ["Ring", "Tree", "NVLS", "NVLSTree"]
NCCL_PROTOS = ["LL", "LL128", "Simple"]


def _port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


# ---- worker -------------------------------------------------------------------

def worker(args) -> None:
    import torch
    import torch.distributed as dist

    from . import harness as H

    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    dev = rank % max(1, torch.cuda.device_count()) if args.device < 0 else args.device
    torch.cuda.set_device(dev)
    torch.zeros(1, device="cuda")  # the CUDA context exists from here on
    if os.environ.get("RB_READY_DIR"):
        open(os.path.join(os.environ["RB_READY_DIR"], f"ready{rank}"), "w").close()
    dist.init_process_group("gloo")
    nodes = args.nodes or (2 if world > 1 else 1)
    stream = torch.cuda.Stream()
    info = {"impl": args.impl, "world": world}
    if args.impl == "nvrar":
        from .comm import ClusterTopology, Communicator
        comm = Communicator.from_process_group(ClusterTopology(nodes, world // nodes),
                                               max(args.sizes), device=dev, timeout_s=30.0)
        if args.algo != "auto":
            comm.set_algo(args.algo)
        if args.blocks:
            from .comm import NvrarConfig
            comm.set_config(NvrarConfig(args.blocks, 65536))
        if args.autotune:
            from .selector import autotune
            autotune(comm, sizes=args.sizes, dtype=torch.bfloat16, calls=30, reps=5)
        info["topology"] = f"{nodes}x{world // nodes}"

        def ar(a, b):
            comm.allreduce(a, b)

        def plan(n):
            return comm.plan(n, torch.bfloat16)
    else:
        from . import nccl_ref
        nc = nccl_ref.Nccl(nccl_ref.lib_path(args.nccl_lib))
        uid = [nc.unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        nc.init_rank(world, uid[0], rank)
        info.update(nccl_version=nc.version(), nccl_lib=args.nccl_lib,
                    nccl_algo=os.environ.get("NCCL_ALGO", "default"),
                    nccl_proto=os.environ.get("NCCL_PROTO", "default"))

        def ar(a, b):
            nc.all_reduce(a, b)

        def plan(n):
            return (info["nccl_algo"], info["nccl_proto"])

    def barrier():
        dist.barrier()

    def max_over_ranks(vals):
        t = torch.tensor(vals, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return t.tolist()

    hidden = 8192
    for size in args.sizes:
        ne = size // 2
        torch.manual_seed(100 + rank)
        if args.profile:
            a = torch.randn(ne, device="cuda").to(torch.bfloat16)
            b = torch.empty_like(a)
            for _ in range(args.calls):
                ar(a, b)
            torch.cuda.synchronize()
            barrier()
            continue
        calls = args.calls or H.calls_for(size, 1)
        src = torch.randn(ne, device="cuda").to(torch.bfloat16)
        bufs = [(src.clone(), torch.empty_like(src)) for _ in range(calls)]
        row = dict(info, bytes=size, calls=calls, producer=args.producer)
        if args.producer == "gemm":
            rows = max(1, ne // hidden)
            k = 1024
            xs = [torch.randn(rows, k, device="cuda").to(torch.bfloat16) for _ in range(4)]
            w = (torch.randn(k, ne // rows, device="cuda") * k ** -0.5).to(torch.bfloat16)

            def prod(i):
                torch.matmul(xs[i % 4], w, out=bufs[i][0].view(rows, ne // rows))
            g0 = H.graph_of(prod, calls, stream)
            t0 = max_over_ranks(H.time_replays(g0.replay, args.steps, args.warmup, barrier, stream))
            del g0
            gr = H.graph_of(lambda i: (prod(i), ar(*bufs[i])), calls, stream)
            ts = max_over_ranks(H.time_replays(gr.replay, args.steps, args.warmup, barrier, stream))
            per = sorted((t - statistics.median(t0)) * 1e3 / calls for t in ts)
            row.update(producer_us=round(statistics.median(t0) * 1e3 / calls, 3),
                       with_producer_us=round(statistics.median(ts) * 1e3 / calls, 3))
        else:
            gr = H.graph_of(lambda i: ar(*bufs[i]), calls, stream)
            ts = max_over_ranks(H.time_replays(gr.replay, args.steps, args.warmup, barrier, stream))
            per = sorted(t * 1e3 / calls for t in ts)
        del gr
        row.update(p50_us=round(statistics.median(per), 3), p10_us=round(per[len(per) // 10], 3),
                   p90_us=round(per[(9 * len(per)) // 10], 3), plan=list(plan(ne)))
        if args.impl == "nvrar":
            comm.check()
        if rank == 0:
            print("RB " + json.dumps(row), flush=True)
    barrier()
    if args.impl == "nvrar":
        comm.close()
    else:
        nc.close()
    dist.destroy_process_group()


# ---- launcher ------------------------------------------------------------------

def launch(args, extra_env=None) -> list:
    """Spawn `world` worker processes; returns rank 0's RB rows."""
    port = _port()
    procs = []
    wargs = ["worker", "--impl", args.impl, "--nodes", str(args.nodes), "--algo", args.algo,
             "--blocks", str(args.blocks),
             "--sizes", ",".join(str(s) for s in args.sizes), "--steps", str(args.steps),
             "--warmup", str(args.warmup), "--calls", str(args.calls), "--producer",
             args.producer, "--nccl-lib", args.nccl_lib]
    if args.autotune:
        wargs.append("--autotune")
    if args.profile:
        wargs.append("--profile")
    import tempfile
    ready = tempfile.mkdtemp(prefix="rb_ready_")
    # with a profiler on rank 0, the other ranks create their CUDA contexts
    # first (a profiled process can hold up another process's CUDA init)
    order = list(range(1, args.world)) + [0] if args.ncu_rank0 else list(range(args.world))
    procs = [None] * args.world
    for r in order:
        env = dict(os.environ, RANK=str(r), WORLD_SIZE=str(args.world), LOCAL_RANK=str(r),
                   MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RB_READY_DIR=ready,
                   **(extra_env or {}))
        cmd = [sys.executable, "-m", "paper_2511_09557_b200.rankbench", *wargs]
        if r == 0 and args.ncu_rank0:
            t0 = time.time()
            while not all(os.path.exists(os.path.join(ready, f"ready{q}"))
                          for q in range(1, args.world)) and time.time() - t0 < 120:
                time.sleep(0.1)
            cmd = shlex.split(args.ncu_rank0) + cmd
        procs[r] = subprocess.Popen(cmd, env=env, cwd=ROOT, stdout=subprocess.PIPE,
                                    stderr=subprocess.STDOUT, text=True)
    rows, outs = [], []
    for p in procs:
        try:
            o, _ = p.communicate(timeout=args.timeout)
        except subprocess.TimeoutExpired:
            for q in procs:
                q.kill()
            o = "TIMEOUT"
        outs.append(o)
    for line in outs[0].splitlines():
        if line.startswith("RB "):
            rows.append(json.loads(line[3:]))
    if any(p.returncode for p in procs):
        sys.stderr.write("\n".join(o[-3000:] for o in outs) + "\n")
    if args.show_output:
        sys.stderr.write(outs[0][-6000:] + "\n")
    return rows


def nccl_best(args) -> None:
    """Every NCCL_ALGO x NCCL_PROTO x library; per size the best p50 and its
    (algo, proto, version) — the strongest NCCL configuration on this box."""
    best = {}
    allrows = []
    libs = args.nccl_libs.split(",")
    args.impl = "nccl"
    for lib in libs:
        for algo in NCCL_ALGOS:
            for proto in NCCL_PROTOS:
                args.nccl_lib = lib
                t = time.time()
                rows = launch(args, {"NCCL_ALGO": algo, "NCCL_PROTO": proto,
                                     "NCCL_DEBUG": "WARN"})
                sys.stderr.write(f"{lib} {algo}/{proto}: {len(rows)} rows in {time.time() - t:.0f}s\n")
                for r in rows:
                    allrows.append(r)
                    k = r["bytes"]
                    if k not in best or r["p50_us"] < best[k]["p50_us"]:
                        best[k] = r
    for r in allrows:
        print("ALL " + json.dumps(r), flush=True)
    for k in sorted(best):
        r = best[k]
        print("BEST " + json.dumps({"bytes": k, "nccl_best_us": r["p50_us"], "algo": r["nccl_algo"],
                                    "proto": r["nccl_proto"], "version": r["nccl_version"],
                                    "lib": r["nccl_lib"], "producer": r["producer"]}), flush=True)


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("mode", choices=["launch", "worker", "nccl-best"])
    ap.add_argument("--world", type=int, default=2)
    ap.add_argument("--nodes", type=int, default=0)
    ap.add_argument("--impl", choices=["nvrar", "nccl"], default="nvrar")
    ap.add_argument("--algo", default="auto")
    ap.add_argument("--autotune", action="store_true")
    ap.add_argument("--blocks", type=int, default=0, help="CTAs per rank (0 = selector)")
    ap.add_argument("--sizes", default=",".join(str(s) for s in SIZES))
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--calls", type=int, default=0, help="0 = enough for rotating buffers > L2")
    ap.add_argument("--producer", choices=["none", "gemm"], default="none")
    ap.add_argument("--nccl-lib", default="torch", help="torch | system | a path")
    ap.add_argument("--nccl-libs", default="system,torch")
    ap.add_argument("--nccl-algo", default="")
    ap.add_argument("--nccl-proto", default="")
    ap.add_argument("--device", type=int, default=-1)
    ap.add_argument("--profile", action="store_true")
    ap.add_argument("--ncu-rank0", default="")
    ap.add_argument("--timeout", type=float, default=900)
    ap.add_argument("--show-output", action="store_true")
    args = ap.parse_args()
    args.sizes = [int(s) for s in str(args.sizes).split(",")]
    if args.mode == "worker":
        worker(args)
    elif args.mode == "launch":
        env = {}
        if args.nccl_algo:
            env["NCCL_ALGO"] = args.nccl_algo
        if args.nccl_proto:
            env["NCCL_PROTO"] = args.nccl_proto
        for r in launch(args, env):
            print("RB " + json.dumps(r), flush=True)
    else:
        nccl_best(args)


if __name__ == "__main__":
    main()
