"""Single-process driver for ncu captures: the N=1 bench workload (2x4 virtual
ranks on cuda:0, one cooperative launch per all-reduce) run eagerly a few
times, so `ncu -k regex:<kernel>` can pick one launch.

    python -m paper_2511_09557_b200.profile_emu --algo twoshot --dtype f32 --bytes 1048576

--rotate: the bench's rotating buffer sets (> L2), launched eagerly twice over:
profile the second pass with `ncu --cache-control none`, so each launch's DRAM
counters include the write-back of earlier calls' outputs that it evicts (a
single cold-cache capture leaves its own writes in L2): sum / launches = the
per-call DRAM traffic in steady state. (--range: the same inside a CUDA graph
between cudaProfilerStart/Stop; ncu's range replay does not accept graph
launches on this driver.)
"""
from __future__ import annotations

import argparse

import torch

from .comm import ClusterTopology, LocalGroup


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--algo", default="auto")
    ap.add_argument("--dtype", default="f32", choices=["f32", "bf16"])
    ap.add_argument("--bytes", type=int, default=1 << 20)
    ap.add_argument("--calls", type=int, default=6)
    ap.add_argument("--nodes", type=int, default=2)
    ap.add_argument("--gpus", type=int, default=4)
    ap.add_argument("--proto", default="auto")
    ap.add_argument("--solo", action="store_true",
                    help="one 1x1 communicator (the single-rank kernel, no virtual ranks)")
    ap.add_argument("--blocks", type=int, default=0)
    ap.add_argument("--range", action="store_true")
    ap.add_argument("--rotate", action="store_true")
    args = ap.parse_args()
    dt = torch.float32 if args.dtype == "f32" else torch.bfloat16
    n = args.bytes // (4 if args.dtype == "f32" else 2)
    if args.solo:
        from .comm import Communicator, NvrarConfig
        c = Communicator(ClusterTopology(1, 1), 0, 0, max(args.bytes, 1 << 20))
        c.connect([c.export()])
        c.set_config(NvrarConfig(args.blocks, 65536))
        x = torch.randn(n, device="cuda").to(dt)
        y = torch.empty_like(x)
        for _ in range(args.calls):
            c.allreduce(x, y)
        c.check()
        print("solo plan", c.plan(n, dt), "ok")
        c.close()
        return
    p = args.nodes * args.gpus
    g = LocalGroup(ClusterTopology(args.nodes, args.gpus), max(args.bytes, 1 << 20), device=0)
    g.set_algo(args.algo)
    g.set_protocol(args.proto)
    if args.rotate:
        from . import harness as H
        calls = H.calls_for(args.bytes, p)
        sets = [([torch.randn(n, device="cuda").to(dt) for _ in range(p)],
                 [torch.empty(n, device="cuda", dtype=dt) for _ in range(p)]) for _ in range(calls)]
        for _ in range(2):
            for i in range(calls):
                g.launch(*sets[i])
        torch.cuda.synchronize()
        g.check()
        print(f"rotate: 2 x {calls} calls, plan {g.plan(n, dt)} ok")
        g.close()
        return
    if args.range:
        from . import harness as H
        calls = H.calls_for(args.bytes, p)
        sets = [([torch.randn(n, device="cuda").to(dt) for _ in range(p)],
                 [torch.empty(n, device="cuda", dtype=dt) for _ in range(p)]) for _ in range(calls)]
        stream = torch.cuda.Stream()
        gr = H.graph_of(lambda i: g.launch(*sets[i], stream=torch.cuda.current_stream()), calls,
                        stream)
        for _ in range(3):
            gr.replay()
        torch.cuda.synchronize()
        torch.cuda.profiler.start()
        gr.replay()
        torch.cuda.synchronize()
        torch.cuda.profiler.stop()
        g.check()
        print(f"range: {calls} calls, plan {g.plan(n, dt)} ok")
        g.close()
        return
    ins = [torch.randn(n, device="cuda").to(dt) for _ in range(p)]
    outs = [torch.empty_like(t) for t in ins]
    for _ in range(args.calls):
        g.launch(ins, outs)
    g.check()
    print("plan", g.plan(n, dt), "ok")
    g.close()


if __name__ == "__main__":
    main()
