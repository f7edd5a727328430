"""Single-process driver for kernel-profiler captures of the real multi-GPU
kernels (one rank per GPU, EMU=false): every rank's communicator lives in
this process (peers mapped directly, peer access enabled), each rank's call
goes to its own GPU's stream, and rank 0's launch is issued LAST. Profile
only device 0 — `ncu --devices 0 ...` — and the other ranks' kernels run
unprofiled and concurrently, so rank 0's kernel completes under the profiler
(a profiler that serialises rank 0 against its peers would deadlock it).
Only single-pass metric sets are valid: a replayed pass of rank 0's kernel
would wait for peers that have moved on (the driver sets a short watchdog).

    ncu --devices 0 -k regex:"flat_kernel|hier_kernel" \
        --metrics gpu__time_duration.sum,nvltx__bytes.sum,nvlrx__bytes.sum \
        python -m paper_2511_09557_b200.nvlprofile --world 2 --algos oneshot,hier \
        --sizes 131072,1048576
"""
from __future__ import annotations

import argparse
import json

import torch


def main() -> None:
    from .comm import ClusterTopology, Communicator

    ap = argparse.ArgumentParser()
    ap.add_argument("--world", type=int, default=2)
    ap.add_argument("--nodes", type=int, default=0)
    ap.add_argument("--algos", default="oneshot,twoshot,hier")
    ap.add_argument("--sizes", default="131072,1048576,2097152")
    ap.add_argument("--calls", type=int, default=3)
    ap.add_argument("--timeout", type=float, default=20.0)
    args = ap.parse_args()
    P = args.world
    nodes = args.nodes or (2 if P > 1 else 1)
    topo = ClusterTopology(nodes, P // nodes)
    sizes = [int(s) for s in args.sizes.split(",")]
    comms = [Communicator(topo, r, r, max(sizes), timeout_s=args.timeout) for r in range(P)]
    handles = [c.export() for c in comms]
    for c in comms:
        c.connect(handles)
    streams = []
    for r in range(P):
        with torch.cuda.device(r):
            streams.append(torch.cuda.Stream(r))
    order = list(range(1, P)) + [0]  # rank 0 last: its peers are already running
    log = []
    for algo in args.algos.split(","):
        for c in comms:
            c.set_algo(algo)
        for size in sizes:
            ne = size // 2
            xs, ys = [], []
            for r in range(P):
                with torch.cuda.device(r):
                    torch.manual_seed(r)
                    xs.append(torch.randn(ne, device=f"cuda:{r}").to(torch.bfloat16))
                    ys.append(torch.empty_like(xs[-1]))
            for r in range(P):
                torch.cuda.synchronize(r)
            for _ in range(args.calls):
                for r in order:
                    comms[r].allreduce(xs[r], ys[r], stream=streams[r])
                for r in range(P):
                    streams[r].synchronize()
            for c in comms:
                c.check()
            want = ys[0].float()
            same = all(torch.equal(ys[r].cpu(), ys[0].cpu()) for r in range(1, P))
            log.append({"world": P, "algo": algo, "bytes": size,
                        "plan": list(comms[0].plan(ne, torch.bfloat16)), "calls": args.calls,
                        "ranks_agree": same, "finite": bool(torch.isfinite(want).all())})
    for c in comms:
        c.close()
    for row in log:
        print("NVLP " + json.dumps(row), flush=True)


if __name__ == "__main__":
    main()
