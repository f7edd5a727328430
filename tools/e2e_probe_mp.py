"""N>1 host-buffer e2e (bench.py's N>1 e2e leg: nvrar_allreduce_host, pinned
bf16 in and out, per step, max over ranks) for each forced schedule — run
under torchrun, one rank per GPU; NVRAR_HOST_CTAS caps the CTAs.

    torchrun --nproc-per-node 2 tools/e2e_probe_mp.py --bytes 1048576
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main() -> None:
    from paper_2511_09557_b200 import ClusterTopology, Communicator
    from paper_2511_09557_b200 import dist as D

    ap = argparse.ArgumentParser()
    ap.add_argument("--bytes", type=int, default=1 << 20)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--algos", default="auto,oneshot,twoshot")
    args = ap.parse_args()
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    rank, world = dist.get_rank(), dist.get_world_size()
    comm = Communicator.from_process_group(ClusterTopology(2 if world > 1 else 1, max(world // 2, 1)),
                                           8 << 20, device=local, timeout_s=30.0)
    dev = torch.device("cuda", local)
    stream = torch.cuda.Stream()
    ne = args.bytes // 2
    host_in = torch.randn(ne).to(torch.bfloat16).pin_memory()
    host_out = torch.empty(ne, dtype=torch.bfloat16).pin_memory()
    res = {}
    for algo in args.algos.split(","):
        comm.set_algo(algo)
        ts = []
        for k in range(5 + args.steps):
            dist.barrier(device_ids=[local])
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            with torch.cuda.stream(stream):
                a.record(stream)
                comm.allreduce_host(host_in, host_out, stream=stream)
                b.record(stream)
            b.synchronize()
            if k >= 5:
                ts.append(a.elapsed_time(b) * 1e3)
        ts = D.max_over_ranks(ts, device=dev)
        comm.check()
        res[algo] = round(statistics.median(ts), 2)
    if rank == 0:
        print("E2EMP " + json.dumps({"world": world, "bytes": args.bytes,
                                     "host_ctas": os.environ.get("NVRAR_HOST_CTAS", "64"),
                                     "us": res}), flush=True)
    comm.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
