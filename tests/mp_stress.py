"""Multi-GPU stress worker: thousands of back-to-back calls that switch schedule,
CTA count, dtype and size between calls (same deterministic sequence on every
rank), each checked against an exactly representable expected sum. A hang is
reported by the device watchdog (DEADLOCK) within `--timeout` seconds.

    python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 \
        tests/mp_stress.py --calls 3000
"""
import argparse
import os
import random
import sys

import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2511_09557_b200 import ClusterTopology, Communicator, NvrarConfig  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--calls", type=int, default=2000)
    ap.add_argument("--timeout", type=float, default=5.0)
    ap.add_argument("--nodes", type=int, default=2)
    ap.add_argument("--graph", action="store_true", help="capture runs of calls in CUDA graphs")
    ap.add_argument("--sync-every", type=int, default=1)
    ap.add_argument("--multicast", action="store_true", help="also the NVLS one-shot")
    ap.add_argument("--registered", action="store_true",
                    help="also in-place all-reduces of registered buffers")
    ap.add_argument("--jitter", type=int, default=0, help="injected delays up to this many ns")
    args = ap.parse_args()
    local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    nodes = min(args.nodes, world)
    comm = Communicator.from_process_group(ClusterTopology(nodes, world // nodes), 4 << 20,
                                           device=local, timeout_s=args.timeout)
    rng = random.Random(1234)
    sizes = [1, 7, 1000, 4099, 65536, 131072, 300001, 1 << 20]
    algos = ["hier", "twoshot", "oneshot", "auto"]
    if args.multicast:
        if not comm.enable_multicast():
            print(f"rank {rank}: multicast unavailable: {getattr(comm, 'mc_error', '')}", flush=True)
        else:
            algos.append("mcast")
    # call kinds: the all-reduce, its fused residual epilogue, the ring / tree orders
    kinds = ["allreduce", "allreduce", "residual", "ring", "tree"]
    regbuf = {}
    if args.registered:
        kinds.append("registered")
        for dt in (torch.bfloat16, torch.float32, torch.int32):
            regbuf[dt] = comm.alloc_symmetric(1 << 20, dt)
    if args.jitter:
        comm.set_jitter(args.jitter, 77 + rank)
    dtypes = [torch.bfloat16, torch.float32, torch.int32]
    total = world * (world + 1) // 2
    bad = 0
    pending = []
    for it in range(args.calls):
        algo = rng.choice(algos)
        blocks = rng.choice([0, 1, 3, 16, 32, 128])
        dt = rng.choice(dtypes)
        n = rng.choice(sizes)
        if dt != torch.int32 and n > (1 << 20) // 2:
            n = (1 << 20) // 2
        kind = rng.choice(kinds)
        if kind == "ring" and world > 8:
            kind = "allreduce"
        comm.set_algo(algo)
        comm.set_config(NvrarConfig(blocks, 65536))
        idx = torch.arange(n, device="cuda", dtype=torch.int64) % 7 + 1
        x = (idx * (rank + 1)).to(dt)
        y = torch.empty_like(x)
        resid = None
        if kind == "residual":
            resid = idx.to(dt)
            comm.allreduce_residual(x, resid, out=y)
        elif kind == "ring":
            comm.ring_allreduce(x, y)
        elif kind == "tree":
            comm.tree_allreduce(x, y)
        elif kind == "registered":
            buf = regbuf[dt][:n]
            buf.copy_(x)
            comm.allreduce_registered(buf, y)
        else:
            comm.allreduce(x, y)
        pending.append((it, f"{kind}:{algo}", blocks, dt, n, idx, y, resid))
        if (it + 1) % args.sync_every == 0 or it == args.calls - 1:
            torch.cuda.synchronize()
            rc = comm.check_status()
            if rc:
                print(f"rank {rank}: call {it} status {rc}: {comm.last_error()}", flush=True)
                bad += 1
                break
            for (i, a, b, d, nn, ix, yy, rr) in pending:
                want = (ix * total).to(d)
                if rr is not None:
                    want = want + rr  # the element type's own add, like the kernel
                if not torch.equal(yy, want):
                    nbad = int((yy != want).sum())
                    print(f"rank {rank}: call {i} {a}/{b} {d} n={nn}: {nbad} wrong", flush=True)
                    bad += 1
            pending = []
            if bad:
                break
    print(f"rank {rank}: {'OK' if bad == 0 else 'FAIL'} after {it + 1} calls", flush=True)
    dist.barrier()
    comm.close()
    dist.destroy_process_group()
    sys.exit(1 if bad else 0)


if __name__ == "__main__":
    main()
