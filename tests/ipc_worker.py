"""One rank of a multi-process NVRAR run whose handles are exchanged through a
directory (paper_2511_09557_b200.bootstrap) instead of a process group. With
--device 0 on every rank the processes share ONE GPU and make progress by
the GPU's time-slicing: the real per-rank kernels (EMU=false: one rank per
launch, peers' regions mapped through CUDA IPC, descriptor by value) run
against each other exactly as over NVLink, only slower. This is how a
1-GPU box (the driver's) executes the multi-GPU path.

    python tests/ipc_worker.py --dir D --rank r --nodes N --gpus G [--ops] [--quick]

Exit code 0 = every result bit-exact against the oracle.
"""
import argparse
import os
import sys

print(f"ipc_worker: interpreter up (pid {os.getpid()})", flush=True)

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

from oracle import oracle as O  # noqa: E402
from paper_2511_09557_b200 import ClusterTopology  # noqa: E402
from paper_2511_09557_b200 import _lib as L  # noqa: E402
from paper_2511_09557_b200 import bootstrap as B  # noqa: E402


def _dev(a, dtype, device):
    t = torch.from_numpy(np.ascontiguousarray(a))
    if dtype == "bf16":
        t = t.view(torch.int16).view(torch.bfloat16)
    return t.to(device)


def _host(t, dtype):
    if dtype == "bf16":
        return t.view(torch.int16).cpu().numpy().view(np.uint16)
    return t.cpu().numpy().view(np.uint32)


def _inputs(dtype, p, n, seed):
    if dtype == "i32":
        return O.random_inputs(p, n, seed, "i32")
    x = O.random_inputs(p, n, seed, "f32")
    return O.bf16_bits_from_f32(x) if dtype == "bf16" else x


def _want(x, nodes, gpus, dtype):
    w = O.nvrar_order_sum(x, nodes, gpus, dtype)
    return w if dtype == "bf16" else w.view(np.uint32)


def parity(comm, rank, nodes, gpus, device, algos, dtypes, sizes, log):
    """Every (schedule, dtype, size) against the oracle's bits."""
    fails = 0
    world = nodes * gpus
    for algo in algos:
        comm.set_algo(algo)
        for dtype in dtypes:
            for n in sizes:
                x = _inputs(dtype, world, n, 5000 + n)
                inp = _dev(x[rank], dtype, device)
                out = torch.empty_like(inp)
                comm.allreduce(inp, out)
                torch.cuda.synchronize(device)
                comm.check()
                bad = int(np.count_nonzero(_host(out, dtype) != _want(x, nodes, gpus, dtype)))
                if bad:
                    fails += 1
                    log(f"{algo} {dtype} n={n}: {bad} mismatches")
    comm.set_algo("auto")
    return fails


def torch_ops(comm, rank, nodes, gpus, device, log):
    """torch.ops.nvrar.* across processes (the TP-decode caller's entry points),
    checked against the oracle: out of place, in place, fused residual, and a
    CUDA graph of the op replayed."""
    from paper_2511_09557_b200 import torch_op  # noqa: F401 (registers the ops)
    world = nodes * gpus
    cid = torch_op.register(comm)
    fails = 0
    try:
        for dtype in ("bf16", "f32"):
            n = 8192 * 3 + 5  # a decode row batch (hidden 8192) plus a ragged tail
            x = _inputs(dtype, world, n, 610)
            want = _want(x, nodes, gpus, dtype)
            y = torch.ops.nvrar.all_reduce(_dev(x[rank], dtype, device), cid)
            torch.cuda.synchronize(device)
            comm.check()
            if not np.array_equal(_host(y, dtype), want):
                fails += 1
                log(f"torch.ops.nvrar.all_reduce {dtype} differs")
            z = _dev(x[rank], dtype, device)
            torch.ops.nvrar.all_reduce_(z, cid)
            torch.cuda.synchronize(device)
            comm.check()
            if not np.array_equal(_host(z, dtype), want):
                fails += 1
                log(f"torch.ops.nvrar.all_reduce_ {dtype} differs")
            res = _inputs(dtype, world, n, 611)
            r_dev = _dev(res[rank], dtype, device)
            torch.ops.nvrar.all_reduce_residual_(_dev(x[rank], dtype, device), r_dev, cid)
            torch.cuda.synchronize(device)
            comm.check()
            if dtype == "f32":
                exp = (O.nvrar_order_sum(x, nodes, gpus, "f32") + res[rank]).view(np.uint32)
            else:
                exp = O.bf16_bits_from_f32(O.f32_from_bf16_bits(want) +
                                           O.f32_from_bf16_bits(res[rank]))
            if not np.array_equal(_host(r_dev, dtype), exp):
                fails += 1
                log(f"torch.ops.nvrar.all_reduce_residual_ {dtype} differs")
        # the op inside a captured graph, replayed: the call counter advances on the device
        x = _inputs("bf16", world, 65536, 612)
        src = _dev(x[rank], "bf16", device)
        buf = torch.empty_like(src)
        s = torch.cuda.Stream(device)
        s.wait_stream(torch.cuda.current_stream(device))
        with torch.cuda.stream(s):
            buf.copy_(src)
            torch.ops.nvrar.all_reduce_(buf, cid)  # warm-up outside capture
        torch.cuda.current_stream(device).wait_stream(s)
        torch.cuda.synchronize(device)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            buf.copy_(src)
            torch.ops.nvrar.all_reduce_(buf, cid)
        for _ in range(3):
            g.replay()
        torch.cuda.synchronize(device)
        comm.check()
        if not np.array_equal(_host(buf, "bf16"), _want(x, nodes, gpus, "bf16")):
            fails += 1
            log("graph-captured torch.ops.nvrar.all_reduce_ differs")
    finally:
        torch_op.unregister(cid)
    return fails


def host_mixed(comm, rank, nodes, gpus, log):
    """nvrar_allreduce_host with even ranks on pinned (zero-copy) and odd ranks
    on pageable (staged) memory: the window schedule must not depend on the
    memory kind (a vector longer than max_bytes -> several windows; then an
    explicit host chunk)."""
    world = nodes * gpus
    fails = 0
    for chunk in (0, 256 << 10):
        comm.set_host_chunk(chunk)
        for dtype in ("f32", "bf16"):
            n = 700001
            x = _inputs(dtype, world, n, 620)
            t = torch.from_numpy(np.ascontiguousarray(x[rank]))
            if dtype == "bf16":
                t = t.view(torch.int16).view(torch.bfloat16)
            out = torch.empty_like(t)
            if rank % 2 == 0:
                t, out = t.pin_memory(), out.pin_memory()
            comm.allreduce_host(t, out)
            torch.cuda.synchronize()
            comm.check()
            got = out.view(torch.int16).numpy().view(np.uint16) if dtype == "bf16" \
                else out.numpy().view(np.uint32)
            if not np.array_equal(got, _want(x, nodes, gpus, dtype)):
                fails += 1
                log(f"host path ({'pinned' if rank % 2 == 0 else 'pageable'}, chunk {chunk}) "
                    f"{dtype} differs")
    comm.set_host_chunk(0)
    return fails


def registered(comm, rank, nodes, gpus, device, log):
    """nvrar_allreduce_registered: inputs in a buffer registered with the comm,
    read in place by the peers. Each call's input is overwritten right after
    the call (stream order) with the next call's — correct only if no launch
    completes before every peer has read its input — and registered calls
    interleave with staged ones on the same call sequence."""
    world = nodes * gpus
    fails = 0
    cap = 70000
    bufs = {dt: comm.alloc_symmetric(cap, dt) for dt in (torch.float32, torch.bfloat16,
                                                         torch.int32)}
    names = {torch.float32: "f32", torch.bfloat16: "bf16", torch.int32: "i32"}
    for dt, buf in bufs.items():
        dtype = names[dt]
        outs, wants = [], []
        for k, n in enumerate((1, 4099, 65539, 65539)):
            x = _inputs(dtype, world, n, 630 + k)
            src = _dev(x[rank], dtype, device)
            off = 8 * k  # a different offset each call, the same on every rank
            buf[off:off + n].copy_(src)
            out = torch.empty_like(src)
            comm.allreduce_registered(buf[off:off + n], out)
            buf[off:off + n].fill_(0)  # overwrite at once: must not reach any peer
            if k == 2:
                extra = torch.empty_like(src)
                comm.allreduce(src, extra)  # a staged call in between
                outs.append(extra)
                wants.append(_want(x, nodes, gpus, dtype))
            outs.append(out)
            wants.append(_want(x, nodes, gpus, dtype))
        torch.cuda.synchronize(device)
        comm.check()
        for i, (o, w) in enumerate(zip(outs, wants)):
            if not np.array_equal(_host(o, dtype), w):
                fails += 1
                log(f"registered all-reduce {dtype} call {i} differs")
    # a peer's registered range is reachable through its mapping here
    peer = (rank + 1) % world
    if world > 1 and comm.buffer_peer_ptr(1, peer) == 0:
        fails += 1
        log("no peer mapping for registered buffer 1")
    # a connected registration is never mapped a second time
    if comm._lib.nvrar_connect_buffer(comm._h, 1, (L.Handle * world)(), world) == 0:
        fails += 1
        log("a second connect of registered buffer 1 was accepted")
    return fails


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--dir", required=True)
    ap.add_argument("--rank", type=int, required=True)
    ap.add_argument("--nodes", type=int, required=True)
    ap.add_argument("--gpus", type=int, required=True)
    ap.add_argument("--device", type=int, default=0)
    ap.add_argument("--quick", action="store_true", help="fewer sizes and dtypes")
    ap.add_argument("--ops", action="store_true", help="also the torch.ops.nvrar entry points")
    ap.add_argument("--mismatch", action="store_true", help="length-mismatch protocol fault")
    ap.add_argument("--registered", action="store_true",
                    help="all-reduce of registered (symmetric) buffers read in place")
    ap.add_argument("--host", action="store_true",
                    help="host-buffer path, pinned on even ranks and pageable on odd ranks")
    ap.add_argument("--timeout", type=float, default=60.0)
    ap.add_argument("--jitter-seeds", type=int, default=0,
                    help="repeat the parity grid under delay injection with this many seeds")
    ap.add_argument("--canary", type=int, default=0,
                    help="word-atomicity canary runs between ranks 0 (writer) and 1 (reader)")
    args = ap.parse_args()
    rank = args.rank
    world = args.nodes * args.gpus
    device = torch.device("cuda", args.device)
    torch.cuda.set_device(device)

    def log(msg):
        print(f"rank {rank}: {msg}", flush=True)

    log(f"started (pid {os.getpid()})")
    torch.zeros(1, device=device)
    log("CUDA context ready")
    topo = ClusterTopology(args.nodes, args.gpus)
    comm = B.communicator_from_dir(args.dir, topo, rank, 1 << 20, device=args.device,
                                   timeout_s=args.timeout)
    if args.mismatch:
        comm.set_algo("hier" if args.nodes > 1 else "twoshot")
        n = 1024 + (1 if rank == 0 else 0)
        x = torch.ones(n, device=device)
        comm.allreduce(x, x)
        rc = comm.check_status()
        log(f"mismatch status {rc} ({comm.last_error()})")
        B.file_barrier(args.dir, rank, world, "done")
        sys.exit(0 if rc in (L.ERR_PROTOCOL_FAULT, L.ERR_DEADLOCK) else 1)
    algos = ("hier", "twoshot", "oneshot") if args.gpus <= 8 else ("hier",)
    dtypes = ("f32", "bf16") if args.quick else ("f32", "bf16", "i32")
    sizes = (4099,) if args.quick else (1, 4099, 65539)
    fails = parity(comm, rank, args.nodes, args.gpus, device, algos, dtypes, sizes, log)
    for seed in range(args.jitter_seeds):
        comm.set_jitter(3000, seed * 7919 + rank)
        fails += parity(comm, rank, args.nodes, args.gpus, device, algos, dtypes, (4099 + seed,),
                        lambda m, s=seed: log(f"jitter seed {s}: {m}"))
        comm.set_jitter(0)
    for seed in range(args.canary):
        if rank in (0, 1) and world > 1:
            comm.canary(1 - rank, 64, writer=rank == 0, jitter_ns=1000, seed=seed)
            torn = comm.canary_result()
            if torn:
                fails += 1
                log(f"canary seed {seed}: {torn} torn cells")
    if args.registered:
        fails += registered(comm, rank, args.nodes, args.gpus, device, log)
    if args.host:
        fails += host_mixed(comm, rank, args.nodes, args.gpus, log)
    if args.ops:
        fails += torch_ops(comm, rank, args.nodes, args.gpus, device, log)
    seq = comm.sequence()
    log(f"{'OK' if fails == 0 else f'{fails} FAILURES'} (sequence {seq})")
    B.file_barrier(args.dir, rank, world, "done")
    comm.close()
    sys.exit(1 if fails else 0)


if __name__ == "__main__":
    main()
