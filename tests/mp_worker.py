"""Multi-process, multi-GPU parity worker (one rank per GPU), launched by
tests/test_multigpu.py through torch.distributed.run. Every rank regenerates
all ranks' inputs with the oracle's generator, runs the CUDA all-reduce over
NVLink (IPC-mapped peer regions), and checks its output against the oracle.

    python -m torch.distributed.run --nproc-per-node 4 --master-addr 127.0.0.1 \
        tests/mp_worker.py --nodes 2 --gpus 2
"""
import argparse
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import oracle as O  # noqa: E402
from paper_2511_09557_b200 import ClusterTopology, Communicator, NvrarConfig  # noqa: E402
from paper_2511_09557_b200 import _lib as L  # noqa: E402
from paper_2511_09557_b200 import dist as D  # noqa: E402


def to_dev(a, dtype):
    t = torch.from_numpy(np.ascontiguousarray(a))
    if dtype == "bf16":
        t = t.view(torch.int16).view(torch.bfloat16)
    return t.cuda()


def from_dev(t, dtype):
    if dtype == "bf16":
        return t.view(torch.int16).cpu().numpy().view(np.uint16)
    return t.cpu().numpy()


def inputs(dtype, p, n, seed):
    if dtype == "i32":
        return O.random_inputs(p, n, seed, "i32")
    x = O.random_inputs(p, n, seed, "f32")
    return O.bf16_bits_from_f32(x) if dtype == "bf16" else x


def parity_loop(comm, args, rank, world, sizes):
    """Every schedule x dtype against the oracle's bits; returns the failures."""
    fails = 0
    for dtype in ("f32", "bf16", "i32"):
        for algo in ("hier", "twoshot", "oneshot"):
            comm.set_algo(algo)
            for n in sizes:
                x = inputs(dtype, world, n, 1000 + n)
                want = O.nvrar_order_sum(x, args.nodes, args.gpus,
                                         {"f32": "f32", "bf16": "bf16", "i32": "i32"}[dtype])
                inp = to_dev(x[rank], dtype)
                out = torch.empty_like(inp)
                plan = D.plan_consensus(comm.plan(n, inp.dtype))
                comm.allreduce(inp, out)
                torch.cuda.synchronize()
                comm.check()
                got = from_dev(out, dtype)
                if dtype == "f32":
                    got, want = got.view(np.uint32), want.view(np.uint32)
                bad = int(np.count_nonzero(got != want))
                if bad:
                    fails += 1
                    print(f"rank {rank}: {dtype} {algo} {plan} n={n}: {bad} mismatches", flush=True)
    comm.set_algo("auto")
    return fails


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--nodes", type=int, required=True)
    ap.add_argument("--gpus", type=int, required=True)
    ap.add_argument("--mismatch", action="store_true", help="length-mismatch protocol fault")
    ap.add_argument("--multicast", action="store_true", help="also test the NVLS one-shot")
    ap.add_argument("--dev-mod", type=int, default=0, help="device = LOCAL_RANK %% dev_mod")
    ap.add_argument("--quick", action="store_true", help="only the schedule x dtype parity loop")
    ap.add_argument("--ag-mismatch", action="store_true",
                    help="all-gather shard-length mismatch (collectives_test.cpp:226-237)")
    args = ap.parse_args()
    local = int(os.environ["LOCAL_RANK"])
    if args.dev_mod:
        # more ranks than GPUs (e.g. the 8-rank layout on 4 GPUs): two processes
        # share a device and progress by time-slicing — a slow but complete run
        # of the P=8 kernel instantiations
        local = local % args.dev_mod
    torch.cuda.set_device(local)
    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    topo = ClusterTopology(args.nodes, args.gpus)
    assert topo.world_size() == world
    comm = Communicator.from_process_group(topo, 4 << 20, device=local, timeout_s=20.0)
    fails = 0
    if args.mismatch:
        comm.set_algo("hier" if args.nodes > 1 else "twoshot")
        n = 1024 + (1 if rank == 0 else 0)
        x = torch.ones(n, device="cuda")
        comm.allreduce(x, x)
        rc = comm.check_status()
        ok = rc in (L.ERR_PROTOCOL_FAULT, L.ERR_DEADLOCK)
        print(f"rank {rank}: mismatch status {rc} ({comm.last_error()})", flush=True)
        dist.barrier()
        sys.exit(0 if ok else 1)

    if args.ag_mismatch:
        shard = torch.ones(4 if rank == 0 else 3, dtype=torch.int32, device="cuda")
        out = torch.empty(shard.numel() * args.gpus, dtype=torch.int32, device="cuda")
        comm.all_gather(shard, out)
        rc = comm.check_status()
        print(f"rank {rank}: ag mismatch status {rc} ({comm.last_error()})", flush=True)
        dist.barrier()
        sys.exit(0 if rc == L.ERR_PROTOCOL_FAULT else 1)

    if args.quick:
        fails += parity_loop(comm, args, rank, world, (1031, 65539))
        print(f"rank {rank}: {'OK' if fails == 0 else f'{fails} FAILURES'}", flush=True)
        dist.barrier()
        comm.close()
        dist.destroy_process_group()
        sys.exit(1 if fails else 0)

    # the phase-only entry points across processes (nvrar.h phase section)
    G = args.gpus
    node = rank // G
    for dtype in ("f32", "i32"):
        n = 4099
        x = inputs(dtype, world, n, 900)
        tdt = torch.float32 if dtype == "f32" else torch.int32
        shard = torch.empty(-(-n // G), dtype=tdt, device="cuda")
        comm.reduce_scatter(to_dev(x[rank], dtype), shard)
        full = torch.empty(shard.numel() * G, dtype=tdt, device="cuda")
        comm.all_gather(shard, full)
        torch.cuda.synchronize()
        comm.check()
        want = O.intra_rs_sum(x[node * G:(node + 1) * G])
        if not np.array_equal(full.cpu().numpy().view(np.uint32), want.view(np.uint32)):
            fails += 1
            print(f"rank {rank}: {dtype} reduce-scatter + all-gather differ", flush=True)
        w = 777
        sh = inputs(dtype, world, w, 901)
        call = comm.sequence() + 1
        packed = torch.from_numpy(O.pack_fused(sh[rank], call).view(np.int64)).cuda()
        red = torch.empty_like(packed)
        comm.rd_inter(packed, red, dtype=tdt)
        torch.cuda.synchronize()
        comm.check()
        got = O.unpack_fused(red.cpu().numpy().view(np.uint64), call,
                             np.float32 if dtype == "f32" else np.int32)
        if not np.array_equal(got.view(np.uint32),
                              O.rd_inter(sh, args.nodes, G)[rank].view(np.uint32)):
            fails += 1
            print(f"rank {rank}: {dtype} rd_inter differs", flush=True)

    # host buffers, pipelined in windows of the whole vector (bits = one call)
    for dtype in ("f32", "bf16"):
        n = 3 * 65536 + 1001
        x = inputs(dtype, world, n, 980)
        if dtype == "bf16":
            hin = torch.from_numpy(x[rank]).view(torch.int16).view(torch.bfloat16).pin_memory()
        else:
            hin = torch.from_numpy(np.ascontiguousarray(x[rank])).pin_memory()
        hout = torch.empty_like(hin).pin_memory()
        comm.set_host_chunk(256 << 10)  # several windows per vector
        comm.allreduce_host(hin, hout)
        comm.set_host_chunk(0)
        hout2 = torch.empty_like(hin).pin_memory()
        comm.allreduce_host(hin, hout2)  # zero-copy: the kernels use the pinned buffers
        torch.cuda.synchronize()
        comm.check()
        if not torch.equal(hout.view(torch.int16) if dtype == "bf16" else hout,
                           hout2.view(torch.int16) if dtype == "bf16" else hout2):
            fails += 1
            print(f"rank {rank}: zero-copy host path {dtype} differs", flush=True)
        torch.cuda.synchronize()
        comm.check()
        want = O.nvrar_order_sum(x, args.nodes, args.gpus, dtype)
        got = hout.view(torch.int16).numpy().view(np.uint16) if dtype == "bf16" else hout.numpy()
        if dtype == "f32":
            got, want = got.view(np.uint32), want.view(np.uint32)
        if not np.array_equal(got, want):
            fails += 1
            print(f"rank {rank}: host pipeline {dtype} differs", flush=True)

    # fused residual epilogue: out = residual + all_reduce(x), in place
    for dtype in ("f32", "bf16"):
        n = 65539
        x = inputs(dtype, world, n, 960)
        res = inputs(dtype, world, n, 961)
        r_dev = to_dev(res[rank], dtype)
        comm.allreduce_residual(to_dev(x[rank], dtype), r_dev)
        torch.cuda.synchronize()
        comm.check()
        want = O.nvrar_order_sum(x, args.nodes, args.gpus, dtype)
        if dtype == "f32":
            exp = (want + res[rank]).view(np.uint32)
            got = from_dev(r_dev, dtype).view(np.uint32)
        else:
            exp = O.bf16_bits_from_f32(O.f32_from_bf16_bits(want) + O.f32_from_bf16_bits(res[rank]))
            got = from_dev(r_dev, dtype)
        if not np.array_equal(got, exp):
            fails += 1
            print(f"rank {rank}: fused residual {dtype} differs", flush=True)

    # the reference's baseline collectives' orders (ring.hpp / tree.hpp)
    for order in ("ring", "tree"):
        if order == "ring" and world > 8:
            continue
        for dtype in ("f32", "bf16"):
            n = 65539
            x = inputs(dtype, world, n, 950)
            inp = to_dev(x[rank], dtype)
            out = torch.empty_like(inp)
            getattr(comm, f"{order}_allreduce")(inp, out)
            torch.cuda.synchronize()
            comm.check()
            want = O.order_sum(x, args.nodes, args.gpus, order, dtype)
            got = from_dev(out, dtype)
            if dtype == "f32":
                got, want = got.view(np.uint32), want.view(np.uint32)
            if not np.array_equal(got, want):
                fails += 1
                print(f"rank {rank}: {order} {dtype} differs", flush=True)

    # NVLS multicast one-shot: same bits as every other schedule
    if args.multicast:
        mc = comm.enable_multicast()
        print(f"rank {rank}: multicast ready={mc} {getattr(comm, 'mc_error', '')}", flush=True)
        if mc:
            comm.set_algo("mcast")
            for dtype in ("f32", "bf16", "i32"):
                for n in (1, 1031, 65539, 262144):
                    x = inputs(dtype, world, n, 970 + n)
                    if dtype == "f32" and n > 1:
                        x.view(np.uint32)[1, 1] = 0xFFFFFFFF  # the Lamport empty pattern as data
                    want = O.nvrar_order_sum(x, args.nodes, args.gpus, dtype)
                    inp = to_dev(x[rank], dtype)
                    out = torch.empty_like(inp)
                    for _ in range(3):  # both parities
                        comm.allreduce(inp, out)
                    torch.cuda.synchronize()
                    comm.check()
                    got = from_dev(out, dtype)
                    if dtype == "f32":
                        ok = np.array_equal(np.isnan(got), np.isnan(want)) and np.array_equal(
                            got[~np.isnan(got)].view(np.uint32), want[~np.isnan(want)].view(np.uint32))
                    else:
                        ok = np.array_equal(got, want)
                    if not ok:
                        fails += 1
                        print(f"rank {rank}: mcast {dtype} n={n} differs", flush=True)
            comm.set_algo("auto")
        elif world > 1:
            fails += 1

    fails += parity_loop(comm, args, rank, world, (1, 1031, 65539, 262144))
    # back-to-back calls captured in a CUDA graph, replayed (seq lives on the device)
    comm.set_algo("auto")
    comm.set_config(NvrarConfig())
    n = 1 << 19
    xs = [inputs("bf16", world, n, 7000 + c) for c in range(4)]
    ins = [to_dev(x[rank], "bf16") for x in xs]
    outs = [torch.empty_like(t) for t in ins]
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        for c in range(4):  # warm-up outside capture
            comm.allreduce(ins[c], outs[c], stream=s)
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    seq0 = comm.sequence()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph):
        for c in range(4):
            comm.allreduce(ins[c], outs[c])
    for _ in range(25):
        for o in outs:
            o.zero_()
        graph.replay()
    torch.cuda.synchronize()
    comm.check()
    seq1 = comm.sequence()
    if seq1 - seq0 != 100:
        fails += 1
        print(f"rank {rank}: sequence advanced by {seq1 - seq0}, expected 100", flush=True)
    for c in range(4):
        want = O.nvrar_order_sum(xs[c], args.nodes, args.gpus, "bf16")
        if not np.array_equal(from_dev(outs[c], "bf16"), want):
            fails += 1
            print(f"rank {rank}: graph replay call {c} differs", flush=True)
    print(f"rank {rank}: {'OK' if fails == 0 else f'{fails} FAILURES'}", flush=True)
    dist.barrier()
    comm.close()
    dist.destroy_process_group()
    sys.exit(1 if fails else 0)


if __name__ == "__main__":
    main()
