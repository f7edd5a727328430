"""NVRAR all-reduce benchmark (driver contract).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl nvrar|reference]
                    [--no-sweep] [--no-autotune] [--no-multicast]

N=1  : BASELINE configs[0] on one B200 — 8 ranks as 2 virtual nodes x 4, 1 MB
       fp32 sum; the 8 ranks are virtual ranks on cuda:0 (one launch for all
       ranks, every buffer in one HBM — the direct schedule), the GPU analogue
       of the reference running all ranks in one process.
N>1  : launched by torch.distributed.run, one rank per GPU; hierarchy 2 x N/2
       (N=8: 2x4, configs[1]); headline message 1 MB bf16, plus the 64 KB-8 MB
       sweep against NCCL all-reduce on the same buffers (configs[1]/[2]).
       The selector is first tuned on the running box (max-over-ranks
       consensus), as the north star's measured selector.

A "step" is one CUDA-graph replay of `calls` back-to-back all-reduces over
rotating buffers whose total exceeds the 126 MB L2 (so no call reads an input
left in L2 by an earlier one). Per-step time comes from CUDA events on the
launching stream, the max over ranks is taken per step, and the per-call
latency is step / calls; `value` is the p50 over the K timed steps.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "all-reduce p50 latency (µs, max over ranks) 128KB–2MB at 2/4/8 B200 vs NCCL"
NVLINK_PEAK_GBS = 770.0     # measured B200 peer copy per direction (B200_PROFILING.md)
NVLINK_NOMINAL_GBS = 900.0  # NVLink 5 per direction per GPU
SWEEP = [64 << 10, 128 << 10, 256 << 10, 512 << 10, 1 << 20, 2 << 20, 4 << 20, 8 << 20]
PRODUCER_SIZES = (128 << 10, 512 << 10, 1 << 20, 2 << 20)


def nccl_best_table(world):
    """Per message size, the best NCCL (algorithm x protocol x library) measured on
    this pool by `rankbench nccl-best` (profiles/*nccl_best_p{world}*.jsonl)."""
    import glob
    out = {}
    for path in sorted(glob.glob(os.path.join(ROOT, "profiles", f"*nccl_best_p{world}*.jsonl")),
                       reverse=True):
        with open(path) as fh:
            for line in fh:
                if line.startswith("BEST "):
                    r = json.loads(line[5:])
                    if r.get("producer", "none") == "none":
                        out.setdefault(int(r["bytes"]), r)
        return out, os.path.basename(path)
    return out, None


def profiled_nvlink_traffic(world, algo, msg):
    """NVLink egress bytes per launch per GPU (nvltx__bytes: payload + link
    protocol) of the schedule's kernel at this size and world, from the committed
    single-pass ncu capture of rank 0 (profiles/*ncu_nvlink*.json), or None.
    Ingress equals the peers' egress (symmetric schedules)."""
    import glob
    for path in sorted(glob.glob(os.path.join(ROOT, "profiles", "*ncu_nvlink*.json")),
                       reverse=True):
        try:
            with open(path) as fh:
                p = json.load(fh)
            for r in p["rows"]:
                if r["world"] == world and r["algo"] == algo and r["bytes"] == msg:
                    return int(r["nvl_tx_bytes"]), os.path.basename(path)
        except Exception:
            continue
    return None, None


def profiled_traffic(kernel_prefix):
    """DRAM bytes (read + write) per launch of the dominant kernel from the newest
    committed ncu --set full capture of that kernel (profiles/*_metrics.json), or None."""
    import glob
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    for path in sorted(glob.glob(os.path.join(ROOT, "profiles", "*ncu*_metrics.json")),
                       reverse=True):
        try:
            with open(path) as fh:
                p = json.load(fh)
            if not p["kernel"].startswith(kernel_prefix):
                continue
            tot = 0.0
            for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
                m = p["metrics"][k]
                tot += float(m["value"]) * scale.get(m["unit"], 1)
            return int(tot), os.path.basename(path)
        except Exception:
            continue
    return None, None


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            p = json.load(fh)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


# ---- the CPU reference path (the reference's own code, compiled in oracle/_ref) -------

def cpu_reference(nodes, gpus, n, budget_s=12.0, max_calls=60):
    """ccsim::NvrarAllreduce<float> on the reference's ConcurrentEngine, pre-generated
    inputs, per-call makespan (bench.hpp:116-122 convention)."""
    from oracle import oracle as O
    x = O.random_inputs(nodes * gpus, n, 1234, "f32")
    kind = "reference" if O.ref_available() else "port"
    if kind == "port":
        # the C restatement (single thread) of the same arithmetic
        t0 = time.perf_counter()
        per = []
        while len(per) < max_calls and time.perf_counter() - t0 < budget_s:
            t = time.perf_counter()
            O.nvrar_order_sum(x, nodes, gpus)
            per.append((time.perf_counter() - t) * 1e6)
        return statistics.median(per), kind, 1, f"{len(per)} calls, {nodes}x{gpus}, n={n} fp32"
    t0 = time.perf_counter()
    per = list(O.ref_time_concurrent(x, nodes, gpus, warmup=2, calls=3))
    one = (time.perf_counter() - t0) / 5
    more = int(max(0, min(max_calls, budget_s / max(one, 1e-6)) - 5))
    if more > 0:
        per += list(O.ref_time_concurrent(x, nodes, gpus, warmup=1, calls=more))
    threads = nodes * gpus  # one std::thread per rank (concurrent_transport.hpp:59-75)
    return (statistics.median(per), kind, min(threads, os.cpu_count() or threads),
            f"{len(per)} calls of NvrarAllreduce<float> on ConcurrentEngine, {nodes}x{gpus}, "
            f"n={n} fp32, B=1, C=65536, p50 of per-call makespan (host nproc={os.cpu_count()})")


def hier_for(world):
    return {1: (2, 4), 2: (2, 1), 4: (2, 2), 8: (2, 4)}[world]


def run_reference(args, rank, world):
    if rank != 0:
        return
    nodes, gpus = hier_for(world)
    n = (1 << 20) // 4 if world == 1 else (1 << 20) // 2
    per = []
    t0 = time.perf_counter()
    for _ in range(args.warmup):
        cpu_reference(nodes, gpus, n, budget_s=2.0, max_calls=3)
    kind, cores, sample = "reference", nodes * gpus, ""
    for _ in range(args.steps):
        v, kind, cores, sample = cpu_reference(nodes, gpus, n, budget_s=4.0, max_calls=10)
        per.append(v)
    total = time.perf_counter() - t0
    val = statistics.median(per)
    line = {
        "impl": "reference", "metric": METRIC, "value": round(val, 3), "unit": "us",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(total * 1e3 / max(1, args.steps + args.warmup), 3),
        "higher_is_better": False, "scaling": "weak", "vs_baseline": None,
        "dtype": "f32", "data": "synthetic (oracles::random_inputs, seed 1234)",
        "config": {"workload": f"reference CPU NVRAR all-reduce, {nodes}x{gpus} ranks as threads, "
                               f"{n} fp32 elements (the element count of the GPU arm's message)",
                   "nodes": nodes, "gpus_per_node": gpus, "elements": n},
        "cpu_baseline": {"value": round(val, 3), "unit": "us", "cores": cores, "kind": kind,
                         "sample": sample},
        "e2e": {"value": round(val, 3), "unit": "us", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---- N = 1: configs[0] with 8 virtual ranks on cuda:0 ----------------------------------

def run_emulated(args):
    import ctypes

    import numpy as np
    import torch

    from oracle import oracle as O
    from paper_2511_09557_b200 import ClusterTopology, LocalGroup, NvrarConfig
    from paper_2511_09557_b200 import _lib as L
    from paper_2511_09557_b200 import harness as H

    nodes, gpus = 2, 4
    P = nodes * gpus
    msg = 1 << 20
    n = msg // 4
    calls = H.calls_for(msg, P)
    g = LocalGroup(ClusterTopology(nodes, gpus), 8 << 20, device=0, timeout_s=30.0)
    x = O.random_inputs(P, n, 1234, "f32")
    base_in = [torch.from_numpy(x[r]).cuda() for r in range(P)]
    sets = [([t.clone() for t in base_in], [torch.empty_like(t) for t in base_in])
            for _ in range(calls)]
    stream = torch.cuda.Stream()

    def graph_for():
        return H.graph_of(lambda i: g.launch(*sets[i], stream=torch.cuda.current_stream()),
                          calls, stream)

    g.set_algo("auto")
    algo, blocks = g.plan(n, torch.float32)
    graph = graph_for()
    hbm, hbm_kind = peaks()
    with H.ClockSampler(0) as clk:
        times = H.time_replays(graph.replay, args.steps, args.warmup, lambda: None, stream)
    g.check()
    want = O.nvrar_order_sum(x, nodes, gpus).view(np.uint32)
    for r in range(P):
        assert np.array_equal(sets[-1][1][r].cpu().numpy().view(np.uint32), want), "parity"
    per_call_us = sorted(t * 1e3 / calls for t in times)
    p50 = statistics.median(per_call_us)
    # roofline: every rank's input read + output written once from HBM (2*P*M)
    alg_bytes = 2 * P * msg
    achieved = alg_bytes / (p50 * 1e-6) / 1e9

    # e2e through the public host-buffer API (the reference's own call shape:
    # host spans in and out): nvrar_allreduce_local_host moves the 8 pinned host
    # inputs in, all-reduces and moves the 8 outputs back, chunk-pipelined, every
    # step; the bits must still equal one all-reduce of the whole vector.
    # The headline goes through the C ABI (include/nvrar.h) with the span
    # pointers held by the caller, as the reference's C++ caller holds its spans;
    # the Python wrapper (LocalGroup.launch_host: per-call tensor checks) is
    # timed beside it.
    host_in = [torch.from_numpy(x[r]).pin_memory() for r in range(P)]
    host_out = [torch.empty(n, dtype=torch.float32).pin_memory() for _ in range(P)]
    c_send = (ctypes.c_void_p * P)(*[t.data_ptr() for t in host_in])
    c_recv = (ctypes.c_void_p * P)(*[t.data_ptr() for t in host_out])
    s_ptr = stream.cuda_stream

    def cabi_call():
        rc = g._lib.nvrar_allreduce_local_host(g._arr, P, c_send, c_recv, n, L.FLOAT32, L.SUM,
                                               s_ptr)
        if rc:
            raise RuntimeError(f"nvrar_allreduce_local_host: {g.comms[0].last_error()}")

    def e2e_of(call):
        out = []
        for t in host_out:
            t.zero_()
        for k in range(args.warmup + args.steps):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            with torch.cuda.stream(stream):
                a.record(stream)
                call()
                b.record(stream)
            b.synchronize()
            if k >= args.warmup:
                out.append(a.elapsed_time(b) * 1e3)
        g.check()
        for r in range(P):
            assert np.array_equal(host_out[r].numpy().view(np.uint32), want), "e2e parity"
        return out

    e2e = e2e_of(cabi_call)
    e2e_py = e2e_of(lambda: g.launch_host(host_in, host_out, stream=stream))

    # each schedule forced (context; after the headline so an ncu launch list of
    # this command starts with the headline's launches)
    by_algo = {}
    for forced in ("hier", "twoshot", "oneshot", "direct"):
        g.set_algo(forced)
        gr = graph_for()
        ts = H.time_replays(gr.replay, max(3, args.steps // 2), 2, lambda: None, stream)
        by_algo[forced] = round(statistics.median(ts) * 1e3 / calls, 3)
        del gr
    g.set_algo("auto")

    sweep = {}
    if not args.no_sweep:
        for size in (128 << 10, 512 << 10, 2 << 20):
            ne = size // 2
            c2 = H.calls_for(size, P)
            xs = [torch.randn(ne, device="cuda").to(torch.bfloat16) for _ in range(P)]
            st = [([t.clone() for t in xs], [torch.empty_like(t) for t in xs]) for _ in range(c2)]
            gr = H.graph_of(lambda i: g.launch(*st[i], stream=torch.cuda.current_stream()),
                            c2, stream)
            ts = H.time_replays(gr.replay, max(5, args.steps // 2), 2, lambda: None, stream)
            sweep[f"{size >> 10}KB_bf16"] = {"p50_us": round(statistics.median(ts) * 1e3 / c2, 3),
                                             "algo": g.plan(ne, torch.bfloat16)[0]}
            del gr, st
    g.check()

    cpu_v, cpu_kind, cpu_cores, cpu_sample = cpu_reference(nodes, gpus, n)
    kname = {"hier": "hier", "twoshot": "flat", "oneshot": "flat", "direct": "direct"}[algo]
    traffic, traffic_src = profiled_traffic(f"nvrar::{kname}_kernel")
    line = {
        "metric": METRIC, "value": round(p50, 3), "unit": "us", "n_gpus": 1,
        "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(statistics.mean(times), 4), "higher_is_better": False,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (oracles::random_inputs, seed 1234); output checked bit-exact vs oracle",
        "config": {"workload": "configs[0]: 2x4 virtual nodes (8 ranks as virtual ranks on one "
                               "B200, one launch per all-reduce), 1 MB fp32 sum",
                   "nodes": nodes, "gpus_per_node": gpus, "message_bytes": msg, "algo": algo,
                   "blocks_per_rank": blocks, "calls_per_step": calls,
                   "per_schedule_us": by_algo,
                   "l2": f"rotating buffers, {calls} x 16 MB per step > 126 MB L2",
                   "p10_us": round(per_call_us[len(per_call_us) // 10], 3),
                   "p90_us": round(per_call_us[(9 * len(per_call_us)) // 10], 3)},
        "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": hbm,
                     "peak_kind": hbm_kind, "unit": "GB/s", "frac": round(achieved / hbm, 4),
                     "traffic": traffic, "traffic_source": traffic_src,
                     "algorithmic_bytes": alg_bytes,
                     "note": "virtual ranks share one HBM: 2*P*M bytes (all inputs read, all "
                             "outputs written) per launch; traffic = DRAM read + write bytes per "
                             "launch of the chosen schedule's kernel in steady state (committed "
                             "ncu capture over rotating buffers without cache flushes, so the "
                             "write-back of earlier outputs is counted)"},
        "cpu_baseline": {"value": round(cpu_v, 3), "unit": "us", "cores": cpu_cores,
                         "kind": cpu_kind, "sample": cpu_sample},
        "e2e": {"value": round(statistics.median(e2e), 3), "unit": "us",
                "h2d_bytes_per_step": P * msg, "d2h_bytes_per_step": P * msg,
                "path": "nvrar_allreduce_local_host through the C ABI (pinned host buffers, "
                        "zero-copy)",
                "python_api_us": round(statistics.median(e2e_py), 3)},
        "gpu_launches": (args.steps + args.warmup) * calls,
        "clocks": clk.summary(),
        "sweep": sweep,
    }
    print(json.dumps(line), flush=True)
    g.close()


# ---- N > 1: one rank per GPU over NVLink ----------------------------------------------

def run_multi(args, rank, world, local):
    import torch
    import torch.distributed as dist

    from paper_2511_09557_b200 import ClusterTopology, Communicator
    from paper_2511_09557_b200 import dist as D
    from paper_2511_09557_b200 import harness as H
    from paper_2511_09557_b200 import selector as S

    torch.cuda.set_device(local)
    os.environ.setdefault("NCCL_DEBUG", "WARN")
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    nodes, gpus = hier_for(world)
    comm = Communicator.from_process_group(ClusterTopology(nodes, gpus), 8 << 20, device=local,
                                           timeout_s=30.0)
    stream = torch.cuda.Stream()
    barrier = lambda: dist.barrier(device_ids=[local])  # noqa: E731
    dev = torch.device("cuda", local)

    alpha = H.alpha_signal_us(comm, rank, world)
    # NVLS multicast one-shot as a selector candidate (collective setup; any
    # rank failing disables it everywhere)
    mc_ok = False if args.no_multicast else comm.enable_multicast()
    tuned = None
    if not args.no_autotune:
        tuned = S.autotune(comm, sizes=SWEEP, dtype=torch.bfloat16, calls=30, reps=5)

    # ncclAllReduce called directly (torch's libnccl, default algorithm and
    # protocol), captured in the same graphs as NVRAR; torch.distributed's
    # all_reduce is kept as the framework-level reference
    from paper_2511_09557_b200 import nccl_ref
    ncc, nccl_version = None, None
    try:
        ncc = nccl_ref.Nccl(nccl_ref.lib_path("torch"))
        uid = [ncc.unique_id() if rank == 0 else None]
    except Exception:  # noqa: BLE001 — no loadable libnccl: torch.distributed's arm only
        ncc, uid = None, [None]
    dist.broadcast_object_list(uid, src=0)
    ok = D.max_over_ranks([0.0 if (ncc is not None and uid[0] is not None) else 1.0],
                          device=torch.device("cuda", local))[0] == 0.0
    if ok:
        ncc.init_rank(world, uid[0], rank)
        nccl_version = ncc.version()
    else:
        ncc = None

    def measure(msg, impl, steps, warmup, producer=False):
        """p50-sorted per-call µs (max over ranks). producer: a cuBLAS GEMM writes
        each call's input first (the decode layer's projection): no PDL chaining
        to the previous all-reduce, L2-hot input; the per-call all-reduce cost is
        (step - GEMM-only step) / calls, the same subtraction for every arm."""
        ne = msg // 2
        calls = H.calls_for(msg, 1)
        torch.manual_seed(1234 + rank)
        src = torch.randn(ne, device="cuda").to(torch.bfloat16)
        bufs = [(src.clone(), torch.empty_like(src)) for _ in range(calls)]
        if impl == "nvrar":
            plan = D.plan_consensus(comm.plan(ne, torch.bfloat16))
            fn = lambda i: comm.allreduce(bufs[i][0], bufs[i][1])  # noqa: E731
        elif impl == "nccl" and ncc is not None:
            plan = ("nccl-direct", 0)
            fn = lambda i: ncc.all_reduce(bufs[i][0], bufs[i][1])  # noqa: E731
        else:
            impl = "torch"
            plan = ("torch.distributed", 0)
            fn = lambda i: dist.all_reduce(bufs[i][1])  # noqa: E731
            for a, b in bufs:
                b.copy_(a)
        base = 0.0
        if producer:
            rows, k = max(1, ne // 8192), 1024
            xs = [torch.randn(rows, k, device="cuda").to(torch.bfloat16) for _ in range(4)]
            w = (torch.randn(k, ne // rows, device="cuda") * k ** -0.5).to(torch.bfloat16)
            dst = 1 if impl == "torch" else 0

            def prod(i):
                torch.matmul(xs[i % 4], w, out=bufs[i][dst].view(rows, ne // rows))
            g0 = H.graph_of(prod, calls, stream)
            t0 = D.max_over_ranks(H.time_replays(g0.replay, steps, warmup, barrier, stream),
                                  device=dev)
            base = statistics.median(t0)
            del g0
            inner = fn
            fn = lambda i: (prod(i), inner(i))  # noqa: E731
        gr = H.graph_of(fn, calls, stream)
        ts = H.time_replays(gr.replay, steps, warmup, barrier, stream)
        ts = D.max_over_ranks(ts, device=dev)
        if impl == "nvrar":
            comm.check()
        del gr
        return sorted((t - base) * 1e3 / calls for t in ts), calls, plan

    hbm, _ = peaks()
    nccl_best, nccl_best_src = nccl_best_table(world)
    msg = 1 << 20
    with H.ClockSampler(local) as clk:
        per, calls, plan = measure(msg, "nvrar", args.steps, args.warmup)
    p50 = statistics.median(per)
    nccl_per, _, _ = measure(msg, "nccl", args.steps, args.warmup)
    nccl50 = statistics.median(nccl_per)
    torch_per, _, _ = measure(msg, "torch", args.steps, args.warmup)
    torch50 = statistics.median(torch_per)

    # e2e: pinned host input -> device, all-reduce, device -> host, per step; max over ranks
    ne = msg // 2
    host_in = torch.randn(ne).to(torch.bfloat16).pin_memory()
    host_out = torch.empty(ne, dtype=torch.bfloat16).pin_memory()
    e2e = []
    for k in range(args.warmup + args.steps):
        barrier()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(stream):
            a.record(stream)
            # nvrar_allreduce_host: H2D, all-reduce and D2H chunk-pipelined
            comm.allreduce_host(host_in, host_out, stream=stream)
            b.record(stream)
        b.synchronize()
        if k >= args.warmup:
            e2e.append(a.elapsed_time(b) * 1e3)
    e2e = D.max_over_ranks(e2e, device=dev)
    comm.check()

    def roof_us(size):
        b_alg = 2 * (world - 1) / world * size
        bw = b_alg / (NVLINK_NOMINAL_GBS * 1e9) * 1e6
        lat = math.log2(world) * alpha if alpha else 0.0
        return max(bw, lat), b_alg

    sweep = {}
    if not args.no_sweep:
        for size in SWEEP:
            s_steps = max(5, args.steps // 2)
            v_per, _, pl = measure(size, "nvrar", s_steps, 2)
            n_per, _, _ = measure(size, "nccl", s_steps, 2)
            v, nv = statistics.median(v_per), statistics.median(n_per)
            rt, b_alg = roof_us(size)
            row = {"nvrar_us": round(v, 3), "nccl_us": round(nv, 3), "algo": pl[0],
                   "blocks": pl[1], "speedup_vs_nccl": round(nv / v, 3),
                   "busbw_GBs": round(b_alg / (v * 1e-6) / 1e9, 1),
                   "roofline_us": round(rt, 3), "roofline_frac": round(rt / v, 3)}
            best = nccl_best.get(size)
            if best:
                row.update(nccl_best_us=best["nccl_best_us"],
                           nccl_best_cfg=f"{best['algo']}/{best['proto']} {best['version']}",
                           speedup_vs_nccl_best=round(best["nccl_best_us"] / v, 3))
            if not args.no_producer and size in PRODUCER_SIZES:
                vp = statistics.median(measure(size, "nvrar", s_steps, 2, producer=True)[0])
                npp = statistics.median(measure(size, "nccl", s_steps, 2, producer=True)[0])
                row.update(nvrar_after_gemm_us=round(vp, 3), nccl_after_gemm_us=round(npp, 3),
                           speedup_after_gemm=round(npp / vp, 3))
            if tuned is not None:
                cands = tuned["measured"][size]
                for a_name in ("hier", "twoshot", "oneshot", "mcast"):
                    vals = [t for k, t in cands.items() if k.startswith(a_name + "/")]
                    if vals:
                        row[f"{a_name}_best_us"] = min(vals)
            sweep[f"{size >> 10}KB"] = row

    rt, b_alg = roof_us(msg)
    busbw = b_alg / (p50 * 1e-6) / 1e9
    # the reference's CPU path on this host, same hierarchy, the message's
    # element count (the reference has fp32 / int32 only), rank 0 only
    cpu = cpu_reference(nodes, gpus, msg // 2, budget_s=10.0, max_calls=30) if rank == 0 else None
    traffic, traffic_src = profiled_nvlink_traffic(world, plan[0], msg)
    if ncc is not None:
        ncc.close()
    if rank == 0:
        line = {
            "metric": METRIC, "value": round(p50, 3), "unit": "us", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(statistics.mean(per) * calls / 1e3, 4),
            "higher_is_better": False, "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic (torch.randn, seed 1234+rank)",
            "config": {"workload": f"NVRAR bf16 sum, {world} B200 as {nodes}x{gpus} virtual "
                                   f"nodes, 1 MB message (configs[1] sweep point)",
                       "nodes": nodes, "gpus_per_node": gpus, "message_bytes": msg,
                       "algo": plan[0], "blocks_per_rank": plan[1], "calls_per_step": calls,
                       "selector": "autotuned on this box" if tuned else "built-in policy",
                       "multicast": mc_ok,
                       "selector_rows": tuned["rows"] if tuned else None,
                       # alpha-beta model fitted to this run
                       "alpha_beta": dict(S.fit_schedules(tuned["measured"]) if tuned else {},
                                          nccl=dict(zip(("alpha_us", "beta_GBs"), [
                                              round(v, 3) for v in S.fit_alpha_beta(
                                                  {int(k[:-2]) << 10: r["nccl_us"]
                                                   for k, r in sweep.items()})])) if sweep
                                          else None),
                       "l2": f"rotating buffers, {calls} x 2 MB per step > 126 MB L2",
                       "p10_us": round(per[len(per) // 10], 3),
                       "p90_us": round(per[(9 * len(per)) // 10], 3),
                       "nccl_p50_us": round(nccl50, 3),
                       "nccl": (f"ncclAllReduce direct (libnccl {nccl_version}, default "
                                f"algorithm/protocol), same graph methodology" if ncc is not None
                                else "torch.distributed.all_reduce (direct libnccl unavailable)"),
                       "speedup_vs_nccl": round(nccl50 / p50, 3),
                       "torch_distributed_p50_us": round(torch50, 3),
                       "nccl_best": nccl_best.get(msg),
                       "nccl_best_source": nccl_best_src,
                       "alpha_signal_us": round(alpha, 3) if alpha else None},
            "roofline": {"bound": "nvlink", "achieved": round(busbw, 1),
                         "peak": NVLINK_PEAK_GBS, "unit": "GB/s",
                         "frac": round(busbw / NVLINK_PEAK_GBS, 4), "traffic": traffic,
                         "traffic_source": traffic_src,
                         "traffic_note": "NVLink egress bytes per launch per GPU (ncu nvltx__bytes, "
                                         "payload + link protocol) vs algorithmic_bytes",
                         "algorithmic_bytes": b_alg,
                         "roofline_us": round(rt, 3), "time_frac": round(rt / p50, 4),
                         "note": "achieved = busbw 2(P-1)/P*M/t vs measured 770 GB/s peer copy; "
                                 "roofline_us = max(B_alg/900 GB/s, log2(P)*alpha_signal)"},
            "cpu_baseline": {"value": round(cpu[0], 3), "unit": "us", "cores": cpu[2],
                             "kind": cpu[1], "sample": cpu[3]},
            "e2e": {"value": round(statistics.median(e2e), 3), "unit": "us",
                    "h2d_bytes_per_step": msg, "d2h_bytes_per_step": msg,
                    "path": "nvrar_allreduce_host (pinned host buffers, zero-copy)"},
            "gpu_launches": (args.steps + args.warmup) * calls,
            "clocks": clk.summary(),
            "sweep": sweep,
        }
        print(json.dumps(line), flush=True)
    barrier()
    comm.close()
    dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["nvrar", "reference"], default="nvrar")
    ap.add_argument("--no-sweep", action="store_true")
    ap.add_argument("--no-autotune", action="store_true")
    ap.add_argument("--no-multicast", action="store_true",
                    help="do not set up the NVLS multicast one-shot candidate")
    ap.add_argument("--no-producer", action="store_true",
                    help="skip the GEMM-producer rows (all-reduce after a non-PDL kernel)")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    if world == 1:
        run_emulated(args)
    else:
        run_multi(args, rank, world, local)


if __name__ == "__main__":
    main()
