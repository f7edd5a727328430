"""Where the N=1 e2e step's time goes (bench.py's e2e leg: 2x4 virtual ranks,
1 MB fp32 each, pinned host buffers in and out, zero-copy direct schedule):

  api     LocalGroup.launch_host, event-timed per step like bench.py
  cabi    nvrar_allreduce_local_host through ctypes with the pointer arrays
          built once (what a C++ caller holding its spans pays)
  graph   the same launch captured in a CUDA graph: the kernel alone
  cpu     host wall time of one LocalGroup.launch_host call (no sync)

    python tools/e2e_probe.py [--steps 50]
"""
from __future__ import annotations

import argparse
import ctypes
import json
import os
import statistics
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main() -> None:
    from paper_2511_09557_b200 import ClusterTopology, LocalGroup
    from paper_2511_09557_b200 import _lib as L
    from paper_2511_09557_b200.comm import _stream_ptr, dtype_code

    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=50)
    args = ap.parse_args()
    nodes, gpus = 2, 4
    P = nodes * gpus
    n = (1 << 20) // 4
    g = LocalGroup(ClusterTopology(nodes, gpus), 8 << 20, device=0, timeout_s=30.0)
    hin = [torch.randn(n).pin_memory() for _ in range(P)]
    hout = [torch.empty(n).pin_memory() for _ in range(P)]
    stream = torch.cuda.Stream()
    lib = g._lib
    send = (ctypes.c_void_p * P)(*[t.data_ptr() for t in hin])
    recv = (ctypes.c_void_p * P)(*[t.data_ptr() for t in hout])
    sp = _stream_ptr(stream)

    def cabi():
        rc = lib.nvrar_allreduce_local_host(g._arr, P, send, recv, n, dtype_code(torch.float32),
                                            L.SUM, sp)
        assert rc == 0

    def api():
        g.launch_host(hin, hout, stream=stream)

    def timed(fn):
        out = []
        for k in range(5 + args.steps):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            with torch.cuda.stream(stream):
                a.record(stream)
                fn()
                b.record(stream)
            b.synchronize()
            if k >= 5:
                out.append(a.elapsed_time(b) * 1e3)
        return statistics.median(out)

    res = {"api_us": timed(api), "cabi_us": timed(cabi)}
    cpu = []
    for k in range(5 + args.steps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        api()
        t1 = time.perf_counter()
        torch.cuda.synchronize()
        if k >= 5:
            cpu.append((t1 - t0) * 1e6)
    res["api_cpu_us"] = statistics.median(cpu)
    cpu = []
    for k in range(5 + args.steps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        cabi()
        t1 = time.perf_counter()
        torch.cuda.synchronize()
        if k >= 5:
            cpu.append((t1 - t0) * 1e6)
    res["cabi_cpu_us"] = statistics.median(cpu)
    graph = torch.cuda.CUDAGraph()
    torch.cuda.synchronize()
    with torch.cuda.graph(graph, stream=stream):
        cabi()
    res["graph_us"] = timed(graph.replay)
    g.check()
    res["upt_env"] = os.environ.get("NVRAR_HOST_UPT", "default")
    print("E2E " + json.dumps({k: (round(v, 2) if isinstance(v, float) else v)
                               for k, v in res.items()}), flush=True)


if __name__ == "__main__":
    main()
