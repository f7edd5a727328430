"""A small, complete workload for compute-sanitizer (memcheck / racecheck /
synccheck): every schedule, dtype and phase entry point on virtual ranks of
one GPU at small sizes, results checked against the oracle. Run as

    compute-sanitizer --tool memcheck python tests/sanitize_emu.py

(the kernels' device watchdog is raised so the sanitizer's slowdown cannot
trip it)."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import oracle as O  # noqa: E402
from paper_2511_09557_b200 import ClusterTopology, LocalGroup, NvrarConfig  # noqa: E402


def main():
    bad = 0
    for nodes, gpus in ((2, 2), (2, 1), (1, 3)):
        P = nodes * gpus
        g = LocalGroup(ClusterTopology(nodes, gpus), 1 << 16, device=0, timeout_s=300.0)
        for algo in ("hier", "twoshot", "oneshot", "direct"):
            g.set_algo(algo)
            g.set_config(NvrarConfig(2, 65536))
            for dtype in ("f32", "bf16", "i32"):
                for n in (1, 37, 1031):
                    x = O.random_inputs(P, n, 77 + n, "i32" if dtype == "i32" else "f32")
                    if dtype == "bf16":
                        x = O.bf16_bits_from_f32(x)
                    want = O.nvrar_order_sum(x, nodes, gpus, dtype)
                    ins = [torch.from_numpy(np.ascontiguousarray(x[r])) for r in range(P)]
                    if dtype == "bf16":
                        ins = [t.view(torch.int16).view(torch.bfloat16) for t in ins]
                    ins = [t.cuda() for t in ins]
                    outs = [torch.empty_like(t) for t in ins]
                    g.run_all(ins, outs)
                    for r in range(P):
                        got = outs[r].cpu()
                        got = got.view(torch.int16).numpy().view(np.uint16) if dtype == "bf16" \
                            else got.numpy().view(np.uint32)
                        exp = want if dtype == "bf16" else want.view(np.uint32)
                        if not np.array_equal(got, exp):
                            bad += 1
                            print(f"{nodes}x{gpus} {algo} {dtype} n={n}: rank {r} differs")
        # phase entry points
        if gpus > 1:
            n = 1031
            x = O.random_inputs(P, n, 5, "f32")
            ins = [torch.from_numpy(x[r]).cuda() for r in range(P)]
            sh = [torch.empty(-(-n // gpus), device="cuda") for _ in range(P)]
            g.run_phase("reduce_scatter", ins, sh)
            full = [torch.empty(sh[0].numel() * gpus, device="cuda") for _ in range(P)]
            g.run_phase("all_gather", sh, full)
        g.close()
    print("sanitize workload:", "OK" if bad == 0 else f"{bad} FAILURES", flush=True)
    return 1 if bad else 0


if __name__ == "__main__":
    sys.exit(main())
