"""Single-GPU twin of tests/mp_stress.py: the same deterministic sequence of
calls (switching schedule, CTA count, dtype, size) on virtual ranks of one GPU,
each checked against an exactly representable expected sum.

    python tests/stress_emu.py --calls 3000 --nodes 2 --gpus 2
"""
import argparse
import os
import random
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2511_09557_b200 import ClusterTopology, LocalGroup, NvrarConfig  # noqa: E402


def dump_cell(g, b, args, world, n, ys, dt):
    """Print the awaited all-gather cell (hier, Lamport, 1 cell/unit) and the peer's output."""
    import ctypes
    c = g.comms[b.global_rank]
    lay = (ctypes.c_uint64 * 8)()
    c._lib.nvrar_debug_read_region(c._h, 0, 0, None, lay)
    parity = b.expected & 1
    src_local = b.peer_rank % args.gpus
    area = {5: (lay[3], lay[4]), 4: (lay[1], lay[2])}.get(b.phase, (lay[3], lay[4]))
    off = area[0] + (parity * world + src_local) * area[1] * 8 + b.word_index * 16
    buf = (ctypes.c_uint32 * 16)()
    c._lib.nvrar_debug_read_region(c._h, off - 16, 64, buf, None)
    print(f"  rank {b.global_rank} phase {b.phase} cta {b.cta}: cells around unit {b.word_index}: "
          + " ".join(f"{v:08x}" for v in buf))
    S = (n + args.gpus - 1) // args.gpus
    peer_chunk = b.peer_rank % args.gpus
    lo = peer_chunk * S + 8 * b.word_index
    print(f"  peer {b.peer_rank} output[{lo}:{lo + 8}] = {ys[b.peer_rank][lo:lo + 8].tolist()}; "
          f"receiver output = {ys[b.global_rank][lo:lo + 8].tolist()}")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--calls", type=int, default=2000)
    ap.add_argument("--nodes", type=int, default=2)
    ap.add_argument("--gpus", type=int, default=2)
    ap.add_argument("--timeout", type=float, default=3.0)
    ap.add_argument("--start", type=int, default=0, help="first call to run (skip earlier ones)")
    ap.add_argument("--verbose", action="store_true")
    ap.add_argument("--check-dirty", action="store_true",
                    help="after every call, every slot word must be empty (all ones)")
    args = ap.parse_args()
    world = args.nodes * args.gpus
    g = LocalGroup(ClusterTopology(args.nodes, args.gpus), 4 << 20, device=0,
                   timeout_s=args.timeout)
    rng = random.Random(1234)
    sizes = [1, 7, 1000, 4099, 65536, 131072, 300001, 1 << 20]
    algos = ["hier", "twoshot", "oneshot", "auto", "direct"]
    dtypes = [torch.bfloat16, torch.float32, torch.int32]
    total = world * (world + 1) // 2
    for it in range(args.calls):
        algo = rng.choice(algos)
        blocks = rng.choice([0, 1, 3, 16, 32, 128])
        dt = rng.choice(dtypes)
        n = rng.choice(sizes)
        if dt != torch.int32 and n > (1 << 20) // 2:
            n = (1 << 20) // 2
        if it < args.start:
            continue
        g.set_algo(algo)
        g.set_config(NvrarConfig(blocks, 65536))
        idx = torch.arange(n, device="cuda", dtype=torch.int64) % 7 + 1
        xs = [(idx * (r + 1)).to(dt) for r in range(world)]
        ys = [torch.empty_like(x) for x in xs]
        if args.verbose:
            print(it, algo, blocks, dt, n, g.plan(n, dt), flush=True)
        try:
            g.run_all(xs, ys)
        except Exception as e:  # noqa: BLE001
            print(f"call {it} ({algo}/{blocks} {dt} n={n} plan={g.plan(n, dt)}): {e}")
            for b in getattr(e, "blocked", lambda: [])():
                dump_cell(g, b, args, world, n, ys, dt)
            return 1
        want = (idx * total).to(dt)
        for r, y in enumerate(ys):
            if not torch.equal(y, want):
                print(f"call {it} ({algo}/{blocks} {dt} n={n}): rank {r} "
                      f"{int((y != want).sum())} wrong")
                return 1
        if args.check_dirty:
            for r, c in enumerate(g.comms):
                cnt, first = c.dirty_cells()
                if cnt:
                    print(f"call {it} ({algo}/{blocks} {dt} n={n} plan={g.plan(n, dt)}): "
                          f"rank {r} left {cnt} non-empty slot words (first at byte {first})")
                    return 1
    print(f"OK after {args.calls} calls")
    return 0


if __name__ == "__main__":
    sys.exit(main())
