"""Repeat one configuration many times on virtual ranks (race hunting).

    python tests/repro_emu.py --algo hier --blocks 16 --dtype bf16 --n 300001 --reps 2000
"""
import argparse
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2511_09557_b200 import ClusterTopology, LocalGroup, NvrarConfig  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--algo", default="hier")
    ap.add_argument("--blocks", type=int, default=16)
    ap.add_argument("--dtype", default="bf16")
    ap.add_argument("--n", type=int, default=300001)
    ap.add_argument("--reps", type=int, default=1000)
    ap.add_argument("--nodes", type=int, default=2)
    ap.add_argument("--gpus", type=int, default=2)
    ap.add_argument("--proto", default="auto")
    ap.add_argument("--batch", type=int, default=50, help="calls enqueued between checks")
    args = ap.parse_args()
    dt = {"bf16": torch.bfloat16, "f32": torch.float32, "i32": torch.int32}[args.dtype]
    world = args.nodes * args.gpus
    g = LocalGroup(ClusterTopology(args.nodes, args.gpus), 4 << 20, device=0, timeout_s=3.0)
    g.set_algo(args.algo)
    g.set_protocol(args.proto)
    g.set_config(NvrarConfig(args.blocks, 65536))
    idx = torch.arange(args.n, device="cuda", dtype=torch.int64) % 7 + 1
    xs = [(idx * (r + 1)).to(dt) for r in range(world)]
    ys = [torch.empty_like(x) for x in xs]
    want = (idx * (world * (world + 1) // 2)).to(dt)
    done = 0
    while done < args.reps:
        for _ in range(args.batch):
            g.launch(xs, ys)
        done += args.batch
        try:
            g.check()
        except Exception as e:  # noqa: BLE001
            print(f"after <= {done} calls: {e}")
            import ctypes
            from collections import Counter
            for r, c in enumerate(g.comms):
                s = (ctypes.c_uint32 * 512)()
                c._lib.nvrar_debug_seq_slots(c._h, s, 512)
                cnt = Counter(list(s))
                odd = [i for i in range(512) if s[i] != cnt.most_common(1)[0][0]]
                print(f"  rank {r} seq slots {dict(cnt)} odd slots {odd[:20]}")
            for b in getattr(e, "blocked", lambda: [])():
                c = g.comms[b.global_rank]
                lay = (ctypes.c_uint64 * 8)()
                c._lib.nvrar_debug_read_region(c._h, 0, 0, None, lay)
                parity = b.expected & 1
                src = b.peer_rank % args.gpus
                base = {5: (lay[3], lay[4]), 4: (lay[1], lay[2])}.get(b.phase, (lay[3], lay[4]))
                off = base[0] + (parity * world + src) * base[1] * 8 + b.word_index * 16
                buf = (ctypes.c_uint32 * 16)()
                c._lib.nvrar_debug_read_region(c._h, off - 16, 64, buf, None)
                print(f"  rank {b.global_rank} cells [u-1..u+2] of src {src} parity {parity}: "
                      + " ".join(f"{v:08x}" for v in buf))
                other = (ctypes.c_uint32 * 16)()
                off2 = base[0] + ((1 - parity) * world + src) * base[1] * 8 + b.word_index * 16
                c._lib.nvrar_debug_read_region(c._h, off2 - 16, 64, other, None)
                print(f"  same cells, other parity: " + " ".join(f"{v:08x}" for v in other))
                cnt2 = ctypes.c_uint64()
                first = ctypes.c_uint64()
                c._lib.nvrar_debug_dirty_cells(c._h, ctypes.byref(cnt2), ctypes.byref(first))
                print(f"  rank {b.global_rank} dirty words {cnt2.value} first at {first.value} "
                      f"(awaited cell at {off})")
            return 1
        for r in range(world):
            if not torch.equal(ys[r], want):
                print(f"after {done} calls: rank {r} wrong")
                return 1
    print(f"OK {done} calls")
    return 0


if __name__ == "__main__":
    sys.exit(main())
