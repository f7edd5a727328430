"""PCIe bandwidth of this box (the e2e path's bound): pinned H2D alone, D2H
alone, both at once (copy engines), and a zero-copy kernel reading/writing
pinned host memory — 8 MB each way, like the N=1 e2e step."""
import json

import torch


def timed(fn, reps=10):
    s = torch.cuda.Event(enable_timing=True)
    e = torch.cuda.Event(enable_timing=True)
    fn()
    torch.cuda.synchronize()
    out = []
    for _ in range(reps):
        s.record()
        fn()
        e.record()
        e.synchronize()
        out.append(s.elapsed_time(e) * 1e3)
    out.sort()
    return out[len(out) // 2]


def main():
    nb = 8 << 20
    h_in = torch.empty(nb, dtype=torch.uint8).pin_memory()
    h_out = torch.empty(nb, dtype=torch.uint8).pin_memory()
    d_in = torch.empty(nb, dtype=torch.uint8, device="cuda")
    d_out = torch.empty(nb, dtype=torch.uint8, device="cuda")
    s2 = torch.cuda.Stream()
    res = {}
    res["h2d_us"] = timed(lambda: d_in.copy_(h_in, non_blocking=True))
    res["d2h_us"] = timed(lambda: h_out.copy_(d_out, non_blocking=True))

    def both():
        cur = torch.cuda.current_stream()
        s2.wait_stream(cur)
        d_in.copy_(h_in, non_blocking=True)
        with torch.cuda.stream(s2):
            h_out.copy_(d_out, non_blocking=True)
        cur.wait_stream(s2)
    res["both_us"] = timed(both)
    for k in ("h2d", "d2h"):
        res[f"{k}_GBs"] = round(nb / (res[f"{k}_us"] * 1e-6) / 1e9, 1)
    res["both_GBs_total"] = round(2 * nb / (res["both_us"] * 1e-6) / 1e9, 1)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
