"""Summarise the rank-0 single-pass ncu captures of the per-rank kernels
(tools/gpu/r8.sh / r9.sh: nvl_<algo>_<bytes>.csv, stall_<algo>_<bytes>.csv)
into profiles/r02_ncu_nvlink_p<P>.json — what bench.py reads for the N>1
roofline.traffic — with B_alg = 2(P-1)/P*M next to the wire bytes.

    python tools/ncu_nvl_summary.py gpurun_out/r8 2 profiles/r02_ncu_nvlink_p2.json
"""
import csv
import glob
import json
import os
import re
import sys


def parse(path):
    rows = list(csv.reader(l for l in open(path) if l.startswith('"')))
    if not rows:
        return None
    head, out = rows[0], {}
    for r in rows[1:]:
        d = dict(zip(head, r))
        out["kernel"], out["grid"] = d["Kernel Name"], d["Grid Size"]
        out[d["Metric Name"]] = float(d["Metric Value"].replace(",", ""))
    return out


def main():
    src, world, dst = sys.argv[1], int(sys.argv[2]), sys.argv[3]
    rows = []
    for path in sorted(glob.glob(os.path.join(src, "nvl_*.csv"))):
        m = re.match(r"nvl_(\w+?)_(\d+)\.csv", os.path.basename(path))
        algo, size = m.group(1), int(m.group(2))
        n = parse(path)
        if not n:
            continue
        dur = n["gpu__time_duration.sum"]
        b_alg = 2 * (world - 1) / world * size
        row = {"world": world, "algo": algo, "bytes": size, "kernel": n["kernel"], "grid": n["grid"],
               "valid": dur < 1e9,  # a capture that hit the 5 s watchdog waited on a paused peer
               "nvl_tx_bytes": n["nvltx__bytes.sum"],
               "nvl_tx_user_bytes": n.get("nvltx__bytes_data_user.sum"),
               "nvl_rx_bytes_in_window": n["nvlrx__bytes.sum"],
               "b_alg_bytes": b_alg,
               "tx_user_over_b_alg": round(n.get("nvltx__bytes_data_user.sum", 0) / b_alg, 3),
               "tx_over_user": round(n["nvltx__bytes.sum"] / max(1.0, n.get("nvltx__bytes_data_user.sum", 1)), 3)}
        sp = os.path.join(src, f"stall_{algo}_{size}.csv")
        if os.path.exists(sp):
            s = parse(sp)
            if s:
                tot = sum(v for k, v in s.items() if k.startswith("smsp__warps_issue_stalled"))
                row["stall_pct"] = {k.replace("smsp__warps_issue_stalled_", "").replace(".sum", ""):
                                    round(100 * v / tot, 1) for k, v in s.items()
                                    if k.startswith("smsp__warps_issue_stalled") and v / tot >= 0.01}
        rows.append(row)
    doc = {"what": "rank 0 of a one-process-per-rank-GPU run, one launch (the 3rd call) per "
                   "(schedule, size), single-pass ncu metrics (ncu --devices 0; other ranks "
                   "unprofiled); NVLink TX = this GPU's egress during its kernel; RX in the "
                   "window misses the peers' pushes that landed before rank 0's kernel started "
                   "(they run first), so per-GPU ingress = the peers' TX by symmetry. Captures "
                   "marked valid=false hit the watchdog: two-round schedules (two-shot) need the "
                   "peer to progress while rank 0 is profiled, which ncu does not allow.",
           "command": "tools/gpu/r8.sh (P=2) / r9.sh (P=4)", "rows": rows}
    with open(dst, "w") as fh:
        json.dump(doc, fh, indent=1)
    print(f"wrote {dst}: {len(rows)} rows")


if __name__ == "__main__":
    main()
