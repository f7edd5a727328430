"""Summarise one kernel of an ncu --set full report into profiles/*_metrics.json
(what bench.py reads for roofline.traffic).

    python tools/ncu_extract.py gpurun_out/direct_emu.ncu-rep profiles/r01_ncu_direct_emu_metrics.json \
        --kernel "nvrar::direct_kernel<F32, N=2> (...)" --command "..."
"""
import argparse
import csv
import io
import json
import subprocess

KEEP = ("dram__bytes", "gpu__time_duration", "sm__throughput", "launch__", "sm__warps_active",
        "lts__t_bytes", "smsp__average_warp_latency_issue_stalled", "l1tex__t_bytes",
        "gpc__cycles_elapsed.max", "sm__cycles_active.avg", "dram__throughput",
        "smsp__warps_issue_stalled", "sm__inst_executed", "achieved_occupancy",
        "sm__maximum_warps_per_active_cycle_pct")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("out")
    ap.add_argument("--kernel", required=True)
    ap.add_argument("--command", default="")
    ap.add_argument("--launch", type=int, default=0, help="row of the report")
    a = ap.parse_args()
    raw = subprocess.run(["ncu", "-i", a.rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    head, units, vals = rows[0], rows[1], rows[2 + a.launch]
    metrics = {}
    for k, u, v in zip(head, units, vals):
        if any(k.startswith(p) or p in k for p in KEEP):
            metrics[k] = {"value": v, "unit": u}
    ver = subprocess.run(["ncu", "--version"], capture_output=True, text=True).stdout.strip()
    with open(a.out, "w") as fh:
        json.dump({"kernel": a.kernel, "command": a.command, "ncu": ver.splitlines()[-1],
                   "metrics": metrics}, fh, indent=1, sort_keys=True)
    print(f"wrote {a.out}: {len(metrics)} metrics")


if __name__ == "__main__":
    main()
