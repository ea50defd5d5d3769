"""Summarise ncu captures into profiles/<tag>_summary.json (development aid).

    python tools/summarize_ncu.py <tag> [gpurun_out]

Reads <dir>/<tag>_apply_<C>.ncu-rep (ncu --set full, one apply launch each) and
<dir>/<tag>_launches_bench_c2.csv (gpu__time_duration.sum launch list of bench.py)
and writes the metrics DESIGN.md quotes plus per-kernel shares of the bench run.
The launch list covers the whole bench process (setup, warm-up, timed steps, e2e);
the shares of the solve kernels are what DESIGN.md compares with the live bench.
"""
import csv
import glob
import io
import json
import os
import subprocess
import sys

METRICS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
    "launch__shared_mem_per_block_dynamic", "launch__occupancy_limit_registers",
    "launch__occupancy_limit_shared_mem", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
    "l1tex__throughput.avg.pct_of_peak_sustained_active",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "smsp__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "smsp__pcsamp_sample_count",
    "smsp__pcsamp_warps_issue_stalled_long_scoreboard", "smsp__pcsamp_warps_issue_stalled_barrier",
    "smsp__pcsamp_warps_issue_stalled_mio_throttle", "smsp__pcsamp_warps_issue_stalled_short_scoreboard",
    "smsp__pcsamp_warps_issue_stalled_wait", "smsp__pcsamp_warps_issue_stalled_math_pipe_throttle",
    "smsp__pcsamp_warps_issue_stalled_lg_throttle", "smsp__pcsamp_warps_issue_stalled_selected",
]


def rep_metrics(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    d = {"kernel": vals[hdr.index("Kernel Name")]}
    for m in METRICS:
        if m in hdr:
            i = hdr.index(m)
            d[m] = f"{vals[i]} {units[i]}".strip()
    return d


def launch_shares(path):
    with open(path) as f:
        lines = [ln for ln in f if ln.startswith('"')]
    rows = list(csv.DictReader(io.StringIO("".join(lines))))
    agg = {}
    for r in rows:
        if r["Metric Name"] != "gpu__time_duration.sum":
            continue
        name = r["Kernel Name"].split("(")[0].replace("void ", "")
        name = name.split("<")[0]
        us = float(r["Metric Value"]) * (1e-3 if r["Metric Unit"] == "ns" else 1.0)
        a = agg.setdefault(name, {"launches": 0, "us": 0.0})
        a["launches"] += 1
        a["us"] += us
    tot = sum(a["us"] for a in agg.values())
    for a in agg.values():
        a["us"] = round(a["us"], 1)
        a["share"] = round(a["us"] / tot, 4)
    return dict(sorted(agg.items(), key=lambda kv: -kv[1]["us"]))


def main():
    tag = sys.argv[1]
    d = sys.argv[2] if len(sys.argv) > 2 else "gpurun_out"
    res = {}
    for p in sorted(glob.glob(os.path.join(d, f"{tag}_*.ncu-rep"))):
        res[os.path.basename(p)[len(tag) + 1:-8]] = rep_metrics(p)
    for lp in sorted(glob.glob(os.path.join(d, f"{tag}_launches_bench_*.csv"))):
        cfg = os.path.basename(lp)[len(tag) + len("_launches_bench_"):-4].upper()
        res[f"bench_{cfg}_launch_shares"] = launch_shares(lp)
    os.makedirs("profiles", exist_ok=True)
    with open(os.path.join("profiles", f"{tag}_summary.json"), "w") as f:
        json.dump(res, f, indent=1)
    print(json.dumps(res, indent=1)[:4000])


if __name__ == "__main__":
    main()
