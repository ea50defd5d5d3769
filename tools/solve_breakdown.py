"""Per-kernel breakdown of ONE GMG-CG solve (development aid, not the bench contract).

    python tools/solve_breakdown.py C2            # run alone: prints the solve time
    ncu --metrics gpu__time_duration.sum,launch__grid_size --profile-from-start off --csv \
        --log-file out.csv python tools/solve_breakdown.py C2
    python tools/solve_breakdown.py --summarize out.csv

Brackets one warm solve with cudaProfilerStart/Stop.  The summary groups the launches by
kernel and grid size (grid size identifies the multigrid level) and compares the sum of
the serialised kernel durations with the solve time measured without the profiler: the
difference is launch latency / dependency gaps.
"""
import collections
import csv
import os

# ncu profiles the kernels of the per-iteration graphs; the single conditional-loop graph of
# the default path hides them, so the breakdown uses the host loop
os.environ.setdefault("FEM_COND_GRAPH", "0")
import re
import sys
import time


def summarize(path):
    with open(path) as f:
        lines = [l for l in f if not l.startswith("==")]
    rows = {}
    for d in csv.DictReader(lines):
        key = d["ID"]
        r = rows.setdefault(key, {"name": re.sub(r"\(.*", "", d["Kernel Name"])})
        v = float(d["Metric Value"].replace(",", ""))
        if d["Metric Name"] == "gpu__time_duration.sum":
            r["us"] = v / 1000.0 if d["Metric Unit"] in ("ns", "nsecond") else (v * 1000 if d["Metric Unit"] in ("ms", "msecond") else v)
        elif d["Metric Name"] == "launch__grid_size":
            r["grid"] = int(v)
    tot = collections.defaultdict(float)
    cnt = collections.Counter()
    for r in rows.values():
        k = (r["name"][-48:], r.get("grid", 0))
        tot[k] += r.get("us", 0.0)
        cnt[k] += 1
    s = sum(tot.values())
    print(f"{len(rows)} launches, sum of kernel durations {s:.1f} us")
    for k, v in sorted(tot.items(), key=lambda x: -x[1]):
        print(f"{k[0]:48s} grid {k[1]:7d} x{cnt[k]:4d} {v:9.1f} us {100 * v / s:5.1f}%  ({v / cnt[k]:.2f} us each)")


def main():
    if sys.argv[1] == "--summarize":
        summarize(sys.argv[2])
        return
    import torch
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import fem_inputs
    from paper_1611_03029_b200 import fem
    w = fem_inputs.CONFIGS[sys.argv[1]]
    F = fem.Fem(w.cells, w.degree, w.method, deform_eps=w.deform_eps, bc=w.bc, penalty_factor=w.penalty_factor)
    b = torch.zeros(F.n_local, dtype=torch.float64, device="cuda")
    F.fem_rhs(b)
    x = torch.zeros_like(b)
    for _ in range(2):
        x.zero_()
        F.cg_solve(b, x)
    torch.cuda.synchronize()
    x.zero_()
    torch.cuda.synchronize()
    torch.cuda.cudart().cudaProfilerStart()
    t0 = time.perf_counter()
    its, rr, ok = F.cg_solve(b, x)
    torch.cuda.synchronize()
    t = time.perf_counter() - t0
    torch.cuda.cudart().cudaProfilerStop()
    print(f"{w.name}: its={its} relres={rr:.2e} solve {t * 1e3:.3f} ms (wall, includes host)")
    F.close()


if __name__ == "__main__":
    main()
