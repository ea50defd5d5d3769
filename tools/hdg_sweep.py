"""N4 degree sweep (development aid): HDG trace / mixed matrix-free apply throughput for k = 1..8
at ~1.6e7 equivalent DoFs (the paper's fig:matvec size class)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402

rows = []
for k in range(1, 9):
    n = max(2, round((1.6e7 / k ** 3) ** (1 / 3)))
    r = bench.hdg_config(cells=(n, n, n), k=k, reps=10, solve=False)
    r.pop("jacobi_pcg")
    r["k"] = k
    rows.append(r)
    print(f"k={k} {n}^3: trace {r['trace_apply_us']:.1f} us {r['trace_equivalent_dofs_per_s']:.3e} eq DoF/s "
          f"FP64 {r['trace_fp64_frac']:.2f}  mixed {r['mixed_apply_us']:.1f} us "
          f"{r['mixed_equivalent_dofs_per_s']:.3e} FP64 {r['mixed_fp64_frac']:.2f} HBM {r['mixed_hbm_frac']:.2f}",
          flush=True)
os.makedirs("gpurun_out", exist_ok=True)
json.dump(rows, open("gpurun_out/hdg_sweep.json", "w"), indent=1)
