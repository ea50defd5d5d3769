"""HDG apply timing probe (development aid): trace / mixed apply at Q<k> on n^3 cells."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402

for spec in (sys.argv[1:] or ["64:4"]):
    n, k = (int(v) for v in spec.split(":"))
    r = bench.hdg_config(cells=(n, n, n), k=k, reps=10, solve=False)
    print(f"{os.environ.get('FEM_LIB', 'libfem.so')} k={k} {n}^3: trace {r['trace_apply_us']:.1f} us "
          f"FP64 {r['trace_fp64_frac']:.3f}  mixed {r['mixed_apply_us']:.1f} us FP64 {r['mixed_fp64_frac']:.3f}",
          flush=True)
