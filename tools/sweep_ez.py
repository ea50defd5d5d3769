"""K1t z-chunk length sweep (development aid): finest-level smoother step and apply time of a
Cartesian CG Q4 mesh for several FEM_ST_EZ (z-element layers per block), one process per value.

    python tools/sweep_ez.py <cells per direction> <ez> [<ez> ...]
"""
import os
import subprocess
import sys

if len(sys.argv) > 1 and sys.argv[1] == "--one":
    import torch
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import fem_inputs
    from paper_1611_03029_b200 import fem
    nc = int(sys.argv[2])
    F = fem.Fem((nc, nc, nc), 4, fem.FEM_CG)
    n = F.n_local
    x = torch.from_numpy(fem_inputs.uniform_pm1(7, n)).cuda()
    b = torch.zeros_like(x)
    y = torch.zeros_like(x)
    F.fem_apply(x, b)

    def timeit(fn, reps):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        fn()
        torch.cuda.synchronize()
        s.record()
        for _ in range(reps):
            fn()
        e.record()
        torch.cuda.synchronize()
        return s.elapsed_time(e) / reps

    L = F.n_levels - 1
    xs = torch.zeros_like(x)
    t_s = timeit(lambda: F.mg_smooth(L, b, xs, False), 10) / 5
    t_a = timeit(lambda: F.fem_apply(x, y), 20)
    print(f"cells {nc}^3 FEM_ST_EZ={os.environ.get('FEM_ST_EZ', 'auto'):>4s}: smoother step {t_s * 1e3:8.1f} us   apply {t_a * 1e3:8.1f} us",
          flush=True)
else:
    nc = sys.argv[1]
    for ez in sys.argv[2:]:
        env = dict(os.environ)
        if ez != "auto":
            env["FEM_ST_EZ"] = ez
        subprocess.run([sys.executable, __file__, "--one", nc], env=env, check=False)
