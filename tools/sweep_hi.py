import sys, os, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import fem_inputs
from paper_1611_03029_b200 import fem
for k in (5, 6, 7, 8):
    for method in (fem.FEM_CG, fem.FEM_SIPG):
        per = k if method == fem.FEM_CG else k + 1
        n = max(2, int(round(1.6e7 ** (1 / 3) / per)))
        F = fem.Fem((n, n, n), k, method, deform_eps=0.05, coarse_cells=n)
        x = torch.from_numpy(fem_inputs.uniform_pm1(0, F.n_local)).cuda(); y = torch.zeros_like(x)
        for _ in range(3): F.fem_apply(x, y)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize(); s.record()
        for _ in range(10): F.fem_apply(x, y)
        e.record(); torch.cuda.synchronize()
        print(f"k={k} {'CG' if method == fem.FEM_CG else 'SIPG'} n={n}: {s.elapsed_time(e)/10*1e3:.1f} us", flush=True)
        F.close()
