"""Solve time vs mesh size (same recipe as C2): how much of a solve is coarse-level latency."""
import sys, time
import torch
sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__file__)))
from paper_1611_03029_b200 import fem  # noqa: E402

for n in (32, 16, 8, 4, 2):
    F = fem.Fem((n, n, n), 4, fem.FEM_CG, deform_eps=0.05)
    b = torch.zeros(F.n_local, dtype=torch.float64, device="cuda")
    F.fem_rhs(b)
    x = torch.zeros_like(b)
    F.cg_solve(b, x)
    ts = []
    for _ in range(5):
        x.zero_()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        its, rr, ok = F.cg_solve(b, x)
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    t = min(ts)
    print(f"{n}^3: levels={F.n_levels} its={its} solve={t*1e3:.3f} ms  per-iteration={t*1e3/its:.3f} ms", flush=True)
    F.close()
