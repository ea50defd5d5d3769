"""Quick timing probe (development aid, not the bench contract): apply and solve times."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__file__)))
import fem_inputs  # noqa: E402
from paper_1611_03029_b200 import fem  # noqa: E402


def timeit(fn, reps=20):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    fn()
    torch.cuda.synchronize()
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps


def run(w, solve=True):
    t0 = time.time()
    cc = __import__("os").environ.get("PROBE_COARSE")
    F = fem.Fem(w.cells, w.degree, w.method, deform_eps=w.deform_eps, coarse_cells=int(cc) if cc else None)
    torch.cuda.synchronize()
    setup = time.time() - t0
    n = F.n_local
    x = torch.from_numpy(fem_inputs.uniform_pm1(w.seed, n)).cuda()
    y = torch.zeros_like(x)
    ms = timeit(lambda: F.fem_apply(x, y))
    n_cells = np.prod(w.cells)
    print(f"{w.name}: n={n} setup={setup:.2f}s apply={ms*1e3:.1f}us  {n/ms/1e6:.2f} GDoF/s "
          f"(equiv {n_cells*w.degree**3/ms/1e6:.2f})", flush=True)
    if __import__("os").environ.get("PROBE_SMOOTH") == "1":   # finest-level smoother (fused Chebyshev launches)
        L = F.n_levels - 1
        b = torch.zeros_like(x)
        F.fem_apply(x, b)
        xs = torch.zeros_like(x)
        ms_s = timeit(lambda: F.mg_smooth(L, b, xs, False), reps=10)
        print(f"   smooth (5 steps from x != 0): {ms_s*1e3:.1f}us = {ms_s*1e3/5:.1f}us per step", flush=True)
    if __import__("os").environ.get("PROBE_TRANSFER") == "1":   # finest-level transfers
        L = F.n_levels - 1
        nc = F.level_info(L - 1)[0]
        xc = torch.from_numpy(fem_inputs.uniform_pm1(3, nc)).cuda()
        rc = torch.zeros_like(xc)
        xf = x.clone()
        ms_p = timeit(lambda: F.mg_prolongate_add(L, xc, xf), reps=10)
        ms_r = timeit(lambda: F.mg_restrict(L, x, rc), reps=10)
        print(f"   transfers: prolongate_add {ms_p*1e3:.1f}us ({(16*n+8*nc)/ms_p/1e6:.0f} GB/s)  "
              f"restrict (incl. zero) {ms_r*1e3:.1f}us ({(8*n+8*nc)/ms_r/1e6:.0f} GB/s)", flush=True)
    if solve:
        b = torch.zeros_like(x)
        F.fem_rhs(b) if w.rhs == "manufactured" else F.fem_apply(x, b)
        xs = torch.zeros_like(x)
        F.cg_solve(b, xs)
        for _ in range(3):
            xs.zero_()
            torch.cuda.synchronize()
            t0 = time.time()
            its, rr, ok = F.cg_solve(b, xs)
            torch.cuda.synchronize()
            t = time.time() - t0
            print(f"   solve: its={its} relres={rr:.2e} t={t*1e3:.2f}ms  {n/t/1e6:.1f} MDoF/s", flush=True)
    F.close()


if __name__ == "__main__":
    import os
    names = sys.argv[1:] or ["C1", "C2", "C4"]
    for nm in names:
        run(fem_inputs.CONFIGS[nm], solve=nm != "C1" and os.environ.get("PROBE_SOLVE", "1") == "1")
