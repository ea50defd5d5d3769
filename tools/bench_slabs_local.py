"""Development check of bench.py's multi-GPU workload on ONE GPU (not a bench number).

    python tools/bench_slabs_local.py [P]

Builds the weak-scaled C2 problem bench.py runs at N = P GPUs (32 x 32 x 32P cells on
[0,1]^2 x [0,P], CG Q4 deformed), solves it once with a single rank and once with P
rank threads sharing this GPU through libfem's in-process transport, and checks that
both converge, that all ranks agree on the iteration count, that it is within +-1 of
the single-rank count, and that the gathered solution matches the single-rank one.
Timings are printed for information only (the ranks share one device).
"""
import os
import sys
import threading
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import fem_inputs  # noqa: E402
from paper_1611_03029_b200 import fem  # noqa: E402

P = int(sys.argv[1]) if len(sys.argv) > 1 else 2
w = fem_inputs.C2
cells = (w.cells[0], w.cells[1], w.cells[2] * P)
hi = (w.hi[0], w.hi[1], w.hi[2] * P)
kw = dict(cells=cells, degree=w.degree, method=w.method, deform_eps=w.deform_eps, bc=w.bc, hi=hi,
          penalty_factor=w.penalty_factor)

F1 = fem.Fem(**kw)
b1 = torch.zeros(F1.n_local, dtype=torch.float64, device="cuda")
F1.fem_rhs(b1)
x1 = torch.zeros_like(b1)
torch.cuda.synchronize()
t0 = time.perf_counter()
its1, rr1, ok1 = F1.cg_solve(b1, x1)
t1 = time.perf_counter() - t0
print(f"1 rank : {F1.n_global} DoFs, its {its1}, relres {rr1:.2e}, {t1 * 1e3:.1f} ms", flush=True)
x1h = x1.cpu().numpy()
F1.close()

group = fem.LocalGroup(P)
res, errs = [None] * P, []


def worker(r):
    try:
        torch.cuda.set_device(0)
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            F = fem.Fem(rank=r, nranks=P, local_group=group, stream=s, **kw)
            b = torch.zeros(F.n_local, dtype=torch.float64, device="cuda")
            F.fem_rhs(b)
            x = torch.zeros_like(b)
            F.cg_solve(b, x)          # warm-up
            x.zero_()
            t0 = time.perf_counter()
            its, rr, ok = F.cg_solve(b, x)
            t = time.perf_counter() - t0
            res[r] = (F.first_global, x.cpu().numpy(), its, rr, ok, t)
            F.close()
    except Exception as e:  # noqa: BLE001
        errs.append((r, repr(e)))


th = [threading.Thread(target=worker, args=(r,)) for r in range(P)]
for t in th:
    t.start()
for t in th:
    t.join()
group.close()
assert not errs, errs
x = np.concatenate([res[r][1] for r in range(P)])
its = {res[r][2] for r in range(P)}
print(f"{P} ranks: its {sorted(its)}, relres {max(res[r][3] for r in range(P)):.2e}, "
      f"max rank time {max(res[r][5] for r in range(P)) * 1e3:.1f} ms (threads on one GPU)", flush=True)
assert all(res[r][4] for r in range(P)) and len(its) == 1 and abs(its.pop() - its1) <= 1
err = np.abs(x - x1h).max() / np.abs(x1h).max()
print(f"max |x_P - x_1| / max |x_1| = {err:.2e}")
assert err <= 1e-8
print("OK")
