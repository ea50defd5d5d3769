"""Small cases for compute-sanitizer (memcheck / racecheck / synccheck).

    compute-sanitizer --tool memcheck python tools/sanitize_cases.py

Runs apply, diagonal, a V-cycle and a PCG solve through the C ABI on C1 (CG Q2 8^3,
through the K1t stencil with FEM_ST_MIN_CELLS=1), a deformed CG Q4 4^3 mesh, and SIPG
Q2/Q6 on 4^3 / 2^3 meshes (Cartesian Kronecker and deformed quadrature kernels), and the
HDG trace / mixed / recovery / Jacobi-PCG entry points (include/fem_hdg.h) at Q2, Q4 and Q6."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("FEM_ST_MIN_CELLS", "1")
import fem_inputs  # noqa: E402
from paper_1611_03029_b200 import fem  # noqa: E402

CASES = [("C1 CG Q2 8^3 (stencil)", (8, 8, 8), 2, fem.FEM_CG, 0.0),
         ("CG Q4 4^3 deformed", (4, 4, 4), 4, fem.FEM_CG, 0.05),
         ("CG Q4 8^3 Cartesian (stencil)", (8, 8, 8), 4, fem.FEM_CG, 0.0),
         ("SIPG Q2 4^3 Cartesian", (4, 4, 4), 2, fem.FEM_SIPG, 0.0),
         ("SIPG Q6 2^3 deformed", (2, 2, 2), 6, fem.FEM_SIPG, 0.05)]

for name, cells, k, method, eps in CASES:
    F = fem.Fem(cells, k, method, deform_eps=eps)
    n = F.n_local
    x = fem_inputs.uniform_pm1(0, n)
    y, d, z = np.zeros(n), np.zeros(n), np.zeros(n)
    F.fem_apply(x, y)
    F.fem_diagonal(d)
    F.mg_vcycle(x, z)
    b = np.zeros(n)
    F.fem_rhs(b)
    xs = np.zeros(n)
    its, rr, ok = F.cg_solve(b, xs, rtol=1e-10)
    F.close()
    print(f"{name}: its {its} relres {rr:.1e} ok {ok}", flush=True)
import torch  # noqa: E402

for cells, k, bc in (((3, 2, 2), 2, (0, 1, 0, 0, 1, 0)), ((2, 2, 2), 4, (0,) * 6), ((2, 2, 1), 6, (1, 0, 0, 1, 0, 0))):
    H = fem.Hdg(cells, k, bc=bc)
    lam = torch.from_numpy(fem_inputs.uniform_pm1(0, H.n_trace)).cuda()
    y = torch.zeros_like(lam)
    H.hdg_apply(lam, y)
    H.hdg_diagonal(y)
    H.hdg_rhs(y)
    u = torch.zeros(H.n_cell_dofs, dtype=torch.float64, device="cuda")
    q = torch.zeros(3 * H.n_cell_dofs, dtype=torch.float64, device="cuda")
    H.hdg_local_solve(lam, u, q)
    qu = torch.from_numpy(fem_inputs.uniform_pm1(1, 4 * H.n_cell_dofs)).cuda()
    H.hdg_mixed_apply(qu, torch.zeros_like(qu))
    x = torch.zeros_like(lam)
    its, rr, ok = H.hdg_cg_solve(y, x, rtol=1e-10)
    torch.cuda.synchronize()
    H.close()
    print(f"HDG Q{k} {cells}: its {its} relres {rr:.1e} ok {ok}", flush=True)
print("sanitize cases done")
