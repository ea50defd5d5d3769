"""The paper's 3-D Gaussian problem on the GPU: L2 errors and iterations
next to the values the paper prints.  RHS from the oracle (test data)."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import gaussians as gs  # noqa: E402
from oracle.mesh import CG, SIPG  # noqa: E402
from paper_1611_03029_b200 import fem  # noqa: E402
from tests.conftest import golden  # noqa: E402

for r in golden("paper_gaussian_errors.json")["rows"]:
    if r["k"] < 2:
        continue
    n = round(r["cells"] ** (1 / 3))
    m = gs.mesh((n, n, n), r["k"])
    for meth, key, itk in ((CG, "FEL2", "qIt"), (SIPG, "dgL2", "dgIt")):
        b = gs.rhs(m, meth)
        F = fem.Fem(m.n, m.k, fem.FEM_CG if meth == CG else fem.FEM_SIPG, lo=tuple(m.lo), hi=tuple(m.hi),
                    bc=m.bc, penalty_factor=gs.PENALTY_FACTOR)
        x = np.zeros_like(b)
        F.cg_solve(b, x, rtol=1e-9)
        x[:] = 0
        t0 = time.perf_counter()
        its, rr, ok = F.cg_solve(b, x, rtol=1e-9)
        t = time.perf_counter() - t0
        F.close()
        e = gs.l2_error_abs(m, meth, x)
        print(f"k={r['k']} {n}^3 {'CG  ' if meth == CG else 'SIPG'}: L2 {e:.4e} (paper {r[key]:.3e}, "
              f"{100 * (e / r[key] - 1):+.2f}%), its {its} (paper {r[itk]}), solve {t * 1e3:.2f} ms", flush=True)
