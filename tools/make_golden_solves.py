"""Write tests/golden/solve_<C>.json: the ORACLE's GMG-PCG run on a full-size config.

Calls only oracle/ and fem_inputs (the seeded generator); never the CUDA path.
Stored per config (SURVEY §8c "Solve parity"; P:L1144-1148 PCG + V-cycle):
  lambda_max estimate of every level, iteration count, the whole
  relative residual history ||r_i|| / ||b|| (recursively updated residual, reading
  R13), the final relative residual and, for the manufactured configs, the relative
  L2 error (O9); for C4 (reading R15: b = A x_7, Dirichlet rows zeroed) the error
  ||x - x_7|| / ||x_7|| on the free DoFs.

Usage: python tools/make_golden_solves.py C4 C5 [C2 C3]   (C4: ~20 min, C5: ~1 h on 8 cores)
"""
from __future__ import annotations

import json
import os
import platform
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import fem_inputs  # noqa: E402
from oracle import multigrid as omg, problem as oprob  # noqa: E402
from oracle.mesh import Mesh, CG  # noqa: E402


def log(*a):
    print(time.strftime("%H:%M:%S"), *a, flush=True)


def run(name: str):
    w = fem_inputs.CONFIGS[name]
    m = Mesh(w.cells, w.degree, eps=w.deform_eps)
    t0 = time.time()
    log(name, "setup (levels, diagonals, lambda estimates, coarse Cholesky)")
    mg = omg.Multigrid(m, w.method, penalty_factor=w.penalty_factor)
    t_setup = time.time() - t0
    lams = [None] + [float(lv.lam) for lv in mg.levels[1:]]
    log(name, f"setup {t_setup:.0f} s, lambdas {lams}")
    extra = {}
    if w.rhs == "random_apply":
        x7 = fem_inputs.uniform_pm1(w.seed, mg.fine.n_dofs)
        b = mg.fine.apply(x7)
        b[~mg.fine.free] = 0.0
    else:
        b = oprob.rhs(m, w.method)
    hist = []
    t1 = time.time()
    x, its, rr = mg.pcg(b, tol=1e-10, history=hist)
    t_solve = time.time() - t1
    bn = float(np.linalg.norm(b))
    log(name, f"solve {t_solve:.0f} s, {its} iterations, relres {rr:.3e}")
    if w.rhs == "random_apply":
        f = mg.fine.free
        extra["err_vs_x7"] = float(np.linalg.norm((x - x7)[f]) / np.linalg.norm(x7[f]))
    else:
        extra["l2_error"] = oprob.l2_error(m, w.method, x)
    out = {
        "config": name,
        "source": "tools/make_golden_solves.py (oracle/ only); SURVEY §8c Solve parity; "
                  "PCG + V-cycle P:L1144-1148, Chebyshev P:L1159-1170",
        "method": "CG" if w.method == CG else "SIPG",
        "degree": w.degree,
        "cells": list(w.cells),
        "deform_eps": w.deform_eps,
        "rhs": w.rhs,
        "n_dofs": int(mg.fine.n_dofs),
        "levels": len(mg.levels),
        "lambda": lams,
        "rtol": 1e-10,
        "iterations": int(its),
        "relres": float(rr),
        "b_norm": bn,
        "history_rel": [float(h) / bn for h in hist],
        **extra,
        "oracle_setup_s": round(t_setup, 1),
        "oracle_solve_s": round(t_solve, 1),
        "host": {"cores": os.cpu_count(), "machine": platform.processor() or platform.machine()},
    }
    path = os.path.join(ROOT, "tests", "golden", f"solve_{name}.json")
    with open(path, "w") as fh:
        json.dump(out, fh, indent=1)
    log(name, "wrote", path, {k: out[k] for k in ("iterations", "relres")}, extra)


if __name__ == "__main__":
    for c in sys.argv[1:] or ["C4", "C5"]:
        run(c)
