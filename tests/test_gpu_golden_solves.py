"""Full-size GMG-CG solves of BASELINE.json configs[1..4] (C2..C5) against the ORACLE's own
run of the same recipe, stored by tools/make_golden_solves.py (oracle/ only) in
tests/golden/solve_<C>.json.

Solve parity (north_star: "iteration counts within +-1 of the oracle's
CG+GMG"; PCG + V-cycle P:L1144-1148, Chebyshev smoother P:L1159-1170):
  * lambda_max estimate of every level within 1e-9 relative (15 Jacobi-PCG steps);
  * PCG iterations within +-1 of the oracle's;
  * the early relative residual history ||r_i||/||b|| (i <= 3) within 1e-8 relative;
  * the final relative residual <= 1e-10;
  * C4 (reading R15, b = A x_7 with the Dirichlet rows zeroed): ||x - x_7|| / ||x_7||
    <= 1e-8 on the free DoFs; manufactured configs: relative L2 error of the GPU solution
    (oracle O9 quadrature) within 3 significant digits of the oracle solution's.
"""
import json
import os

import numpy as np
import pytest
import torch

import fem_inputs
from oracle import problem as oprob
from oracle.mesh import Mesh, CG

pytestmark = [pytest.mark.gpu, pytest.mark.slow]
GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load(name):
    p = os.path.join(GOLDEN, f"solve_{name}.json")
    if not os.path.exists(p):
        pytest.skip(f"{p} not generated (tools/make_golden_solves.py {name})")
    with open(p) as f:
        return json.load(f)


def dirichlet_mask(w, n):
    k = w.degree
    nn = [k * c + 1 for c in w.cells]
    i = torch.arange(n, device="cuda")
    g = [i % nn[0], (i // nn[0]) % nn[1], i // (nn[0] * nn[1])]
    m = torch.zeros(n, dtype=torch.bool, device="cuda")
    for d in range(3):
        m |= (g[d] == 0) | (g[d] == nn[d] - 1)
    return m


@pytest.mark.parametrize("name", ["C2", "C3", "C4", "C5"])
def test_full_size_solve_matches_oracle_run(name):
    from paper_1611_03029_b200 import fem
    g = load(name)
    w = fem_inputs.CONFIGS[name]
    F = fem.Fem(w.cells, w.degree, w.method, deform_eps=w.deform_eps, bc=w.bc, penalty_factor=w.penalty_factor)
    assert F.n_global == g["n_dofs"] and F.n_levels == g["levels"]
    for l in range(1, F.n_levels):
        lam = F.fem_level_lambda(l)
        assert abs(lam - g["lambda"][l]) <= 1e-9 * g["lambda"][l], (l, lam, g["lambda"][l])
    n = F.n_local
    b = torch.zeros(n, dtype=torch.float64, device="cuda")
    xs = None
    if w.rhs == "manufactured":
        F.fem_rhs(b)
    else:
        xs = torch.from_numpy(fem_inputs.uniform_pm1(w.seed, n)).cuda()
        F.fem_apply(xs, b)
        b[dirichlet_mask(w, n)] = 0.0
    assert abs(b.norm().item() - g["b_norm"]) <= 1e-12 * g["b_norm"]
    x = torch.zeros_like(b)
    its, rr, ok = F.cg_solve(b, x, rtol=1e-10)
    hist = F.cg_history()
    assert ok and rr <= 1e-10
    assert abs(its - g["iterations"]) <= 1, (its, g["iterations"])
    for i in range(1, min(4, len(hist), len(g["history_rel"]))):
        ho = g["history_rel"][i]
        assert abs(hist[i] - ho) <= 1e-8 * ho, (i, hist[i], ho)
    if xs is not None:
        free = ~dirichlet_mask(w, n)
        err = ((x - xs)[free].norm() / xs[free].norm()).item()
        assert err <= 1e-8, err
    else:
        m = Mesh(w.cells, w.degree, eps=w.deform_eps, bc=w.bc)
        e = oprob.l2_error(m, w.method, x.cpu().numpy())
        assert abs(e - g["l2_error"]) <= 5e-4 * g["l2_error"], (e, g["l2_error"])
    F.close()
