"""GPU parity of the SIPG path (element-centric cell + face kernel) against the CPU oracle.

Same bars as the CG tests: operator/diagonal <= 1e-12 relative max-norm, V-cycle
<= 1e-11 with lambda pinned, PCG iterations +-1, true residual and L2 error.
"""
import numpy as np
import pytest
import torch

import fem_inputs
from oracle import multigrid as omg, problem as oprob, sipg as osipg
from oracle.mesh import Mesh, SIPG, DIRICHLET, NEUMANN

pytestmark = pytest.mark.gpu

MIXED = (DIRICHLET, NEUMANN, DIRICHLET, DIRICHLET, NEUMANN, DIRICHLET)


def fem_mod():
    from paper_1611_03029_b200 import fem
    return fem


def relmax(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return np.abs(a - b).max() / max(np.abs(b).max(), 1e-300)


def make(cells, k, eps=0.0, bc=(DIRICHLET,) * 6, pf=2.0, **kw):
    f = fem_mod()
    return (f.Fem(cells, k, f.FEM_SIPG, deform_eps=eps, bc=bc, penalty_factor=pf, **kw),
            Mesh(cells, k, eps=eps, bc=bc))


@pytest.mark.parametrize("k,cells,eps,bc", [
    (1, (5, 3, 4), 0.0, MIXED),
    (2, (3, 4, 5), 0.05, MIXED),
    (3, (4, 3, 2), 0.05, (DIRICHLET,) * 6),
    (4, (6, 4, 3), 0.0, (DIRICHLET,) * 6),       # C3 recipe, several batches + ragged tail
    (4, (5, 3, 4), 0.05, MIXED),
    (5, (3, 2, 3), 0.05, (DIRICHLET,) * 6),
    (6, (3, 2, 2), 0.05, MIXED),                 # C5 recipe
    (7, (2, 2, 1), 0.05, (DIRICHLET,) * 6),
    (8, (2, 1, 2), 0.0, MIXED),
    (2, (1, 1, 1), 0.05, (NEUMANN,) * 6),        # single cell, all Neumann
])
def test_apply_and_diagonal_match_oracle(k, cells, eps, bc):
    F, m = make(cells, k, eps, bc)
    x = fem_inputs.uniform_pm1(0, m.dg_n_dofs())
    y = np.zeros_like(x)
    F.fem_apply(x, y)
    yo = osipg.apply(m, x)
    assert relmax(y, yo) <= 1e-12
    d = np.zeros_like(x)
    F.fem_diagonal(d)
    assert relmax(d, osipg.diagonal(m)) <= 1e-12
    F.close()


@pytest.mark.parametrize("k,cells,bc", [(1, (5, 3, 4), MIXED), (4, (6, 4, 3), (DIRICHLET,) * 6),
                                        (3, (2, 5, 1), MIXED), (8, (2, 1, 2), MIXED)])
def test_cartesian_quadrature_kernel_matches_oracle(k, cells, bc, monkeypatch):
    """Cartesian levels run the Kronecker kernel (K2c) by default; the quadrature
    cell+face kernel (FEM_DG_KRON=0) stays pinned too."""
    monkeypatch.setenv("FEM_DG_KRON", "0")
    F, m = make(cells, k, 0.0, bc)
    x = fem_inputs.uniform_pm1(6, m.dg_n_dofs())
    y = np.zeros_like(x)
    F.fem_apply(x, y)
    assert relmax(y, osipg.apply(m, x)) <= 1e-12
    F.close()


@pytest.mark.parametrize("eps", [0.05, 0.0])
def test_penalty_factor_is_honoured(eps):
    F, m = make((3, 2, 2), 2, eps, MIXED, pf=3.0)
    x = fem_inputs.uniform_pm1(4, m.dg_n_dofs())
    y = np.zeros_like(x)
    F.fem_apply(x, y)
    assert relmax(y, osipg.apply(m, x, 3.0)) <= 1e-12


def test_rhs_matches_oracle():
    F, m = make((4, 2, 4), 3, 0.05)
    b = np.zeros(m.dg_n_dofs())
    F.fem_rhs(b)
    assert relmax(b, oprob.rhs(m, SIPG)) <= 1e-12


@pytest.mark.parametrize("k,cells,eps", [(2, (8, 4, 4), 0.05), (4, (4, 4, 8), 0.0)])
def test_levels_transfers_coarse_lambda(k, cells, eps):
    F, m = make(cells, k, eps, MIXED)
    mg = omg.Multigrid(m, SIPG)
    assert F.n_levels == len(mg.levels)
    for l, lev in enumerate(mg.levels):
        n, c = F.level_info(l)
        assert c == lev.mesh.n and n == lev.n_dofs
        x = fem_inputs.uniform_pm1(l, n)
        y = np.zeros(n)
        F.fem_level_apply(l, x, y)
        assert relmax(y, lev.apply(x)) <= 1e-12
        d = np.zeros(n)
        F.fem_level_diagonal(l, d)
        assert relmax(d, lev.diagonal()) <= 1e-12
        if l >= 1:
            assert abs(F.fem_level_lambda(l) - lev.lam) <= 1e-10 * lev.lam
            cm = mg.levels[l - 1]
            xc = fem_inputs.uniform_pm1(100 + l, cm.n_dofs)
            xf = fem_inputs.uniform_pm1(200 + l, n)
            out = xf.copy()
            F.mg_prolongate_add(l, xc, out)
            assert relmax(out, xf + mg.prolongate(l, xc)) <= 1e-12
            rc = np.zeros(cm.n_dofs)
            F.mg_restrict(l, xf, rc)
            assert relmax(rc, mg.restrict(l, xf)) <= 1e-12
    b0 = fem_inputs.uniform_pm1(9, mg.levels[0].n_dofs)
    x0 = np.zeros_like(b0)
    F.mg_coarse_solve(b0, x0)
    assert relmax(x0, mg.coarse_solve(b0)) <= 1e-11


def test_vcycle_with_pinned_lambda():
    cells, k, eps = (4, 4, 8), 3, 0.05
    m = Mesh(cells, k, eps=eps, bc=MIXED)
    mg = omg.Multigrid(m, SIPG)
    lam = [0.0] + [lev.lam for lev in mg.levels[1:]]
    F = fem_mod().Fem(cells, k, fem_mod().FEM_SIPG, deform_eps=eps, bc=MIXED, lambda_override=lam)
    b = fem_inputs.uniform_pm1(3, mg.fine.n_dofs)
    z = np.zeros_like(b)
    F.mg_vcycle(b, z)
    assert relmax(z, mg.vcycle(b)) <= 1e-11


@pytest.mark.parametrize("k,cells,eps", [(4, (8, 8, 8), 0.0), (6, (4, 4, 4), 0.05), (2, (8, 8, 4), 0.05)])
def test_pcg_matches_oracle(k, cells, eps):
    F, m = make(cells, k, eps)
    mg = omg.Multigrid(m, SIPG)
    b = oprob.rhs(m, SIPG)
    xo, its_o, _ = mg.pcg(b, tol=1e-10)
    x = np.zeros_like(b)
    its, rr, ok = F.cg_solve(b, x, rtol=1e-10)
    assert ok and rr <= 1e-10
    assert abs(its - its_o) <= 1
    assert np.linalg.norm(b - mg.fine.apply(x)) / np.linalg.norm(b) <= 1e-9
    e_gpu, e_or = oprob.l2_error(m, SIPG, x), oprob.l2_error(m, SIPG, xo)
    assert abs(e_gpu - e_or) <= 5e-4 * e_or


@pytest.mark.slow
def test_c3_full_solve_matches_oracle():
    w = fem_inputs.C3
    F, m = make(w.cells, w.degree, w.deform_eps)
    b = np.zeros(m.dg_n_dofs())
    F.fem_rhs(b)
    mg = omg.Multigrid(m, SIPG)
    assert relmax(b, oprob.rhs(m, SIPG)) <= 1e-12
    xo, its_o, _ = mg.pcg(b, tol=1e-10)
    x = np.zeros_like(b)
    its, rr, ok = F.cg_solve(b, x, rtol=1e-10)
    assert ok and abs(its - its_o) <= 1
    assert np.linalg.norm(b - mg.fine.apply(x)) / np.linalg.norm(b) <= 1e-9
    e_gpu, e_or = oprob.l2_error(m, SIPG, x), oprob.l2_error(m, SIPG, xo)
    assert abs(e_gpu - e_or) <= 5e-4 * e_or


@pytest.mark.slow
def test_c5_full_size_sampled_apply_and_solve_properties():
    w = fem_inputs.C5
    F, m = make(w.cells, w.degree, w.deform_eps)
    n = m.dg_n_dofs()
    x = torch.from_numpy(fem_inputs.uniform_pm1(0, n)).cuda()
    y = torch.zeros_like(x)
    F.fem_apply(x, y)
    xs = x.cpu().numpy()
    rng = np.random.default_rng(5)
    cells = np.unique(np.concatenate([rng.integers(0, m.n_cells, 40),
                                      [0, m.n_cells - 1, 63, 64 * 64 - 1, 64 * 64 * 32 + 64 * 10 + 5]]))
    m3 = (w.degree + 1) ** 3
    yo = osipg.apply_cells(m, xs, cells)
    yc = y.cpu().numpy().reshape(-1, m3)[cells]
    assert np.abs(yc - yo).max() <= 1e-12 * np.abs(yo).max()
    # the GMG-CG solve converges; its residual is re-checked by the oracle on sampled cells
    b = torch.zeros_like(x)
    F.fem_rhs(b)
    xsol = torch.zeros_like(b)
    its, rr, ok = F.cg_solve(b, xsol, rtol=1e-10)
    assert ok and rr <= 1e-10 and its <= 20
    bh, xh = b.cpu().numpy(), xsol.cpu().numpy()
    r_cells = bh.reshape(-1, m3)[cells] - osipg.apply_cells(m, xh, cells)
    assert np.abs(r_cells).max() <= 1e-7 * np.abs(bh).max()


@pytest.mark.parametrize("k,cells,bc", [(2, (3, 4, 5), MIXED), (4, (5, 3, 4), MIXED), (6, (3, 2, 2), (DIRICHLET,) * 6)])
def test_face_geometry_recomputed_on_the_fly_matches_oracle(k, cells, bc, monkeypatch):
    """FEM_DG_FGEO_FLY=1: the deformed kernel recomputes JxW and J^-1 n at the face points
    from the analytic map instead of reading the face records (same operator)."""
    monkeypatch.setenv("FEM_DG_FGEO_FLY", "1")
    F, m = make(cells, k, 0.05, bc)
    x = fem_inputs.uniform_pm1(2, m.dg_n_dofs())
    y = np.zeros_like(x)
    F.fem_apply(x, y)
    assert relmax(y, osipg.apply(m, x)) <= 1e-12
    F.close()
