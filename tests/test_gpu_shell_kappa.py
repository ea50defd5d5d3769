"""GPU parity of the SURVEY §8f N3 path: shell patch, degree-l polynomial mappings and
variable kappa (eq:diffusivity_shell), through the C ABI against the oracle.

Same bars as the Cartesian/deformed tests: operator, diagonal and geometry table to
relative 1e-12 in the max norm, PCG iterations within +-1 of the oracle's, true residual
below the tolerance.  kappa amplitude 1e6 (the paper's) is exercised on the
apply and diagonal only: kappa is negative on part of the domain (DESIGN.md reading
N3-c), so it is not a PCG problem.
"""
import numpy as np
import pytest

import fem_inputs
from oracle import cg as ocg, sipg as osipg, multigrid as omg, problem as oprob, gaussians as gs
from oracle.mesh import Mesh, CG, SIPG, SHELL, BOX, DIRICHLET, NEUMANN

pytestmark = pytest.mark.gpu

MIXED = (DIRICHLET, NEUMANN, DIRICHLET, DIRICHLET, NEUMANN, DIRICHLET)


def fem_mod():
    from paper_1611_03029_b200 import fem
    return fem


def relmax(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return np.abs(a - b).max() / max(np.abs(b).max(), 1e-300)


def make(method, cells, k, geometry=BOX, mapping_degree=0, kappa_amp=0.0, eps=0.0, bc=(DIRICHLET,) * 6, **kw):
    f = fem_mod()
    F = f.Fem(cells, k, f.FEM_CG if method == CG else f.FEM_SIPG, deform_eps=eps, bc=bc, geometry=geometry,
              mapping_degree=mapping_degree, kappa_amplitude=kappa_amp, **kw)
    m = Mesh(cells, k, eps=eps, bc=bc, geometry=geometry, mapping_degree=mapping_degree, kappa_amp=kappa_amp)
    return F, m


CASES = [
    # geometry, l, kappa amplitude, eps, k, cells, bc
    (SHELL, 5, 0.0, 0.0, 2, (3, 4, 5), (DIRICHLET,) * 6),
    (SHELL, 5, 1e6, 0.0, 4, (3, 2, 3), (DIRICHLET,) * 6),
    (SHELL, 0, 0.5, 0.0, 3, (4, 3, 2), MIXED),
    (SHELL, 2, 0.5, 0.0, 1, (5, 3, 4), MIXED),
    (BOX, 0, 0.5, 0.0, 4, (5, 3, 4), MIXED),          # variable kappa on the Cartesian box
    (BOX, 3, 0.0, 0.05, 3, (4, 4, 3), (DIRICHLET,) * 6),  # deformed box, cubic mapping
    (SHELL, 5, 0.5, 0.0, 6, (2, 2, 2), (DIRICHLET,) * 6),
    (SHELL, 4, 0.5, 0.0, 8, (1, 2, 1), MIXED),
]


@pytest.mark.parametrize("method", [CG, SIPG])
@pytest.mark.parametrize("geometry,l,amp,eps,k,cells,bc", CASES)
def test_apply_diagonal_geometry_match_oracle(method, geometry, l, amp, eps, k, cells, bc):
    F, m = make(method, cells, k, geometry, l, amp, eps, bc, coarse_cells=max(cells))
    n = m.cg_n_dofs() if method == CG else m.dg_n_dofs()
    x = fem_inputs.uniform_pm1(7, n)
    y = np.zeros_like(x)
    F.fem_apply(x, y)
    yo = ocg.apply(m, x) if method == CG else osipg.apply(m, x, 2.0)
    assert relmax(y, yo) <= 1e-12
    d = np.zeros_like(x)
    F.fem_diagonal(d)
    do = ocg.diagonal(m) if method == CG else osipg.diagonal(m, 2.0)
    assert relmax(d, do) <= 1e-12
    nq = (k + 1) ** 3
    G = np.zeros(m.n_cells * 6 * nq)
    F.fem_level_geometry(F.n_levels - 1, G)
    Go = ocg.metric(m, np.arange(m.n_cells), ocg.CellQuadrature(k))
    comp = [(0, 0), (0, 1), (0, 2), (1, 1), (1, 2), (2, 2)]
    Gr = np.stack([Go[:, :, a, b] for a, b in comp], axis=1).reshape(-1)
    assert relmax(G, Gr) <= 1e-12
    F.close()


@pytest.mark.parametrize("method", [CG, SIPG])
@pytest.mark.parametrize("geometry,amp", [(SHELL, 0.5), (BOX, 0.5)])
def test_rhs_matches_oracle(method, geometry, amp):
    F, m = make(method, (4, 3, 5), 3, geometry, 5 if geometry == SHELL else 0, amp, 0.05 if geometry == BOX else 0.0)
    b = np.zeros(m.cg_n_dofs() if method == CG else m.dg_n_dofs())
    F.fem_rhs(b)
    assert relmax(b, oprob.rhs(m, method)) <= 1e-12
    F.close()


@pytest.mark.parametrize("method,k,cells", [(CG, 4, (8, 8, 8)), (SIPG, 3, (8, 8, 4)), (CG, 2, (8, 4, 8))])
def test_pcg_shell_variable_kappa_matches_oracle(method, k, cells):
    """GMG-PCG on the shell patch, degree-5 mapping on every level, kappa amplitude 0.5."""
    F, m = make(method, cells, k, SHELL, 5, 0.5)
    mg = omg.Multigrid(m, method)
    b = gs.rhs(m, method, penalty_factor=2.0) if method == SIPG else gs.rhs(m, method)
    x0 = np.where(m.cg_dirichlet_mask(), b, 0.0) if method == CG else None
    xo, its_o, _ = mg.pcg(b, tol=1e-10, x0=x0) if method == CG else mg.pcg(b, tol=1e-10)
    x = np.zeros_like(b)
    its, rr, ok = F.cg_solve(b, x, rtol=1e-10)
    assert ok and rr <= 1e-10
    assert abs(its - its_o) <= 1
    assert relmax(x, xo) <= 1e-7
    F.close()


def test_shell_volume_from_gpu_geometry():
    """Trace of the CG operator on linear functions = the patch volume 7 pi / 36 (all-Neumann)."""
    k, cells = 4, (4, 4, 4)
    F, m = make(CG, cells, k, SHELL, 4, 0.0, bc=(NEUMANN,) * 6, coarse_cells=4)
    X = gs.node_coords(m)
    a, b = np.array([0.3, -1.1, 0.7]), np.array([-0.4, 0.25, 1.3])
    y = np.zeros(m.cg_n_dofs())
    F.fem_apply(X @ a, y)
    assert abs((X @ b) @ y / (a @ b) - 7 * np.pi / 36) < 1e-9
    F.close()


def test_negative_kappa_is_accepted_by_the_apply_and_errors_are_reported():
    fem = fem_mod()
    with pytest.raises(fem.FemError):
        fem.Fem((2, 2, 2), 2, fem.FEM_CG, geometry=7)
    with pytest.raises(fem.FemError):
        fem.Fem((2, 2, 2), 2, fem.FEM_CG, mapping_degree=9)
