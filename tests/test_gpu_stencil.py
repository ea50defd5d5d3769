"""GPU parity of the warp-specialised assembled stencil (K1t, kernels_stencil.cu) on
Cartesian CG levels: the operator, its fused Chebyshev epilogue (smoother), the V-cycle
and PCG against the CPU oracle.

FEM_ST_MIN_CELLS=1 routes every single-rank Cartesian level with k in 2..4 through K1t
(the default threshold keeps the smallest levels on the cell kernel); FEM_ST_EZ sets the
z-element layers per block so that several z-chunks (and their halo layers) are covered.
Tolerances as in test_gpu_cg.py: apply 1e-12 relative max-norm (north_star), smoother
1e-12, V-cycle 1e-11 with lambda pinned, PCG iterations +-1 and the true residual.
"""
import numpy as np
import pytest
import torch

import fem_inputs
from oracle import cg as ocg, multigrid as omg, problem as oprob, transfer as otr
from oracle.mesh import Mesh, CG, DIRICHLET, NEUMANN

pytestmark = pytest.mark.gpu

MIXED = (DIRICHLET, NEUMANN, DIRICHLET, DIRICHLET, NEUMANN, DIRICHLET)
NEUM = (NEUMANN,) * 6
DIRI = (DIRICHLET,) * 6


def fem_mod():
    from paper_1611_03029_b200 import fem
    return fem


def relmax(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return np.abs(a - b).max() / max(np.abs(b).max(), 1e-300)


@pytest.fixture
def st_env(monkeypatch):
    monkeypatch.setenv("FEM_ST_MIN_CELLS", "1")
    monkeypatch.setenv("FEM_STENCIL2", "1")
    return monkeypatch


@pytest.mark.parametrize("k,cells,bc,ez", [
    (4, (8, 8, 8), DIRI, 32),      # exactly one full tile: far vertex column/row on the edge warps
    (4, (8, 8, 8), MIXED, 3),      # + z-chunks with halo layers, ragged last chunk
    (4, (9, 17, 5), MIXED, 2),     # partial tiles in x and y
    (4, (16, 8, 7), NEUM, 4),      # two full x tiles; pure Neumann (vertex rows at the boundary)
    (4, (3, 2, 4), DIRI, 1),       # one partial tile, one layer per block
    (4, (1, 1, 1), MIXED, 1),
    (3, (10, 8, 3), MIXED, 2),     # k = 3: 10 x slots (30 columns) per tile
    (3, (11, 9, 4), DIRI, 32),
    (2, (16, 8, 6), MIXED, 5),     # k = 2: 16 x slots per tile
    (2, (17, 9, 2), NEUM, 1),
    (1, (33, 17, 5), MIXED, 2),    # k = 1: 32 x slots, 8 rows per tile
    (1, (40, 9, 3), NEUM, 1),
])
def test_stencil2_apply_matches_oracle(k, cells, bc, ez, st_env):
    st_env.setenv("FEM_ST_EZ", str(ez))
    f = fem_mod()
    F = f.Fem(cells, k, f.FEM_CG, bc=bc)
    m = Mesh(cells, k, bc=bc)
    x = fem_inputs.uniform_pm1(0, m.cg_n_dofs())
    y = torch.zeros(m.cg_n_dofs(), dtype=torch.float64, device="cuda")
    F.fem_apply(torch.from_numpy(x).cuda(), y)
    yo = ocg.apply(m, x)
    assert relmax(y.cpu().numpy(), yo) <= 1e-12
    # every level of the hierarchy goes through K1t as well (MIN_CELLS = 1)
    for l, ml in enumerate(otr.hierarchy(m)):
        xl = fem_inputs.uniform_pm1(l + 1, ml.cg_n_dofs())
        yl = np.zeros(ml.cg_n_dofs())
        F.fem_level_apply(l, xl, yl)
        assert relmax(yl, ocg.apply(ml, xl)) <= 1e-12, l
    F.close()


@pytest.mark.parametrize("k,cells,bc", [(4, (16, 8, 8), MIXED), (3, (12, 8, 8), DIRI), (2, (16, 16, 8), MIXED),
                                        (1, (32, 16, 16), MIXED)])
def test_stencil2_fused_chebyshev_and_vcycle(k, cells, bc, st_env):
    st_env.setenv("FEM_ST_EZ", "3")
    m = Mesh(cells, k, bc=bc)
    mg = omg.Multigrid(m, CG)
    lam = [0.0] + [lev.lam for lev in mg.levels[1:]]
    f = fem_mod()
    F = f.Fem(cells, k, f.FEM_CG, bc=bc, lambda_override=lam)
    L = len(mg.levels) - 1
    b = fem_inputs.uniform_pm1(3, mg.fine.n_dofs) * mg.fine.free
    x = np.zeros_like(b)
    F.mg_smooth(L, b, x, True)
    xo = omg.chebyshev(mg.fine, b, None, 5, 0.06, 1.2, True)
    assert relmax(x, xo) <= 1e-12
    x2 = x.copy()
    F.mg_smooth(L, b, x2, False)
    assert relmax(x2, omg.chebyshev(mg.fine, b, xo, 5, 0.06, 1.2, False)) <= 1e-12
    z = np.zeros_like(b)
    F.mg_vcycle(b, z)
    assert relmax(z, mg.vcycle(b)) <= 1e-11
    F.close()


@pytest.mark.parametrize("k,cells", [(4, (16, 16, 16)), (2, (16, 8, 8))])
def test_stencil2_pcg_matches_oracle(k, cells, st_env):
    m = Mesh(cells, k)
    mg = omg.Multigrid(m, CG)
    b = oprob.rhs(m, CG)
    xo, its_o, _ = mg.pcg(b, tol=1e-10)
    f = fem_mod()
    F = f.Fem(cells, k, f.FEM_CG)
    x = np.zeros_like(b)
    its, rr, ok = F.cg_solve(b, x, rtol=1e-10)
    assert ok and abs(its - its_o) <= 1
    assert np.linalg.norm(b - mg.fine.apply(x)) / np.linalg.norm(b) <= 1e-9
    hist = F.cg_history()
    assert len(hist) == its + 1
    F.close()


def test_stencil2_matches_cell_kernel_bitwise_structure(st_env):
    """Same operator through K1t and through the Cartesian cell kernel (K1c): agreement
    to rounding on a multi-tile mesh with mixed boundaries."""
    cells, k = (20, 12, 9), 4
    f = fem_mod()
    x = fem_inputs.uniform_pm1(9, (k * 20 + 1) * (k * 12 + 1) * (k * 9 + 1))
    F1 = f.Fem(cells, k, f.FEM_CG, bc=MIXED)
    y1 = np.zeros_like(x)
    F1.fem_apply(x, y1)
    F1.close()
    st_env.setenv("FEM_STENCIL2", "0")
    F2 = f.Fem(cells, k, f.FEM_CG, bc=MIXED)
    y2 = np.zeros_like(x)
    F2.fem_apply(x, y2)
    F2.close()
    assert relmax(y1, y2) <= 1e-13
