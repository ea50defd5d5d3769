"""GPU parity of the CG path (libfem through the C ABI) against the CPU oracle.

Tolerances: operator/diagonal/transfer/geometry relative max-norm <= 1e-12
(north_star: per-apply agreement within relative 1e-12 in the max norm);
V-cycle with lambda pinned <= 1e-11; PCG iterations within +-1,
both true residuals <= tol, L2 errors within 3 significant digits.
"""
import numpy as np
import pytest
import torch

import fem_inputs
from oracle import cg as ocg, multigrid as omg, problem as oprob, transfer as otr
from oracle.mesh import Mesh, CG, DIRICHLET, NEUMANN

pytestmark = pytest.mark.gpu

MIXED = (DIRICHLET, NEUMANN, DIRICHLET, DIRICHLET, NEUMANN, DIRICHLET)


def fem_mod():
    from paper_1611_03029_b200 import fem
    return fem


def relmax(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return np.abs(a - b).max() / max(np.abs(b).max(), 1e-300)


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def host(t):
    return t.cpu().numpy()


def make(cells, k, eps=0.0, bc=(DIRICHLET,) * 6, **kw):
    f = fem_mod()
    return f.Fem(cells, k, f.FEM_CG, deform_eps=eps, bc=bc, **kw), Mesh(cells, k, eps=eps, bc=bc)


@pytest.mark.parametrize("variant,k,cells", [
    ("FEM_PLANE", 1, (5, 3, 4)), ("FEM_PLANE", 2, (3, 4, 5)), ("FEM_PLANE", 3, (9, 4, 3)),
    ("FEM_PLANE", 4, (11, 5, 3)),                # > 32 cells: several groups + ragged tail
    ("FEM_DBASIS", 1, (5, 3, 4)), ("FEM_DBASIS", 2, (3, 4, 5)), ("FEM_DBASIS", 4, (6, 4, 3)),
    ("FEM_DBASIS", 6, (2, 3, 2)), ("FEM_DBASIS", 8, (2, 1, 2)),
])
def test_alternative_deformed_kernels_match_oracle(variant, k, cells, monkeypatch):
    """The plane kernel (K1p) and the derivative-basis line kernel (K1d) are
    selectable at fem_setup (env); same operator, geometry table and diagonal."""
    monkeypatch.setenv(variant, "1")
    F, m = make(cells, k, 0.05, MIXED)
    x = fem_inputs.uniform_pm1(3, m.cg_n_dofs())
    y = np.zeros_like(x)
    F.fem_apply(x, y)
    assert relmax(y, ocg.apply(m, x)) <= 1e-12
    d = np.zeros_like(x)
    F.fem_diagonal(d)
    assert relmax(d, ocg.diagonal(m)) <= 1e-12
    nq = (k + 1) ** 3
    G = np.zeros(m.n_cells * 6 * nq)
    F.fem_level_geometry(F.n_levels - 1, G)
    Go = ocg.metric(m, np.arange(m.n_cells), ocg.CellQuadrature(k))
    comp = [(0, 0), (0, 1), (0, 2), (1, 1), (1, 2), (2, 2)]
    Gr = np.stack([Go[:, :, a, b] for a, b in comp], axis=1).reshape(-1)
    assert relmax(G, Gr) <= 1e-13
    F.close()


@pytest.mark.parametrize("k,cells,bc", [
    (1, (5, 3, 4), MIXED), (2, (8, 8, 8), (DIRICHLET,) * 6), (3, (7, 5, 3), MIXED),
    (4, (37, 9, 3), (DIRICHLET,) * 6),           # several x and y tiles, ragged
    (5, (3, 2, 3), MIXED), (8, (2, 1, 2), (DIRICHLET,) * 6),
])
def test_stencil_kernel_matches_oracle(k, cells, bc, monkeypatch):
    """Atomic-free global Kronecker stencil (K1s, FEM_STENCIL=1) on Cartesian CG levels."""
    monkeypatch.setenv("FEM_STENCIL", "1")
    F, m = make(cells, k, 0.0, bc)
    x = fem_inputs.uniform_pm1(5, m.cg_n_dofs())
    y = np.zeros_like(x)
    F.fem_apply(x, y)
    assert relmax(y, ocg.apply(m, x)) <= 1e-12
    F.close()


@pytest.mark.parametrize("k,cells,eps,bc", [
    (2, (8, 8, 8), 0.0, (DIRICHLET,) * 6),       # C1
    (1, (5, 3, 4), 0.05, MIXED),
    (2, (3, 4, 5), 0.05, MIXED),
    (3, (4, 3, 2), 0.05, (DIRICHLET,) * 6),
    (4, (6, 4, 3), 0.05, MIXED),                 # several cell batches + ragged tail
    (4, (5, 3, 3), 0.05, MIXED),                 # 45 cells: last 8-cell G block partial (TMA copy)
    (4, (3, 1, 1), 0.05, (DIRICHLET,) * 6),      # a single partial block
    (7, (3, 1, 1), 0.05, (DIRICHLET,) * 6),      # TMA-staged G, ragged 2-cell block
    (8, (1, 3, 1), 0.05, MIXED),
    (4, (7, 5, 3), 0.0, (DIRICHLET,) * 6),
    (5, (3, 2, 3), 0.05, MIXED),
    (6, (2, 3, 2), 0.05, (DIRICHLET,) * 6),
    (7, (2, 2, 2), 0.05, MIXED),
    (8, (2, 1, 2), 0.0, (DIRICHLET,) * 6),
])
def test_apply_and_diagonal_match_oracle(k, cells, eps, bc):
    F, m = make(cells, k, eps, bc)
    x = fem_inputs.uniform_pm1(0, m.cg_n_dofs())
    y = torch.zeros(m.cg_n_dofs(), dtype=torch.float64, device="cuda")
    F.fem_apply(dev(x), y)
    torch.cuda.synchronize()
    yo = ocg.apply(m, x)
    assert relmax(host(y), yo) <= 1e-12
    d = torch.zeros_like(y)
    F.fem_diagonal(d)
    assert relmax(host(d), ocg.diagonal(m)) <= 1e-12
    F.close()


def test_c1_exact_diagonal_and_host_vectors():
    from tests.conftest import golden
    g = golden("c1_diagonal.json")
    w = fem_inputs.C1
    F, m = make(w.cells, w.degree)
    d = np.zeros(m.cg_n_dofs())
    F.fem_diagonal(d)                          # host vector path
    gc = m.cg_node_coords()
    n_mid = (gc % 2 == 1).sum(axis=1)
    vals = np.array([g["free_values"][kk] for kk in ("vvv", "one_m", "two_m", "mmm")])[n_mid]
    mask = m.cg_dirichlet_mask()
    assert np.all(d[mask] == 1.0)
    assert np.allclose(d[~mask], vals[~mask], rtol=1e-14, atol=0)
    # host and device apply agree bit for bit (same kernels)
    x = fem_inputs.uniform_pm1(w.seed, m.cg_n_dofs())
    yh = np.zeros_like(x)
    F.fem_apply(x, yh)
    assert relmax(yh, ocg.apply(m, x)) <= 1e-12


def test_geometry_table_matches_oracle_metric():
    F, m = make((3, 4, 2), 3, 0.05, MIXED)
    nl = F.n_levels
    n_dofs, cells = F.level_info(nl - 1)
    N = 4
    G = np.zeros(np.prod(cells) * 6 * N ** 3)
    F.fem_level_geometry(nl - 1, G)
    Go = ocg.metric(m, np.arange(m.n_cells), ocg.CellQuadrature(3))     # [C, q, 3, 3]
    comps = [(0, 0), (0, 1), (0, 2), (1, 1), (1, 2), (2, 2)]
    Gr = G.reshape(m.n_cells, 6, N ** 3)
    for c, (a, b) in enumerate(comps):
        assert relmax(Gr[:, c, :], Go[:, :, a, b]) <= 1e-13


def test_rhs_matches_oracle():
    F, m = make((4, 4, 2), 4, 0.05)
    b = np.zeros(m.cg_n_dofs())
    F.fem_rhs(b)
    assert relmax(b, oprob.rhs(m, CG)) <= 1e-12


def test_errors():
    f = fem_mod()
    F, m = make((2, 2, 2), 2)
    with pytest.raises(f.FemError) as e:
        F.fem_apply(np.zeros(5), np.zeros(m.cg_n_dofs()))
    assert e.value.code == -2
    with pytest.raises(f.FemError) as e:
        F.fem_level_apply(17, np.zeros(5), np.zeros(5))
    assert e.value.code == -1
    with pytest.raises(f.FemError) as e:
        f.Fem((2, 2, 2), 2, f.FEM_CG, deform_eps=-0.9)   # folds cells: det J <= 0
    assert e.value.code == -3 and "cell" in str(e.value)


@pytest.mark.parametrize("k,cells,eps", [(2, (8, 4, 4), 0.05), (4, (4, 4, 8), 0.0), (3, (4, 2, 4), 0.05)])
def test_levels_transfers_coarse_lambda(k, cells, eps):
    F, m = make(cells, k, eps, MIXED)
    mg = omg.Multigrid(m, CG)
    assert F.n_levels == len(mg.levels)
    for l, lev in enumerate(mg.levels):
        n, c = F.level_info(l)
        assert c == lev.mesh.n and n == lev.n_dofs
        x = fem_inputs.uniform_pm1(l, n) * lev.free
        y = np.zeros(n)
        F.fem_level_apply(l, x, y)
        assert relmax(y, lev.apply(x)) <= 1e-12
        d = np.zeros(n)
        F.fem_level_diagonal(l, d)
        assert relmax(d, lev.diagonal()) <= 1e-12
        if l >= 1:
            assert abs(F.fem_level_lambda(l) - lev.lam) <= 1e-10 * lev.lam
            cm = mg.levels[l - 1]
            xc = fem_inputs.uniform_pm1(100 + l, cm.n_dofs) * cm.free
            xf = fem_inputs.uniform_pm1(200 + l, n) * lev.free
            out = xf.copy()
            F.mg_prolongate_add(l, xc, out)
            assert relmax(out, xf + mg.prolongate(l, xc)) <= 1e-12
            rc = np.zeros(cm.n_dofs)
            F.mg_restrict(l, xf, rc)
            assert relmax(rc, mg.restrict(l, xf)) <= 1e-12
    b0 = fem_inputs.uniform_pm1(9, mg.levels[0].n_dofs) * mg.levels[0].free
    x0 = np.zeros_like(b0)
    F.mg_coarse_solve(b0, x0)
    assert relmax(x0, mg.coarse_solve(b0)) <= 1e-11


def test_smoother_and_vcycle_with_pinned_lambda():
    cells, k, eps = (8, 8, 4), 3, 0.05
    m = Mesh(cells, k, eps=eps, bc=MIXED)
    mg = omg.Multigrid(m, CG)
    lam = [0.0] + [lev.lam for lev in mg.levels[1:]]
    F = fem_mod().Fem(cells, k, fem_mod().FEM_CG, deform_eps=eps, bc=MIXED, lambda_override=lam)
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


@pytest.mark.parametrize("cells,eps", [((8, 8, 8), 0.05), ((8, 8, 8), 0.0)])
def test_pcg_matches_oracle(cells, eps):
    k = 4
    F, m = make(cells, k, eps)
    mg = omg.Multigrid(m, CG)
    b = oprob.rhs(m, CG)
    hist = []
    xo, its_o, rr_o = mg.pcg(b, tol=1e-10, history=hist)
    x = np.zeros_like(b)
    its, rr, ok = F.cg_solve(b, x, rtol=1e-10)
    assert ok and rr <= 1e-10
    assert abs(its - its_o) <= 1
    true_res = np.linalg.norm(b - mg.fine.apply(x)) / np.linalg.norm(b)
    assert true_res <= 1e-9
    e_gpu, e_or = oprob.l2_error(m, CG, x), oprob.l2_error(m, CG, xo)
    assert abs(e_gpu - e_or) <= 5e-4 * e_or


@pytest.mark.slow
def test_c2_full_solve_matches_oracle():
    w = fem_inputs.C2
    F, m = make(w.cells, w.degree, w.deform_eps)
    b = np.zeros(m.cg_n_dofs())
    F.fem_rhs(b)
    assert relmax(b, oprob.rhs(m, CG)) <= 1e-12
    mg = omg.Multigrid(m, CG)
    for l in range(1, len(mg.levels)):
        assert abs(F.fem_level_lambda(l) - mg.levels[l].lam) <= 1e-9 * mg.levels[l].lam
    xo, its_o, _ = mg.pcg(b, tol=1e-10)
    x = np.zeros_like(b)
    its, rr, ok = F.cg_solve(b, x, rtol=1e-10)
    assert ok and abs(its - its_o) <= 1
    assert np.linalg.norm(b - mg.fine.apply(x)) / np.linalg.norm(b) <= 1e-9
    e_gpu, e_or = oprob.l2_error(m, CG, x), oprob.l2_error(m, CG, xo)
    assert abs(e_gpu - e_or) <= 5e-4 * e_or


@pytest.mark.slow
def test_c4_full_size_sampled_apply_and_exact_solution():
    w = fem_inputs.C4
    F, m = make(w.cells, w.degree)
    n = m.cg_n_dofs()
    x7 = fem_inputs.uniform_pm1(w.seed, n)
    xd = dev(x7)
    y = torch.zeros_like(xd)
    F.fem_apply(xd, y)
    rows = np.unique(np.concatenate([
        np.random.default_rng(0).integers(0, n, 400),
        [0, 1, m.nn[0], n // 2, n - 1, n - 2],
    ]))
    yo = ocg.apply_rows(m, x7, rows)
    yh = host(y)
    assert np.abs(yh[rows] - yo).max() <= 1e-12 * np.abs(yo).max()
    # R15: b = A x7 with Dirichlet rows zeroed -> the solution is x7 on free DoFs
    b = y.clone()
    bm = torch.from_numpy(m.cg_dirichlet_mask()).cuda()
    b[bm] = 0.0
    xs = torch.zeros_like(b)
    its, rr, ok = F.cg_solve(b, xs, rtol=1e-10)
    assert ok and its <= 8
    err = (xs - xd)[~bm]
    assert (err.norm() / xd[~bm].norm()).item() < 1e-8
    del xs, b, y
    # finest-level transfers at full size, in the launch configuration of the bench (node-grid
    # kernels): sampled fine / coarse nodes against P = P1 (x) P1 (x) P1 built from the oracle's
    # 1-D embedding, constrained nodes ignored on input and untouched on output
    L = F.n_levels - 1
    ncd, ccells = F.level_info(L - 1)
    P1 = otr._cg_1d(w.degree, ccells[0])            # [fine nodes, coarse nodes] per direction
    NF, NC = P1.shape
    assert NF ** 3 == n and NC ** 3 == ncd
    rng = np.random.default_rng(1)

    def interior(a):
        g = np.zeros(a.shape, bool)
        g[1:-1, 1:-1, 1:-1] = True
        return np.where(g, a, 0.0)

    xc = fem_inputs.uniform_pm1(11, ncd)
    xcm, xfm = interior(xc.reshape(NC, NC, NC)), interior(x7.reshape(NF, NF, NF))
    out = xd.clone()
    F.mg_prolongate_add(L, dev(xc), out)
    fs = np.vstack([rng.integers(0, NF, (300, 3)), [[0, 0, 0], [NF - 1, 5, 7], [1, 1, 1], [NF - 2, NF - 2, NF - 2],
                                                    [128, 256, 8], [129, NF - 2, 1]]])
    idx = fs[:, 0] + NF * (fs[:, 1] + NF * fs[:, 2])
    got = host(out[torch.from_numpy(idx).cuda()])
    for (fx, fy, fz), g, i in zip(fs, got, idx):
        e = x7[i]
        if 0 < fx < NF - 1 and 0 < fy < NF - 1 and 0 < fz < NF - 1:
            ix, iy, iz = (np.nonzero(P1[f])[0] for f in (fx, fy, fz))
            e += np.einsum("c,b,a,cba->", P1[fz, iz], P1[fy, iy], P1[fx, ix], xcm[np.ix_(iz, iy, ix)])
        assert abs(g - e) <= 1e-12 * 4, (fx, fy, fz)
    del out
    rc = torch.full((ncd,), 3.0, dtype=torch.float64, device="cuda")
    F.mg_restrict(L, xd, rc)
    cs = np.vstack([rng.integers(0, NC, (300, 3)), [[0, 0, 0], [NC - 1, 3, 3], [1, 1, 1], [NC - 2, NC - 2, NC - 2],
                                                    [64, 128, 4], [65, 1, NC - 2]]])
    idx = cs[:, 0] + NC * (cs[:, 1] + NC * cs[:, 2])
    got = host(rc[torch.from_numpy(idx).cuda()])
    for (cx, cy, cz), g in zip(cs, got):
        e = 0.0
        if 0 < cx < NC - 1 and 0 < cy < NC - 1 and 0 < cz < NC - 1:
            jx, jy, jz = (np.nonzero(P1[:, c])[0] for c in (cx, cy, cz))
            e = np.einsum("c,b,a,cba->", P1[jz, cz], P1[jy, cy], P1[jx, cx], xfm[np.ix_(jz, jy, jx)])
        assert abs(g - e) <= 1e-12 * 30, (cx, cy, cz)


@pytest.mark.parametrize("k", [1, 2, 4, 6, 8])
def test_cartesian_fast_path_and_general_quadrature_path_agree(k, monkeypatch):
    """The Kronecker (App. B) kernel and the quadrature kernel give the same operator."""
    cells = (5, 3, 2) if k < 6 else (2, 2, 1)
    x = fem_inputs.uniform_pm1(11, (k * cells[0] + 1) * (k * cells[1] + 1) * (k * cells[2] + 1))
    F1, m = make(cells, k, 0.0, MIXED)
    y1 = np.zeros_like(x)
    F1.fem_apply(x, y1)
    monkeypatch.setenv("FEM_GENERAL_PATH", "1")
    F2, _ = make(cells, k, 0.0, MIXED)
    y2 = np.zeros_like(x)
    F2.fem_apply(x, y2)
    yo = ocg.apply(m, x)
    assert relmax(y1, yo) <= 1e-12 and relmax(y2, yo) <= 1e-12


@pytest.mark.parametrize("env,val", [("FEM_G_DIRECT", "1"), ("FEM_FUSE_CHEB", "0"), ("FEM_FUSE_CELLS", "100000000")])
def test_layout_and_fusion_switches_keep_parity(env, val, monkeypatch):
    """Q4 deformed: G read directly from global memory instead of the default TMA-staged
    8-cell blocks; Chebyshev fusion off / on every level.  Same operator,
    PCG iterations within +-1 of the oracle's, true residual below tolerance."""
    monkeypatch.setenv(env, val)
    k, cells = 4, (8, 8, 8)
    F, m = make(cells, k, 0.05, MIXED)
    x = fem_inputs.uniform_pm1(5, m.cg_n_dofs())
    y = np.zeros_like(x)
    F.fem_apply(x, y)
    assert relmax(y, ocg.apply(m, x)) <= 1e-12
    mg = omg.Multigrid(m, CG)
    b = oprob.rhs(m, CG)
    xo, its_o, _ = mg.pcg(b, tol=1e-10)
    xs = np.zeros_like(b)
    its, rr, ok = F.cg_solve(b, xs, rtol=1e-10)
    assert ok and abs(its - its_o) <= 1
    assert np.linalg.norm(b - mg.fine.apply(xs)) / np.linalg.norm(b) <= 1e-9
    F.close()


@pytest.mark.parametrize("k,cells", [(2, (5, 3, 4)), (4, (6, 4, 3)), (7, (2, 2, 2))])
def test_metric_recomputed_on_the_fly_matches_oracle(k, cells, monkeypatch):
    """FEM_CG_GEO_FLY=1: the deformed line kernel evaluates G_q from the analytic map in its
    q-point phase instead of reading the table (same operator)."""
    monkeypatch.setenv("FEM_CG_GEO_FLY", "1")
    F, m = make(cells, k, 0.05, MIXED)
    x = fem_inputs.uniform_pm1(6, m.cg_n_dofs())
    y = np.zeros_like(x)
    F.fem_apply(x, y)
    assert relmax(y, ocg.apply(m, x)) <= 1e-12
    F.close()


def test_profile_mode_2_times_the_finest_smoother_steps(monkeypatch):
    # fem_options.profile = 2: every finest-level Chebyshev step is bracketed by events and
    # carries its algorithmic bytes (x, x_old if any, b read; x_new written): one mg_smooth from
    # x != 0 is p = 5 steps, the first without x_old -> 8 n (3 + 4 * 4) bytes
    fem = fem_mod()
    monkeypatch.setenv("FEM_ST_MIN_CELLS", "1")
    F = fem.Fem((8, 8, 8), 4, fem.FEM_CG, profile=2)
    n = F.n_local
    b = torch.ones(n, dtype=torch.float64, device="cuda")
    x = torch.zeros_like(b)
    F.mg_smooth(F.n_levels - 1, b, x, False)
    ms, launches, nbytes = F.fem_profile_read_bytes(reset=True)
    assert launches == 5 and ms > 0 and nbytes == 8.0 * n * (3 + 4 * 4)
    F.fem_profile_mode(1)                      # back to the PCG-apply channel: smoothing not timed
    F.mg_smooth(F.n_levels - 1, b, x, False)
    assert F.fem_profile_read_bytes(reset=True)[1] == 0
    F.close()


def test_conditional_graph_loop_equals_host_loop(monkeypatch):
    # the single-graph PCG loop (conditional WHILE node, on-device stopping test) and the host
    # loop run the same kernels: same iteration count, residual history and solution
    import torch
    fem = fem_mod()
    res = {}
    for cond in ("1", "0"):
        monkeypatch.setenv("FEM_COND_GRAPH", cond)
        F = fem.Fem((8, 8, 8), 3, fem.FEM_CG, deform_eps=0.05, bc=MIXED)
        b = torch.zeros(F.n_local, dtype=torch.float64, device="cuda")
        F.fem_rhs(b)
        x = torch.zeros_like(b)
        its, rr, ok = F.cg_solve(b, x, rtol=1e-10)
        x.zero_()
        its2, rr2, ok2 = F.cg_solve(b, x, rtol=1e-10)     # second call: the cached graph
        assert ok and ok2 and its == its2
        res[cond] = (its, F.cg_history(), x.cpu().numpy())
        F.close()
    assert res["1"][0] == res["0"][0]
    assert np.allclose(res["1"][1], res["0"][1], rtol=1e-9, atol=0)
    assert relmax(res["1"][2], res["0"][2]) <= 1e-11


# node-grid CG transfers (kernels_mg.cu prolongate_grid_kernel / restrict_grid_kernel): forced onto
# every level (FEM_GT_MIN_CELLS=1), several x strips with a ragged last strip (coarse n_x > 64/k),
# unmasked inputs (constrained entries must be ignored on input and left alone on output), and
# the element form (FEM_GT_MIN_CELLS huge) on the same inputs
@pytest.mark.parametrize("k,cells,bc", [
    (4, (40, 4, 2), MIXED), (4, (8, 6, 4), (DIRICHLET,) * 6), (3, (48, 2, 4), MIXED),
    (2, (72, 4, 2), MIXED), (1, (136, 2, 2), (DIRICHLET,) * 6),
    (4, (4, 2, 6), (NEUMANN, NEUMANN, DIRICHLET, NEUMANN, NEUMANN, NEUMANN)),
])
@pytest.mark.parametrize("min_cells", ["1", "1000000000"])
def test_grid_and_element_transfers_match_oracle(k, cells, bc, min_cells, monkeypatch):
    monkeypatch.setenv("FEM_GT_MIN_CELLS", min_cells)
    F, m = make(cells, k, 0.0, bc)
    mg = omg.Multigrid(m, CG)
    for l in range(1, F.n_levels):
        lev, cm = mg.levels[l], mg.levels[l - 1]
        xc = fem_inputs.uniform_pm1(300 + l, cm.n_dofs)
        xf = fem_inputs.uniform_pm1(400 + l, lev.n_dofs)
        out = xf.copy()
        F.mg_prolongate_add(l, xc, out)
        assert relmax(out, xf + mg.prolongate(l, xc)) <= 1e-12, ("prolongate", l)
        rc = np.full(cm.n_dofs, 7.0)          # the restriction overwrites its output
        F.mg_restrict(l, xf, rc)
        assert relmax(rc, mg.restrict(l, xf)) <= 1e-12, ("restrict", l)
    F.close()


def test_cg_solve_zero_ignores_x_on_entry_and_equals_cg_solve_from_zero():
    F, m = make((8, 8, 8), 3, 0.05, MIXED)
    n = m.cg_n_dofs()
    b = torch.zeros(n, dtype=torch.float64, device="cuda")
    F.fem_rhs(b)
    x1 = torch.zeros_like(b)
    its1, rr1, ok1 = F.cg_solve(b, x1, rtol=1e-10)
    h1 = F.cg_history()
    x2 = torch.full_like(b, float("nan"))            # contents on entry must not matter
    its2, rr2, ok2 = F.cg_solve_zero(b, x2, rtol=1e-10)
    assert ok1 and ok2 and its1 == its2
    assert np.allclose(F.cg_history(), h1, rtol=1e-9, atol=0)
    assert relmax(host(x2), host(x1)) <= 1e-12
    xh = np.full(n, 1e300)                            # host vectors: x is not uploaded
    its3, rr3, ok3 = F.cg_solve_zero(host(b), xh, rtol=1e-10)
    assert ok3 and its3 == its1 and relmax(xh, host(x1)) <= 1e-12
    F.close()
