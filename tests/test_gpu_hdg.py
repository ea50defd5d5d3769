"""HDG matrix-free operators on the GPU (include/fem_hdg.h) against the oracle (oracle/hdg.py).

SURVEY §8f N4; P:L257-326 (discretization), P:L435-480 (trace / mixed matrix-free).  Parity:
trace operator, diagonal, condensed right-hand side, local recovery and the mixed operator to
1e-12 relative max-norm (north_star's per-apply tolerance); Jacobi-PCG iterations +-1 and the
L2 error of the recovered u against the oracle's.  Degrees whose quadrature-built oracle
matrices are too large to form (k >= 6) are pinned by properties that hold exactly: the
trace of a linear function is annihilated at every interior face node and its local
recovery is the function itself (the patch test), symmetry, and constants in the kernel of
the pure-Neumann operator.
"""
import numpy as np
import pytest
import torch

import fem_inputs
from oracle import hdg as ohdg, problem
from oracle.basis import gll_nodes
from oracle.mesh import Mesh, DIRICHLET as D, NEUMANN as N, SIPG

pytestmark = pytest.mark.gpu

fem = pytest.importorskip("paper_1611_03029_b200.fem")


def rel(a, b):
    return np.abs(a - b).max() / max(np.abs(b).max(), 1e-300)


def cuda(x):
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


CASES = [((3, 2, 4), 1, (1.0, 0.6, 1.4), (D, N, D, N, N, D)),
         ((2, 3, 2), 2, (0.8, 1.0, 1.2), (D,) * 6),
         ((3, 3, 2), 3, (1.0, 1.0, 1.0), (N, D, D, N, D, N)),
         ((2, 2, 3), 4, (1.0, 1.3, 0.7), (D, D, N, N, D, D)),
         ((2, 2, 2), 5, (1.0, 1.0, 1.0), (D, N, N, D, D, N))]


@pytest.mark.parametrize("cells,k,hi,bc", CASES)
def test_trace_apply_diagonal_rhs_match_oracle(cells, k, hi, bc):
    mesh = Mesh(cells, k, hi=hi, bc=bc)
    op = ohdg.HdgOperator(mesh)
    H = fem.Hdg(cells, k, hi=hi, bc=bc)
    assert H.n_trace == op.n
    x = fem_inputs.uniform_pm1(0, op.n)
    y = torch.zeros(op.n, dtype=torch.float64, device="cuda")
    H.hdg_apply(cuda(x), y)
    assert rel(y.cpu().numpy(), op.apply(x)) <= 1e-12
    d = torch.zeros_like(y)
    H.hdg_diagonal(d)
    assert rel(d.cpu().numpy(), op.diagonal()) <= 1e-12
    r = torch.zeros_like(y)
    H.hdg_rhs(r)
    assert rel(r.cpu().numpy(), op.rhs(ohdg.load(mesh))) <= 1e-12
    H.close()


@pytest.mark.parametrize("cells,k,hi,bc", CASES[:4])
def test_local_solve_and_mixed_apply_match_oracle(cells, k, hi, bc):
    mesh = Mesh(cells, k, hi=hi, bc=bc)
    op = ohdg.HdgOperator(mesh)
    H = fem.Hdg(cells, k, hi=hi, bc=bc)
    m = (k + 1) ** 3
    lam = fem_inputs.uniform_pm1(3, op.n)
    Qo, Uo = op.local_solve(lam, ohdg.load(mesh))
    u = torch.zeros(mesh.n_cells * m, dtype=torch.float64, device="cuda")
    q = torch.zeros(3 * mesh.n_cells * m, dtype=torch.float64, device="cuda")
    H.hdg_local_solve(cuda(lam), u, q, with_f=True)
    assert rel(u.cpu().numpy(), Uo.ravel()) <= 1e-12
    qg = q.cpu().numpy().reshape(3, mesh.n_cells, m).transpose(1, 0, 2)
    assert rel(qg, Qo) <= 1e-12
    # mixed operator on random cell unknowns
    qu = fem_inputs.uniform_pm1(5, 4 * mesh.n_cells * m)
    Q = qu[:3 * mesh.n_cells * m].reshape(3, mesh.n_cells, m).transpose(1, 0, 2)
    U = qu[3 * mesh.n_cells * m:].reshape(mesh.n_cells, m)
    yq, yu = ohdg.mixed_apply(mesh, Q, U)
    y = torch.zeros(4 * mesh.n_cells * m, dtype=torch.float64, device="cuda")
    H.hdg_mixed_apply(cuda(qu), y)
    ref = np.concatenate([yq.transpose(1, 0, 2).ravel(), yu.ravel()])
    assert rel(y.cpu().numpy(), ref) <= 1e-12
    H.close()


@pytest.mark.parametrize("k", [1, 2, 3, 4, 5, 6, 7, 8])
def test_patch_test_and_invariants_all_degrees(k):
    # lambda = trace of u = a.x + c: K lambda = 0 at every interior face node (no Dirichlet
    # sides, so nothing is constrained), the local recovery (f = 0) returns u itself with
    # q = -a; K symmetric; K 1 = 0 on the pure-Neumann operator
    cells, hi = (3, 2, 2), (1.0, 0.8, 1.1)
    mesh = Mesh(cells, k, hi=hi, bc=(N,) * 6)
    H = fem.Hdg(cells, k, hi=hi, bc=(N,) * 6)
    a, c = np.array([0.4, -0.9, 1.3]), -0.2
    lam = ohdg.trace_node_points(mesh) @ a + c
    y = torch.zeros(H.n_trace, dtype=torch.float64, device="cuda")
    H.hdg_apply(cuda(lam), y)
    yv = y.cpu().numpy()
    nf = (k + 1) ** 2
    fid = ohdg.cell_face_ids(mesh)
    counts = np.bincount(fid.ravel(), minlength=sum(ohdg.n_faces(mesh)))
    interior = np.repeat(counts == 2, nf)
    scale = np.abs(yv).max()
    assert np.abs(yv[interior]).max() <= 1e-11 * max(scale, 1.0)
    m = (k + 1) ** 3
    u = torch.zeros(mesh.n_cells * m, dtype=torch.float64, device="cuda")
    q = torch.zeros(3 * mesh.n_cells * m, dtype=torch.float64, device="cuda")
    H.hdg_local_solve(cuda(lam), u, q, with_f=False)
    nodes = gll_nodes(k)
    xi = np.stack([nodes[np.arange(m) % (k + 1)], nodes[(np.arange(m) // (k + 1)) % (k + 1)],
                   nodes[np.arange(m) // (k + 1) ** 2]], -1)
    xn = mesh.points(mesh.cell_coords(), xi)
    assert np.abs(u.cpu().numpy().reshape(mesh.n_cells, m) - (xn @ a + c)).max() <= 1e-11
    assert np.abs(q.cpu().numpy().reshape(3, -1) + a[:, None]).max() <= 1e-9
    H.hdg_apply(cuda(np.ones(H.n_trace)), y)
    assert np.abs(y.cpu().numpy()).max() <= 1e-11
    x1, x2 = fem_inputs.uniform_pm1(1, H.n_trace), fem_inputs.uniform_pm1(2, H.n_trace)
    y1, y2 = torch.zeros_like(y), torch.zeros_like(y)
    H.hdg_apply(cuda(x1), y1)
    H.hdg_apply(cuda(x2), y2)
    s12, s21 = x2 @ y1.cpu().numpy(), x1 @ y2.cpu().numpy()
    assert abs(s12 - s21) <= 1e-12 * np.abs(y1.cpu().numpy()).max() * np.abs(x2).sum()
    H.close()


@pytest.mark.parametrize("n,k", [(4, 2), (4, 3)])
def test_jacobi_pcg_solve_matches_oracle(n, k):
    mesh = Mesh((n,) * 3, k)
    op = ohdg.HdgOperator(mesh)
    F = ohdg.load(mesh)
    b = op.rhs(F)
    xo, its_o, hist_o = ohdg.jacobi_pcg(op, b, tol=1e-10)
    H = fem.Hdg((n,) * 3, k)
    bg = torch.zeros(H.n_trace, dtype=torch.float64, device="cuda")
    H.hdg_rhs(bg)
    lam = torch.zeros_like(bg)
    its, rr, ok = H.hdg_cg_solve(bg, lam, rtol=1e-10)
    assert ok and abs(its - its_o) <= 1, (its, its_o)
    assert rel(lam.cpu().numpy(), xo) <= 1e-7
    u = torch.zeros(mesh.n_cells * (k + 1) ** 3, dtype=torch.float64, device="cuda")
    H.hdg_local_solve(lam, u, with_f=True)
    _, Uo = op.local_solve(xo, F)
    e_gpu = problem.l2_error(mesh, SIPG, u.cpu().numpy())
    e_or = problem.l2_error(mesh, SIPG, Uo.ravel())
    assert abs(e_gpu - e_or) <= 1e-6 * e_or
    H.close()


def test_errors():
    with pytest.raises(fem.FemError) as e:
        fem.Hdg((2, 2, 2), 9)
    assert e.value.code == -1
    H = fem.Hdg((2, 2, 2), 2)
    with pytest.raises(fem.FemError) as e:
        H.hdg_apply(np.zeros(H.n_trace), np.zeros(H.n_trace))     # host pointers
    assert e.value.code == -1
    with pytest.raises(fem.FemError) as e:
        H.hdg_apply(torch.zeros(3, dtype=torch.float64, device="cuda"),
                    torch.zeros(H.n_trace, dtype=torch.float64, device="cuda"))
    assert e.value.code == -2
    H.close()


# ---- the paper's design: inner Schur complement inverse stored per cell (deformed meshes, and
# Cartesian ones with FEM_HDG_DENSE=1)
CURVED = [((2, 2, 2), 1, 0.05, (D, N, D, N, N, D)),
          ((2, 3, 2), 2, 0.05, (D,) * 6),
          ((2, 2, 2), 3, 0.05, (N, D, D, N, D, N)),
          ((2, 2, 2), 4, 0.05, (D, D, N, N, D, D)),
          ((3, 2, 2), 2, 0.0, (D, N, D, D, N, D))]


@pytest.mark.parametrize("cells,k,eps,bc", CURVED)
def test_stored_inverse_path_matches_oracle(cells, k, eps, bc, monkeypatch):
    monkeypatch.setenv("FEM_HDG_DENSE", "1")
    mesh = Mesh(cells, k, eps=eps, bc=bc)
    op = ohdg.HdgOperator(mesh)
    H = fem.Hdg(cells, k, bc=bc, deform_eps=eps)
    x = fem_inputs.uniform_pm1(0, op.n)
    y = torch.zeros(op.n, dtype=torch.float64, device="cuda")
    H.hdg_apply(cuda(x), y)
    assert rel(y.cpu().numpy(), op.apply(x)) <= 1e-11
    d = torch.zeros_like(y)
    H.hdg_diagonal(d)
    assert rel(d.cpu().numpy(), op.diagonal()) <= 1e-11
    r = torch.zeros_like(y)
    H.hdg_rhs(r)
    F = ohdg.load(mesh)
    assert rel(r.cpu().numpy(), op.rhs(F)) <= 1e-11
    m = (k + 1) ** 3
    Qo, Uo = op.local_solve(x, F)
    u = torch.zeros(mesh.n_cells * m, dtype=torch.float64, device="cuda")
    q = torch.zeros(3 * mesh.n_cells * m, dtype=torch.float64, device="cuda")
    H.hdg_local_solve(cuda(x), u, q, with_f=True)
    assert rel(u.cpu().numpy(), Uo.ravel()) <= 1e-11
    assert rel(q.cpu().numpy().reshape(3, mesh.n_cells, m).transpose(1, 0, 2), Qo) <= 1e-11
    H.close()


def test_deformed_solve_converges_at_order_k_plus_1():
    errs = []
    for n in (2, 4, 8):
        mesh = Mesh((n,) * 3, 2, eps=0.05)
        H = fem.Hdg((n,) * 3, 2, deform_eps=0.05)
        b = torch.zeros(H.n_trace, dtype=torch.float64, device="cuda")
        H.hdg_rhs(b)
        lam = torch.zeros_like(b)
        its, rr, ok = H.hdg_cg_solve(b, lam, rtol=1e-12)
        assert ok
        u = torch.zeros(H.n_cell_dofs, dtype=torch.float64, device="cuda")
        H.hdg_local_solve(lam, u, with_f=True)
        errs.append(problem.l2_error(mesh, SIPG, u.cpu().numpy()))
        H.close()
    rate = np.log2(errs[-2] / errs[-1])
    assert rate >= 3 - 0.3, errs


@pytest.mark.parametrize("cells,k,hi,bc", CASES[:4])
def test_postprocessing_matches_oracle(cells, k, hi, bc):
    mesh = Mesh(cells, k, hi=hi, bc=bc)
    m = (k + 1) ** 3
    rng = np.random.default_rng(k)
    Q = rng.uniform(-1, 1, (mesh.n_cells, 3, m))
    U = rng.uniform(-1, 1, (mesh.n_cells, m))
    ref = ohdg.postprocess(mesh, Q, U)
    H = fem.Hdg(cells, k, hi=hi, bc=bc)
    us = torch.zeros(mesh.n_cells * (k + 2) ** 3, dtype=torch.float64, device="cuda")
    H.hdg_postprocess(cuda(Q.transpose(1, 0, 2).ravel()), cuda(U.ravel()), us)
    assert rel(us.cpu().numpy(), ref.ravel()) <= 1e-11
    H.close()


def test_postprocessed_solution_superconverges():
    # GPU solve -> local recovery -> post-processing: order k + 2
    k, errs = 2, []
    for n in (4, 8, 16):
        H = fem.Hdg((n,) * 3, k)
        b = torch.zeros(H.n_trace, dtype=torch.float64, device="cuda")
        H.hdg_rhs(b)
        lam = torch.zeros_like(b)
        its, rr, ok = H.hdg_cg_solve(b, lam, rtol=1e-12)
        assert ok
        u = torch.zeros(H.n_cell_dofs, dtype=torch.float64, device="cuda")
        q = torch.zeros(3 * H.n_cell_dofs, dtype=torch.float64, device="cuda")
        H.hdg_local_solve(lam, u, q, with_f=True)
        us = torch.zeros(H.n_cells * (k + 2) ** 3, dtype=torch.float64, device="cuda")
        H.hdg_postprocess(q, u, us)
        errs.append(problem.l2_error(Mesh((n,) * 3, k + 1), SIPG, us.cpu().numpy()))
        H.close()
    rate = np.log2(errs[-2] / errs[-1])
    assert rate >= k + 2 - 0.3, errs
