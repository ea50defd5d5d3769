"""Pins of the HDG oracle (oracle/hdg.py).

CPU only.  Each pin is fixed by the mathematics, not by re-evaluating the oracle's formulas:
symmetry and definiteness of the condensed trace operator, constants in the kernel of the
pure-Neumann operator on affine meshes, exact reproduction of linear solutions (the HDG
patch test: lambda = u on the faces, u_h = u, q_h = -grad u), L2 convergence of order
k+1, the Cartesian inner Schur complement as a Kronecker sum of independently derived
1-D matrices, and the mixed form's residual vanishing at the trace solution.
"""
import numpy as np
import pytest
import scipy.sparse.linalg as spla

from oracle import hdg, problem
from oracle.basis import gauss_rule, gll_nodes, lagrange, lagrange_deriv
from oracle.mesh import Mesh, DIRICHLET as D, NEUMANN as N, SIPG


@pytest.mark.parametrize("k,eps,bc", [(1, 0.0, (D,) * 6), (2, 0.05, (D, N, D, N, N, D)),
                                      (3, 0.0, (N, D, N, D, D, N))])
def test_trace_operator_symmetric_positive_definite(k, eps, bc):
    op = hdg.HdgOperator(Mesh((2, 2, 2), k, eps=eps, bc=bc))
    K = op.assemble().toarray()
    assert np.abs(K - K.T).max() <= 1e-13 * np.abs(K).max()
    assert np.linalg.eigvalsh(0.5 * (K + K.T)).min() > 1e-4
    x = np.random.default_rng(k).standard_normal(op.n)
    assert np.allclose(op.apply(x), K @ x, rtol=0, atol=1e-13 * np.abs(K @ x).max())


@pytest.mark.parametrize("k", [1, 2, 3])
def test_pure_neumann_constants_in_kernel(k):
    # affine (Cartesian, anisotropic) cells: lambda = 1 gives u = 1, q = 0 exactly
    op = hdg.HdgOperator(Mesh((2, 3, 2), k, hi=(1.0, 0.7, 1.3), bc=(N,) * 6))
    y = op.apply(np.ones(op.n))
    assert np.abs(y).max() <= 1e-13
    K = op.assemble().toarray()
    ev = np.linalg.eigvalsh(K)
    assert abs(ev[0]) < 1e-12 and ev[1] > 1e-4      # one-dimensional kernel


@pytest.mark.parametrize("k", [1, 2, 3])
def test_patch_test_linear_solution_reproduced(k):
    # u = a.x + c with g_D = u on all faces, f = 0: HDG returns lambda = u|_F,
    # u_h = u and q_h = -a exactly (u is in every local space)
    mesh = Mesh((2, 2, 3), k, hi=(1.0, 1.2, 0.9))
    a, c = np.array([0.3, -1.1, 0.7]), 0.25
    op = hdg.HdgOperator(mesh)
    K = op.assemble(identity_dirichlet=False).tocsc()
    lam_exact = hdg.trace_node_points(mesh) @ a + c
    dm = op.dmask
    lam = lam_exact.copy()
    lam[~dm] = spla.spsolve(K[~dm][:, ~dm], -K[~dm][:, dm] @ lam_exact[dm])
    assert np.abs(lam - lam_exact).max() <= 1e-12
    # local recovery with the full trace (Dirichlet values included)
    op_nd = hdg.HdgOperator(Mesh((2, 2, 3), k, hi=(1.0, 1.2, 0.9), bc=(N,) * 6))
    Q, U = op_nd.local_solve(lam)
    xn = mesh.points(mesh.cell_coords(), np.stack(np.meshgrid(*(gll_nodes(k),) * 3, indexing='ij'),
                                                   -1)[..., ::-1].reshape(-1, 3))
    assert np.abs(U - (xn @ a + c)).max() <= 1e-12
    assert np.abs(Q + a[None, :, None]).max() <= 1e-11   # derivatives: rounding x (k+1)^2 / h


def _solve(mesh):
    op = hdg.HdgOperator(mesh)
    F = hdg.load(mesh)
    r = op.rhs(F)
    lam = spla.spsolve(op.assemble().tocsc(), r)
    return op, lam, F


@pytest.mark.parametrize("k,eps", [(1, 0.0), (2, 0.0), (2, 0.05)])
def test_l2_convergence_order_k_plus_1(k, eps):
    errs = []
    for n in (2, 4, 8):
        mesh = Mesh((n,) * 3, k, eps=eps)
        op, lam, F = _solve(mesh)
        _, U = op.local_solve(lam, F)
        errs.append(problem.l2_error(mesh, SIPG, U.ravel()))
    rates = np.log2(np.array(errs[:-1]) / np.array(errs[1:]))
    assert rates[-1] >= k + 1 - 0.3, (errs, rates)


def test_cartesian_inner_schur_complement_is_kronecker_sum():
    # S = D + E A^-1 E^T on an affine cell = J sum_d L_d (x) M (x) M (slot d), with the 1-D
    # L_d = (2/h_d)^2 Dm M^-1 Dm^T + tau (2/h_d) (e0 e0^T + eK eK^T), M_ij = int phi_i phi_j,
    # Dm_ij = int phi_i phi_j' on [-1, 1] (GLL Lagrange basis, Gauss k+1) -- derived by hand
    # from the tensor structure, independent of the quadrature-built 3-D matrices
    k, h = 3, np.array([0.5, 0.25, 0.4])
    mesh = Mesh((2, 4, 1), k, hi=tuple(h * np.array([2, 4, 1])))
    loc = hdg.LocalMatrices(mesh, np.array([0]))
    m = (k + 1) ** 3
    S = loc.D[0] + loc.E[0] @ np.linalg.solve(loc.A[0], loc.E[0].T)
    x, w = gauss_rule(k + 1)
    nodes = gll_nodes(k)
    phi, dphi = lagrange(nodes, x), lagrange_deriv(nodes, x)
    M = phi.T @ (w[:, None] * phi)
    Dm = phi.T @ (w[:, None] * dphi)
    B = np.zeros((k + 1, k + 1))
    B[0, 0] = B[k, k] = 1.0
    J = np.prod(h / 2)
    L = [(2 / h[d]) ** 2 * Dm @ np.linalg.solve(M, Dm.T) + hdg.TAU * (2 / h[d]) * B for d in range(3)]
    Sk = J * (np.kron(M, np.kron(M, L[0])) + np.kron(M, np.kron(L[1], M)) + np.kron(L[2], np.kron(M, M)))
    assert S.shape == (m, m)
    assert np.abs(S - Sk).max() <= 1e-12 * np.abs(Sk).max()


@pytest.mark.parametrize("eps", [0.0, 0.05])
def test_mixed_form_residual_vanishes_at_trace_solution(eps):
    # lambda = H_F^-1 sum_K (C q + G u) holds at the solution of the trace system, so the
    # mixed operator maps the recovered (q, u) to (0, F)
    mesh = Mesh((2, 2, 2), 2, eps=eps, bc=(D, N, D, D, N, D))
    op, lam, F = _solve(mesh)
    Q, U = op.local_solve(lam, F)
    yq, yu = hdg.mixed_apply(mesh, Q, U)
    assert np.abs(yq).max() <= 1e-11 * np.abs(F).max()
    assert np.abs(yu - F).max() <= 1e-11 * np.abs(F).max()


def test_jacobi_pcg_matches_direct_solve():
    mesh = Mesh((3, 3, 3), 2)
    op, lam, _ = _solve(mesh)
    x, its, hist = hdg.jacobi_pcg(op, op.rhs(hdg.load(mesh)), tol=1e-12)
    assert hist[-1] <= 1e-12 and its < 200
    assert np.abs(x - lam).max() <= 1e-9 * np.abs(lam).max()


@pytest.mark.parametrize("eps", [0.0, 0.05])
def test_diagonal_is_the_assembled_diagonal(eps):
    # diag(K) gathered per face node == the diagonal of the assembled K (pinned above by
    # symmetry, definiteness and the patch test); constrained rows 1
    op = hdg.HdgOperator(Mesh((2, 3, 2), 2, eps=eps, bc=(D, N, N, D, D, N)))
    assert np.abs(op.diagonal() - op.assemble().diagonal()).max() <= 1e-14 * np.abs(op.diagonal()).max()


@pytest.mark.parametrize("k,eps", [(1, 0.0), (2, 0.0), (2, 0.05)])
def test_postprocessing_superconverges_at_order_k_plus_2(k, eps):
    # the element-by-element post-processed u* converges at rate k+2 (observed on
    # hexahedra by the paper, "superconvergence ... for all constant-coefficient elliptic test
    # cases"); its cell means equal those of u_h
    errs, errs_u = [], []
    for n in (2, 4, 8):
        mesh = Mesh((n,) * 3, k, eps=eps)
        op, lam, F = _solve(mesh)
        Q, U = op.local_solve(lam, F)
        us = hdg.postprocess(mesh, Q, U)
        errs.append(problem.l2_error(Mesh((n,) * 3, k + 1, eps=eps), SIPG, us.ravel()))
        errs_u.append(problem.l2_error(mesh, SIPG, U.ravel()))
    rates = np.log2(np.array(errs[:-1]) / np.array(errs[1:]))
    assert rates[-1] >= k + 2 - 0.3, (errs, rates)
    assert errs[-1] < errs_u[-1]


def test_postprocessing_reproduces_linear_u_and_keeps_cell_means():
    # u = a.x + c: q = -a, u_h = u, so u* = u exactly; and (u*, 1)_K = (u_h, 1)_K on every cell
    from oracle.cg import CellQuadrature
    k = 2
    mesh = Mesh((2, 2, 3), k, hi=(1.0, 1.2, 0.9))
    a, c = np.array([0.3, -1.1, 0.7]), 0.25
    m = (k + 1) ** 3
    nodes = gll_nodes(k)
    xi = np.stack([nodes[np.arange(m) % (k + 1)], nodes[(np.arange(m) // (k + 1)) % (k + 1)],
                   nodes[np.arange(m) // (k + 1) ** 2]], -1)
    U = mesh.points(mesh.cell_coords(), xi) @ a + c
    Q = np.broadcast_to(-a[None, :, None], (mesh.n_cells, 3, m)).copy()
    us = hdg.postprocess(mesh, Q, U)
    m2 = (k + 2) ** 3
    n2 = gll_nodes(k + 1)
    xi2 = np.stack([n2[np.arange(m2) % (k + 2)], n2[(np.arange(m2) // (k + 2)) % (k + 2)],
                    n2[np.arange(m2) // (k + 2) ** 2]], -1)
    assert np.abs(us - (mesh.points(mesh.cell_coords(), xi2) @ a + c)).max() <= 1e-12
    # means with a random (non-linear) input
    rng = np.random.default_rng(3)
    U = rng.standard_normal((mesh.n_cells, m))
    Q = rng.standard_normal((mesh.n_cells, 3, m))
    us = hdg.postprocess(mesh, Q, U)
    q1, q2 = CellQuadrature(k + 1), CellQuadrature(k + 1)
    from oracle.mesh import eval_basis_3d
    v_lo, _ = eval_basis_3d(gll_nodes(k), q1.pts)
    W = q1.w * np.prod(mesh.h / 2)
    assert np.allclose(us @ (q2.val.T @ W), U @ (v_lo.T @ W), rtol=1e-12, atol=1e-12)
