"""Pins of the CPU oracle against closed forms, invariants, golden values and
brute force (no GPU).  Each test names the fact it pins; none retypes the
oracle's own formula."""
import numpy as np
import pytest
import scipy.sparse.linalg as spla
from numpy.polynomial import chebyshev as C

import fem_inputs
from oracle import basis, cg, sipg, transfer, multigrid, problem
from oracle.mesh import Mesh, CG, SIPG, DIRICHLET, NEUMANN, tensor_points
from tests.conftest import golden


# ------------------------------------------------------------------ inputs
def test_splitmix64_reference_vector():
    g = golden("splitmix64.json")
    out = fem_inputs.splitmix64(g["seed"], 0, len(g["outputs"]))
    assert [int(v) for v in out] == [int(s) for s in g["outputs"]]


def test_uniform_is_partition_independent_and_in_range():
    full = fem_inputs.uniform_pm1(7, 1000)
    part = np.concatenate([fem_inputs.uniform_pm1(7, 300, 0), fem_inputs.uniform_pm1(7, 700, 300)])
    assert np.array_equal(full, part)
    assert full.min() >= -1.0 and full.max() < 1.0 and abs(full.mean()) < 0.1


# ------------------------------------------------------------------ 1-D rules
def test_gauss_and_gll_closed_forms():
    g = golden("rules_1d.json")
    for n, ref in g["gauss"].items():
        x, w = basis.gauss_rule(int(n))
        assert np.allclose(x, ref["x"], atol=1e-15) and np.allclose(w, ref["w"], atol=1e-15)
    for k, ref in g["gll"].items():
        assert np.allclose(basis.gll_nodes(int(k)), ref, atol=1e-15)


@pytest.mark.parametrize("n", range(1, 10))
def test_gauss_exact_to_degree_2n_minus_1(n):
    x, w = basis.gauss_rule(n)
    for p in range(2 * n):
        exact = 0.0 if p % 2 else 2.0 / (p + 1)
        assert abs(w @ x ** p - exact) < 1e-13


@pytest.mark.parametrize("k", range(1, 9))
def test_lagrange_delta_partition_of_unity_derivative(k):
    nodes = basis.gll_nodes(k)
    assert np.allclose(basis.lagrange(nodes, nodes), np.eye(k + 1), atol=1e-13)
    xi = np.linspace(-1, 1, 17)
    assert np.allclose(basis.lagrange(nodes, xi).sum(1), 1.0, atol=1e-13)
    assert np.allclose(basis.lagrange_deriv(nodes, xi).sum(1), 0.0, atol=1e-11)
    # derivative of the interpolant of xi^k is k xi^(k-1) exactly
    d = basis.lagrange_deriv(nodes, xi) @ nodes ** k
    assert np.allclose(d, k * xi ** (k - 1), atol=1e-11)
    # GLL nodes are the roots of (1-x^2) P_k'
    from numpy.polynomial import legendre as L
    assert np.allclose((1 - nodes ** 2) * L.Legendre.basis(k).deriv()(nodes), 0, atol=1e-12)


@pytest.mark.parametrize("k", [1, 2])
def test_1d_mass_stiffness_closed_forms(k):
    g = golden("rules_1d.json")
    b = basis.Basis1D(k)
    M = (b.val * b.qw[:, None]).T @ b.val
    S = (b.der * b.qw[:, None]).T @ b.der
    assert np.allclose(M, g["mass"][str(k)]["scale"] * np.array(g["mass"][str(k)]["M"]), atol=1e-15)
    assert np.allclose(S, g["stiffness"][str(k)]["scale"] * np.array(g["stiffness"][str(k)]["S"]),
                       atol=1e-14)


# ------------------------------------------------------------------ geometry
@pytest.mark.parametrize("eps", [0.0, 0.05, 0.1])
def test_jacobian_matches_finite_differences_and_det_lemma(eps):
    m = Mesh((3, 2, 4), 3, eps=eps)
    cc = m.cell_coords(np.array([0, 5, 23]))
    xi = np.array([[0.3, -0.7, 0.1], [-1, 1, 0.5], [0.9, 0.2, -0.4]])
    J = m.jacobian(cc, xi)
    hstep = 1e-6
    for e in range(3):
        dp, dm = xi.copy(), xi.copy()
        dp[:, e] += hstep
        dm[:, e] -= hstep
        fd = (m.phys(m.xhat(cc, dp)) - m.phys(m.xhat(cc, dm))) / (2 * hstep)
        assert np.allclose(J[..., e], fd, atol=1e-9)
    # det(I + eps 1 grad s^T) = 1 + eps (grad s . 1)  (matrix determinant lemma)
    xh = m.xhat(cc, xi)
    s = [np.sin(np.pi * xh[..., d]) for d in range(3)]
    c = [np.cos(np.pi * xh[..., d]) for d in range(3)]
    gs = np.pi * (c[0] * s[1] * s[2] + s[0] * c[1] * s[2] + s[0] * s[1] * c[2])
    assert np.allclose(np.linalg.det(J), (1 + eps * gs) * np.prod(m.h / 2), rtol=1e-14)


@pytest.mark.parametrize("k,n", [(2, 4), (4, 8), (6, 3)])
def test_volume_sums_to_one_on_deformed_mesh(k, n):
    m = Mesh((n, n, n), k, eps=0.05)
    q = cg.CellQuadrature(k)
    _, detJ = cg.cell_geometry(m, np.arange(m.n_cells), q)
    assert abs(np.sum(detJ @ q.w) - 1.0) < 1e-13


# ------------------------------------------------------------------ CG operator
def _kron_element(M, S, h):
    # local index i0 + n i1 + n^2 i2 => kron order (z, y, x)
    return (h / 2) * (np.kron(M, np.kron(M, S)) + np.kron(M, np.kron(S, M)) + np.kron(S, np.kron(M, M)))


@pytest.mark.parametrize("k", [1, 2])
def test_cartesian_element_matrix_equals_kronecker_closed_form(k):
    g = golden("rules_1d.json")
    M = g["mass"][str(k)]["scale"] * np.array(g["mass"][str(k)]["M"])
    S = g["stiffness"][str(k)]["scale"] * np.array(g["stiffness"][str(k)]["S"])
    m = Mesh((4, 4, 4), k)
    assert np.allclose(cg.element_matrix(m, 9), _kron_element(M, S, 0.25), atol=1e-15)


def test_q1_element_and_stencil():
    g = golden("q1_stencil.json")
    h = 0.25
    m = Mesh((4, 4, 4), 1)
    Ke = cg.element_matrix(m, 0) / h
    el = g["element_over_h"]
    assert np.isclose(Ke[0, 0], el["diagonal"])
    assert np.isclose(Ke[0, 1], el["edge_adjacent"], atol=1e-15)
    assert np.isclose(Ke[0, 3], el["face_diagonal"])
    assert np.isclose(Ke[0, 7], el["body_diagonal"])
    A = cg.assemble(m)
    st = g["stencil_over_h"]
    nn = m.nn[0]
    c = 2 + nn * (2 + nn * 2)
    row = A[c].toarray().ravel() / h
    assert np.isclose(row[c], st["centre"])
    assert np.isclose(row[c + 1], st["face_neighbour"], atol=1e-15)
    assert np.isclose(row[c + 1 + nn], st["edge_neighbour"])
    assert np.isclose(row[c + 1 + nn + nn * nn], st["corner_neighbour"])


def test_c1_diagonal_exact():
    g = golden("c1_diagonal.json")
    w = fem_inputs.C1
    m = Mesh(w.cells, w.degree)
    d = cg.diagonal(m)
    mask = m.cg_dirichlet_mask()
    assert len(d) == g["n_dofs"] and mask.sum() == g["n_constrained"]
    assert np.all(d[mask] == g["constrained"])
    gc = m.cg_node_coords()
    n_mid = (gc % 2 == 1).sum(axis=1)
    vals = [g["free_values"][kk] for kk in ("vvv", "one_m", "two_m", "mmm")]
    expect = np.array(vals)[n_mid]
    assert np.allclose(d[~mask], expect[~mask], rtol=1e-14, atol=0)


def test_cg_cartesian_stored_element_matrix_mode_equals_dense_b():
    """Mode O3-ii (one stored K^e on a Cartesian mesh, used by Operator.apply) against the
    dense-B quadrature evaluation B^T (G o (B x_e)) of every row (apply_rows), k = 4."""
    m = Mesh((3, 2, 2), 4, bc=(DIRICHLET, NEUMANN, DIRICHLET, DIRICHLET, NEUMANN, DIRICHLET))
    x = np.random.default_rng(5).standard_normal(m.cg_n_dofs())
    y = cg.apply(m, x)
    rows = np.arange(m.cg_n_dofs())
    assert np.abs(cg.apply_rows(m, x, rows) - y).max() <= 1e-13 * np.abs(y).max()


@pytest.mark.parametrize("k,eps", [(1, 0.0), (2, 0.05), (3, 0.05), (4, 0.0)])
def test_cg_apply_modes_agree_symmetric_positive(k, eps):
    m = Mesh((3, 2, 4), k, eps=eps, bc=(DIRICHLET, NEUMANN, DIRICHLET, DIRICHLET, NEUMANN, DIRICHLET))
    rng = np.random.default_rng(1)
    x, z = rng.standard_normal((2, m.cg_n_dofs()))
    A = cg.assemble(m)
    y = cg.apply(m, x)
    assert np.abs(A @ x - y).max() <= 1e-13 * np.abs(y).max()
    assert abs(z @ cg.apply(m, x) - x @ cg.apply(m, z)) < 1e-12 * np.linalg.norm(x) * np.linalg.norm(z) * 10
    assert np.allclose(A.diagonal(), cg.diagonal(m), rtol=1e-13)
    rows = np.array([0, 7, 33, m.cg_n_dofs() // 2, m.cg_n_dofs() - 1])
    assert np.allclose(cg.apply_rows(m, x, rows), y[rows], rtol=1e-13, atol=1e-13)
    assert spla.eigsh(A, k=1, which="SA", return_eigenvectors=False)[0] > 0


@pytest.mark.parametrize("method", [CG, SIPG])
@pytest.mark.parametrize("eps", [0.0, 0.05])
def test_constants_in_kernel_of_pure_neumann_operator(method, eps):
    m = Mesh((3, 3, 2), 3, eps=eps, bc=(NEUMANN,) * 6)
    if method == CG:
        y = cg.apply(m, np.ones(m.cg_n_dofs()))
    else:
        y = sipg.apply(m, np.ones(m.dg_n_dofs()))
    assert np.abs(y).max() < 1e-12


# ------------------------------------------------------------------ SIPG operator
def _sipg_1d(k, N, c_pen, dirichlet=True):
    """1-D SIPG matrix on [0,1], N cells (independent 1-D assembly) and the 1-D mass."""
    b = basis.Basis1D(k)
    n, h = k + 1, 1.0 / N
    Mref = (b.val * b.qw[:, None]).T @ b.val
    Sref = (b.der * b.qw[:, None]).T @ b.der
    l0, l1 = basis.lagrange(b.nodes, [-1.0])[0], basis.lagrange(b.nodes, [1.0])[0]
    d0, d1 = basis.lagrange_deriv(b.nodes, [-1.0])[0] * 2 / h, basis.lagrange_deriv(b.nodes, [1.0])[0] * 2 / h
    sigma = c_pen * (k + 1) ** 2 / h
    A = np.zeros((N * n, N * n))
    Mm = np.zeros_like(A)
    for c in range(N):
        s = slice(c * n, (c + 1) * n)
        A[s, s] += (2 / h) * Sref
        Mm[s, s] += (h / 2) * Mref
    for c in range(N - 1):   # point between c (minus, n=+1) and c+1
        vm, vp, gm, gp = l1, l0, d1, d0
        blocks = {(0, 0): (vm, gm, vm, gm, 1, 1), (0, 1): (vm, gm, vp, gp, 1, -1),
                  (1, 0): (vp, gp, vm, gm, -1, 1), (1, 1): (vp, gp, vp, gp, -1, -1)}
        for (s_, t_), (v, dv, u, du, ss, st) in blocks.items():
            blk = (-ss * np.outer(v, 0.5 * du) - np.outer(0.5 * dv, st * u) + sigma * ss * st * np.outer(v, u))
            A[(c + s_) * n:(c + s_ + 1) * n, (c + t_) * n:(c + t_ + 1) * n] += blk
    if dirichlet:
        for c, v, dv, nrm in ((0, l0, d0, -1.0), (N - 1, l1, d1, 1.0)):
            dn = nrm * dv
            A[c * n:(c + 1) * n, c * n:(c + 1) * n] += -np.outer(v, dn) - np.outer(dn, v) + 2 * sigma * np.outer(v, v)
    return A, Mm


@pytest.mark.parametrize("k,N", [(1, 3), (2, 2), (3, 2)])
def test_cartesian_sipg_is_kronecker_sum_of_1d_sipg(k, N):
    A1, M1 = _sipg_1d(k, N, 2.0)
    # 1-D DG index (cell, local) -> the 3-D DG numbering (cells lexicographic, local x fastest)
    n = k + 1
    A = sipg.assemble(Mesh((N, N, N), k), 2.0).toarray()
    Ak = (np.kron(M1, np.kron(M1, A1)) + np.kron(M1, np.kron(A1, M1)) + np.kron(A1, np.kron(M1, M1)))
    # permutation: tensor index (gz, gy, gx) with g = cell*n + l  ->  DG index
    g = np.arange((N * n) ** 3)
    gx, gy, gz = g % (N * n), (g // (N * n)) % (N * n), g // (N * n) ** 2
    cell = gx // n + N * (gy // n + N * (gz // n))
    dgi = cell * n ** 3 + gx % n + n * (gy % n + n * (gz % n))
    P = np.zeros_like(Ak)
    P[dgi, g] = 1.0
    assert np.abs(P @ Ak @ P.T - A).max() < 1e-12 * np.abs(A).max()


@pytest.mark.parametrize("k,eps", [(1, 0.0), (2, 0.05), (3, 0.05)])
def test_sipg_apply_modes_agree_symmetric_positive(k, eps):
    m = Mesh((3, 2, 2), k, eps=eps, bc=(DIRICHLET, NEUMANN, DIRICHLET, DIRICHLET, NEUMANN, DIRICHLET))
    x = np.random.default_rng(2).standard_normal(m.dg_n_dofs())
    A = sipg.assemble(m)
    y = sipg.apply(m, x)
    assert np.abs(A @ x - y).max() <= 1e-13 * np.abs(y).max()
    assert np.abs(A - A.T).max() < 1e-12 * np.abs(A).max()
    assert np.allclose(A.diagonal(), sipg.diagonal(m), rtol=1e-13)
    cells = np.array([0, 5, 11])
    assert np.allclose(sipg.apply_cells(m, x, cells), y.reshape(m.n_cells, -1)[cells], rtol=1e-13, atol=1e-12)
    assert spla.eigsh(A, k=1, which="SA", return_eigenvectors=False)[0] > 0


def test_sipg_penalty_on_cartesian_config():
    m = Mesh((32, 32, 32), 4)
    q = cg.CellQuadrature(4)
    fd = sipg.InteriorFaces(m, 0, np.array([0]), np.array([1]), q, 2.0)
    assert np.isclose(fd.sigma[0], 1600.0)   # 2 (k+1)^2 / h = 2*25*32


# ------------------------------------------------------------------ transfers
@pytest.mark.parametrize("method", [CG, SIPG])
@pytest.mark.parametrize("k", [1, 2, 3, 4])
def test_transfer_explicit_equals_tensorial_and_transpose(method, k):
    f = Mesh((4, 2, 4), k, bc=(DIRICHLET, NEUMANN, DIRICHLET, DIRICHLET, NEUMANN, DIRICHLET))
    c = transfer.coarsen(f)
    P = transfer.prolongation_matrix(c, f, method)
    rng = np.random.default_rng(3)
    nc, nf = P.shape[1], P.shape[0]
    xc, xf = rng.standard_normal(nc), rng.standard_normal(nf)
    if method == CG:
        xc[c.cg_dirichlet_mask()] = 0
        xf[f.cg_dirichlet_mask()] = 0
    pc = transfer.prolongate(c, f, method, xc)
    rf = transfer.restrict(c, f, method, xf)
    assert np.abs(P @ xc - pc).max() < 1e-13 and np.abs(P.T @ xf - rf).max() < 1e-12
    assert abs(pc @ xf - xc @ rf) < 1e-11


@pytest.mark.parametrize("method", [CG, SIPG])
def test_prolongation_reproduces_polynomials(method):
    k = 3
    f = Mesh((4, 4, 2), k, bc=(NEUMANN,) * 6)
    c = transfer.coarsen(f)
    poly = lambda p: p[:, 0] ** 3 - 2 * p[:, 1] ** 2 * p[:, 0] + p[:, 2] ** 3 * p[:, 1] ** 0 + 0.5

    def nodal(m):
        nodes = basis.gll_nodes(k)
        if method == CG:
            g = m.cg_node_coords()
            fc = np.minimum(g // k, np.asarray(m.n) - 1)
            t = (fc + 0.5 * (nodes[g - k * fc] + 1)) / np.asarray(m.n)
        else:
            cc = np.repeat(m.cell_coords(), (k + 1) ** 3, axis=0)
            loc = np.tile(tensor_points(nodes), (m.n_cells, 1))
            t = (cc + 0.5 * (loc + 1)) / np.asarray(m.n)
        return poly(t)
    assert np.abs(transfer.prolongate(c, f, method, nodal(c)) - nodal(f)).max() < 1e-12


# ------------------------------------------------------------------ Chebyshev / lambda / V-cycle / PCG
def test_chebyshev_error_polynomial_is_scaled_chebyshev():
    m = Mesh((3, 3, 3), 1, bc=(DIRICHLET,) * 6)
    lev = multigrid.Level(m, CG, 2.0)
    A = cg.assemble(m).toarray()
    free = lev.free
    Af = A[np.ix_(free, free)]
    D = np.diag(Af)
    lam = np.linalg.eigvals(np.diag(1 / D) @ Af).real
    lev.lam = lam.max() / 1.2 * 1.0001
    p = 5
    a, c = 1.2 * lev.lam, 0.06 * lev.lam
    theta, delta = (a + c) / 2, (a - c) / 2
    # error propagation on an eigenvector of D^-1 A:  b = 0, x0 = v -> x_p = E v
    w, V = np.linalg.eig(np.diag(1 / D) @ Af)
    for j in range(len(w)):
        v = np.zeros(m.cg_n_dofs())
        v[free] = V[:, j].real
        xp = multigrid.chebyshev(lev, np.zeros_like(v), v, p, 0.06, 1.2, False)
        expect = C.chebval((theta - w[j].real) / delta, [0] * p + [1]) / C.chebval(theta / delta, [0] * p + [1])
        assert np.allclose(xp[free], expect * v[free], atol=1e-12)


def test_chebyshev_damping_bound():
    # worst-case damping of the degree-5 polynomial on [0.06, 1.2]: 1/T5(1.26/1.14)
    assert abs(1 / C.chebval(1.26 / 1.14, [0] * 5 + [1]) - 0.2035) < 1e-4


@pytest.mark.parametrize("n,lam_exact", [(4, 1.21339), (8, 1.41053)])
def test_jacobi_spectrum_q1_closed_form_and_lanczos_estimate(n, lam_exact):
    h = 1.0 / n
    th = np.arange(1, n) * np.pi / n
    s, mm = (2 - 2 * np.cos(th)) / h, h * (4 + 2 * np.cos(th)) / 6
    lam = (3 / (8 * h)) * (s[:, None, None] * mm[None, :, None] * mm[None, None, :]
                           + mm[:, None, None] * s[None, :, None] * mm[None, None, :]
                           + mm[:, None, None] * mm[None, :, None] * s[None, None, :])
    assert abs(lam.max() - lam_exact) < 1e-5
    m = Mesh((n, n, n), 1)
    A = cg.assemble(m).toarray()
    free = ~m.cg_dirichlet_mask()
    Af = A[np.ix_(free, free)]
    dense = np.linalg.eigvals(np.diag(1 / np.diag(Af)) @ Af).real.max()
    assert abs(dense - lam.max()) < 1e-10
    est, _ = multigrid.estimate_lambda_max(multigrid.Level(m, CG, 2.0))
    assert 0.9 * dense <= est <= dense * (1 + 1e-12)


@pytest.mark.parametrize("method,k", [(CG, 2), (SIPG, 2)])
def test_vcycle_linear_symmetric_and_two_level_contraction(method, k):
    m = Mesh((4, 4, 4), k, eps=0.05)
    mg = multigrid.Multigrid(m, method)
    N = mg.fine.n_dofs
    rng = np.random.default_rng(4)
    b1, b2 = rng.standard_normal((2, N)) * mg.fine.free
    v1, v2 = mg.vcycle(b1), mg.vcycle(b2)
    assert abs(v1 @ b2 - b1 @ v2) < 1e-11 * abs(v1 @ b2)
    assert np.allclose(mg.vcycle(2 * b1 + b2), 2 * v1 + v2, atol=1e-11 * np.abs(v1).max())


def test_two_level_error_propagation_spectral_radius():
    m = Mesh((4, 4, 4), 2)
    mg = multigrid.Multigrid(m, CG)
    free = np.nonzero(mg.fine.free)[0]
    A = cg.assemble(m).toarray()[np.ix_(free, free)]
    E = np.zeros((len(free), len(free)))
    for j in range(len(free)):
        e = np.zeros(mg.fine.n_dofs)
        e[free[j]] = 1.0
        r = np.zeros(mg.fine.n_dofs)
        r[free] = A @ e[free]
        E[:, j] = (e - mg.vcycle(r))[free]
    assert np.max(np.abs(np.linalg.eigvals(E))) < 0.5


def test_pcg_identity_like_and_exact_solution_pin():
    m = Mesh((8, 8, 8), 4)
    mg = multigrid.Multigrid(m, CG)
    xr = fem_inputs.uniform_pm1(7, mg.fine.n_dofs) * mg.fine.free
    b = mg.fine.apply(xr)
    b[~mg.fine.free] = 0
    x, its, rr = mg.pcg(b, tol=1e-10)
    assert rr <= 1e-10 and its <= 8
    assert np.linalg.norm(x - xr) / np.linalg.norm(xr) < 1e-9


def test_galerkin_exactness_quadratic_solution():
    # u = prod x_d(1 - x_d) in Q_k (k >= 2): the discrete solution is its interpolant
    for method in (CG, SIPG):
        m = Mesh((3, 3, 3), 2)
        mg = multigrid.Multigrid(m, method, coarse_cells=3)
        q = cg.CellQuadrature(2)
        cells = np.arange(m.n_cells)
        xq = m.phys(m.xhat(m.cell_coords(cells), q.pts))
        u = lambda p: np.prod(p * (1 - p), axis=-1)
        f = 2 * (xq[..., 1] * (1 - xq[..., 1]) * xq[..., 2] * (1 - xq[..., 2])
                 + xq[..., 0] * (1 - xq[..., 0]) * xq[..., 2] * (1 - xq[..., 2])
                 + xq[..., 0] * (1 - xq[..., 0]) * xq[..., 1] * (1 - xq[..., 1]))
        be = (f * (np.prod(m.h) / 8) * q.w) @ q.val
        nodes = basis.gll_nodes(2)
        if method == CG:
            dm = m.cg_dofmap()
            b = np.bincount(dm.ravel(), be.ravel(), m.cg_n_dofs())
            b[m.cg_dirichlet_mask()] = 0
            g = m.cg_node_coords()
            ui = u(g / (2 * np.asarray(m.n)))
        else:
            b = be.ravel()
            cc = np.repeat(m.cell_coords(), 27, axis=0)
            ui = u((cc + 0.5 * (np.tile(tensor_points(nodes), (m.n_cells, 1)) + 1)) / 3)
        x, _, _ = mg.pcg(b, tol=1e-13)
        assert np.abs(x - ui).max() < 1e-12


@pytest.mark.parametrize("method", [CG, SIPG])
@pytest.mark.parametrize("eps", [0.0, 0.05])
def test_l2_convergence_order(method, eps):
    k = 2
    errs = []
    for n in (4, 8):
        m = Mesh((n, n, n), k, eps=eps)
        mg = multigrid.Multigrid(m, method)
        x, _, _ = mg.pcg(problem.rhs(m, method), tol=1e-12)
        errs.append(problem.l2_error(m, method, x))
    assert np.log2(errs[0] / errs[1]) > k + 1 - 0.3


@pytest.mark.slow
def test_pcg_iteration_counts_match_independent_prototype():
    g = golden("prototype_iterations.json")
    for case in g["cases"]:
        method = CG if case["method"] == "CG" else SIPG
        m = Mesh((case["n"],) * 3, case["k"])
        mg = multigrid.Multigrid(m, method)
        _, its, rr = mg.pcg(problem.rhs(m, method), tol=1e-10)
        assert rr <= 1e-10
        assert abs(its - case["iterations"]) <= g["tolerance_iterations"], case


# ---------------------------------------------------------------- the paper's own problem (N2)
@pytest.mark.parametrize("k", [2, 3, 4])
def test_paper_gaussian_problem_errors_match_printed_values(k):
    """eq:pois_analytic on (-1,1)^3 (Neumann at x_e=-1, Dirichlet at +1, sigma with d=3,
    tol 1e-9): the oracle's CG and SIPG solutions reproduce the L2 errors the paper
    prints for 8^3 cells (tests/golden/paper_gaussian_errors.json) to 2%,
    and the iteration counts within the +-2 envelope (the paper's multigrid setup differs:
    coarse solver, smoother degree, residual norm)."""
    from oracle import gaussians as gs, multigrid as omg
    from oracle.mesh import CG, SIPG
    row = next(r for r in golden("paper_gaussian_errors.json")["rows"] if r["k"] == k and r["cells"] == 512)
    m = gs.mesh((8, 8, 8), k)
    b = gs.rhs(m, CG)
    x0 = np.where(m.cg_dirichlet_mask(), b, 0.0)
    x, its, rr = omg.Multigrid(m, CG).pcg(b, tol=1e-9, x0=x0)
    assert rr <= 1e-9
    assert abs(gs.l2_error_abs(m, CG, x) / row["FEL2"] - 1.0) <= 0.02
    assert abs(its - row["qIt"]) <= 2
    bd = gs.rhs(m, SIPG)
    xd, itd, rd = omg.Multigrid(m, SIPG, penalty_factor=gs.PENALTY_FACTOR).pcg(bd, tol=1e-9)
    assert rd <= 1e-9
    assert abs(gs.l2_error_abs(m, SIPG, xd) / row["dgL2"] - 1.0) <= 0.02
    assert abs(itd - row["dgIt"]) <= 2


def test_paper_gaussian_problem_data():
    """The problem data is what eq:pois_analytic states: f = -Laplace u checked by finite
    differences, g_N = -n.grad u, the Gaussian normalisation (integral of one Gaussian
    over R^3 = alpha^3 (pi)^(3/2) (alpha sqrt(2 pi))^-3 = 2^(-3/2))."""
    from oracle import gaussians as gs
    rng = np.random.default_rng(3)
    x = rng.uniform(-1, 1, (20, 3))
    h = 1e-4
    lap = sum((gs.exact_u(x + h * e) - 2 * gs.exact_u(x) + gs.exact_u(x - h * e)) / h ** 2 for e in np.eye(3))
    assert np.allclose(-lap, gs.exact_f(x), rtol=1e-5, atol=1e-6 * np.abs(gs.exact_f(x)).max())
    g = np.stack([(gs.exact_u(x + h * e) - gs.exact_u(x - h * e)) / (2 * h) for e in np.eye(3)], axis=-1)
    assert np.allclose(g, gs.grad_u(x), rtol=1e-6, atol=1e-8 * np.abs(g).max())
    # one Gaussian integrates to 2^-1.5 over R^3 (its mass lies well inside the cube)
    t = np.linspace(-3, 3, 601)
    w = np.full_like(t, t[1] - t[0])
    X, Y, Z = np.meshgrid(t, t, t, indexing="ij")
    c = (1 / (gs.ALPHA * np.sqrt(2 * np.pi))) ** 3
    one = c * np.exp(-(X ** 2 + Y ** 2 + Z ** 2) / gs.ALPHA ** 2)
    assert abs(np.einsum("ijk,i,j,k->", one, w, w, w) - 2 ** -1.5) <= 1e-6
