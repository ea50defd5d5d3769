"""The paper's own 3-D test problem: three Gaussians on (-1,1)^3.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

eq:pois_analytic:
    u(x) = (1/(alpha sqrt(2 pi)))^3 sum_{j=1..3} exp(-|x - x_j|^2 / alpha^2),
    x_j = (-0.5, 0.5, 0.25), (-0.6, -0.5, -0.125), (0.5, -0.5, 0.5),  alpha = 1/5,
on the cube (-1,1)^3 with Neumann conditions on the faces x_e = -1 and Dirichlet
conditions on x_e = +1, kappa = 1; g_D, g_N and f "set such that the
analytic solution is obtained":
    f = -Laplace u,  g_D = u on Gamma_D,  g_N = -n . grad u on Gamma_N (eq:poisson).
Per Gaussian G = c exp(-r^2/alpha^2): grad G = -2 (x - x_j)/alpha^2 G,
Laplace G = (4 r^2/alpha^4 - 6/alpha^2) G.

Right-hand sides (all with the cell / face Gauss rules of the operator):
* CG, eq:poisson_fem: b_i = (phi_i, f) - <phi_i, g_N>_{Gamma_N} on free rows;
  the solution space satisfies g_D by interpolation at the nodes, so the
  constrained rows carry g_D(x_i) and the free rows subtract the coupling
  sum_{j constrained} A_ij g_D(x_j) (the unconstrained operator, i.e. the same mesh
  with every side Neumann, applied to the nodal g_D).
* SIPG, eq:poisson_dgsip with the extension values of eq:bc_dgsip:
  Dirichlet u+ = -u- + 2 g_D moves  int g_D (2 sigma phi_i - d_n phi_i)  to the right;
  Neumann d_n u+ = -d_n u- - 2 g_N gives {d_n u} = -g_N, i.e. -<phi_i, g_N>.
Error: absolute L2 norm ||u - u_h|| with (k+2)^3 Gauss points (the paper's plots list
absolute errors: 3.5 on the coarsest k = 1 mesh).

The shell case: `shell_mesh` = one cube-sphere patch of
the shell (oracle/mesh.py), Dirichlet on all sides, degree-5 mapping, variable kappa;
with kappa the data become f = -div(kappa grad u) = -kappa Laplace u - grad kappa . grad u,
g_N = -kappa n . grad u, and the SIPG Dirichlet term carries kappa:
int g_D kappa (2 sigma phi_i - d_n phi_i).
"""
from __future__ import annotations

import numpy as np

from .basis import Basis1D
from .cg import CellQuadrature, cell_geometry
from .cg import apply as cg_apply
from .mesh import Mesh, CG, DIRICHLET, NEUMANN, SHELL, tensor_points, tensor_weights, eval_basis_3d
from .sipg import FaceRef, face_geometry, boundary_cells, cell_volume

ALPHA = 0.2
CENTERS = np.array([[-0.5, 0.5, 0.25], [-0.6, -0.5, -0.125], [0.5, -0.5, 0.5]])
BC = (NEUMANN, DIRICHLET, NEUMANN, DIRICHLET, NEUMANN, DIRICHLET)   # -x,+x,-y,+y,-z,+z
PENALTY_FACTOR = 3.0   # sigma = (k+1)^2 d / h with d = 3


def mesh(cells, k) -> Mesh:
    return Mesh(cells, k, lo=(-1.0, -1.0, -1.0), hi=(1.0, 1.0, 1.0), bc=BC)


def shell_mesh(cells, k, mapping_degree=5, kappa_amp=0.0) -> Mesh:
    """One cube-sphere patch of the shell 0.5 < r < 1, Dirichlet everywhere."""
    return Mesh(cells, k, geometry=SHELL, mapping_degree=mapping_degree, kappa_amp=kappa_amp)


def _gauss(x):
    c = (1.0 / (ALPHA * np.sqrt(2.0 * np.pi))) ** 3
    d = x[..., None, :] - CENTERS                    # [..., 3 centers, 3]
    r2 = np.sum(d * d, axis=-1)
    return c * np.exp(-r2 / ALPHA ** 2), d, r2


def exact_u(x):
    g, _, _ = _gauss(x)
    return g.sum(axis=-1)


def grad_u(x):
    g, d, _ = _gauss(x)
    return np.sum(-2.0 / ALPHA ** 2 * d * g[..., None], axis=-2)


def exact_f(x):
    g, _, r2 = _gauss(x)
    return -np.sum((4.0 * r2 / ALPHA ** 4 - 6.0 / ALPHA ** 2) * g, axis=-1)


class Solution:
    """An exact solution u with its gradient and -Laplace u (the problem's data follow)."""

    def __init__(self, u, grad, minus_lap):
        self.u, self.grad, self.minus_lap = u, grad, minus_lap


GAUSSIANS = Solution(exact_u, grad_u, exact_f)


def linear(a, c=0.0):
    """u = a . x + c: the patch test (any kappa: f = -grad kappa . a)."""
    a = np.asarray(a, dtype=np.float64)
    return Solution(lambda x: x @ a + c, lambda x: np.broadcast_to(a, x.shape), lambda x: np.zeros(x.shape[:-1]))


def exact_f_kappa(m: Mesh, x, sol: Solution = GAUSSIANS):
    """-div(kappa grad u) = kappa (-Laplace u) - grad kappa . grad u."""
    return m.kappa(x) * sol.minus_lap(x) - np.sum(m.grad_kappa(x) * sol.grad(x), axis=-1)


def _cell_load(m: Mesh, method, b, sol):
    quad = CellQuadrature(m.k)
    nm = (m.k + 1) ** 3
    cells = np.arange(m.n_cells)
    _, detJ = cell_geometry(m, cells, quad)
    xq = m.points(m.cell_coords(cells), quad.pts)
    be = (exact_f_kappa(m, xq, sol) * detJ * quad.w[None, :]) @ quad.val
    if method == CG:
        dm = m.cg_dofmap(cells)
        b += np.bincount(dm.ravel(), weights=be.ravel(), minlength=len(b))
    else:
        b += be.ravel()
    return nm


def _face_terms(m: Mesh, method, b, penalty_factor, sol):
    quad = CellQuadrature(m.k)
    for side in range(6):
        d, sign = side // 2, (1.0 if side % 2 else -1.0)
        cells = boundary_cells(m, side)
        ref = FaceRef(m.k, d, sign)
        Jinv, nrm, JxW, xf = face_geometry(m, cells, ref)
        dm = m.cg_dofmap(cells) if method == CG else m.dg_dofmap(cells)
        if m.bc[side] == NEUMANN:
            gN = -m.kappa(xf) * np.sum(nrm * sol.grad(xf), axis=-1)   # -n . kappa grad u
            be = -(gN * JxW) @ ref.val
        elif method == CG:
            continue                                                # interpolated g_D (below)
        else:
            gD = sol.u(xf)
            area = JxW.sum(axis=1)
            sigma = penalty_factor * (m.k + 1) ** 2 * area / cell_volume(m, cells, quad)
            Jn = np.einsum('fqed,fqd->fqe', Jinv, nrm)
            dn = np.einsum('fqe,qei->fqi', Jn, ref.grad)            # d_n phi_i at the face points
            be = np.einsum('fq,fqi->fi', gD * m.kappa(xf) * JxW,
                           2.0 * sigma[:, None, None] * ref.val[None] - dn)
        b += np.bincount(dm.ravel(), weights=be.ravel(), minlength=len(b))


def node_coords(m: Mesh):
    """Physical coordinates of the CG nodes (GLL support points of the cells, mapped)."""
    b1 = Basis1D(m.k)
    g = m.cg_node_coords()
    cell = np.minimum(g // m.k, np.asarray(m.n) - 1)
    return m.points_each(cell, b1.nodes[g - m.k * cell])


def rhs(m: Mesh, method: int, penalty_factor: float = PENALTY_FACTOR, sol: Solution = GAUSSIANS):
    """Right-hand side of the linear system (CG: constrained rows hold g_D)."""
    n = m.cg_n_dofs() if method == CG else m.dg_n_dofs()
    b = np.zeros(n)
    _cell_load(m, method, b, sol)
    _face_terms(m, method, b, penalty_factor, sol)
    if method == CG:
        mask = m.cg_dirichlet_mask()
        g = np.where(mask, sol.u(node_coords(m)), 0.0)
        free_op = Mesh(m.n, m.k, lo=m.lo, hi=m.hi, eps=m.eps, bc=(NEUMANN,) * 6, geometry=m.geometry,
                       mapping_degree=m.mapping_degree, kappa_amp=m.kappa_amp)
        b -= cg_apply(free_op, g)
        b[mask] = g[mask]
    return b


def l2_error_abs(m: Mesh, method: int, uh, sol: Solution = GAUSSIANS):
    """||u_h - u||_{L2(Omega)} with (k+2)^3 Gauss points."""
    b1 = Basis1D(m.k, m.k + 2)
    pts, w = tensor_points(b1.qp), tensor_weights(b1.qw)
    val, _ = eval_basis_3d(b1.nodes, pts)
    cells = np.arange(m.n_cells)
    cc = m.cell_coords(cells)
    detJ = np.linalg.det(m.jacobian(cc, pts))
    xq = m.points(cc, pts)
    dm = m.cg_dofmap(cells) if method == CG else m.dg_dofmap(cells)
    err = uh[dm] @ val.T - sol.u(xq)
    return float(np.sqrt(np.sum(err ** 2 * detJ * w[None, :])))
