"""Manufactured right-hand side and L2 error.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

u = prod_d sin(pi t_d), t = (x - lo)/(hi - lo) (BASELINE.json configs[1..4]:
"manufactured u = sin(pi x) sin(pi y) sin(pi z)" on the unit cube),
f = -div(kappa grad u) = kappa pi^2 sum_d (hi_d-lo_d)^-2 u - grad kappa . grad u
(= 3 pi^2 u on [0,1]^3 with kappa = 1), eq:poisson; kappa of mesh.kappa (N3).
Load vector (v_h, f) of eq:poisson_fem / eq:poisson_dgsip with (k+1)^3 Gauss
points in physical coordinates; CG Dirichlet rows set to 0 (g_D = 0); SIPG has
no boundary term for g_D = 0.
"""
from __future__ import annotations

import numpy as np

from .basis import Basis1D
from .cg import CellQuadrature, cell_geometry
from .mesh import Mesh, CG, tensor_points, tensor_weights, eval_basis_3d


def exact_u(mesh: Mesh, x):
    t = (x - mesh.lo) / (mesh.hi - mesh.lo)
    return np.prod(np.sin(np.pi * t), axis=-1)


def grad_u(mesh: Mesh, x):
    t = (x - mesh.lo) / (mesh.hi - mesh.lo)
    sn, cs = np.sin(np.pi * t), np.cos(np.pi * t)
    g = np.empty(x.shape)
    for d in range(3):
        o = [e for e in range(3) if e != d]
        g[..., d] = np.pi / (mesh.hi[d] - mesh.lo[d]) * cs[..., d] * sn[..., o[0]] * sn[..., o[1]]
    return g


def exact_f(mesh: Mesh, x):
    f = mesh.kappa(x) * np.pi ** 2 * np.sum((mesh.hi - mesh.lo) ** -2.0) * exact_u(mesh, x)
    if mesh.kappa_amp != 0.0:
        f -= np.sum(mesh.grad_kappa(x) * grad_u(mesh, x), axis=-1)
    return f


def rhs(mesh: Mesh, method: int, chunk: int = 4096):
    quad = CellQuadrature(mesh.k)
    m = (mesh.k + 1) ** 3
    b = np.zeros(mesh.cg_n_dofs() if method == CG else mesh.dg_n_dofs())
    for c0 in range(0, mesh.n_cells, chunk):
        cells = np.arange(c0, min(c0 + chunk, mesh.n_cells))
        _, detJ = cell_geometry(mesh, cells, quad)
        xq = mesh.points(mesh.cell_coords(cells), quad.pts)
        fq = exact_f(mesh, xq) * detJ * quad.w[None, :]       # [C, q]
        be = fq @ quad.val                                    # [C, n^3]
        if method == CG:
            dm = mesh.cg_dofmap(cells)
            lo, hi = int(dm.min()), int(dm.max()) + 1
            b[lo:hi] += np.bincount(dm.ravel() - lo, weights=be.ravel(), minlength=hi - lo)
        else:
            b[c0 * m:(c0 + len(cells)) * m] = be.ravel()
    if method == CG:
        b[mesh.cg_dirichlet_mask()] = 0.0
    return b


def l2_error(mesh: Mesh, method: int, uh, chunk: int = 4096):
    """||u_h - u|| / ||u|| with (k+2)^3 Gauss points."""
    b1 = Basis1D(mesh.k, mesh.k + 2)
    pts, w = tensor_points(b1.qp), tensor_weights(b1.qw)
    val, _ = eval_basis_3d(b1.nodes, pts)
    num = den = 0.0
    for c0 in range(0, mesh.n_cells, chunk):
        cells = np.arange(c0, min(c0 + chunk, mesh.n_cells))
        cc = mesh.cell_coords(cells)
        detJ = np.linalg.det(mesh.jacobian(cc, pts))
        xq = mesh.points(cc, pts)
        dm = mesh.cg_dofmap(cells) if method == CG else mesh.dg_dofmap(cells)
        uq = uh[dm] @ val.T
        ue = exact_u(mesh, xq)
        JxW = detJ * w[None, :]
        num += np.sum((uq - ue) ** 2 * JxW)
        den += np.sum(ue ** 2 * JxW)
    return float(np.sqrt(num / den))
