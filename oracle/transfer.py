"""Geometric level transfer: prolongation P = nodal interpolation, restriction R = P^T.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

P:L1181-1182: "The level transfer is based on the usual geometric embedding
operations and also implemented by tensorial techniques."  Reading R12: the
level spaces are {vhat o Phi^-1 : vhat piecewise Q_k on the Cartesian level
grid}, nested, so P_ij = phi_j^coarse(xhat_i^fine) evaluated in undeformed
coordinates and P does not depend on the deformation.  With a per-level polynomial
mapping or the shell patch (N3) the level spaces are no longer exactly nested; the
same reference-coordinate P is used (reading N3-d: it is the preconditioner's
transfer, the paper's geometric multigrid on curved meshes does the same).

Two forms, pinned against each other in tests:
  prolongation_matrix()  explicit sparse P by POINTWISE 3-D evaluation of the
                         coarse basis at every fine node (small meshes);
  prolongate()/restrict() the same P applied as the Kronecker product of the
                         1-D interpolation matrices (valid because the nodes
                         and the basis are tensor products); used at scale.
CG: constrained (Dirichlet) rows and columns are removed (zero), as in the
eliminated operator.  DG: P maps every coarse cell to its 2^3 children.
"""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp

from .basis import gll_nodes, lagrange
from .mesh import Mesh, CG, eval_basis_3d


def coarsen(mesh: Mesh) -> Mesh:
    return mesh.like(tuple(m // 2 for m in mesh.n))


def hierarchy(mesh: Mesh, coarse_cells: int = 1):
    """Meshes level 0 (coarsest) .. L (= mesh): halve while every n_d is even and
    max(n_d) > coarse_cells."""
    out = [mesh]
    while all(m % 2 == 0 for m in out[-1].n) and max(out[-1].n) > coarse_cells:
        out.append(coarsen(out[-1]))
    return out[::-1]


# ---------------------------------------------------------------- 1-D pieces
def _cg_1d(k: int, n_coarse: int) -> np.ndarray:
    """1-D CG interpolation [k*2Nc+1, k*Nc+1]: coarse nodal basis at fine node positions."""
    nodes = gll_nodes(k)
    nf = 2 * n_coarse
    # fine node g: fine cell g//k (last node -> last cell), local g%k
    g = np.arange(k * nf + 1)
    fc = np.minimum(g // k, nf - 1)
    fl = g - k * fc
    t = (fc + 0.5 * (nodes[fl] + 1.0)) / nf               # position in [0,1]
    cc = np.minimum((t * n_coarse).astype(int), n_coarse - 1)
    xi = 2.0 * (t * n_coarse - cc) - 1.0
    phi = lagrange(nodes, xi)                              # [fine, k+1]
    P = np.zeros((k * nf + 1, k * n_coarse + 1))
    for i in range(len(g)):
        P[i, k * cc[i]:k * cc[i] + k + 1] = phi[i]
    return P


def _dg_1d(k: int, n_coarse: int) -> np.ndarray:
    """1-D DG interpolation [(2Nc)(k+1), Nc(k+1)]: child c of parent p gets
    phi_j((xi_i + 2c - 1)/2) of the parent."""
    nodes = gll_nodes(k)
    n = k + 1
    P = np.zeros((2 * n_coarse * n, n_coarse * n))
    for c in (0, 1):
        E = lagrange(nodes, 0.5 * (nodes + 2 * c - 1))     # [i fine, j coarse]
        for p in range(n_coarse):
            f = 2 * p + c
            P[f * n:(f + 1) * n, p * n:(p + 1) * n] = E
    return P


def _kron_apply(mats, arr):
    """Apply 1-D matrices along axes (x, y, z) of arr shaped [z, y, x]."""
    arr = np.einsum('ij,zyj->zyi', mats[0], arr)
    arr = np.einsum('ij,zjx->zix', mats[1], arr)
    return np.einsum('ij,jyx->iyx', mats[2], arr)


def _dg_to_grid(mesh: Mesh, v):
    n = mesh.k + 1
    nx, ny, nz = mesh.n
    a = v.reshape(nz, ny, nx, n, n, n)                     # [cz,cy,cx,lz,ly,lx]
    return a.transpose(0, 3, 1, 4, 2, 5).reshape(nz * n, ny * n, nx * n)


def _grid_to_dg(mesh: Mesh, g):
    n = mesh.k + 1
    nx, ny, nz = mesh.n
    a = g.reshape(nz, n, ny, n, nx, n).transpose(0, 2, 4, 1, 3, 5)
    return a.reshape(-1)


# ---------------------------------------------------------------- tensorial form
def prolongate(coarse: Mesh, fine: Mesh, method: int, xc: np.ndarray) -> np.ndarray:
    k = fine.k
    if method == CG:
        mats = [_cg_1d(k, coarse.n[d]) for d in range(3)]
        xcm = np.where(coarse.cg_dirichlet_mask(), 0.0, xc)
        arr = xcm.reshape(coarse.nn[2], coarse.nn[1], coarse.nn[0])
        xf = _kron_apply(mats, arr).reshape(-1)
        return np.where(fine.cg_dirichlet_mask(), 0.0, xf)
    mats = [_dg_1d(k, coarse.n[d]) for d in range(3)]
    return _grid_to_dg(fine, _kron_apply(mats, _dg_to_grid(coarse, xc)))


def restrict(coarse: Mesh, fine: Mesh, method: int, xf: np.ndarray) -> np.ndarray:
    k = fine.k
    if method == CG:
        mats = [_cg_1d(k, coarse.n[d]).T for d in range(3)]
        xfm = np.where(fine.cg_dirichlet_mask(), 0.0, xf)
        arr = xfm.reshape(fine.nn[2], fine.nn[1], fine.nn[0])
        xc = _kron_apply(mats, arr).reshape(-1)
        return np.where(coarse.cg_dirichlet_mask(), 0.0, xc)
    mats = [_dg_1d(k, coarse.n[d]).T for d in range(3)]
    return _grid_to_dg(coarse, _kron_apply(mats, _dg_to_grid(fine, xf)))


# ---------------------------------------------------------------- explicit form
def prolongation_matrix(coarse: Mesh, fine: Mesh, method: int) -> sp.csr_matrix:
    """Explicit P by pointwise 3-D evaluation phi_j^coarse(xhat_i^fine) (small meshes)."""
    k = fine.k
    nodes = gll_nodes(k)
    n = k + 1
    rows, cols, vals = [], [], []
    if method == CG:
        g = fine.cg_node_coords()
        fc = np.minimum(g // k, np.asarray(fine.n) - 1)       # fine cell (last node -> last cell)
        t = (fc + 0.5 * (nodes[g - k * fc] + 1.0)) / np.asarray(fine.n)   # in [0,1]^3
    else:
        fc = fine.cell_coords()
        loc = np.arange(n ** 3)
        l3 = np.stack([loc % n, (loc // n) % n, loc // (n * n)], axis=-1)
        t = (fc[:, None, :] + 0.5 * (nodes[l3][None] + 1.0)) / np.asarray(fine.n)
        t = t.reshape(-1, 3)
    ncs = np.asarray(coarse.n)
    if method == CG:   # any coarse cell whose closure holds the node gives the same value
        cc = np.minimum((t * ncs).astype(int), ncs - 1)
    else:              # DG: the parent cell of the fine cell
        cc = np.repeat(fine.cell_coords() // 2, n ** 3, axis=0)
    xi = 2.0 * (t * ncs - cc) - 1.0
    val, _ = eval_basis_3d(nodes, xi)                           # [fine, n^3]
    if method == CG:
        cdm, n_coarse = coarse.cg_dofmap(coarse.cell_id(cc)), coarse.cg_n_dofs()
    else:
        cdm, n_coarse = coarse.dg_dofmap(coarse.cell_id(cc)), coarse.dg_n_dofs()
    for i in range(len(t)):
        rows.append(np.full(n ** 3, i))
        cols.append(cdm[i])
        vals.append(val[i])
    P = sp.coo_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))),
                      shape=(len(t), n_coarse))
    P = P.tocsr()
    P.data[np.abs(P.data) < 1e-14] = 0.0     # exact zeros at non-matching nodes
    P.eliminate_zeros()
    if method == CG:
        P = sp.diags((~fine.cg_dirichlet_mask()).astype(float)) @ P @ \
            sp.diags((~coarse.cg_dirichlet_mask()).astype(float))
    return P.tocsr()
