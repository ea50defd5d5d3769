"""Continuous Galerkin Q_k Laplace operator: element matrices by full quadrature.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Definition followed:
  weak form (grad v, kappa grad u) = (v, f), eq:poisson_fem, P:L184-189;
  element matrix K^e_ij = sum_q w_q det J_q kappa(x_q) (J_q^-T grad_xi phi_i(xi_q)) . (J_q^-T grad_xi phi_j(xi_q)),
  which is eq:mf_eval written as a matrix, with (k+1)^3 Gauss points
   and grad_xi phi evaluated pointwise in 3-D (no sum factorization).
  Assembly "in the usual finite element way, including the elimination of
  Dirichlet rows and columns"; reading R5: a constrained row is the
  identity (y_c = x_c, diag = 1), constrained columns are dropped.

Three evaluation modes:
  assemble()      global CSR (tiny meshes);
  apply()         y = sum_e P_e^T K^e P_e x, with K^e x_e evaluated as
                  B^T (G o (B x_e)) where B is the dense [3 n^3_q x n^3] reference
                  gradient matrix (mathematically K^e x_e; O((k+1)^6) per cell);
  apply_rows()    the same for a sample of rows (full-size configs).
"""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp

from .basis import Basis1D
from .mesh import Mesh, tensor_points, tensor_weights, eval_basis_3d


class CellQuadrature:
    """Reference data: Gauss points (k+1)^3, weights, dense B [q, 3, i]."""

    def __init__(self, k: int, n_q: int | None = None):
        self.b1 = Basis1D(k, n_q)
        self.pts = tensor_points(self.b1.qp)
        self.w = tensor_weights(self.b1.qw)
        self.val, self.grad = eval_basis_3d(self.b1.nodes, self.pts)


def cell_geometry(mesh: Mesh, cells, quad: CellQuadrature):
    """Jinv [C,q,3,3], detJ [C,q] at the cell quadrature points (numpy.linalg)."""
    cc = mesh.cell_coords(cells)
    J = mesh.jacobian(cc, quad.pts)
    detJ = np.linalg.det(J)
    if np.any(detJ <= 0):
        bad = np.argwhere(detJ <= 0)[0]
        raise ValueError(f"det J <= 0 in cell {np.asarray(cells).ravel()[bad[0]]}")
    return np.linalg.inv(J), detJ


def cell_kappa(mesh, cells, quad):
    """kappa at the physical quadrature points [C, q] (1 unless mesh.kappa_amp)."""
    if mesh.kappa_amp == 0.0:
        return np.ones((len(np.atleast_1d(cells)), len(quad.w)))
    return mesh.kappa(mesh.points(mesh.cell_coords(cells), quad.pts))


def metric(mesh, cells, quad):
    """G_q = J_q^-1 (w_q det J_q kappa(x_q)) J_q^-T  [C, q, 3, 3] (eq:mf_eval)."""
    Jinv, detJ = cell_geometry(mesh, cells, quad)
    wk = quad.w[None, :] * detJ * cell_kappa(mesh, cells, quad)
    return wk[..., None, None] * np.einsum('cqde,cqfe->cqdf', Jinv, Jinv)


def element_matrix(mesh: Mesh, cell: int, quad: CellQuadrature | None = None):
    """K^e of one cell by full tensor quadrature, [n^3, n^3]."""
    quad = quad or CellQuadrature(mesh.k)
    Jinv, detJ = cell_geometry(mesh, np.array([cell]), quad)
    kap = cell_kappa(mesh, np.array([cell]), quad)[0]
    # physical gradients J^-T grad_xi phi_i : [q, 3, i]
    pg = np.einsum('qed,qei->qdi', Jinv[0], quad.grad)
    return np.einsum('q,qdi,qdj->ij', quad.w * detJ[0] * kap, pg, pg)


def element_apply_G(G, xe, quad):
    """K^e x_e for a batch of cells via dense B: B^T (G (B x_e)); xe [C, n^3], G [C,q,3,3]."""
    nq, m = len(quad.w), quad.grad.shape[2]
    B = quad.grad.reshape(nq * 3, m)                      # rows (q, d)
    gu = (xe @ B.T).reshape(len(xe), nq, 3)               # grad_xi u at q
    flux = np.einsum('cqde,cqe->cqd', G, gu)
    return flux.reshape(len(xe), nq * 3) @ B


def cell_diagonals(G, quad):
    """K^e_ii = sum_q sum_de grad_d phi_i(q) G_q,de grad_e phi_i(q) for a batch of cells,
    G [C, q, 3, 3]: the same sum as einsum('qdi,cqde,qei->ci'), evaluated as one matrix
    product with H[q, de, i] = grad_d phi_i(q) grad_e phi_i(q)."""
    g = quad.grad
    H = (g[:, :, None, :] * g[:, None, :, :]).reshape(-1, g.shape[2])     # [(q, d, e), i]
    return np.ascontiguousarray(G).reshape(len(G), -1) @ H


def element_apply(mesh, cells, xe, quad):
    return element_apply_G(metric(mesh, cells, quad), xe, quad)


def assemble(mesh: Mesh) -> sp.csr_matrix:
    """Global CSR with Dirichlet rows/columns eliminated (tiny meshes)."""
    quad = CellQuadrature(mesh.k)
    dm = mesh.cg_dofmap()
    N = mesh.cg_n_dofs()
    mask = mesh.cg_dirichlet_mask()
    rows, cols, vals = [], [], []
    for c in range(mesh.n_cells):
        Ke = element_matrix(mesh, c, quad)
        rows.append(np.repeat(dm[c], len(dm[c])))
        cols.append(np.tile(dm[c], len(dm[c])))
        vals.append(Ke.ravel())
    A = sp.coo_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))),
                      shape=(N, N)).tocsr()
    free = sp.diags((~mask).astype(np.float64))
    A = free @ A @ free + sp.diags(mask.astype(np.float64))
    return A.tocsr()


def _scatter_add(y, dm, ye):
    """y[dm] += ye with repeated indices summed (np.bincount over the index range the
    chunk touches: the same sums as a full-length bincount, without allocating len(y))."""
    lo, hi = int(dm.min()), int(dm.max()) + 1
    y[lo:hi] += np.bincount(dm.ravel() - lo, weights=ye.ravel(), minlength=hi - lo)


class Operator:
    """y = A x with the geometry factors G_q of every cell cached (mode O3-iii).

    Cartesian meshes (mesh.uniform: eps = 0, exact map, kappa = 1): J is the same on
    every cell, so every cell has the same element matrix; it is computed once by full
    tensor quadrature (element_matrix, cell 0) and applied as y_e = K^e x_e (mode O3-ii,
    SURVEY §8c: "Stored K^e -- one per level if Cartesian"; the same definition,
    K^e = B^T G B, evaluated once instead of per cell)."""

    def __init__(self, mesh: Mesh, chunk: int = 8192):
        self.mesh, self.chunk = mesh, chunk
        self.quad = CellQuadrature(mesh.k)
        self.mask = mesh.cg_dirichlet_mask()
        self.uniform = mesh.uniform
        if self.uniform:
            self.G0 = metric(mesh, np.array([0]), self.quad)
            self.Ke = element_matrix(mesh, 0, self.quad)
        else:
            self.G = [metric(mesh, np.arange(c0, min(c0 + chunk, mesh.n_cells)), self.quad)
                      for c0 in range(0, mesh.n_cells, chunk)]

    def _chunks(self):
        for j, c0 in enumerate(range(0, self.mesh.n_cells, self.chunk)):
            cells = np.arange(c0, min(c0 + self.chunk, self.mesh.n_cells))
            G = np.broadcast_to(self.G0, (len(cells),) + self.G0.shape[1:]) \
                if self.uniform else self.G[j]
            yield cells, G

    def apply(self, x):
        """Constrained inputs read as 0; y_c = x_c."""
        xf = np.where(self.mask, 0.0, x)
        y = np.zeros(self.mesh.cg_n_dofs())
        for cells, G in self._chunks():
            dm = self.mesh.cg_dofmap(cells)
            ye = xf[dm] @ self.Ke if self.uniform else element_apply_G(G, xf[dm], self.quad)
            _scatter_add(y, dm, ye)
        return np.where(self.mask, x, y)

    def diagonal(self):
        """sum over cells of K^e_ii = sum_q w det J |J^-T grad phi_i|^2; 1 on constrained rows."""
        d = np.zeros(self.mesh.cg_n_dofs())
        for cells, G in self._chunks():
            if self.uniform:   # mode O3-ii: K^e_ii of the one stored element matrix
                de = np.broadcast_to(np.diag(self.Ke), (len(cells), self.Ke.shape[0]))
            else:
                de = cell_diagonals(G, self.quad)
            dm = self.mesh.cg_dofmap(cells)
            _scatter_add(d, dm, de)
        return np.where(self.mask, 1.0, d)


def apply(mesh: Mesh, x: np.ndarray) -> np.ndarray:
    return Operator(mesh).apply(x)


def diagonal(mesh: Mesh) -> np.ndarray:
    return Operator(mesh).diagonal()


def cells_of_node(mesh: Mesh, g):
    """All (cell id, local index) pairs whose closure contains node g = (gx, gy, gz)."""
    k, out = mesh.k, []
    cand = []
    for d in range(3):
        cs = {g[d] // k, (g[d] - 1) // k}
        cand.append([c for c in cs if 0 <= c < mesh.n[d] and 0 <= g[d] - k * c <= k])
    n = k + 1
    for cx in cand[0]:
        for cy in cand[1]:
            for cz in cand[2]:
                loc = (g[0] - k * cx) + n * ((g[1] - k * cy) + n * (g[2] - k * cz))
                out.append((cx + mesh.n[0] * (cy + mesh.n[1] * cz), loc))
    return out


def apply_rows(mesh: Mesh, x, rows) -> np.ndarray:
    """(A x)[rows] for sampled rows (full-size configs); x may be a memmap/array."""
    quad = CellQuadrature(mesh.k)
    rows = np.asarray(rows)
    nn0, nn1 = mesh.nn[0], mesh.nn[1]
    g_all = np.stack([rows % nn0, (rows // nn0) % nn1, rows // (nn0 * nn1)], axis=-1)
    mask = _mask_rows(mesh, g_all)
    pairs = [cells_of_node(mesh, g) for g in g_all]
    cells = np.unique(np.array([c for p in pairs for c, _ in p], dtype=np.int64))
    dm = mesh.cg_dofmap(cells)
    full_mask = _mask_rows(mesh, np.stack([dm % nn0, (dm // nn0) % nn1, dm // (nn0 * nn1)], -1))
    xe = np.where(full_mask, 0.0, np.asarray(x)[dm])
    ye = element_apply(mesh, cells, xe, quad)
    pos = {int(c): i for i, c in enumerate(cells)}
    y = np.array([sum(ye[pos[c], l] for c, l in p) for p in pairs])
    return np.where(mask, np.asarray(x)[rows], y)


def _mask_rows(mesh, g):
    m = np.zeros(g.shape[:-1], dtype=bool)
    for d in range(3):
        if mesh.bc[2 * d] == 0:
            m |= g[..., d] == 0
        if mesh.bc[2 * d + 1] == 0:
            m |= g[..., d] == mesh.nn[d] - 1
    return m
