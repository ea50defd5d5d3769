"""Symmetric interior penalty DG (SIPG) Q_k Laplace operator: cell + face terms.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Definition followed, eq:poisson_dgsip:
  (grad v, kappa grad u)_T - <v n, kappa {grad u}> - <grad v / 2, kappa n [u]> + <v, kappa sigma [u]>,
  kappa continuous, so every face term carries kappa(x_q) at the face point (folded into
  JxW below after sigma has been computed from the geometric |F| and |K|),
  both face terms visiting every interior face twice.  Summing the two visits of
  an interior face F (minus side K- = lower cell index, n = n-) gives
      a_F(u, v) = int_F ( -[v]{d_n u} - {d_n v}[u] + sigma [u][v] ),
  [u] = u- - u+,  {d_n u} = (grad u- + grad u+)/2 . n.
Boundary faces use the mirror values of eq:bc_dgsip with g = 0:
  Dirichlet u+ = -u-, grad u+ = grad u-:   -v d_n u - d_n v u + 2 sigma u v
  Neumann   u+ = u-,  d_n u+ = -d_n u-:     0.
Penalty (BASELINE.json configs[2]): sigma_F = c (k+1)^2 / h_F,
  interior 1/h_F = (|F|/|K-| + |F|/|K+|)/2, boundary 1/h_F = |F|/|K-|, with |F|,
  |K| quadrature sums of JxW; c = penalty_factor (2.0 for the configs).
Face quadrature: (k+1)^2 Gauss points (reading R4).  Face normal and surface
element by Nanson's formula: n = J^-T nhat / |J^-T nhat|, JxW_F = w detJ |J^-T nhat|,
computed from both sides and checked equal.  d_n phi = n . J^-T grad_xi phi
= (J^-1 n) . grad_xi phi, with grad_xi phi evaluated pointwise in 3-D on the face.
"""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp

from .basis import Basis1D
from .cg import CellQuadrature, cell_geometry, metric, element_matrix, element_apply_G, cell_diagonals
from .mesh import Mesh, eval_basis_3d, DIRICHLET


class FaceRef:
    """Reference face points of the face xi_d = sign (sign = +1 or -1)."""

    def __init__(self, k: int, d: int, sign: float):
        b1 = Basis1D(k)
        n = k + 1
        t1, t2 = [e for e in range(3) if e != d]
        a = np.arange(n * n) % n
        b = np.arange(n * n) // n
        pts = np.zeros((n * n, 3))
        pts[:, t1] = b1.qp[a]
        pts[:, t2] = b1.qp[b]
        pts[:, d] = sign
        self.d, self.sign, self.pts = d, sign, pts
        self.w = b1.qw[a] * b1.qw[b]
        self.val, self.grad = eval_basis_3d(b1.nodes, pts)     # [q, i], [q, 3, i]


def cell_volume(mesh, cells, quad):
    _, detJ = cell_geometry(mesh, cells, quad)
    return detJ @ quad.w


def face_geometry(mesh: Mesh, cells, ref: FaceRef):
    """Jinv [F,q,3,3], outward unit normal [F,q,3], JxW [F,q], physical points [F,q,3]."""
    cc = mesh.cell_coords(cells)
    J = mesh.jacobian(cc, ref.pts)
    detJ = np.linalg.det(J)
    Jinv = np.linalg.inv(J)
    nhat = np.zeros(3)
    nhat[ref.d] = ref.sign
    m = np.einsum('fqed,e->fqd', Jinv, nhat)        # J^-T nhat
    norm = np.linalg.norm(m, axis=-1)
    return Jinv, m / norm[..., None], ref.w * detJ * norm, mesh.points(cc, ref.pts)


def interior_faces(mesh: Mesh, d: int):
    cc = mesh.cell_coords()
    cm = np.nonzero(cc[:, d] < mesh.n[d] - 1)[0]
    step = [1, mesh.n[0], mesh.n[0] * mesh.n[1]][d]
    return cm, cm + step


def boundary_cells(mesh: Mesh, side: int):
    d, hi = side // 2, side % 2
    cc = mesh.cell_coords()
    return np.nonzero(cc[:, d] == (mesh.n[d] - 1 if hi else 0))[0]


class InteriorFaces:
    """Interior faces normal to d: minus cells cm, plus cells cp, with
    JxW [F,q], Jn_s = J_s^-1 n [F,q,3] for both sides and sigma [F]."""

    def __init__(self, mesh, d, cm, cp, quad, penalty_factor):
        self.cm, self.cp = cm, cp
        self.rm, self.rp = FaceRef(mesh.k, d, +1.0), FaceRef(mesh.k, d, -1.0)
        Jm, nm, Wm, xm = face_geometry(mesh, cm, self.rm)
        Jp, np_, Wp, xp = face_geometry(mesh, cp, self.rp)
        scale = max(1.0, float(np.max(np.abs(xm)))) if len(xm) else 1.0
        assert np.allclose(xm, xp, rtol=0, atol=1e-13 * scale), "face points differ"
        assert np.allclose(nm, -np_, rtol=0, atol=1e-12), "normals not opposite"
        assert np.allclose(Wm, Wp, rtol=1e-12, atol=0), "face JxW differs"
        self.Jn_m = np.einsum('fqed,fqd->fqe', Jm, nm)
        self.Jn_p = np.einsum('fqed,fqd->fqe', Jp, nm)
        area = Wm.sum(axis=1)
        inv_h = 0.5 * (area / cell_volume(mesh, cm, quad) + area / cell_volume(mesh, cp, quad))
        self.sigma = penalty_factor * (mesh.k + 1) ** 2 * inv_h
        self.JxW = Wm * mesh.kappa(xm)


class BoundaryFaces:
    def __init__(self, mesh, side, cells, quad, penalty_factor):
        d, sign = side // 2, (1.0 if side % 2 else -1.0)
        self.cells = cells
        self.r = FaceRef(mesh.k, d, sign)
        Jb, nb, Wb, xb = face_geometry(mesh, cells, self.r)
        self.Jn = np.einsum('fqed,fqd->fqe', Jb, nb)
        area = Wb.sum(axis=1)
        self.sigma = penalty_factor * (mesh.k + 1) ** 2 * area / cell_volume(mesh, cells, quad)
        self.JxW = Wb * mesh.kappa(xb)


def _dn(Jn, ref, xs):
    """d_n u at the face points: sum_e (J^-1 n)_e (grad_e phi . x)  -> [F, q]."""
    return sum(Jn[..., e] * (xs @ ref.grad[:, e, :].T) for e in range(3))


def _dn_test(c, Jn, ref):
    """sum_q c_q d_n phi_i(q)  -> [F, i]."""
    return sum((c * Jn[..., e]) @ ref.grad[:, e, :] for e in range(3))


def face_residual(fd: InteriorFaces, xm, xp):
    """Interior-face contributions (y-, y+) for nodal values xm, xp [F, n^3]."""
    um, up = xm @ fd.rm.val.T, xp @ fd.rp.val.T                  # u at face points
    jump = um - up
    avg = 0.5 * (_dn(fd.Jn_m, fd.rm, xm) + _dn(fd.Jn_p, fd.rp, xp))
    cu = fd.JxW * (fd.sigma[:, None] * jump - avg)               # tests +v- / -v+
    cg = fd.JxW * (-0.5 * jump)                                  # tests d_n v on both sides
    ym = cu @ fd.rm.val + _dn_test(cg, fd.Jn_m, fd.rm)
    yp = -cu @ fd.rp.val + _dn_test(cg, fd.Jn_p, fd.rp)
    return ym, yp


def boundary_residual(bd: BoundaryFaces, xb):
    """Dirichlet mirror-face contribution -v d_n u - d_n v u + 2 sigma u v."""
    u = xb @ bd.r.val.T
    cu = bd.JxW * (2.0 * bd.sigma[:, None] * u - _dn(bd.Jn, bd.r, xb))
    return cu @ bd.r.val + _dn_test(bd.JxW * (-u), bd.Jn, bd.r)


class Operator:
    """y = A x with cell metric and face data cached (cells by dense B, faces by traces)."""

    def __init__(self, mesh: Mesh, penalty_factor: float = 2.0, chunk: int = 8192):
        self.mesh, self.pf, self.chunk = mesh, penalty_factor, chunk
        self.quad = CellQuadrature(mesh.k)
        self.m = (mesh.k + 1) ** 3
        self.uniform = mesh.uniform
        if self.uniform:
            self.G0 = metric(mesh, np.array([0]), self.quad)
        else:
            self.G = [metric(mesh, np.arange(c0, min(c0 + chunk, mesh.n_cells)), self.quad)
                      for c0 in range(0, mesh.n_cells, chunk)]
        self.faces = []
        for d in range(3):
            cm, cp = interior_faces(mesh, d)
            if len(cm):
                self.faces.append(InteriorFaces(mesh, d, cm, cp, self.quad, penalty_factor))
        self.bfaces = [BoundaryFaces(mesh, s, boundary_cells(mesh, s), self.quad, penalty_factor)
                       for s in range(6) if mesh.bc[s] == DIRICHLET]

    def _cell_chunks(self):
        for j, c0 in enumerate(range(0, self.mesh.n_cells, self.chunk)):
            cells = np.arange(c0, min(c0 + self.chunk, self.mesh.n_cells))
            G = np.broadcast_to(self.G0, (len(cells),) + self.G0.shape[1:]) \
                if self.uniform else self.G[j]
            yield cells, G

    def apply(self, x):
        X = x.reshape(self.mesh.n_cells, self.m)
        Y = np.zeros_like(X)
        for cells, G in self._cell_chunks():
            Y[cells] += element_apply_G(G, X[cells], self.quad)
        for fd in self.faces:          # within one direction every cell is at most once minus/plus
            ym, yp = face_residual(fd, X[fd.cm], X[fd.cp])
            Y[fd.cm] += ym
            Y[fd.cp] += yp
        for bd in self.bfaces:
            Y[bd.cells] += boundary_residual(bd, X[bd.cells])
        return Y.reshape(-1)

    def diagonal(self):
        """cell sum_q w detJ |J^-T grad phi_i|^2, plus per face side s
        sum_q JxW (-sg_s phi_i d_n phi_i + sigma phi_i^2); Dirichlet boundary
        sum_q JxW (-2 phi_i d_n phi_i + 2 sigma phi_i^2)."""
        D = np.zeros((self.mesh.n_cells, self.m))
        for cells, G in self._cell_chunks():
            D[cells] += cell_diagonals(G, self.quad)
        for fd in self.faces:
            for cells, ref, Jn, sg in ((fd.cm, fd.rm, fd.Jn_m, 1.0), (fd.cp, fd.rp, fd.Jn_p, -1.0)):
                phidn = sum((fd.JxW * Jn[..., e]) @ (ref.val * ref.grad[:, e, :]) for e in range(3))
                D[cells] += -sg * phidn + (fd.sigma[:, None] * fd.JxW) @ (ref.val ** 2)
        for bd in self.bfaces:
            phidn = sum((bd.JxW * bd.Jn[..., e]) @ (bd.r.val * bd.r.grad[:, e, :]) for e in range(3))
            D[bd.cells] += -2.0 * phidn + 2.0 * (bd.sigma[:, None] * bd.JxW) @ (bd.r.val ** 2)
        return D.reshape(-1)


def apply(mesh: Mesh, x: np.ndarray, penalty_factor: float = 2.0):
    return Operator(mesh, penalty_factor).apply(x)


def diagonal(mesh: Mesh, penalty_factor: float = 2.0):
    return Operator(mesh, penalty_factor).diagonal()


def assemble(mesh: Mesh, penalty_factor: float = 2.0) -> sp.csr_matrix:
    """Global SIPG matrix (tiny meshes): cell K^e plus the four (test, trial) face
    blocks A_F[s,t] = sum_q JxW ( -sg_s v_s (d_n u_t)/2 - (d_n v_s)/2 sg_t u_t
                                  + sigma sg_s sg_t v_s u_t ),  sg_- = +1, sg_+ = -1."""
    quad = CellQuadrature(mesh.k)
    m = (mesh.k + 1) ** 3
    N = mesh.dg_n_dofs()
    rows, cols, vals = [], [], []
    loc = np.arange(m)

    def add(ci, cj, blk):
        rows.append(np.repeat(ci * m + loc, m))
        cols.append(np.tile(cj * m + loc, m))
        vals.append(blk.ravel())

    def dn_matrix(Jn, ref):             # d_n phi_i at face points, [F, q, i]
        return np.einsum('fqe,qei->fqi', Jn, ref.grad)

    for c in range(mesh.n_cells):
        add(c, c, element_matrix(mesh, c, quad))
    sg = (1.0, -1.0)
    for d in range(3):
        cm, cp = interior_faces(mesh, d)
        if len(cm) == 0:
            continue
        fd = InteriorFaces(mesh, d, cm, cp, quad, penalty_factor)
        V = (fd.rm.val, fd.rp.val)
        Dn = (dn_matrix(fd.Jn_m, fd.rm), dn_matrix(fd.Jn_p, fd.rp))
        cel = (cm, cp)
        for s in (0, 1):
            for t in (0, 1):
                blk = (-sg[s] * 0.5 * np.einsum('fq,qi,fqj->fij', fd.JxW, V[s], Dn[t])
                       - 0.5 * sg[t] * np.einsum('fq,fqi,qj->fij', fd.JxW, Dn[s], V[t])
                       + sg[s] * sg[t] * np.einsum('f,fq,qi,qj->fij', fd.sigma, fd.JxW, V[s], V[t]))
                for f in range(len(cm)):
                    add(cel[s][f], cel[t][f], blk[f])
    for side in range(6):
        if mesh.bc[side] != DIRICHLET:
            continue
        cb = boundary_cells(mesh, side)
        bd = BoundaryFaces(mesh, side, cb, quad, penalty_factor)
        V, Dn = bd.r.val, dn_matrix(bd.Jn, bd.r)
        blk = (-np.einsum('fq,qi,fqj->fij', bd.JxW, V, Dn)
               - np.einsum('fq,fqi,qj->fij', bd.JxW, Dn, V)
               + 2.0 * np.einsum('f,fq,qi,qj->fij', bd.sigma, bd.JxW, V, V))
        for f in range(len(cb)):
            add(cb[f], cb[f], blk[f])
    return sp.coo_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))),
                         shape=(N, N)).tocsr()


def apply_cells(mesh: Mesh, x, cells, penalty_factor: float = 2.0):
    """(A x) restricted to the DoFs of the given cells -> [C, n^3] (full-size sampled parity)."""
    quad = CellQuadrature(mesh.k)
    m = (mesh.k + 1) ** 3
    cells = np.asarray(cells)
    X = x.reshape(-1, m)
    cc = mesh.cell_coords(cells)
    out = element_apply_G(metric(mesh, cells, quad), np.asarray(X[cells]), quad)
    step = (1, mesh.n[0], mesh.n[0] * mesh.n[1])
    for i, c in enumerate(cells):
        for d in range(3):
            for sgn in (+1, -1):
                if 0 <= cc[i, d] + sgn < mesh.n[d]:
                    cm, cp = (c, c + step[d]) if sgn > 0 else (c - step[d], c)
                    fd = InteriorFaces(mesh, d, np.array([cm]), np.array([cp]), quad,
                                       penalty_factor)
                    ym, yp = face_residual(fd, np.asarray(X[[cm]]), np.asarray(X[[cp]]))
                    out[i] += ym[0] if sgn > 0 else yp[0]
                elif mesh.bc[2 * d + (1 if sgn > 0 else 0)] == DIRICHLET:
                    side = 2 * d + (1 if sgn > 0 else 0)
                    bd = BoundaryFaces(mesh, side, np.array([c]), quad, penalty_factor)
                    out[i] += boundary_residual(bd, np.asarray(X[[c]]))[0]
    return out
