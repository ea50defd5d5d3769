"""Hybridizable DG (HDG) for the Poisson problem: local matrices, the condensed trace
operator, its right-hand side, local recovery and the mixed (flux-substituted) operator.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Discretization, sec:discret_hdg: q = -kappa grad u, u_h in V_h^DG (Q_k,
GLL nodal, reading R3), q_h in (V_h^DG)^3, trace lambda_h in Q_k(F) on every face
(eq:trace_space; nodal in the GLL points of the face's two reference
directions, lower direction fastest), numerical fluxes u^ = lambda,
q^.n = q.n + tau (u - lambda), tau = 5 max kappa on the face (
kappa = 1 -> tau = 5).  Per cell K (eq:hdg, with the volume term of the second equation
written as in the standard derivation; reading HDG-1 in DESIGN.md):
    (kappa^-1 q, w)_K - (u, div w)_K + <lambda, w.n>_dK            = 0
    -(q, grad v)_K + <q.n + tau (u - lambda), v>_dK                = (f, v)_K
    sum_K <q.n + tau (u - lambda), mu>_dK                           = <g_N, mu>_Gamma_N
Matrices (eq:hdg_matrix; signs of this reading), per cell with m = (k+1)^3:
    A_{w,q} = (kappa^-1 q, w)            (3m x 3m, block diagonal)
    E_{v,(d,j)} = (d phi_j / d x_d, v)    (m x 3m; -(q, grad v) + <q.n, v> = (div q, v))
    C_{mu,(d,j)} = <mu, phi_j n_d>_F      per face F of K
    G_{mu,v} = <tau mu, v>_F,  D = sum_F <tau u, v>_F,  H_F^K = <tau lambda, mu>_F
so that, for the local unknowns of one cell,
    [ A  -E^T ] [q]   [ -C^T lambda         ]
    [ E   D   ] [u] = [  G^T lambda + F     ],
and the third equation is sum_K (H^K lambda - C q - G u) = <g_N, mu> (= 0 here).
Eliminating (q, u) cell by cell gives the statically condensed trace system
eq:hdg_matrix_condensed: K lambda = r with
    K = sum_K ( H^K - [C G] L^-1 [-C^T; G^T] ),   r = sum_K [C G] L^-1 [0; F],
L the 4m x 4m local matrix above, evaluated here exactly as written: quadrature-built
matrices and a dense local solve (no inner Schur complement, no sum factorization).
Dirichlet faces (homogeneous, "imposed strongly on the trace space"):
zero-in / identity-out rows as for CG (reading R5).  Homogeneous Neumann faces are free
trace unknowns with one adjacent cell.
Quadrature: Gauss (k+1)^3 in cells, (k+1)^2 on faces (readings R4), geometry and Nanson
normals of oracle.sipg.face_geometry.

Mixed form ("HDG mixed matrix-free"): lambda eliminated face by face instead,
lambda = H_F^-1 sum_K (C q + G u), with H_F = sum_K H_F^K:
    y_q = A q - E^T u + C^T lambda(q, u),   y_u = E q + D u - G^T lambda(q, u)
(the local residual of the first two equations with the trace from the third); solving
it for the cell unknowns gives the same (q, u) as the trace solve plus local recovery.

Trace numbering: faces normal to x first ((n_x+1) n_y n_z, index i_x + (n_x+1)(c_y + n_y c_z)),
then y (n_x (n_y+1) n_z), then z (n_x n_y (n_z+1)); each face (k+1)^2 nodes.
"""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp

from .basis import Basis1D, lagrange
from .cg import CellQuadrature, cell_geometry, cell_kappa
from .mesh import Mesh, DIRICHLET, SIPG
from .problem import rhs as load_vector
from .sipg import FaceRef, face_geometry

TAU = 5.0   # tau = 5 max kappa on the face, kappa = 1


def n_faces(mesh: Mesh):
    nx, ny, nz = mesh.n
    return ((nx + 1) * ny * nz, nx * (ny + 1) * nz, nx * ny * (nz + 1))


def n_trace_dofs(mesh: Mesh):
    return sum(n_faces(mesh)) * (mesh.k + 1) ** 2


def cell_face_ids(mesh: Mesh, cells=None):
    """[C, 6] global face index of the sides -x, +x, -y, +y, -z, +z of each cell."""
    cc = mesh.cell_coords(cells)
    nx, ny, nz = mesh.n
    fx, fy, _ = n_faces(mesh)
    cx, cy, cz = cc[:, 0], cc[:, 1], cc[:, 2]
    out = np.empty((len(cc), 6), dtype=np.int64)
    for hi in (0, 1):
        out[:, 0 + hi] = (cx + hi) + (nx + 1) * (cy + ny * cz)
        out[:, 2 + hi] = fx + cx + nx * ((cy + hi) + (ny + 1) * cz)
        out[:, 4 + hi] = fx + fy + cx + nx * (cy + ny * (cz + hi))
    return out


def dirichlet_faces(mesh: Mesh):
    """Boolean [n_faces]: the face lies on a Dirichlet side."""
    nx, ny, nz = mesh.n
    fx, fy, fz = n_faces(mesh)
    mask = np.zeros(fx + fy + fz, dtype=bool)
    ix = np.arange(fx) % (nx + 1)
    iy = (np.arange(fy) // nx) % (ny + 1)
    iz = np.arange(fz) // (nx * ny)
    for hi in (0, 1):
        if mesh.bc[0 + hi] == DIRICHLET:
            mask[:fx] |= ix == (nx if hi else 0)
        if mesh.bc[2 + hi] == DIRICHLET:
            mask[fx:fx + fy] |= iy == (ny if hi else 0)
        if mesh.bc[4 + hi] == DIRICHLET:
            mask[fx + fy:] |= iz == (nz if hi else 0)
    return mask


def dirichlet_mask(mesh: Mesh):
    return np.repeat(dirichlet_faces(mesh), (mesh.k + 1) ** 2)


class LocalMatrices:
    """Quadrature-built HDG matrices of a batch of cells (see the module docstring)."""

    def __init__(self, mesh: Mesh, cells, tau: float = TAU):
        k, n = mesh.k, mesh.k + 1
        m = n ** 3
        quad = CellQuadrature(k)
        cells = np.asarray(cells)
        Jinv, detJ = cell_geometry(mesh, cells, quad)
        wdet = quad.w[None, :] * detJ                                   # [C, q]
        kap = cell_kappa(mesh, cells, quad)
        phys = np.einsum('cqed,qei->cqdi', Jinv, quad.grad)             # d phi_i / d x_d
        Mk = np.einsum('cq,qi,qj->cij', wdet / kap, quad.val, quad.val)
        C_ = len(cells)
        self.A = np.zeros((C_, 3 * m, 3 * m))
        for d in range(3):
            self.A[:, d * m:(d + 1) * m, d * m:(d + 1) * m] = Mk
        self.E = np.einsum('cq,qv,cqdj->cvdj', wdet, quad.val, phys).reshape(C_, m, 3 * m)
        self.C, self.G, self.H = [], [], []
        self.D = np.zeros((C_, m, m))
        for side in range(6):
            d, sign = side // 2, (1.0 if side % 2 else -1.0)
            ref = FaceRef(k, d, sign)
            _, nrm, JxW, _ = face_geometry(mesh, cells, ref)
            t1, t2 = [e for e in range(3) if e != d]
            a = np.arange(n * n) % n
            b = np.arange(n * n) // n
            nodes = Basis1D(k).nodes
            mu = lagrange(nodes, ref.pts[:, t1])[:, a] * lagrange(nodes, ref.pts[:, t2])[:, b]
            self.C.append(np.einsum('cq,qa,qj,cqd->cadj', JxW, mu, ref.val, nrm).reshape(C_, n * n, 3 * m))
            self.G.append(tau * np.einsum('cq,qa,qj->caj', JxW, mu, ref.val))
            self.D += tau * np.einsum('cq,qi,qj->cij', JxW, ref.val, ref.val)
            self.H.append(tau * np.einsum('cq,qa,qb->cab', JxW, mu, mu))
        Z = np.zeros((C_, 4 * m, 4 * m))
        Z[:, :3 * m, :3 * m] = self.A
        Z[:, :3 * m, 3 * m:] = -np.transpose(self.E, (0, 2, 1))
        Z[:, 3 * m:, :3 * m] = self.E
        Z[:, 3 * m:, 3 * m:] = self.D
        self.L = Z
        self.m, self.nf = m, n * n

    def trace_rhs(self, lam):
        """[-C^T lambda; G^T lambda] for lam [C, 6, n^2] -> [C, 4m]."""
        rq = -sum(np.einsum('caj,ca->cj', self.C[s], lam[:, s]) for s in range(6))
        ru = sum(np.einsum('caj,ca->cj', self.G[s], lam[:, s]) for s in range(6))
        return np.concatenate([rq, ru], axis=1)

    def solve(self, R):
        return np.linalg.solve(self.L, R[..., None])[..., 0]

    def trace_out(self, lam, qu):
        """y_s = H^K_s lambda_s - C_s q - G_s u  -> [C, 6, n^2]."""
        m = self.m
        q, u = qu[:, :3 * m], qu[:, 3 * m:]
        return np.stack([np.einsum('cab,cb->ca', self.H[s], lam[:, s])
                         - np.einsum('caj,cj->ca', self.C[s], q)
                         - np.einsum('caj,cj->ca', self.G[s], u) for s in range(6)], axis=1)

    def element_trace_matrix(self):
        """K^e = H^e - [C G] L^-1 [-C^T; G^T]  [C, 6 n^2, 6 n^2] (eq:hdg_matrix_condensed per cell)."""
        C_, nf = len(self.L), self.nf
        cols = []
        for s in range(6):
            for a in range(nf):
                lam = np.zeros((C_, 6, nf))
                lam[:, s, a] = 1.0
                cols.append(self.trace_out(lam, self.solve(self.trace_rhs(lam))).reshape(C_, 6 * nf))
        return np.stack(cols, axis=2)


class HdgOperator:
    """The condensed trace operator K, its right-hand side and the local recovery."""

    def __init__(self, mesh: Mesh, tau: float = TAU, chunk: int = 512):
        self.mesh, self.tau, self.chunk = mesh, tau, chunk
        self.nf = (mesh.k + 1) ** 2
        self.fid = cell_face_ids(mesh)
        self.n = n_trace_dofs(mesh)
        self.dmask = dirichlet_mask(mesh)
        self.uniform = mesh.uniform
        if self.uniform:
            self.loc0 = LocalMatrices(mesh, np.array([0]), tau)
            self.Ke0 = self.loc0.element_trace_matrix()[0]

    def _chunks(self):
        for c0 in range(0, self.mesh.n_cells, self.chunk):
            cells = np.arange(c0, min(c0 + self.chunk, self.mesh.n_cells))
            loc = self.loc0 if self.uniform else LocalMatrices(self.mesh, cells, self.tau)
            yield cells, loc

    def _gather(self, x, cells):
        idx = self.fid[cells][:, :, None] * self.nf + np.arange(self.nf)[None, None, :]
        return x[idx], idx

    def _bcast(self, loc, ncell):
        """The shared matrices of a uniform mesh for a batch of ncell cells."""
        if not self.uniform:
            return loc

        class B:
            pass
        b = B()
        for name in ('L', 'H', 'C', 'G'):
            v = getattr(loc, name)
            setattr(b, name, [np.broadcast_to(t, (ncell,) + t.shape[1:]) for t in v]
                    if isinstance(v, list) else np.broadcast_to(v, (ncell,) + v.shape[1:]))
        b.m, b.nf = loc.m, loc.nf
        b.trace_rhs = lambda lam: LocalMatrices.trace_rhs(b, lam)
        b.solve = lambda R: np.linalg.solve(np.broadcast_to(loc.L[0], (len(R),) + loc.L.shape[1:]),
                                            R[..., None])[..., 0]
        b.trace_out = lambda lam, qu: LocalMatrices.trace_out(b, lam, qu)
        return b

    def apply(self, x, identity_dirichlet=True):
        """y = K x (Dirichlet rows: y = x, Dirichlet entries of x read as 0)."""
        x = np.asarray(x, dtype=np.float64)
        xin = np.where(self.dmask, 0.0, x) if identity_dirichlet else x
        y = np.zeros(self.n)
        for cells, loc in self._chunks():
            lam, idx = self._gather(xin, cells)
            if self.uniform:
                ye = lam.reshape(len(cells), -1) @ self.Ke0.T
            else:
                ye = loc.trace_out(lam, loc.solve(loc.trace_rhs(lam))).reshape(len(cells), -1)
            np.add.at(y, idx.reshape(len(cells), -1), ye)
        if identity_dirichlet:
            y[self.dmask] = x[self.dmask]
        return y

    def local_solve(self, lam_vec, F=None):
        """(q, u) of every cell from the trace (and the load vector F [n_cells, m] or None):
        returns q [n_cells, 3, m], u [n_cells, m] (u in the DG layout of oracle.sipg)."""
        mesh = self.mesh
        m = (mesh.k + 1) ** 3
        Q = np.zeros((mesh.n_cells, 3, m))
        U = np.zeros((mesh.n_cells, m))
        lam_vec = np.where(self.dmask, 0.0, lam_vec)
        for cells, loc in self._chunks():
            lam, _ = self._gather(lam_vec, cells)
            bl = self._bcast(loc, len(cells))
            R = bl.trace_rhs(lam)
            if F is not None:
                R[:, 3 * m:] += F[cells]
            qu = bl.solve(R)
            Q[cells] = qu[:, :3 * m].reshape(len(cells), 3, m)
            U[cells] = qu[:, 3 * m:]
        return Q, U

    def rhs(self, F):
        """r = sum_K [C G] L^-1 [0; F] (Dirichlet rows 0), F [n_cells, m]."""
        mesh = self.mesh
        m = (mesh.k + 1) ** 3
        r = np.zeros(self.n)
        for cells, loc in self._chunks():
            bl = self._bcast(loc, len(cells))
            R = np.zeros((len(cells), 4 * m))
            R[:, 3 * m:] = F[cells]
            qu = bl.solve(R)
            zero = np.zeros((len(cells), 6, self.nf))
            ye = -bl.trace_out(zero, qu)                         # C q + G u
            _, idx = self._gather(r, cells)
            np.add.at(r, idx.reshape(len(cells), -1), ye.reshape(len(cells), -1))
        r[self.dmask] = 0.0
        return r

    def diagonal(self):
        """diag(K) (1 on Dirichlet rows)."""
        d = np.zeros(self.n)
        for cells, loc in self._chunks():
            Ke = np.broadcast_to(self.Ke0, (len(cells),) + self.Ke0.shape) if self.uniform \
                else loc.element_trace_matrix()
            _, idx = self._gather(d, cells)
            np.add.at(d, idx.reshape(len(cells), -1), np.diagonal(Ke, axis1=1, axis2=2))
        d[self.dmask] = 1.0
        return d

    def assemble(self, identity_dirichlet=True) -> sp.csr_matrix:
        """Global K (tiny meshes) from the per-cell K^e."""
        rows, cols, vals = [], [], []
        for cells, loc in self._chunks():
            Ke = np.broadcast_to(self.Ke0, (len(cells),) + self.Ke0.shape) if self.uniform \
                else loc.element_trace_matrix()
            _, idx = self._gather(np.zeros(self.n), cells)
            idx = idx.reshape(len(cells), -1)
            rows.append(np.repeat(idx, idx.shape[1], axis=1).ravel())
            cols.append(np.tile(idx, (1, idx.shape[1])).ravel())
            vals.append(np.asarray(Ke).ravel())
        K = sp.coo_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))),
                          shape=(self.n, self.n)).tocsr()
        if identity_dirichlet:
            keep = sp.diags((~self.dmask).astype(float))
            K = keep @ K @ keep + sp.diags(self.dmask.astype(float))
        return K.tocsr()


def load(mesh: Mesh):
    """F = (f, v) per cell [n_cells, m] for the manufactured f of oracle.problem (O8)."""
    return load_vector(mesh, SIPG).reshape(mesh.n_cells, -1)


def jacobi_pcg(op: HdgOperator, b, tol=1e-10, maxit=5000):
    """PCG with the diagonal of K (Dirichlet rows identity), x0 = 0; stopping test
    ||r|| <= tol ||b|| on the updated residual (reading R13).  Returns x, its, relres history."""
    dinv = 1.0 / op.diagonal()
    x = np.zeros_like(b)
    r = b.copy()
    nb = np.linalg.norm(b)
    z = dinv * r
    p = z.copy()
    rz = r @ z
    hist = [1.0]
    for it in range(1, maxit + 1):
        q = op.apply(p)
        alpha = rz / (p @ q)
        x += alpha * p
        r -= alpha * q
        hist.append(np.linalg.norm(r) / nb)
        if hist[-1] <= tol:
            return x, it, hist
        z = dinv * r
        rz_new = r @ z
        p = z + (rz_new / rz) * p
        rz = rz_new
    return x, maxit, hist


def mixed_apply(mesh: Mesh, q, u, tau: float = TAU):
    """Mixed (flux-substituted) HDG operator on cell unknowns q [n_cells, 3, m], u [n_cells, m]:
    lambda_F = H_F^-1 sum_K (C q + G u) on every non-Dirichlet face (0 on Dirichlet faces),
    y_q = A q - E^T u + C^T lambda,  y_u = E q + D u - G^T lambda  (see the docstring)."""
    k = mesh.k
    nf = (k + 1) ** 2
    m = (k + 1) ** 3
    fid = cell_face_ids(mesh)
    nfaces = sum(n_faces(mesh))
    dmf = dirichlet_faces(mesh)
    cells = np.arange(mesh.n_cells)
    loc = LocalMatrices(mesh, np.array([0]) if mesh.uniform else cells, tau)
    bc = (lambda t: np.broadcast_to(t, (mesh.n_cells,) + t.shape[1:])) if mesh.uniform else (lambda t: t)
    qf = q.reshape(mesh.n_cells, 3 * m)
    S = np.zeros((nfaces, nf))
    Hs = np.zeros((nfaces, nf, nf))
    for s in range(6):
        np.add.at(S, fid[:, s], np.einsum('caj,cj->ca', bc(loc.C[s]), qf) + np.einsum('caj,cj->ca', bc(loc.G[s]), u))
        np.add.at(Hs, fid[:, s], bc(loc.H[s]))
    lam_f = np.zeros((nfaces, nf))
    free = ~dmf
    lam_f[free] = np.linalg.solve(Hs[free], S[free][..., None])[..., 0]
    lam = lam_f[fid]                                                    # [C, 6, nf]
    yq = np.einsum('cij,cj->ci', bc(loc.A), qf) - np.einsum('cji,cj->ci', bc(loc.E), u) \
        + sum(np.einsum('caj,ca->cj', bc(loc.C[s]), lam[:, s]) for s in range(6))
    yu = np.einsum('cij,cj->ci', bc(loc.E), qf) + np.einsum('cij,cj->ci', bc(loc.D), u) \
        - sum(np.einsum('caj,ca->cj', bc(loc.G[s]), lam[:, s]) for s in range(6))
    return yq.reshape(mesh.n_cells, 3, m), yu


def trace_node_points(mesh: Mesh):
    """Physical coordinates [n_trace, 3] of the trace nodes (GLL points of each face)."""
    k, n = mesh.k, mesh.k + 1
    nodes = Basis1D(k).nodes
    fid = cell_face_ids(mesh)
    pts = np.zeros((sum(n_faces(mesh)), n * n, 3))
    a = np.arange(n * n) % n
    b = np.arange(n * n) // n
    cc = mesh.cell_coords()
    for side in range(6):
        d = side // 2
        t1, t2 = [e for e in range(3) if e != d]
        xi = np.zeros((n * n, 3))
        xi[:, d] = 1.0 if side % 2 else -1.0
        xi[:, t1], xi[:, t2] = nodes[a], nodes[b]
        pts[fid[:, side]] = mesh.points(cc, xi)
    return pts.reshape(-1, 3)


def postprocess(mesh: Mesh, Q, U):
    """Element-by-element post-processing ([cgl09]): u* in Q_{k+1}(K) with
        (grad u*, grad w)_K = -(q, grad w)_K   for all w in Q_{k+1}(K),   (u*, 1)_K = (u, 1)_K,
    q = -grad u in the HDG sense (Q [n_cells, 3, m], U [n_cells, m] from local_solve).  GLL-nodal
    Q_{k+1} basis, Gauss (k+2)^3 quadrature, the singular Neumann system closed by the mean
    condition (one row replaced).  Returns u* [n_cells, (k+2)^3] (DG layout of degree k+1)."""
    from .cg import CellQuadrature as CQ
    from .mesh import eval_basis_3d
    k = mesh.k
    quad = CQ(k + 1)                                        # Gauss (k+2)^3, basis degree k+1
    lo_nodes = Basis1D(k).nodes
    val_lo, _ = eval_basis_3d(lo_nodes, quad.pts)           # degree-k basis at the points [q, m]
    ms = (k + 2) ** 3
    out = np.zeros((mesh.n_cells, ms))
    for c0 in range(0, mesh.n_cells, 256):
        cells = np.arange(c0, min(c0 + 256, mesh.n_cells))
        Jinv, detJ = cell_geometry(mesh, cells, quad)
        W = quad.w[None, :] * detJ                                          # [C, q]
        phys = np.einsum('cqed,qei->cqdi', Jinv, quad.grad)                 # grad w_i at q [C, q, 3, i]
        Kst = np.einsum('cq,cqdi,cqdj->cij', W, phys, phys)
        qq = np.einsum('qj,cdj->cqd', val_lo, Q[cells])                     # q at the points
        rhs = -np.einsum('cq,cqd,cqdi->ci', W, qq, phys)
        mean_w = np.einsum('cq,qi->ci', W, quad.val)                        # (w_i, 1)
        mean_u = np.einsum('cq,qj,cj->c', W, val_lo, U[cells])              # (u, 1)
        A = Kst.copy()
        A[:, 0, :] = mean_w                                                 # replace row 0: the mean
        rhs[:, 0] = mean_u
        out[cells] = np.linalg.solve(A, rhs[..., None])[..., 0]
    return out
