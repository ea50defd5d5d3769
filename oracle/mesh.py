"""Structured hexahedral mesh, deformation map, Jacobians and DoF numbering.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

* Cells are images of [-1,1]^3.  The configs use the box [0,1]^3
  split into n[0] x n[1] x n[2] cells, optionally deformed by
  x_d = xhat_d + eps * s(xhat),  s = prod_e sin(pi t_e),  t_e = (xhat_e-lo_e)/(hi_e-lo_e)
  (BASELINE.json configs[1], configs[4]; SURVEY §8c reading R2: s is evaluated at
  the undeformed point, same map on every multigrid level).
* J = dx/dxi is the analytic derivative of that composed map (chain rule);
  the oracle inverts it with numpy.linalg (no closed form shared with the GPU).
* SURVEY §8f N3 (readings N3-a..c):
  - geometry SHELL: one of the six cube-sphere patches of the paper's spherical shell
    with inner radius 0.5 and outer radius 1.0, t = (c + (xi+1)/2)/n in
    [0,1]^3, a = tan(pi/2 (t_0 - 1/2)), b = tan(pi/2 (t_1 - 1/2)) (equiangular
    gnomonic coordinates of the +x cap), r = 0.5 + 0.5 t_2,  x = r (1, a, b)/|(1, a, b)|;
  - mapping_degree l > 0: "a polynomial mapping of degree l ... on GLL support
    points": per cell x(xi) = sum_j X_j phi^l_j(xi) with
    X_j the exact map (manifold) at the tensor GLL(l) points; J its derivative;
  - kappa_amp A != 0: variable diffusivity eq:diffusivity_shell
    kappa(x) = 1 + A prod_{e=1..3} cos(2 pi x_e + 0.1 e) at the physical point
    (the paper's A = 1e6 makes kappa negative in places: reading N3-c).
* CG numbering: node (k*cx+i, k*cy+j, k*cz+l), x fastest.
  DG numbering: cell*(k+1)^3 + (i + n*j + n^2*l), cells lexicographic, x fastest.
* Boundary sides are ordered -x,+x,-y,+y,-z,+z; 0 = Dirichlet, 1 = Neumann.
"""
from __future__ import annotations

import numpy as np

from .basis import lagrange, lagrange_deriv

CG, SIPG = 0, 1
DIRICHLET, NEUMANN = 0, 1
BOX, SHELL = 0, 1
SHELL_R = (0.5, 1.0)        # inner / outer radius


class Mesh:
    def __init__(self, n, k, lo=(0.0, 0.0, 0.0), hi=(1.0, 1.0, 1.0), eps=0.0,
                 bc=(DIRICHLET,) * 6, geometry=BOX, mapping_degree=0, kappa_amp=0.0):
        self.n = tuple(int(v) for v in n)
        self.k = int(k)
        self.lo = np.asarray(lo, dtype=np.float64)
        self.hi = np.asarray(hi, dtype=np.float64)
        self.eps = float(eps)
        self.bc = tuple(int(b) for b in bc)
        self.geometry = int(geometry)
        self.mapping_degree = int(mapping_degree)
        self.kappa_amp = float(kappa_amp)
        # same G on every cell: Cartesian box, exact map, kappa = 1
        self.uniform = (self.geometry == BOX and self.eps == 0.0 and self.kappa_amp == 0.0
                        and self.mapping_degree == 0)
        self.h = (self.hi - self.lo) / np.asarray(self.n, dtype=np.float64)
        self.n_cells = self.n[0] * self.n[1] * self.n[2]
        self.nn = tuple(self.k * m + 1 for m in self.n)       # CG nodes per direction

    # ---- cells -------------------------------------------------------------
    def cell_coords(self, cells=None):
        """(cx, cy, cz) of lexicographic cell ids (x fastest)."""
        if cells is None:
            cells = np.arange(self.n_cells)
        cells = np.asarray(cells)
        cx = cells % self.n[0]
        cy = (cells // self.n[0]) % self.n[1]
        cz = cells // (self.n[0] * self.n[1])
        return np.stack([cx, cy, cz], axis=-1)

    def cell_id(self, c):
        c = np.asarray(c)
        return c[..., 0] + self.n[0] * (c[..., 1] + self.n[1] * c[..., 2])

    # ---- geometry ----------------------------------------------------------
    def xhat(self, cc, xi):
        """Undeformed point of reference point xi [P,3] in cells cc [C,3] -> [C,P,3]."""
        return self.lo + self.h * (cc[:, None, :] + 0.5 * (xi[None, :, :] + 1.0))

    def _t(self, xh):
        return (xh - self.lo) / (self.hi - self.lo)

    def phys(self, xh):
        """x = xhat + eps * s(xhat) * (1,1,1)."""
        s = np.prod(np.sin(np.pi * self._t(xh)), axis=-1)
        return xh + self.eps * s[..., None]

    def like(self, n):
        """The same geometry, coefficient and boundary conditions on n cells."""
        return Mesh(n, self.k, self.lo, self.hi, self.eps, self.bc, self.geometry,
                    self.mapping_degree, self.kappa_amp)

    def kappa(self, x):
        """eq:diffusivity_shell, kappa = 1 + A prod_{e=1}^{3} cos(2 pi x_e + 0.1 e)."""
        if self.kappa_amp == 0.0:
            return np.ones(x.shape[:-1])
        e = np.arange(1, 4)
        return 1.0 + self.kappa_amp * np.prod(np.cos(2.0 * np.pi * x + 0.1 * e), axis=-1)

    def grad_kappa(self, x):
        if self.kappa_amp == 0.0:
            return np.zeros(x.shape)
        e = np.arange(1, 4)
        c = np.cos(2.0 * np.pi * x + 0.1 * e)
        s = np.sin(2.0 * np.pi * x + 0.1 * e)
        g = np.empty(x.shape)
        for d in range(3):
            o = [f for f in range(3) if f != d]
            g[..., d] = -2.0 * np.pi * self.kappa_amp * s[..., d] * c[..., o[0]] * c[..., o[1]]
        return g

    # exact map ("manifold") and its analytic Jacobian
    def _shell_t(self, cc, xi):
        return (cc[:, None, :] + 0.5 * (xi[None, :, :] + 1.0)) / np.asarray(self.n, dtype=np.float64)

    def _map_t(self, t):
        """Exact map of patch coordinates t in [0,1]^3 (any leading shape)."""
        if self.geometry == BOX:
            return self.phys(self.lo + (self.hi - self.lo) * t)
        a = np.tan(0.5 * np.pi * (t[..., 0] - 0.5))
        b = np.tan(0.5 * np.pi * (t[..., 1] - 0.5))
        r = SHELL_R[0] + (SHELL_R[1] - SHELL_R[0]) * t[..., 2]
        q = np.stack([np.ones_like(a), a, b], axis=-1)
        return (r / np.linalg.norm(q, axis=-1))[..., None] * q

    def manifold(self, cc, xi):
        """Exact physical point of reference points xi [P,3] in cells cc [C,3] -> [C,P,3]."""
        if self.geometry == BOX:
            return self.phys(self.xhat(cc, xi))
        return self._map_t(self._shell_t(cc, xi))

    def points_each(self, cc, xi, chunk=20000):
        """x(xi_i) in cell cc_i, one reference point per cell: cc, xi [P,3] -> [P,3]."""
        out = np.empty((len(cc), 3))
        for c0 in range(0, len(cc), chunk):
            sl = slice(c0, c0 + chunk)
            if self.mapping_degree == 0:
                t = (cc[sl] + 0.5 * (xi[sl] + 1.0)) / np.asarray(self.n, dtype=np.float64)
                out[sl] = self._map_t(t)
            else:
                X, nodes = self._support(cc[sl])
                n = len(nodes)
                v = [lagrange(nodes, xi[sl][:, d]) for d in range(3)]
                j = np.arange(n ** 3)
                val = v[0][:, j % n] * v[1][:, (j // n) % n] * v[2][:, j // (n * n)]
                out[sl] = np.einsum('pj,pjd->pd', val, X)
        return out

    def manifold_jacobian(self, cc, xi):
        if self.geometry == BOX:
            return self._box_jacobian(cc, xi)
        t = self._shell_t(cc, xi)
        a = np.tan(0.5 * np.pi * (t[..., 0] - 0.5))
        b = np.tan(0.5 * np.pi * (t[..., 1] - 0.5))
        r = SHELL_R[0] + (SHELL_R[1] - SHELL_R[0]) * t[..., 2]
        q = np.stack([np.ones_like(a), a, b], axis=-1)
        s = np.linalg.norm(q, axis=-1)
        u = q / s[..., None]
        J = np.empty(t.shape + (3,))
        # du/da = (e_1 - u u_1)/s, da/dt_0 = (pi/2)(1 + a^2); likewise b with e_2
        for col, (par, e) in enumerate(((a, 1), (b, 2))):
            du = -u * u[..., e, None]
            du[..., e] += 1.0
            du /= s[..., None]
            J[..., :, col] = (r * 0.5 * np.pi * (1.0 + par * par))[..., None] * du
        J[..., :, 2] = (SHELL_R[1] - SHELL_R[0]) * u
        return J * (0.5 / np.asarray(self.n, dtype=np.float64))[None, None, None, :]

    def _support(self, cc):
        """Support points X_j [C, (l+1)^3, 3] of the degree-l mapping and the GLL(l) nodes."""
        from .basis import gll_nodes
        nodes = gll_nodes(self.mapping_degree)
        return self.manifold(cc, tensor_points(nodes)), nodes

    def points(self, cc, xi):
        """Physical points x(xi) of the cells' mapping -> [C,P,3]."""
        if self.mapping_degree == 0:
            return self.manifold(cc, xi)
        X, nodes = self._support(cc)
        val, _ = eval_basis_3d(nodes, xi)
        return np.einsum('pj,cjd->cpd', val, X)

    def jacobian(self, cc, xi):
        """J[c, p, d, e] = d x_d / d xi_e  at reference points xi [P,3] of cells cc."""
        if self.mapping_degree == 0:
            return self.manifold_jacobian(cc, xi)
        X, nodes = self._support(cc)
        _, grad = eval_basis_3d(nodes, xi)
        return np.einsum('pej,cjd->cpde', grad, X)

    def _box_jacobian(self, cc, xi):
        xh = self.xhat(cc, xi)
        t = self._t(xh)
        sn = np.sin(np.pi * t)
        cs = np.cos(np.pi * t)
        # ds/dxhat_e = pi/(hi_e-lo_e) cos(pi t_e) prod_{f != e} sin(pi t_f)
        grad_s = np.empty_like(xh)
        for e in range(3):
            others = [f for f in range(3) if f != e]
            grad_s[..., e] = (np.pi / (self.hi[e] - self.lo[e])) * cs[..., e] \
                * sn[..., others[0]] * sn[..., others[1]]
        dxdxh = np.eye(3)[None, None] + self.eps * grad_s[..., None, :]  # [.., d, e]
        return dxdxh * (0.5 * self.h)[None, None, None, :]

    # ---- numbering ---------------------------------------------------------
    def cg_n_dofs(self):
        return self.nn[0] * self.nn[1] * self.nn[2]

    def dg_n_dofs(self):
        return self.n_cells * (self.k + 1) ** 3

    def cg_dofmap(self, cells=None):
        """[C, n^3] global CG indices of the local nodes (i + n j + n^2 l)."""
        cc = self.cell_coords(cells)
        n, k = self.k + 1, self.k
        l0 = np.arange(n)
        gx = k * cc[:, 0, None] + l0[None, :]
        gy = k * cc[:, 1, None] + l0[None, :]
        gz = k * cc[:, 2, None] + l0[None, :]
        idx = (gx[:, None, None, :] + self.nn[0] * (gy[:, None, :, None]
               + self.nn[1] * gz[:, :, None, None]))
        return idx.reshape(len(cc), n ** 3)

    def dg_dofmap(self, cells=None):
        if cells is None:
            cells = np.arange(self.n_cells)
        cells = np.asarray(cells)
        m = (self.k + 1) ** 3
        return cells[:, None] * m + np.arange(m)[None, :]

    def cg_node_coords(self):
        """Integer node coordinates (gx, gy, gz) of all CG nodes."""
        i = np.arange(self.cg_n_dofs())
        gx = i % self.nn[0]
        gy = (i // self.nn[0]) % self.nn[1]
        gz = i // (self.nn[0] * self.nn[1])
        return np.stack([gx, gy, gz], axis=-1)

    def cg_dirichlet_mask(self):
        """True on CG nodes lying on a Dirichlet side."""
        g = self.cg_node_coords()
        mask = np.zeros(len(g), dtype=bool)
        for d in range(3):
            if self.bc[2 * d] == DIRICHLET:
                mask |= g[:, d] == 0
            if self.bc[2 * d + 1] == DIRICHLET:
                mask |= g[:, d] == self.nn[d] - 1
        return mask


def tensor_points(p1d):
    """3-D tensor grid of a 1-D point set, x fastest: [n^3, 3]."""
    n = len(p1d)
    q = np.arange(n ** 3)
    return np.stack([p1d[q % n], p1d[(q // n) % n], p1d[q // (n * n)]], axis=-1)


def tensor_weights(w1d):
    n = len(w1d)
    q = np.arange(n ** 3)
    return w1d[q % n] * w1d[(q // n) % n] * w1d[q // (n * n)]


def eval_basis_3d(nodes, pts):
    """Tensor Lagrange basis phi_i(xi) = phi_i0(a) phi_i1(b) phi_i2(c) and its
    reference gradient, evaluated POINTWISE at arbitrary points pts [P,3].
    Returns val [P, n^3] and grad [P, 3, n^3]; local index i = i0 + n i1 + n^2 i2."""
    n = len(nodes)
    v = [lagrange(nodes, pts[:, d]) for d in range(3)]          # [P, n]
    g = [lagrange_deriv(nodes, pts[:, d]) for d in range(3)]
    i = np.arange(n ** 3)
    i0, i1, i2 = i % n, (i // n) % n, i // (n * n)
    val = v[0][:, i0] * v[1][:, i1] * v[2][:, i2]
    grad = np.stack([g[0][:, i0] * v[1][:, i1] * v[2][:, i2],
                     v[0][:, i0] * g[1][:, i1] * v[2][:, i2],
                     v[0][:, i0] * v[1][:, i1] * g[2][:, i2]], axis=1)
    return val, grad
