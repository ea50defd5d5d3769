"""Geometric multigrid V-cycle with Chebyshev-Jacobi smoothing inside CG.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Follows P:L1144-1185 (sec:comparison, sec:mg_cg) step by step:
* PCG with a multigrid V-cycle preconditioner, stopped once the residual norm
  is below tol x the right-hand-side norm (tol = 1e-10 from
  BASELINE.json, reading R13: recursively updated residual, checked after each
  update, iterations = number of x updates).
* "polynomial Chebyshev accelerated pointwise Jacobi smoother" on
  [0.06 lam, 1.2 lam] of the Jacobi-preconditioned matrix, with
  lam from "15 iterations with the conjugate gradient method".
  Reading O5/R9: Saad Alg. 12.1 form, p = degree of the error polynomial, the
  same polynomial pre and post; p-1 operator applies from a zero start.
  Reading O6/R10: Jacobi-PCG on A x = s, s = splitmix64 seed 0x5eed (global
  index, Dirichlet entries zero), Lanczos matrix from the CG coefficients
  T_jj = 1/a_j + b_{j-1}/a_{j-1}, T_j,j+1 = sqrt(b_j)/a_j; lam = lambda_max(T).
* level transfer = nodal interpolation and its transpose (oracle.transfer).
* coarse level: exact dense Cholesky of the level-0 matrix on free DoFs
  (reading R11; the paper uses Chebyshev to 1e-3 there).
Level operators are re-discretised on every level (reading R12).
"""
from __future__ import annotations

import numpy as np
import scipy.linalg as sla

import fem_inputs
from . import cg as cgop
from . import sipg as sipgop
from . import transfer
from .mesh import Mesh, CG


class Level:
    def __init__(self, mesh: Mesh, method: int, penalty_factor: float):
        self.mesh, self.method, self.pf = mesh, method, penalty_factor
        if method == CG:
            self.free = ~mesh.cg_dirichlet_mask()
            self.n_dofs = mesh.cg_n_dofs()
        else:
            self.free = np.ones(mesh.dg_n_dofs(), dtype=bool)
            self.n_dofs = mesh.dg_n_dofs()
        self.op = (cgop.Operator(mesh) if method == CG
                   else sipgop.Operator(mesh, penalty_factor))
        self._diag = None
        self.lam = None

    def apply(self, x):
        return self.op.apply(x)

    def diagonal(self):
        if self._diag is None:
            self._diag = self.op.diagonal()
        return self._diag

    def assemble(self):
        return (cgop.assemble(self.mesh) if self.method == CG
                else sipgop.assemble(self.mesh, self.pf))


def estimate_lambda_max(level: Level, iters: int = 15, seed: int = 0x5EED):
    """lam_max(D^-1 A) from `iters` Jacobi-PCG iterations (Lanczos from CG coefficients).
    Returns (lam, T)."""
    s = fem_inputs.uniform_pm1(seed, level.n_dofs)
    s = np.where(level.free, s, 0.0)
    Dinv = np.where(level.free, 1.0 / level.diagonal(), 0.0)
    x = np.zeros_like(s)
    r = s.copy()
    z = Dinv * r
    p = z.copy()
    rz = r @ z
    alphas, betas = [], []
    for _ in range(iters):
        q = level.apply(p)
        pq = p @ q
        if pq <= 0 or rz <= 0:
            break
        alpha = rz / pq
        x += alpha * p
        r -= alpha * q
        z = Dinv * r
        rz_new = r @ z
        beta = rz_new / rz
        alphas.append(alpha)
        betas.append(beta)
        rz = rz_new
        if rz_new == 0.0:
            break
        p = z + beta * p
    m = len(alphas)
    T = np.zeros((m, m))
    for j in range(m):
        T[j, j] = 1.0 / alphas[j] + (betas[j - 1] / alphas[j - 1] if j > 0 else 0.0)
        if j + 1 < m:
            T[j, j + 1] = T[j + 1, j] = np.sqrt(betas[j]) / alphas[j]
    return float(np.max(np.linalg.eigvalsh(T))), T


def chebyshev(level: Level, b, x, degree, lo, hi, x_is_zero):
    """Saad Alg. 12.1 Chebyshev acceleration of Jacobi on [lo*lam, hi*lam] (reading O5).

    Error propagation: T_p((theta - lam_i)/delta) / T_p(theta/delta) on the
    eigenvalues lam_i of D^-1 A; applies: p-1 from x = 0, p otherwise."""
    a, c = hi * level.lam, lo * level.lam
    theta, delta = 0.5 * (a + c), 0.5 * (a - c)
    sigma = theta / delta
    rho = 1.0 / sigma
    Dinv = np.where(level.free, 1.0 / level.diagonal(), 0.0)
    r = b.copy() if x_is_zero else b - level.apply(x)
    x = np.zeros_like(b) if x_is_zero else x.copy()
    d = Dinv * r / theta
    for i in range(1, degree + 1):
        x += d
        if i == degree:
            break
        r -= level.apply(d)
        rho_new = 1.0 / (2.0 * sigma - rho)
        d = rho_new * rho * d + (2.0 * rho_new / delta) * (Dinv * r)
        rho = rho_new
    return x


class Multigrid:
    def __init__(self, mesh: Mesh, method: int, penalty_factor: float = 2.0,
                 cheb_degree: int = 5, cheb_lo: float = 0.06, cheb_hi: float = 1.2,
                 eig_iters: int = 15, coarse_cells: int = 1, eig_seed: int = 0x5EED,
                 lambda_override=None):
        self.method = method
        self.levels = [Level(m, method, penalty_factor) for m in transfer.hierarchy(mesh, coarse_cells)]
        self.degree, self.lo, self.hi = cheb_degree, cheb_lo, cheb_hi
        for l, lev in enumerate(self.levels):
            if l == 0:
                continue
            if lambda_override is not None:
                lev.lam = float(lambda_override[l])
            else:
                lev.lam, _ = estimate_lambda_max(lev, eig_iters, eig_seed)
        A0 = self.levels[0].assemble().toarray()
        f0 = self.levels[0].free
        self.coarse_free = np.nonzero(f0)[0]
        self.coarse_chol = np.linalg.cholesky(A0[np.ix_(self.coarse_free, self.coarse_free)])

    @property
    def fine(self):
        return self.levels[-1]

    def coarse_solve(self, b):
        L = self.coarse_chol
        x = np.zeros_like(b)
        y = sla.solve_triangular(L, b[self.coarse_free], lower=True)
        x[self.coarse_free] = sla.solve_triangular(L.T, y, lower=False)
        return x

    def prolongate(self, l, xc):
        return transfer.prolongate(self.levels[l - 1].mesh, self.levels[l].mesh, self.method, xc)

    def restrict(self, l, xf):
        return transfer.restrict(self.levels[l - 1].mesh, self.levels[l].mesh, self.method, xf)

    def vcycle(self, b, l=None):
        """V(l, b) per SURVEY §8a R10."""
        if l is None:
            l = len(self.levels) - 1
        if l == 0:
            return self.coarse_solve(b)
        lev = self.levels[l]
        x = chebyshev(lev, b, None, self.degree, self.lo, self.hi, x_is_zero=True)
        r = b - lev.apply(x)
        x = x + self.prolongate(l, self.vcycle(self.restrict(l, r), l - 1))
        return chebyshev(lev, b, x, self.degree, self.lo, self.hi, x_is_zero=False)

    def pcg(self, b, tol=1e-10, maxit=1000, x0=None, history=None):
        """PCG per SURVEY §8a R11; returns (x, iterations, ||r||/||b||)."""
        A = self.fine.apply
        x = np.zeros_like(b) if x0 is None else x0.copy()
        r = b - A(x) if x0 is not None else b.copy()
        bnorm = np.linalg.norm(b)
        rn = np.linalg.norm(r)
        if history is not None:
            history.append(rn)
        if rn <= tol * bnorm:
            return x, 0, rn / bnorm
        z = self.vcycle(r)
        p = z.copy()
        rz = r @ z
        it = 0
        while it < maxit:
            q = A(p)
            pq = p @ q
            if not pq > 0:
                raise FloatingPointError(f"breakdown p^T A p = {pq} at iteration {it + 1}")
            alpha = rz / pq
            x += alpha * p
            r -= alpha * q
            it += 1
            rn = np.linalg.norm(r)
            if history is not None:
                history.append(rn)
            if rn <= tol * bnorm:
                break
            z = self.vcycle(r)
            rz_new = r @ z
            p = z + (rz_new / rz) * p
            rz = rz_new
        return x, it, rn / bnorm
