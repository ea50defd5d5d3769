"""1-D quadrature rules and the Lagrange basis in Gauss-Lobatto nodes.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

* Basis: Lagrange polynomials in the (k+1) Gauss-Lobatto-Legendre nodes,
  P:L175-179 (sec:discret_fem, "basis representation by Lagrange polynomials in
  the nodes of the (k+1)-point Gauss--Lobatto--Legendre quadrature rule").
* Quadrature: Gauss-Legendre with k+1 points per direction
  (after eq:mf_eval).
Reference interval [-1, 1] as in P:L154-155 ("image of the reference domain
[-1,1]^d").
"""
from __future__ import annotations

import numpy as np
from numpy.polynomial import legendre as L


def gauss_rule(n: int):
    """n-point Gauss-Legendre points and weights on [-1, 1] (library routine)."""
    if n < 1:
        raise ValueError("n >= 1")
    x, w = L.leggauss(n)
    return np.asarray(x, dtype=np.float64), np.asarray(w, dtype=np.float64)


def gll_nodes(k: int) -> np.ndarray:
    """The k+1 Gauss-Lobatto-Legendre nodes: -1, +1 and the roots of P_k'.

    Roots from the companion matrix, polished by Newton on P_k' (tol 1e-15).
    """
    if k < 1:
        raise ValueError("k >= 1")
    if k == 1:
        return np.array([-1.0, 1.0])
    dPk = L.Legendre.basis(k).deriv()
    d2Pk = dPk.deriv()
    r = np.sort(np.real(dPk.roots()))
    for _ in range(50):
        step = dPk(r) / d2Pk(r)
        r = r - step
        if np.max(np.abs(step)) < 1e-15:
            break
    r = 0.5 * (r - r[::-1])           # enforce exact symmetry about 0
    return np.concatenate(([-1.0], r, [1.0]))


def lagrange(nodes: np.ndarray, xi) -> np.ndarray:
    """phi_i(xi) = prod_{j!=i} (xi - x_j)/(x_i - x_j); returns [len(xi), n]."""
    xi = np.atleast_1d(np.asarray(xi, dtype=np.float64))
    n = len(nodes)
    out = np.ones((len(xi), n))
    for i in range(n):
        for j in range(n):
            if j != i:
                out[:, i] *= (xi - nodes[j]) / (nodes[i] - nodes[j])
    return out


def lagrange_deriv(nodes: np.ndarray, xi) -> np.ndarray:
    """phi_i'(xi) by the product rule (no tables):
    sum_{m!=i} 1/(x_i-x_m) prod_{j!=i,m} (xi-x_j)/(x_i-x_j); returns [len(xi), n]."""
    xi = np.atleast_1d(np.asarray(xi, dtype=np.float64))
    n = len(nodes)
    out = np.zeros((len(xi), n))
    for i in range(n):
        for m in range(n):
            if m == i:
                continue
            term = np.full(len(xi), 1.0 / (nodes[i] - nodes[m]))
            for j in range(n):
                if j != i and j != m:
                    term *= (xi - nodes[j]) / (nodes[i] - nodes[j])
            out[:, i] += term
    return out


class Basis1D:
    """Nodes, Gauss rule and basis tables for degree k (n = k+1 points)."""

    def __init__(self, k: int, n_q: int | None = None):
        self.k = k
        self.n = k + 1
        self.nodes = gll_nodes(k)
        self.n_q = n_q or (k + 1)
        self.qp, self.qw = gauss_rule(self.n_q)
        self.val = lagrange(self.nodes, self.qp)          # [q, i]
        self.der = lagrange_deriv(self.nodes, self.qp)    # [q, i]
