// 1-D tables of the tensor-product Lagrange basis (host, FP64).
//
// Basis: Lagrange polynomials in the k+1 Gauss-Lobatto-Legendre nodes.
// Quadrature: (k+1)-point Gauss-Legendre.  Collocation derivative on
// the Gauss points (values interpolated to the Gauss points are differentiated
// exactly by the Lagrange basis of the Gauss points, since both represent the
// same degree-k polynomial).  Transfer tables: nodal interpolation of the
// parent basis at the children's nodes (reading R12).
#include <cmath>

#include "internal.h"

namespace fem {

namespace {

// P_n(x) and P_n'(x) by the three-term recurrence.
void legendre(int n, double x, double& p, double& dp) {
  double p0 = 1.0, p1 = x;
  if (n == 0) { p = 1.0; dp = 0.0; return; }
  for (int m = 2; m <= n; ++m) {
    double p2 = ((2 * m - 1) * x * p1 - (m - 1) * p0) / m;
    p0 = p1;
    p1 = p2;
  }
  p = p1;
  // derivative: (1-x^2) P_n' = n (P_{n-1} - x P_n); valid for |x| < 1
  dp = n * (p0 - x * p1) / (1.0 - x * x);
}

void gauss_rule(int n, double* x, double* w) {
  for (int i = 0; i < n; ++i) {
    double z = -std::cos(M_PI * (i + 0.75) / (n + 0.5));
    for (int it = 0; it < 100; ++it) {
      double p, dp;
      legendre(n, z, p, dp);
      double dz = p / dp;
      z -= dz;
      if (std::fabs(dz) < 1e-16) break;
    }
    double p, dp;
    legendre(n, z, p, dp);
    x[i] = z;
    w[i] = 2.0 / ((1.0 - z * z) * dp * dp);
  }
  for (int i = 0; i < n / 2; ++i) {  // exact symmetry
    double a = 0.5 * (x[n - 1 - i] - x[i]);
    x[i] = -a;
    x[n - 1 - i] = a;
    double b = 0.5 * (w[i] + w[n - 1 - i]);
    w[i] = w[n - 1 - i] = b;
  }
  if (n % 2) x[n / 2] = 0.0;
}

// GLL nodes: -1, the k-1 roots of P_k', +1.  Newton on P_k' with
// P_k'' = (2 x P_k' - k(k+1) P_k) / (1 - x^2).
void gll_nodes(int k, double* x) {
  x[0] = -1.0;
  x[k] = 1.0;
  for (int i = 1; i < k; ++i) {
    double z = -std::cos(M_PI * i / k);
    for (int it = 0; it < 100; ++it) {
      double p, dp;
      legendre(k, z, p, dp);
      double d2p = (2.0 * z * dp - k * (k + 1.0) * p) / (1.0 - z * z);
      double dz = dp / d2p;
      z -= dz;
      if (std::fabs(dz) < 1e-16) break;
    }
    x[i] = z;
  }
  for (int i = 1; i < (k + 1) / 2; ++i) {
    double a = 0.5 * (x[k - i] - x[i]);
    x[i] = -a;
    x[k - i] = a;
  }
  if (k % 2 == 0) x[k / 2] = 0.0;
}

double lagr(const double* nodes, int n, int i, double z) {
  double v = 1.0;
  for (int j = 0; j < n; ++j)
    if (j != i) v *= (z - nodes[j]) / (nodes[i] - nodes[j]);
  return v;
}

double lagr_d(const double* nodes, int n, int i, double z) {
  double s = 0.0;
  for (int m = 0; m < n; ++m) {
    if (m == i) continue;
    double t = 1.0 / (nodes[i] - nodes[m]);
    for (int j = 0; j < n; ++j)
      if (j != i && j != m) t *= (z - nodes[j]) / (nodes[i] - nodes[j]);
    s += t;
  }
  return s;
}

}  // namespace

void gll_points(int l, double* x) { gll_nodes(l, x); }

void build_tables(int k, Tables1D& t) {
  t = Tables1D{};
  t.k = k;
  t.n = k + 1;
  const int n = k + 1;
  gll_nodes(k, t.gll);
  gauss_rule(n, t.qp, t.qw);
  for (int q = 0; q < n; ++q)
    for (int i = 0; i < n; ++i) {
      t.val[q][i] = lagr(t.gll, n, i, t.qp[q]);
      t.der[q][i] = lagr_d(t.gll, n, i, t.qp[q]);
      t.colloc[q][i] = lagr_d(t.qp, n, i, t.qp[q]);
    }
  for (int i = 0; i < n; ++i) {
    t.dface[0][i] = lagr_d(t.gll, n, i, -1.0);
    t.dface[1][i] = lagr_d(t.gll, n, i, 1.0);
  }
  // CG: fine node r in [0, 2k] of the two children of a parent cell [-1,1];
  // child 0 covers [-1,0] (eta = (xi-1)/2), child 1 covers [0,1] (eta = (xi+1)/2).
  for (int r = 0; r <= 2 * k; ++r) {
    double eta = (r <= k) ? 0.5 * (t.gll[r] - 1.0) : 0.5 * (t.gll[r - k] + 1.0);
    for (int j = 0; j < n; ++j) t.cg_embed[r][j] = lagr(t.gll, n, j, eta);
  }
  for (int c = 0; c < 2; ++c)
    for (int i = 0; i < n; ++i)
      for (int j = 0; j < n; ++j)
        t.dg_embed[c][i][j] = lagr(t.gll, n, j, 0.5 * (t.gll[i] + (2 * c - 1)));
}

}  // namespace fem
