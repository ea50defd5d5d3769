// Device-side helpers shared by the libfem kernels (sm_100a, FP64).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "internal.h"

namespace fem {

// Even-odd form of a (k+1)x(k+1) 1-D matrix M that is centro-symmetric
// (M[N-1-q][N-1-p] = M[q][p]: the GLL -> Gauss interpolation, both point sets symmetric
// about 0) or anti-centro-symmetric (= -M[q][p]: the collocation derivative): with
// e_j = x_j + x_{N-1-j}, o_j = x_j - x_{N-1-j} (j < N/2; e_h = x_h for odd N),
//   y_q = sum_j E[q][j] e_j + sum_j O[q][j] o_j,  E = (M[q][j] + M[q][N-1-j])/2,
//   O = (M[q][j] - M[q][N-1-j])/2, and the mirrored row y_{N-1-q} = +-(E part) -+ (O part),
// so half the rows need computing: (h+1)^2 + h^2 FMA instead of N^2 (N = 7: 25 vs 49) plus
// 2h adds before and after -- the paper's "even-odd decomposition".
// ET/OT: the same for M^T (the transposed sweeps).
template <int N>
struct EO {
  double E[N][N], O[N][N], ET[N][N], OT[N][N];
};

// Per-degree 1-D tables passed by value (they live in the kernel-parameter
// constant bank, so the sweeps' DFMAs read them as broadcast constant operands).
template <int N>
struct Tab {
  double val[N][N];     // [q][i] GLL basis at Gauss points
  double der[N][N];     // [q][i] GLL basis derivative at Gauss points
  double colloc[N][N];  // [q][p] derivative of the Gauss-point Lagrange basis
  double w[N];          // Gauss weights
  double qp[N];         // Gauss points
  double gll[N];        // GLL nodes
  double dface[2][N];   // phi_i'(-1), phi_i'(+1)
  EO<N> valeo;          // even-odd form of val (centro-symmetric)
  EO<N> coleo;          // even-odd form of colloc (anti-centro-symmetric)
};

template <int N, int LD>
inline void make_eo(const double (&M)[LD][LD], EO<N>& t) {
  constexpr int h = N / 2;
  for (int q = 0; q < N; ++q)
    for (int j = 0; j < N; ++j) {
      t.E[q][j] = t.O[q][j] = t.ET[q][j] = t.OT[q][j] = 0.0;
      if (j < h) {
        t.E[q][j] = 0.5 * (M[q][j] + M[q][N - 1 - j]);
        t.O[q][j] = 0.5 * (M[q][j] - M[q][N - 1 - j]);
        t.ET[q][j] = 0.5 * (M[j][q] + M[N - 1 - j][q]);
        t.OT[q][j] = 0.5 * (M[j][q] - M[N - 1 - j][q]);
      } else if (j == h && (N & 1)) {
        t.E[q][j] = M[q][j];
        t.ET[q][j] = M[j][q];
      }
    }
}

template <int N>
inline Tab<N> make_tab(const Tables1D& t) {
  Tab<N> r;
  for (int q = 0; q < N; ++q) {
    for (int i = 0; i < N; ++i) {
      r.val[q][i] = t.val[q][i];
      r.der[q][i] = t.der[q][i];
      r.colloc[q][i] = t.colloc[q][i];
    }
    r.w[q] = t.qw[q];
    r.qp[q] = t.qp[q];
    r.gll[q] = t.gll[q];
    r.dface[0][q] = t.dface[0][q];
    r.dface[1][q] = t.dface[1][q];
  }
  make_eo<N>(t.val, r.valeo);
  make_eo<N>(t.colloc, r.coleo);
  return r;
}

// out = M in  (out_i = sum_j M[i][j] in_j)
template <int N>
__device__ __forceinline__ void mv(const double (&M)[N][N], const double (&in)[N], double (&out)[N]) {
#pragma unroll
  for (int i = 0; i < N; ++i) {
    double s = 0.0;
#pragma unroll
    for (int j = 0; j < N; ++j) s = fma(M[i][j], in[j], s);
    out[i] = s;
  }
}

// out = M^T in  (out_j = sum_i M[i][j] in_i)
template <int N>
__device__ __forceinline__ void mvt(const double (&M)[N][N], const double (&in)[N], double (&out)[N]) {
#pragma unroll
  for (int j = 0; j < N; ++j) {
    double s = 0.0;
#pragma unroll
    for (int i = 0; i < N; ++i) s = fma(M[i][j], in[i], s);
    out[j] = s;
  }
}

// out += M^T in
template <int N>
__device__ __forceinline__ void mvt_add(const double (&M)[N][N], const double (&in)[N], double (&out)[N]) {
#pragma unroll
  for (int j = 0; j < N; ++j) {
    double s = out[j];
#pragma unroll
    for (int i = 0; i < N; ++i) s = fma(M[i][j], in[i], s);
    out[j] = s;
  }
}

// out (+)= M in (T = false) or M^T in (T = true) in even-odd form; ANTI: M is
// anti-centro-symmetric.  FEM_EVEN_ODD=0 at build time restores the dense sweeps.
#ifndef FEM_EVEN_ODD
#define FEM_EVEN_ODD 1
#endif
template <int N, bool ANTI, bool TR, bool ADD>
__device__ __forceinline__ void mv_eo(const EO<N>& t, const double (&in)[N], double (&out)[N]) {
  constexpr int h = N / 2;
  constexpr bool odd = N & 1;
  const double(&E)[N][N] = TR ? t.ET : t.E;
  const double(&O)[N][N] = TR ? t.OT : t.O;
  double e[h + 1], o[h + 1];
#pragma unroll
  for (int j = 0; j < h; ++j) {
    e[j] = in[j] + in[N - 1 - j];
    o[j] = in[j] - in[N - 1 - j];
  }
  if (odd) e[h] = in[h];
  // centro: even rows q < h (+ the middle), odd rows q < h; anti: even rows q < h, odd
  // rows q < h (+ the middle)
#pragma unroll
  for (int q = 0; q < h + (odd ? 1 : 0); ++q) {
    double ye = 0.0, yo = 0.0;
    const bool mid = odd && q == h;
    if (!(ANTI && mid)) {
#pragma unroll
      for (int j = 0; j < h + (odd ? 1 : 0); ++j) ye = fma(E[q][j], e[j], ye);
    }
    if (!(!ANTI && mid)) {
#pragma unroll
      for (int j = 0; j < h; ++j) yo = fma(O[q][j], o[j], yo);
    }
    double lo, hi;
    if (mid) {
      lo = ANTI ? yo : ye;
      hi = lo;
    } else if (!ANTI) {
      lo = ye + yo;
      hi = ye - yo;
    } else {
      lo = ye + yo;
      hi = yo - ye;
    }
    if (ADD) {
      out[q] += lo;
      if (!mid) out[N - 1 - q] += hi;
    } else {
      out[q] = lo;
      if (!mid) out[N - 1 - q] = hi;
    }
  }
}
// drop-in replacements of mv / mvt / mvt_add for the val and colloc tables of Tab
#if FEM_EVEN_ODD
#define MV_VAL(T, in, out) mv_eo<N, false, false, false>((T).valeo, in, out)
#define MVT_VAL(T, in, out) mv_eo<N, false, true, false>((T).valeo, in, out)
#define MV_COL(T, in, out) mv_eo<N, true, false, false>((T).coleo, in, out)
#define MVT_COL(T, in, out) mv_eo<N, true, true, false>((T).coleo, in, out)
#define MVT_ADD_COL(T, in, out) mv_eo<N, true, true, true>((T).coleo, in, out)
#else
#define MV_VAL(T, in, out) mv<N>((T).val, in, out)
#define MVT_VAL(T, in, out) mvt<N>((T).val, in, out)
#define MV_COL(T, in, out) mv<N>((T).colloc, in, out)
#define MVT_COL(T, in, out) mvt<N>((T).colloc, in, out)
#define MVT_ADD_COL(T, in, out) mvt_add<N>((T).colloc, in, out)
#endif

// Programmatic dependent launch (launch_pdl, internal.h): wait for the predecessor
// grid (no-op when launched without the attribute), then let the successor launch.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
#define FEM_PDL_ENTRY() \
  do {                  \
    pdl_wait();         \
    pdl_trigger();      \
  } while (0)

// Mesh map (reading R2): xhat = lo + h (c + (xi+1)/2), x = xhat + eps s(xhat) (1,1,1),
// s = prod_e sin(pi t_e), t = (xhat - lo)/(hi - lo).
struct MapArgs {
  double lo[3], L[3], h[3];
  double eps;
  int cz0;  // global z offset of the rank's slab (cells)
  // SURVEY §8f N3 (fem_mesh.geometry / mapping_degree / kappa_amplitude)
  int general;      // 1: any of the three below is set -> geo_point() path
  int geom;         // FEM_GEOM_BOX / FEM_GEOM_SHELL
  int mdeg;         // 0: exact map; l: degree-l polynomial through GLL(l) support points
  int ng[3];        // global cells per direction of the level (shell patch coordinates)
  double kamp;      // kappa = 1 + kamp prod_e cos(2 pi x_e + 0.1 e)
  double gll[9];    // GLL(l) nodes
};

struct PointGeo {
  double xh[3];     // undeformed point
  double g[3];      // grad s (w.r.t. xhat)
  double s;         // s(xhat)
  double det;       // det J
  double beta;      // eps / (1 + eps sum g)
  double fac;       // 1 + eps sum g  (det J / prod(h/2))
};

__device__ __forceinline__ PointGeo map_point(const MapArgs& m, int cx, int cy, int cz,
                                              double xi0, double xi1, double xi2) {
  PointGeo p;
  const int c[3] = {cx, cy, cz + m.cz0};
  const double xi[3] = {xi0, xi1, xi2};
  double sn[3], cs[3];
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    p.xh[d] = m.lo[d] + m.h[d] * (c[d] + 0.5 * (xi[d] + 1.0));
    double t = (p.xh[d] - m.lo[d]) / m.L[d];
    sincospi(t, &sn[d], &cs[d]);
  }
  p.s = sn[0] * sn[1] * sn[2];
  p.g[0] = M_PI / m.L[0] * cs[0] * sn[1] * sn[2];
  p.g[1] = M_PI / m.L[1] * sn[0] * cs[1] * sn[2];
  p.g[2] = M_PI / m.L[2] * sn[0] * sn[1] * cs[2];
  p.fac = 1.0 + m.eps * (p.g[0] + p.g[1] + p.g[2]);
  p.det = p.fac * (0.5 * m.h[0]) * (0.5 * m.h[1]) * (0.5 * m.h[2]);
  p.beta = m.eps / p.fac;
  return p;
}

// ---- general geometry (N3): point and Jacobian dx/dxi of the level's cell map
struct GeoPt {
  double x[3];
  double J[3][3];   // J[d][e] = d x_d / d xi_e
};

// exact map ("manifold") at reference point xi of global cell c; J only if want_j
__device__ __forceinline__ void manifold_point(const MapArgs& m, const int c[3], const double xi[3], double x[3],
                                               double (*J)[3]) {
  if (m.geom == 1) {   // cube-sphere patch of the shell 0.5 < r < 1
    double t[3];
#pragma unroll
    for (int d = 0; d < 3; ++d) t[d] = (c[d] + 0.5 * (xi[d] + 1.0)) / m.ng[d];
    const double a = tan(0.5 * M_PI * (t[0] - 0.5)), b = tan(0.5 * M_PI * (t[1] - 0.5));
    const double r = 0.5 + 0.5 * t[2];
    const double is = rsqrt(1.0 + a * a + b * b);
    const double u[3] = {is, a * is, b * is};
#pragma unroll
    for (int d = 0; d < 3; ++d) x[d] = r * u[d];
    if (J) {
      // du/da = (e1 - u u1)/s, da/dt0 = (pi/2)(1 + a^2); likewise b; dx/dt2 = 0.5 u
      const double fa = r * 0.5 * M_PI * (1.0 + a * a) * is, fb = r * 0.5 * M_PI * (1.0 + b * b) * is;
#pragma unroll
      for (int d = 0; d < 3; ++d) {
        J[d][0] = fa * ((d == 1 ? 1.0 : 0.0) - u[d] * u[1]) * (0.5 / m.ng[0]);
        J[d][1] = fb * ((d == 2 ? 1.0 : 0.0) - u[d] * u[2]) * (0.5 / m.ng[1]);
        J[d][2] = 0.5 * u[d] * (0.5 / m.ng[2]);
      }
    }
    return;
  }
  // box with the sine deformation (reading R2): x = xhat + eps s(xhat) (1,1,1)
  double xh[3], sn[3], cs[3];
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    xh[d] = m.lo[d] + m.h[d] * (c[d] + 0.5 * (xi[d] + 1.0));
    sincospi((xh[d] - m.lo[d]) / m.L[d], &sn[d], &cs[d]);
  }
  const double s = sn[0] * sn[1] * sn[2];
#pragma unroll
  for (int d = 0; d < 3; ++d) x[d] = xh[d] + m.eps * s;
  if (J) {
    const double g[3] = {M_PI / m.L[0] * cs[0] * sn[1] * sn[2], M_PI / m.L[1] * sn[0] * cs[1] * sn[2],
                         M_PI / m.L[2] * sn[0] * sn[1] * cs[2]};
#pragma unroll
    for (int d = 0; d < 3; ++d)
#pragma unroll
      for (int e = 0; e < 3; ++e) J[d][e] = ((d == e ? 1.0 : 0.0) + m.eps * g[e]) * 0.5 * m.h[e];
  }
}

// fills the N3 fields of m for level L (global cells per direction: slabs split z)
inline void set_general_map(const fem_ctx* h, const Level& L, MapArgs& m) {
  m.general = mesh_general(h->mesh) ? 1 : 0;
  m.geom = h->mesh.geometry;
  m.mdeg = h->mesh.mapping_degree;
  m.kamp = h->mesh.kappa_amplitude;
  m.ng[0] = L.n[0];
  m.ng[1] = L.n[1];
  m.ng[2] = L.nzg;
  for (int i = 0; i < 9; ++i) m.gll[i] = 0.0;
  if (m.mdeg > 0) gll_points(m.mdeg, m.gll);
}

// Lagrange basis of the GLL(l) nodes and its derivative at t
__device__ __forceinline__ void gll_lagrange(const MapArgs& m, double t, double* v, double* dv) {
  const int n = m.mdeg + 1;
  for (int i = 0; i < n; ++i) {
    double p = 1.0, dp = 0.0;
    for (int j = 0; j < n; ++j) {
      if (j == i) continue;
      const double den = 1.0 / (m.gll[i] - m.gll[j]);
      dp = dp * (t - m.gll[j]) * den + p * den;
      p *= (t - m.gll[j]) * den;
    }
    v[i] = p;
    dv[i] = dp;
  }
}

// point and Jacobian of local cell (cx, cy, cz) at xi: exact map, or the degree-l
// polynomial through the exact map at the GLL(l) support points
static __device__ __noinline__ GeoPt geo_point(const MapArgs& m, int cx, int cy, int cz, double xi0, double xi1,
                                        double xi2) {
  GeoPt p;
  const int c[3] = {cx, cy, cz + m.cz0};
  if (m.mdeg == 0) {
    const double xi[3] = {xi0, xi1, xi2};
    manifold_point(m, c, xi, p.x, p.J);
    return p;
  }
  double v0[9], d0[9], v1[9], d1[9], v2[9], d2[9];
  gll_lagrange(m, xi0, v0, d0);
  gll_lagrange(m, xi1, v1, d1);
  gll_lagrange(m, xi2, v2, d2);
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    p.x[d] = 0.0;
    p.J[d][0] = p.J[d][1] = p.J[d][2] = 0.0;
  }
  const int n = m.mdeg + 1;
  for (int k = 0; k < n; ++k)
    for (int j = 0; j < n; ++j)
      for (int i = 0; i < n; ++i) {
        const double s[3] = {m.gll[i], m.gll[j], m.gll[k]};
        double X[3];
        manifold_point(m, c, s, X, nullptr);
        const double w = v0[i] * v1[j] * v2[k];
        const double w0 = d0[i] * v1[j] * v2[k], w1 = v0[i] * d1[j] * v2[k], w2 = v0[i] * v1[j] * d2[k];
#pragma unroll
        for (int d = 0; d < 3; ++d) {
          p.x[d] = fma(w, X[d], p.x[d]);
          p.J[d][0] = fma(w0, X[d], p.J[d][0]);
          p.J[d][1] = fma(w1, X[d], p.J[d][1]);
          p.J[d][2] = fma(w2, X[d], p.J[d][2]);
        }
      }
  return p;
}

// det J and J^-1 by cofactors
__device__ __forceinline__ double geo_inverse(const GeoPt& p, double Ji[3][3]) {
  const double (*J)[3] = p.J;
  Ji[0][0] = J[1][1] * J[2][2] - J[1][2] * J[2][1];
  Ji[0][1] = J[0][2] * J[2][1] - J[0][1] * J[2][2];
  Ji[0][2] = J[0][1] * J[1][2] - J[0][2] * J[1][1];
  Ji[1][0] = J[1][2] * J[2][0] - J[1][0] * J[2][2];
  Ji[1][1] = J[0][0] * J[2][2] - J[0][2] * J[2][0];
  Ji[1][2] = J[0][2] * J[1][0] - J[0][0] * J[1][2];
  Ji[2][0] = J[1][0] * J[2][1] - J[1][1] * J[2][0];
  Ji[2][1] = J[0][1] * J[2][0] - J[0][0] * J[2][1];
  Ji[2][2] = J[0][0] * J[1][1] - J[0][1] * J[1][0];
  const double det = J[0][0] * Ji[0][0] + J[0][1] * Ji[1][0] + J[0][2] * Ji[2][0];
  const double id = 1.0 / det;
#pragma unroll
  for (int a = 0; a < 3; ++a)
#pragma unroll
    for (int b = 0; b < 3; ++b) Ji[a][b] *= id;
  return det;
}

// eq:diffusivity_shell and its gradient
__device__ __forceinline__ double kappa_at(const MapArgs& m, const double x[3], double* grad = nullptr) {
  if (m.kamp == 0.0) {
    if (grad) grad[0] = grad[1] = grad[2] = 0.0;
    return 1.0;
  }
  double sn[3], cs[3];
#pragma unroll
  for (int e = 0; e < 3; ++e) sincos(2.0 * M_PI * x[e] + 0.1 * (e + 1), &sn[e], &cs[e]);
  if (grad) {
    grad[0] = -2.0 * M_PI * m.kamp * sn[0] * cs[1] * cs[2];
    grad[1] = -2.0 * M_PI * m.kamp * cs[0] * sn[1] * cs[2];
    grad[2] = -2.0 * M_PI * m.kamp * cs[0] * cs[1] * sn[2];
  }
  return 1.0 + m.kamp * cs[0] * cs[1] * cs[2];
}

// J^-1 = H^-1 (I - beta 1 g^T)  (Sherman-Morrison):  Jinv[d][e] = (2/h_d)(delta_de - beta g_e)
__device__ __forceinline__ double jinv(const MapArgs& m, const PointGeo& p, int d, int e) {
  return (2.0 / m.h[d]) * ((d == e ? 1.0 : 0.0) - p.beta * p.g[e]);
}

// ---- TMA bulk copy (cp.async.bulk, SASS UBLKCP) with an mbarrier transaction count
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(phase)
      : "memory");
}

// global -> shared bulk copy of `bytes` (multiple of 16, 16-byte aligned), completes on bar
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// ---- geometry-table layouts (R2), entry (cell, comp, q), q = q0 + N q1 + N^2 q2
//   kGLayoutCell  [cell][comp][q]                        (SIPG, line kernel)
//   kGLayoutXLine [cell][comp][q0][q1 + N q2]            (CG x-line kernel: in its
//                 quadrature phase thread t = q1 + N q2 owns the x-line q0 = 0..N-1,
//                 so a warp's loads of one (comp, q0) are consecutive addresses)
//   kGLayoutPlane groups of kGroupCells cells, [group][comp][e][cell-in-group][q2],
//                 e = q0 + N q1 (CG plane kernel: lane = q2 + N cell; a row q1 of all
//                 six components is six contiguous chunks -> TMA bulk copies)
//   kGLayoutCell8 blocks of kCell8 cells, [block][comp][q][cell-in-block] (CG line kernel
//                 at Q4 with the cells-fastest thread layout: a warp's 4 points x 8 cells
//                 of one component are 32 consecutive doubles)
constexpr int kGroupCells = 12;
constexpr int kCell8 = 8;
enum { kGLayoutCell = 0, kGLayoutPlane = 1, kGLayoutXLine = 2, kGLayoutCell8 = 3 };

template <int N>
__host__ __device__ __forceinline__ int64_t g_index(int layout, int64_t cell, int comp, int q) {
  constexpr int N2 = N * N, N3 = N2 * N;
  if (layout == kGLayoutXLine) return (cell * 6 + comp) * N3 + (q % N) * N2 + q / N;
  if (layout == kGLayoutCell8) return (((cell / kCell8) * 6 + comp) * N3 + q) * kCell8 + cell % kCell8;
  if (layout != kGLayoutPlane) return (cell * 6 + comp) * N3 + q;
  const int64_t g = cell / kGroupCells;
  const int c = (int)(cell % kGroupCells);
  const int pz = q / N2, e = q % N2;
  return (((g * 6 + comp) * N2 + e) * kGroupCells + c) * N + pz;
}

// global -> L2 bulk prefetch (no destination, no completion tracking); bytes % 16 == 0
__device__ __forceinline__ void bulk_prefetch_l2(const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}

// L2 prefetch of an arbitrary byte range (bulk prefetch needs 16-byte aligned start and size)
__device__ __forceinline__ void prefetch_l2_range(const void* p, size_t bytes) {
  const uintptr_t a = reinterpret_cast<uintptr_t>(p), b = a & ~(uintptr_t)15;
  const size_t n = (a + bytes - b + 15) & ~(size_t)15;
  bulk_prefetch_l2(reinterpret_cast<const void*>(b), (uint32_t)n);
}

__device__ __forceinline__ bool cg_constrained(int bcmask, int gx, int gy, int gz, int nn0, int nn1,
                                               int nn2) {
  return ((bcmask & 1) && gx == 0) || ((bcmask & 2) && gx == nn0 - 1) ||
         ((bcmask & 4) && gy == 0) || ((bcmask & 8) && gy == nn1 - 1) ||
         ((bcmask & 16) && gz == 0) || ((bcmask & 32) && gz == nn2 - 1);
}

}  // namespace fem
