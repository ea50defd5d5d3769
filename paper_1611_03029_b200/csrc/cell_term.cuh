// Sum-factorized cell term of the Laplace operator (eq:mf_eval),
// shared by the CG (K1) and SIPG (K2) kernels.
//
// A cell is handled by (k+1)^2 threads; thread t = ta + N tb owns one 1-D line of
// the cell per phase (z-line (x=ta,y=tb), y-line (x=ta,z=tb) or x-line (y=ta,z=tb)),
// held in registers; direction changes are transposes through the cell's three
// shared-memory buffers s0, s1, s2 (N^3 doubles each).
//   in : u[] = the thread's z-line of nodal values (constrained entries already 0)
//   out: v[] = the thread's z-line of the cell residual  sum_q grad phi . G_q grad u
// The caller must __syncthreads() before reusing s0..s2.
#pragma once

#include "device_common.cuh"

namespace fem {

// Analytic geometry of the deformed box (reading R2) at the thread's z-line of quadrature
// points: x = xhat + eps s(xhat) (1,1,1), s = prod_d sin(pi t_d).  With g = grad s,
// fac = 1 + eps sum g, beta = eps / fac, J^-1 = diag(2/h) (I - beta 1 g^T), the metric is
//   G_ab = w det J (4 / (h_a h_b)) (delta_ab - beta (g_a + g_b) + beta^2 |g|^2),
// det J = fac prod(h/2) -- the geometry_kernel formula, evaluated in the q-point phase
// instead of read from the 48-byte-per-point table.
struct GeoFlyC {             // level constants (kernel parameter)
  double pl[3];              // pi / L_d
  double eps, hh;            // eps, prod(h/2)
  double ih[6];              // 4 / (h_a h_b) for (00, 01, 02, 11, 12, 22)
};
template <int N>
struct GeoFlyPt {
  double sx, cx, sy, cy;     // sin / cos (pi t) of the thread's x and y quadrature coordinates
  const double* scz;         // shared: sin (pi t_z) at [0, N), cos at [N, 2N) of the cell's z points
  const GeoFlyC* c;
};

template <int N>
struct CellGeo {
  const double* G;  // deformed: &G[cell][0][0] of layout [6][N^3] (global or shared)
  double c0, c1, c2;
  bool active;
  uint64_t* bar;    // if set: mbarrier of a bulk copy that fills G, waited on before the q-point phase
  int gq = 1;       // G stride between quadrature points ([cell][comp][q]: 1)
  int gc = N * N * N;  // G stride between components
  const GeoFlyPt<N>* fly = nullptr;   // analytic geometry instead of G (FLY kernels)
};

// RT_STRIDES: G strides from geo.gq / geo.gc (the Q4 line kernel's 8-cell block order);
// else [cell][comp][q] (1, N^3).  (Compile-time strides at Q4 measured slower: 67 vs 59 us.)
// B, S: row and plane strides of the shared-memory buffers (element (i0, i1, i2) at
// i0 + B i1 + S i2; dense: N, N^2).  Z pattern: thread line (ta, tb) along i2; Y: along
// i1 with (i0, i2) = (ta, tb); X: along i0 with (i1, i2) = (ta, tb).
template <int N, bool DEFORMED, bool RT_STRIDES = false, int B = N, int S = N * N>
__device__ __forceinline__ void cell_laplace(const Tab<N>& T, const CellGeo<N>& geo, double* s0,
                                             double* s1, double* s2, int t, double (&u)[N],
                                             double (&v)[N]) {
  constexpr int N2 = N * N, N3 = N2 * N;
  const int ta = t % N, tb = t / N;
  const int zi = ta + B * tb;   // Z-pattern word of the thread's line
  double g[N], w[N];
  // Z: interpolate in z
  MV_VAL(T, u, v);
#pragma unroll
  for (int l = 0; l < N; ++l) s0[zi + S * l] = v[l];
  __syncthreads();
  // Y: interpolate in y
#pragma unroll
  for (int l = 0; l < N; ++l) w[l] = s0[ta + B * l + S * tb];
  MV_VAL(T, w, v);
#pragma unroll
  for (int l = 0; l < N; ++l) s0[ta + B * l + S * tb] = v[l];
  __syncthreads();
  // X: interpolate in x, d/dxi_x by collocation
#pragma unroll
  for (int l = 0; l < N; ++l) w[l] = s0[l + B * ta + S * tb];
  MV_VAL(T, w, v);
  MV_COL(T, v, g);
#pragma unroll
  for (int l = 0; l < N; ++l) {
    s0[l + B * ta + S * tb] = v[l];
    s2[l + B * ta + S * tb] = g[l];
  }
  __syncthreads();
  // Y: d/dxi_y
#pragma unroll
  for (int l = 0; l < N; ++l) w[l] = s0[ta + B * l + S * tb];
  MV_COL(T, w, g);
#pragma unroll
  for (int l = 0; l < N; ++l) s1[ta + B * l + S * tb] = g[l];
  __syncthreads();
  // Z: d/dxi_z, quadrature-point operation, transposed d/dxi_z
#pragma unroll
  for (int l = 0; l < N; ++l) w[l] = s0[zi + S * l];
  MV_COL(T, w, g);
  if (DEFORMED && geo.bar) mbar_wait(geo.bar, 0);
#pragma unroll
  for (int l = 0; l < N; ++l) {
    const int q = t + N2 * l;                 // quadrature point (G index)
    const int zq = zi + S * l;                // its shared-memory word
    const double gxq = s2[zq], gyq = s1[zq], gzq = g[l];
    double fx, fy, fz;
    if (DEFORMED) {
      double G00 = 0, G01 = 0, G02 = 0, G11 = 0, G12 = 0, G22 = 0;
      if (geo.fly) {
        const GeoFlyPt<N>& f = *geo.fly;
        const GeoFlyC& k = *f.c;
        const double szl = f.scz[l], czl = f.scz[N + l];
        const double g0 = k.pl[0] * f.cx * f.sy * szl, g1 = k.pl[1] * f.sx * f.cy * szl,
                     g2 = k.pl[2] * f.sx * f.sy * czl;
        const double fac = 1.0 + k.eps * (g0 + g1 + g2);
        const double beta = k.eps / fac;
        const double W = T.w[ta] * T.w[tb] * T.w[l] * fac * k.hh;
        const double bb = beta * beta * (g0 * g0 + g1 * g1 + g2 * g2);
        G00 = W * k.ih[0] * (1.0 - 2.0 * beta * g0 + bb);
        G01 = W * k.ih[1] * (bb - beta * (g0 + g1));
        G02 = W * k.ih[2] * (bb - beta * (g0 + g2));
        G11 = W * k.ih[3] * (1.0 - 2.0 * beta * g1 + bb);
        G12 = W * k.ih[4] * (bb - beta * (g1 + g2));
        G22 = W * k.ih[5] * (1.0 - 2.0 * beta * g2 + bb);
      } else if (geo.active) {
        const int gq = RT_STRIDES ? geo.gq : 1, gc = RT_STRIDES ? geo.gc : N3;
        const double* Gc = geo.G + q * gq;
        G00 = Gc[0];
        G01 = Gc[gc];
        G02 = Gc[2 * gc];
        G11 = Gc[3 * gc];
        G12 = Gc[4 * gc];
        G22 = Gc[5 * gc];
      }
      fx = G00 * gxq + G01 * gyq + G02 * gzq;
      fy = G01 * gxq + G11 * gyq + G12 * gzq;
      fz = G02 * gxq + G12 * gyq + G22 * gzq;
    } else {
      const double w3 = T.w[ta] * T.w[tb] * T.w[l];
      fx = geo.c0 * w3 * gxq;
      fy = geo.c1 * w3 * gyq;
      fz = geo.c2 * w3 * gzq;
    }
    s2[zq] = fx;
    s1[zq] = fy;
    v[l] = fz;
  }
  MVT_COL(T, v, w);
#pragma unroll
  for (int l = 0; l < N; ++l) s0[zi + S * l] = w[l];
  __syncthreads();
  // Y: += colloc^T f_y
#pragma unroll
  for (int l = 0; l < N; ++l) {
    v[l] = s1[ta + B * l + S * tb];
    w[l] = s0[ta + B * l + S * tb];
  }
  MVT_ADD_COL(T, v, w);
#pragma unroll
  for (int l = 0; l < N; ++l) s0[ta + B * l + S * tb] = w[l];
  __syncthreads();
  // X: += colloc^T f_x, then interpolate back in x
#pragma unroll
  for (int l = 0; l < N; ++l) {
    v[l] = s2[l + B * ta + S * tb];
    w[l] = s0[l + B * ta + S * tb];
  }
  MVT_ADD_COL(T, v, w);
  MVT_VAL(T, w, v);
#pragma unroll
  for (int l = 0; l < N; ++l) s0[l + B * ta + S * tb] = v[l];
  __syncthreads();
  // Y: interpolate back in y
#pragma unroll
  for (int l = 0; l < N; ++l) w[l] = s0[ta + B * l + S * tb];
  MVT_VAL(T, w, v);
#pragma unroll
  for (int l = 0; l < N; ++l) s0[ta + B * l + S * tb] = v[l];
  __syncthreads();
  // Z: interpolate back in z
#pragma unroll
  for (int l = 0; l < N; ++l) w[l] = s0[zi + S * l];
  MVT_VAL(T, w, v);
}

}  // namespace fem
