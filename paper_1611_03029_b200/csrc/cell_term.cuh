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

template <int N>
struct CellGeo {
  const double* G;  // deformed: &G[cell][0][0] of layout [6][N^3] (global or shared)
  double c0, c1, c2;
  bool active;
  uint64_t* bar;    // if set: mbarrier of a bulk copy that fills G, waited on before the q-point phase
  int gq = 1;       // G stride between quadrature points ([cell][comp][q]: 1)
  int gc = N * N * N;  // G stride between components
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
      if (geo.active) {
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
