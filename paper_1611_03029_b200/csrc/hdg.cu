// HDG matrix-free operators on Cartesian meshes (sec:discret_hdg,
// P:L257-326; "HDG trace matrix-free" and "HDG mixed matrix-free").
//
// Per cell K (affine, h_d, J = prod h_d / 2, a_d = 2 / h_d), with the 1-D GLL-basis matrices
// M_ij = int phi_i phi_j, Dm_ij = int phi_i phi_j' on [-1, 1] (Gauss k+1), the HDG matrices of
// eq:hdg_matrix are Kronecker products:
//   A = J M(x)M(x)M per q component,  E_d = J a_d (Dm in slot d, M elsewhere),
//   face s (direction d, layer l_s = 0 | k, outward sign sg_s = -1 | +1):
//   C_s = sg_s J a_d (e_l^T in slot d) (x) M(x)M,  G_s = tau J a_d (e_l^T) (x) M(x)M,
//   H_s = tau J a_d M(x)M,  D = sum_s tau J a_d (e_l e_l^T) (x) M(x)M.
// The trace operator K lambda = sum_K (H lambda - C q - G u) with (q, u) the local solution of
//   A q - E^T u = -C^T lambda,   E q + D u = G^T lambda (+ F)
// is applied in the paper's three steps:
//  (1) R_q = -C^T lambda, R_u = G^T lambda: with l_s = (M(x)M) lambda_s the face-mass-weighted
//      trace, E A^-1 R_q is again a sum of rank-one tensors, and
//      t = R_u - E A^-1 R_q = sum_s w_s (x) l_s,  w_s = J (tau a_d e_l + sg_s a_d^2 Dm M^-1 e_l);
//  (2) u = S^-1 t with the inner Schur complement S = D + E A^-1 E^T = J sum_d L_d (x) M (x) M,
//      L_d = a_d^2 Dm M^-1 Dm^T + tau a_d (e_0 e_0^T + e_k e_k^T) (pinned against the quadrature
//      matrices in tests/test_oracle_hdg.py), applied by fast diagonalization:
//      L_d V_d = M V_d Lambda_d, V_d^T M V_d = I  =>  S^-1 = J^-1 V^(3) (sum Lambda)^-1 V^(3)T
//      (6 sweeps of (k+1)^4 instead of the paper's stored (k+1)^3 x (k+1)^3 dense inverse);
//      q_d = A^-1 (R_q + E^T u) = a_d (P u)_d - sum_{s' in d} sg_s' a_d M^-1 e_l' (x) lambda_s',
//      P = M^-1 Dm^T, needed only on the d-face layers;
//  (3) y_s = H_s lambda_s - C_s q - G_s u = J a_d (M(x)M) [tau lambda_s - sg_s q_d(l_s) - tau u(l_s)].
// Every interior face receives two cell contributions: cells are processed in two colour
// passes (c_x + c_y + c_z even, then odd; neighbours always differ in colour): the first
// stores, the second adds (no atomics, no zero fill, deterministic).
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <string>
#include <vector>

#include "device_common.cuh"
#include "../../include/fem_hdg.h"

#pragma nv_diag_suppress 128   // code after the kRecover early return in the other modes

// minimum resident blocks per SM requested from ptxas (register cap); 0 = none
#ifndef FEM_HDG_MINB
#define FEM_HDG_MINB 6
#endif
#ifndef FEM_HDG_MINB_MIX
#define FEM_HDG_MINB_MIX 0
#endif

namespace fem {
namespace {

struct HdgTab {                    // host-built 1-D tables (padded to kMaxN)
  double M[kMaxN][kMaxN];          // mass
  double Minv[kMaxN][kMaxN];       // inverse mass
  double P[kMaxN][kMaxN];          // M^-1 Dm^T  ([l][i])
  double Dm[kMaxN][kMaxN];         // [i][j] int phi_i phi_j'
  double V[3][kMaxN][kMaxN];       // generalized eigenvectors of (L_d, M), columns
  double lam[3][kMaxN];            // eigenvalues
  double w[6][kMaxN];              // t-tensor weights per side
  double J, a[3], tau;
};
constexpr int kTabDoubles = sizeof(HdgTab) / sizeof(double);

enum { kApply = 0, kRhs = 1, kRecover = 2, kDiag = 3 };

struct HdgArgs {
  const double* lam;   // trace input (kApply, kRecover)
  const double* F;     // cell load vector (kRhs, kRecover with F) or nullptr
  double* y;           // trace output (kApply, kRhs), diag_e (kDiag)
  double* u;           // kRecover: u (cell vector)
  double* q;           // kRecover: q (3 cell vectors) or nullptr
  const HdgTab* tab;
  int nx, ny, nz;
  int64_t fx, fy;      // faces normal to x, y
  int bc;              // Dirichlet side mask (bit s)
  int color;           // 0 / 1: colour pass; -1: all cells
  int64_t n_work;      // cells (or virtual cells) of this launch
};

template <int N>
struct HdgCfg {
  static constexpr int NF = N * N, N3 = N * N * N;
  static constexpr int CPB = std::max(1, 128 / NF);          // cells per block
  static constexpr int PER_CELL = 3 * 6 * NF + 2 * N3;       // lam, fz, ell, T1, T2
  static constexpr int SMEM = CPB * PER_CELL;  // doubles
};

template <int K, int MODE>
__global__ void __launch_bounds__(HdgCfg<K + 1>::CPB * (K + 1) * (K + 1), FEM_HDG_MINB)
    hdg_cell_kernel(HdgArgs a, const __grid_constant__ HdgTab T) {
  // T: kernel parameter (constant bank): every compile-time-indexed coefficient is a uniform
  // operand, no shared-memory load; the thread-indexed rows are preloaded from a.tab below
  constexpr int N = K + 1, NF = N * N, N3 = N * N * N;
  using Cfg = HdgCfg<N>;
  extern __shared__ double sm[];
  const int t = threadIdx.x, ta = t % N, tb = t / N;
  double Ma[N], Mb[N];
#pragma unroll
  for (int jj = 0; jj < N; ++jj) {
    Ma[jj] = __ldg(&a.tab->M[ta][jj]);
    Mb[jj] = __ldg(&a.tab->M[tb][jj]);
  }
  const double w2a = __ldg(&a.tab->w[2][ta]), w3a = __ldg(&a.tab->w[3][ta]), w4b = __ldg(&a.tab->w[4][tb]),
               w5b = __ldg(&a.tab->w[5][tb]);
  const double lxy = __ldg(&a.tab->lam[0][ta]) + __ldg(&a.tab->lam[1][tb]);
  double* base = sm + threadIdx.y * Cfg::PER_CELL;
  double* lam = base;              // [6][NF]
  double* fz = lam + 6 * NF;       // [6][NF]
  double* ell = fz + 6 * NF;       // [6][NF]
  double* T1 = ell + 6 * NF;       // [N3]
  double* T2 = T1 + N3;            // [N3]
  const int64_t j = (int64_t)blockIdx.x * Cfg::CPB + threadIdx.y;
  bool active = j < a.n_work;
  int cx = 0, cy = 0, cz = 0, s0 = -1, t0 = -1;
  if (MODE == kDiag) {             // virtual cell: unit trace entry (s0, t0) of the reference cell
    s0 = (int)(j / NF);
    t0 = (int)(j % NF);
    active = active && s0 < 6;
  } else if (a.color >= 0) {
    const int cpr = (a.nx + 1) / 2;
    const int64_t row = j / cpr;
    cy = (int)(row % a.ny);
    cz = (int)(row / a.ny);
    cx = 2 * (int)(j % cpr) + ((cy + cz + a.color) & 1);
    active = active && cz < a.nz && cx < a.nx;
  } else {
    cx = (int)(j % a.nx);
    cy = (int)((j / a.nx) % a.ny);
    cz = (int)(j / ((int64_t)a.nx * a.ny));
  }
  int64_t fid[6];
  bool inter[6], dir[6];
  {
    const int c3[3] = {cx, cy, cz}, n3[3] = {a.nx, a.ny, a.nz};
    for (int s = 0; s < 6; ++s) {
      const int d = s / 2, hi = s & 1;
      fid[s] = d == 0 ? (cx + hi) + (int64_t)(a.nx + 1) * (cy + (int64_t)a.ny * cz)
             : d == 1 ? a.fx + cx + (int64_t)a.nx * ((cy + hi) + (int64_t)(a.ny + 1) * cz)
                      : a.fx + a.fy + cx + (int64_t)a.nx * (cy + (int64_t)a.ny * (cz + hi));
      inter[s] = hi ? c3[d] < n3[d] - 1 : c3[d] > 0;
      dir[s] = !inter[s] && ((a.bc >> s) & 1);
    }
  }
  // ---- inputs: the six faces' traces (constrained faces read as 0) and the load vector
  for (int s = 0; s < 6; ++s) {
    double v = 0.0;
    if (MODE == kDiag) v = (s == s0 && t == t0) ? 1.0 : 0.0;
    else if ((MODE == kApply || MODE == kRecover) && active && !dir[s]) v = a.lam[fid[s] * NF + t];
    lam[s * NF + t] = v;
  }
  const int64_t cell = cx + (int64_t)a.nx * (cy + (int64_t)a.ny * cz);
  if (a.F && (MODE == kRhs || MODE == kRecover))
    for (int i = t; i < N3; i += NF) T2[i] = active ? a.F[cell * N3 + i] : 0.0;
  __syncthreads();
  // ---- (1) l_s = (M (x) M) lambda_s, then t = sum_s w_s (x) l_s (+ F) on x-lines
#pragma unroll
  for (int s = 0; s < 6; ++s) {
    double v = 0.0;
#pragma unroll
    for (int jj = 0; jj < N; ++jj) v = fma(Ma[jj], lam[s * NF + jj + N * tb], v);
    fz[s * NF + t] = v;
  }
  __syncthreads();
#pragma unroll
  for (int s = 0; s < 6; ++s) {
    double v = 0.0;
#pragma unroll
    for (int jj = 0; jj < N; ++jj) v = fma(Mb[jj], fz[s * NF + ta + N * jj], v);
    ell[s * NF + t] = v;
  }
  __syncthreads();
  double line[N];
  {   // thread = x-line (i1, i2) = (ta, tb)
    const double l0 = ell[0 * NF + t], l1 = ell[1 * NF + t];
#pragma unroll
    for (int i0 = 0; i0 < N; ++i0) {
      double v = T.w[0][i0] * l0 + T.w[1][i0] * l1;
      v = fma(w2a, ell[2 * NF + i0 + N * tb], v);
      v = fma(w3a, ell[3 * NF + i0 + N * tb], v);
      v = fma(w4b, ell[4 * NF + i0 + N * ta], v);
      v = fma(w5b, ell[5 * NF + i0 + N * ta], v);
      if (a.F && (MODE == kRhs || MODE == kRecover)) v += T2[i0 + N * ta + NF * tb];
      line[i0] = v;
    }
  }
  __syncthreads();   // T2 (F) consumed
  // ---- (2) u = S^-1 t: V_x^T, V_y^T, V_z^T, scale, V_z, V_y, V_x
#pragma unroll
  for (int i = 0; i < N; ++i) {
    double v = 0.0;
#pragma unroll
    for (int jj = 0; jj < N; ++jj) v = fma(T.V[0][jj][i], line[jj], v);
    T1[i + N * ta + NF * tb] = v;
  }
  __syncthreads();
  {   // y-line (i0, i2) = (ta, tb)
    double g[N];
#pragma unroll
    for (int jj = 0; jj < N; ++jj) g[jj] = T1[ta + N * jj + NF * tb];
#pragma unroll
    for (int i = 0; i < N; ++i) {
      double v = 0.0;
#pragma unroll
      for (int jj = 0; jj < N; ++jj) v = fma(T.V[1][jj][i], g[jj], v);
      T2[ta + N * i + NF * tb] = v;
    }
  }
  __syncthreads();
  {   // z-line (i0, i1) = (ta, tb): V_z^T, divide, V_z
    double g[N], hh[N];
#pragma unroll
    for (int jj = 0; jj < N; ++jj) g[jj] = T2[ta + N * tb + NF * jj];
#pragma unroll
    for (int i = 0; i < N; ++i) {
      double v = 0.0;
#pragma unroll
      for (int jj = 0; jj < N; ++jj) v = fma(T.V[2][jj][i], g[jj], v);
      hh[i] = v / (T.J * (lxy + T.lam[2][i]));
    }
#pragma unroll
    for (int l = 0; l < N; ++l) {
      double v = 0.0;
#pragma unroll
      for (int i = 0; i < N; ++i) v = fma(T.V[2][l][i], hh[i], v);
      T1[ta + N * tb + NF * l] = v;
    }
  }
  __syncthreads();
  {   // y-line back
    double g[N];
#pragma unroll
    for (int jj = 0; jj < N; ++jj) g[jj] = T1[ta + N * jj + NF * tb];
#pragma unroll
    for (int l = 0; l < N; ++l) {
      double v = 0.0;
#pragma unroll
      for (int i = 0; i < N; ++i) v = fma(T.V[1][l][i], g[i], v);
      T2[ta + N * l + NF * tb] = v;
    }
  }
  __syncthreads();
  {   // x-line back: u
    double g[N];
#pragma unroll
    for (int jj = 0; jj < N; ++jj) g[jj] = T2[jj + N * ta + NF * tb];
#pragma unroll
    for (int l = 0; l < N; ++l) {
      double v = 0.0;
#pragma unroll
      for (int i = 0; i < N; ++i) v = fma(T.V[0][l][i], g[i], v);
      T1[l + N * ta + NF * tb] = v;
      if (MODE == kRecover && active) a.u[cell * N3 + l + N * ta + NF * tb] = v;
    }
  }
  __syncthreads();   // u complete in T1
  auto uat = [&](int d, int i) -> double {   // u on the d-line through the thread's face point
    return d == 0 ? T1[i + N * ta + NF * tb] : d == 1 ? T1[ta + N * i + NF * tb] : T1[ta + N * tb + NF * i];
  };
  if (MODE == kRecover) {
    if (a.q && active) {   // q_d on every node of the thread's d-line
#pragma unroll
      for (int d = 0; d < 3; ++d) {
        const double ad = T.a[d];
        double g[N];
#pragma unroll
        for (int i = 0; i < N; ++i) g[i] = uat(d, i);
        const double lm = lam[(2 * d) * NF + t], lp = lam[(2 * d + 1) * NF + t];
#pragma unroll
        for (int l = 0; l < N; ++l) {
          double v = 0.0;
#pragma unroll
          for (int i = 0; i < N; ++i) v = fma(T.P[l][i], g[i], v);
          v += T.Minv[l][0] * lm - T.Minv[l][K] * lp;   // -sum sg_s' M^-1 e_l' lambda_s'
          const int idx = d == 0 ? l + N * ta + NF * tb : d == 1 ? ta + N * l + NF * tb : ta + N * tb + NF * l;
          a.q[(int64_t)d * a.n_work * N3 + cell * N3 + idx] = ad * v;
        }
      }
    }
    return;
  }
  // ---- (3) z_s = tau lambda_s - sg_s q_d(l_s) - tau u(l_s) at the face points
#pragma unroll
  for (int s = 0; s < 6; ++s) {
    const int d = s / 2, ly = (s & 1) ? K : 0;
    const double sg = (s & 1) ? 1.0 : -1.0, ad = T.a[d];
    double pu = 0.0;
#pragma unroll
    for (int i = 0; i < N; ++i) pu = fma(T.P[ly][i], uat(d, i), pu);
    const double corr = T.Minv[ly][K] * lam[(2 * d + 1) * NF + t] - T.Minv[ly][0] * lam[(2 * d) * NF + t];
    const double qn = ad * (pu - corr);
    fz[s * NF + t] = T.tau * (lam[s * NF + t] - uat(d, ly)) - sg * qn;
  }
  __syncthreads();
#pragma unroll
  for (int s = 0; s < 6; ++s) {
    double v = 0.0;
#pragma unroll
    for (int jj = 0; jj < N; ++jj) v = fma(Ma[jj], fz[s * NF + jj + N * tb], v);
    ell[s * NF + t] = v;
  }
  __syncthreads();
#pragma unroll
  for (int s = 0; s < 6; ++s) {
    double v = 0.0;
#pragma unroll
    for (int jj = 0; jj < N; ++jj) v = fma(Mb[jj], ell[s * NF + ta + N * jj], v);
    v *= T.J * T.a[s / 2];
    if (MODE == kDiag) {
      if (active && s == s0 && t == t0) a.y[j] = v;
      continue;
    }
    if (!active) continue;
    double* yp = a.y + fid[s] * NF + t;
    if (dir[s]) {
      *yp = MODE == kApply ? a.lam[fid[s] * NF + t] : 0.0;   // y_c = x_c (apply), 0 (rhs)
    } else {
      if (MODE == kRhs) v = -v;                               // r = sum_K (C q + G u)
      if (a.color == 1 && inter[s]) *yp += v;                 // second colour: the face's other cell
      else *yp = v;
    }
  }
}


// ---- "HDG mixed matrix-free" on Cartesian cells:
//   lambda^_s = (sum over the face's cells of (sg q_d(l) + tau u(l))) / (tau x number of cells)
//   (H_F^-1 sum_K (C q + G u): M(x)M cancels, a point-wise flux; 0 on constrained faces)
//   y_q,d = J [ M(x)M(x)M q_d - a_d (Dm^T in slot d) (x) M(x)M u + sum_{s in d} sg_s a_d e_l (x) M(x)M lambda^_s ]
//   y_u   = J [ sum_d a_d (Dm in slot d) (x) M(x)M q_d + sum_s tau a_d e_l (x) M(x)M (u(l) - lambda^_s) ]
template <int N>
struct MixCfg {
  static constexpr int NF = N * N, N3 = N * N * N;
  static constexpr int CPB = std::max(1, 128 / NF);
  static constexpr int PER_CELL = 9 * N3 + 6 * NF;   // Q[3], U, W[2], X[2], Yu; lambda^[6]
  static constexpr int SMEM = CPB * PER_CELL;
};

template <int N>
__device__ __forceinline__ int tidx(int e, int i, int ta, int tb) {   // node i on the e-line at (ta, tb)
  return e == 0 ? i + N * ta + N * N * tb : e == 1 ? ta + N * i + N * N * tb : ta + N * tb + N * N * i;
}

template <int K>
__global__ void __launch_bounds__(MixCfg<K + 1>::CPB * (K + 1) * (K + 1), FEM_HDG_MINB_MIX) hdg_mixed_kernel(
    const double* __restrict__ qu, double* __restrict__ y, const __grid_constant__ HdgTab T, int nx, int ny, int nz,
    int bc, int64_t ncells) {
  constexpr int N = K + 1, NF = N * N, N3 = N * N * N;
  using Cfg = MixCfg<N>;
  extern __shared__ double sm[];
  const int t = threadIdx.x, ta = t % N, tb = t / N;
  double* Q = sm + threadIdx.y * Cfg::PER_CELL;   // [3][N3]
  double* U = Q + 3 * N3;
  double* W = U + N3;       // [2][N3]
  double* X = W + 2 * N3;   // [2][N3]
  double* Yu = X + 2 * N3;
  double* lh = Yu + N3;     // [6][NF]
  const int64_t cell = (int64_t)blockIdx.x * Cfg::CPB + threadIdx.y;
  const bool active = cell < ncells;
  const int cx = (int)(cell % nx), cy = (int)((cell / nx) % ny), cz = (int)(cell / ((int64_t)nx * ny));
  for (int i = t; i < N3; i += NF) {
    for (int d = 0; d < 3; ++d) Q[d * N3 + i] = active ? qu[(int64_t)d * ncells * N3 + cell * N3 + i] : 0.0;
    U[i] = active ? qu[3 * ncells * N3 + cell * N3 + i] : 0.0;
    Yu[i] = 0.0;
  }
  __syncthreads();
  {   // lambda^ on the six faces at the thread's face point
    const int c3[3] = {cx, cy, cz}, n3[3] = {nx, ny, nz};
    const int64_t step[3] = {1, nx, (int64_t)nx * ny};
#pragma unroll
    for (int s = 0; s < 6; ++s) {
      const int d = s / 2, hi = s & 1, l = hi ? K : 0;
      const double sg = hi ? 1.0 : -1.0;
      const bool inter = hi ? c3[d] < n3[d] - 1 : c3[d] > 0;
      double v = 0.0;
      if (inter) {
        const int64_t nb = cell + (hi ? step[d] : -step[d]);
        const int ni = tidx<N>(d, K - l, ta, tb);
        const double qn = active ? qu[(int64_t)d * ncells * N3 + nb * N3 + ni] : 0.0;
        const double un = active ? qu[3 * ncells * N3 + nb * N3 + ni] : 0.0;
        v = (sg * Q[d * N3 + tidx<N>(d, l, ta, tb)] + T.tau * U[tidx<N>(d, l, ta, tb)] - sg * qn + T.tau * un) /
            (2.0 * T.tau);
      } else if (!((bc >> s) & 1)) {   // Neumann face
        v = (sg * Q[d * N3 + tidx<N>(d, l, ta, tb)] + T.tau * U[tidx<N>(d, l, ta, tb)]) / T.tau;
      }
      lh[s * NF + t] = v;
    }
  }
  __syncthreads();
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    const int e1 = d == 0 ? 1 : 0, e2 = d == 2 ? 1 : 2;   // tangential directions
    const double ad = T.a[d];
    {   // slot-d operators along the d-line (ta, tb) and the layer terms
      double qd[N], ud[N];
#pragma unroll
      for (int i = 0; i < N; ++i) {
        qd[i] = Q[d * N3 + tidx<N>(d, i, ta, tb)];
        ud[i] = U[tidx<N>(d, i, ta, tb)];
      }
      const double lm = lh[(2 * d) * NF + t], lp = lh[(2 * d + 1) * NF + t];
#pragma unroll
      for (int l = 0; l < N; ++l) {
        double wq = 0.0, wu = 0.0;
#pragma unroll
        for (int j = 0; j < N; ++j) {
          wq = fma(T.M[l][j], qd[j], wq);
          wq = fma(-ad * T.Dm[j][l], ud[j], wq);
          wu = fma(ad * T.Dm[l][j], qd[j], wu);
        }
        if (l == 0) {
          wq -= ad * lm;
          wu += T.tau * ad * (ud[0] - lm);
        }
        if (l == K) {
          wq += ad * lp;
          wu += T.tau * ad * (ud[K] - lp);
        }
        W[tidx<N>(d, l, ta, tb)] = wq;
        W[N3 + tidx<N>(d, l, ta, tb)] = wu;
      }
    }
    __syncthreads();
    // M in the tangential directions e1 (thread = e1-line) then e2
#pragma unroll
    for (int pass = 0; pass < 2; ++pass) {
      const int e = pass == 0 ? e1 : e2;
      const double* src = pass == 0 ? W : X;
      double* dst = pass == 0 ? X : W;
      // the e-line of the thread: the other two directions in increasing order = (ta, tb)
      for (int f = 0; f < 2; ++f) {
        double g[N];
#pragma unroll
        for (int i = 0; i < N; ++i) g[i] = src[f * N3 + tidx<N>(e, i, ta, tb)];
#pragma unroll
        for (int l = 0; l < N; ++l) {
          double v = 0.0;
#pragma unroll
          for (int j = 0; j < N; ++j) v = fma(T.M[l][j], g[j], v);
          dst[f * N3 + tidx<N>(e, l, ta, tb)] = v;
        }
      }
      __syncthreads();
    }
    // W now holds y_q,d / J and this direction's part of y_u / J
    for (int i = t; i < N3; i += NF) {
      if (active) y[(int64_t)d * ncells * N3 + cell * N3 + i] = T.J * W[i];
      Yu[i] += W[N3 + i];
    }
    __syncthreads();
  }
  for (int i = t; i < N3; i += NF)
    if (active) y[3 * ncells * N3 + cell * N3 + i] = T.J * Yu[i];
}


// ---- element-by-element post-processing on Cartesian cells: u* in Q_{k+1} with
//   (grad u*, grad w)_K = -(q, grad w)_K,  (u*, 1)_K = (u, 1)_K.
// With the degree-(k+1) GLL basis (P = k+2 points, Gauss P-point rule) the stiffness is the
// Kronecker sum J sum_d a_d^2 S* (x) M* (x) M* and the right-hand side
//   -sum_d J a_d (C in slot d, X elsewhere) q_d,  C_ij = int phi*_i' phi_j,  X_ij = int phi*_i phi_j
// (phi_j the degree-k basis of q); S* V = M* V Lambda (V^T M* V = I, Lambda_z = 0 for the constant
// mode) gives u* = J^-1 V^(3) (sum a_d^2 Lambda)^-1 V^(3)T rhs on the other modes, plus the
// constant mode fixed by the cell mean.
struct PostTab {
  double V[kMaxN + 1][kMaxN + 1];     // [i][mode] generalized eigenvectors (degree k+1)
  double lam[kMaxN + 1];
  double C[kMaxN + 1][kMaxN];         // [i*][j]
  double X[kMaxN + 1][kMaxN];
  double mk[kMaxN];                   // int phi_j (degree k)
  double a2[3], a[3], J;
  double vzsum;                       // (1^T M* v_z) for the constant mode
  int z;                              // index of the constant mode
};

template <int K>
__global__ void __launch_bounds__((K + 2) * (K + 2)) hdg_post_kernel(const double* __restrict__ q,
                                                                       const double* __restrict__ u,
                                                                       double* __restrict__ us,
                                                                       const __grid_constant__ PostTab T,
                                                                       int64_t ncells) {
  constexpr int N = K + 1, P = K + 2, N3 = N * N * N, P3 = P * P * P;
  __shared__ double A[P3], B[P3], R[P3], Qs[N3];
  const int t = threadIdx.x, ta = t % P, tb = t / P;
  const int64_t cell = blockIdx.x;
  for (int i = t; i < P3; i += P * P) R[i] = 0.0;
  // mean of u
  __shared__ double umean;
  if (t == 0) umean = 0.0;
  __syncthreads();
  for (int d = 0; d < 3; ++d) {
    for (int i = t; i < N3; i += P * P) Qs[i] = q[(int64_t)d * ncells * N3 + cell * N3 + i];
    __syncthreads();
    // x: n -> P (lines over (y, z) in n^2)
    if (ta < N && tb < N) {
      double g[N];
#pragma unroll
      for (int j = 0; j < N; ++j) g[j] = Qs[j + N * ta + N * N * tb];
#pragma unroll
      for (int i = 0; i < P; ++i) {
        double v = 0.0;
#pragma unroll
        for (int j = 0; j < N; ++j) v = fma(d == 0 ? T.C[i][j] : T.X[i][j], g[j], v);
        A[i + P * ta + P * N * tb] = v;   // [P][N][N]
      }
    }
    __syncthreads();
    // y: n -> P (lines over (x*, z) in P x n)
    if (tb < N) {
      double g[N];
#pragma unroll
      for (int j = 0; j < N; ++j) g[j] = A[ta + P * j + P * N * tb];
#pragma unroll
      for (int i = 0; i < P; ++i) {
        double v = 0.0;
#pragma unroll
        for (int j = 0; j < N; ++j) v = fma(d == 1 ? T.C[i][j] : T.X[i][j], g[j], v);
        B[ta + P * i + P * P * tb] = v;   // [P][P][N]
      }
    }
    __syncthreads();
    // z: n -> P (lines over (x*, y*))
    {
      double g[N];
#pragma unroll
      for (int j = 0; j < N; ++j) g[j] = B[ta + P * tb + P * P * j];
      const double f = -T.J * T.a[d];
#pragma unroll
      for (int i = 0; i < P; ++i) {
        double v = 0.0;
#pragma unroll
        for (int j = 0; j < N; ++j) v = fma(d == 2 ? T.C[i][j] : T.X[i][j], g[j], v);
        R[ta + P * tb + P * P * i] += f * v;
      }
    }
    __syncthreads();
  }
  {   // (u, 1)_K = J sum_j mk x mk x mk u_j
    double s = 0.0;
    for (int i = t; i < N3; i += P * P) s += T.mk[i % N] * T.mk[(i / N) % N] * T.mk[i / (N * N)] * u[cell * N3 + i];
    atomicAdd(&umean, s);   // shared-memory atomic (one block)
  }
  // FD: V^T in x, y, z; scale; V in z, y, x
  auto sweep = [&](int e, const double* src, double* dst, bool trans) {
    double g[P];
#pragma unroll
    for (int i = 0; i < P; ++i)
      g[i] = src[e == 0 ? i + P * ta + P * P * tb : e == 1 ? ta + P * i + P * P * tb : ta + P * tb + P * P * i];
#pragma unroll
    for (int o = 0; o < P; ++o) {
      double v = 0.0;
#pragma unroll
      for (int i = 0; i < P; ++i) v = fma(trans ? T.V[i][o] : T.V[o][i], g[i], v);
      dst[e == 0 ? o + P * ta + P * P * tb : e == 1 ? ta + P * o + P * P * tb : ta + P * tb + P * P * o] = v;
    }
  };
  sweep(0, R, A, true);
  __syncthreads();
  sweep(1, A, B, true);
  __syncthreads();
  sweep(2, B, A, true);
  __syncthreads();
  for (int i = t; i < P3; i += P * P) {
    const int i0 = i % P, i1 = (i / P) % P, i2 = i / (P * P);
    if (i0 == T.z && i1 == T.z && i2 == T.z) {
      A[i] = umean / (T.vzsum * T.vzsum * T.vzsum);   // the constant mode: (u*, 1)_K = (u, 1)_K (J cancels)
    } else {
      A[i] /= T.J * (T.a2[0] * T.lam[i0] + T.a2[1] * T.lam[i1] + T.a2[2] * T.lam[i2]);
    }
  }
  __syncthreads();
  sweep(2, A, B, false);
  __syncthreads();
  sweep(1, B, A, false);
  __syncthreads();
  sweep(0, A, B, false);
  __syncthreads();
  for (int i = t; i < P3; i += P * P) us[cell * P3 + i] = B[i];
}

// manufactured load F = (f, v), f = pi^2 sum_d (hi_d - lo_d)^-2 prod_d sin(pi t_d)
__global__ void hdg_load_kernel(double* F, const double* qp, const double* qw, const double* val, int N,
                                int nx, int ny, int nz, double lx, double ly, double lz, double hx, double hy,
                                double hz, double c, int64_t total) {
  const int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (g >= total) return;
  const int N3 = N * N * N;
  const int64_t cell = g / N3;
  const int i = (int)(g % N3);
  const int idx[3] = {i % N, (i / N) % N, i / (N * N)};
  const int cc[3] = {(int)(cell % nx), (int)((cell / nx) % ny), (int)(cell / ((int64_t)nx * ny))};
  const double h[3] = {hx, hy, hz}, len[3] = {hx * nx, hy * ny, hz * nz};
  (void)lx, (void)ly, (void)lz;
  double f = c * (hx / 2) * (hy / 2) * (hz / 2);
  for (int d = 0; d < 3; ++d) {
    double s = 0.0;
    for (int q = 0; q < N; ++q) {
      const double xr = h[d] * (cc[d] + 0.5 * (qp[q] + 1.0));   // x - lo
      s += qw[q] * val[q * N + idx[d]] * sin(M_PI * xr / len[d]);
    }
    f *= s;
  }
  F[g] = f;
}

// diag(K) from the element diagonal de[6][NF]: a face node gets the lo-side entry of the
// cell above it and the hi-side entry of the cell below it (constrained: 1)
__global__ void hdg_diag_kernel(double* d, const double* de, int N, int nx, int ny, int nz, int64_t fx,
                                int64_t fy, int bc, int64_t n) {
  const int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (g >= n) return;
  const int NF = N * N;
  const int64_t f = g / NF;
  const int t = (int)(g % NF);
  int dd, i, nn;
  if (f < fx) {
    dd = 0;
    i = (int)(f % (nx + 1));
    nn = nx;
  } else if (f < fx + fy) {
    dd = 1;
    i = (int)(((f - fx) / nx) % (ny + 1));
    nn = ny;
  } else {
    dd = 2;
    i = (int)((f - fx - fy) / ((int64_t)nx * ny));
    nn = nz;
  }
  const bool has_hi = i < nn, has_lo = i > 0;   // cell above (face = its lo side) / below
  if ((!has_lo && ((bc >> (2 * dd)) & 1)) || (!has_hi && ((bc >> (2 * dd + 1)) & 1))) {
    d[g] = 1.0;
    return;
  }
  d[g] = (has_hi ? de[(2 * dd) * NF + t] : 0.0) + (has_lo ? de[(2 * dd + 1) * NF + t] : 0.0);
}

__global__ void hdg_dot_kernel(const double* x, const double* y, int64_t n, double* part) {
  __shared__ double s[256];
  double v = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    v = fma(x[i], y[i], v);
  s[threadIdx.x] = v;
  __syncthreads();
  for (int w = blockDim.x / 2; w > 0; w >>= 1) {
    if ((int)threadIdx.x < w) s[threadIdx.x] += s[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) part[blockIdx.x] = s[0];
}

__global__ void hdg_sum_kernel(const double* part, int n, double* out) {   // one block of 256
  __shared__ double s[256];
  double v = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) v += part[i];
  s[threadIdx.x] = v;
  __syncthreads();
  for (int w = blockDim.x / 2; w > 0; w >>= 1) {
    if ((int)threadIdx.x < w) s[threadIdx.x] += s[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = s[0];
}

// x += alpha p, r -= alpha q, z = Dinv r
__global__ void hdg_upd_kernel(double* x, double* r, double* z, const double* p, const double* q, const double* dinv,
                               double alpha, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    x[i] = fma(alpha, p[i], x[i]);
    const double ri = fma(-alpha, q[i], r[i]);
    r[i] = ri;
    z[i] = dinv[i] * ri;
  }
}
// p = z + beta p (beta = 0: p = z)
__global__ void hdg_axpy_kernel(double* p, const double* z, double beta, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    p[i] = fma(beta, p[i], z[i]);
}
// r = b, z = Dinv b (x = 0 start) or r = b - y
__global__ void hdg_res_kernel(double* r, double* z, const double* b, const double* y, const double* dinv, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double ri = y ? b[i] - y[i] : b[i];
    r[i] = ri;
    z[i] = dinv[i] * ri;
  }
}
__global__ void hdg_inv_kernel(double* dinv, const double* d, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    dinv[i] = 1.0 / d[i];
}

// ---------------------------------------------------------------- host 1-D algebra
void invert(int n, const double (&A)[kMaxN][kMaxN], double (&X)[kMaxN][kMaxN]) {   // Gauss-Jordan, pivoting
  double W[kMaxN][2 * kMaxN] = {};
  for (int i = 0; i < n; ++i) {
    for (int j = 0; j < n; ++j) W[i][j] = A[i][j];
    W[i][n + i] = 1.0;
  }
  for (int c = 0; c < n; ++c) {
    int p = c;
    for (int r = c + 1; r < n; ++r)
      if (std::fabs(W[r][c]) > std::fabs(W[p][c])) p = r;
    for (int j = 0; j < 2 * n; ++j) std::swap(W[c][j], W[p][j]);
    const double piv = W[c][c];
    for (int j = 0; j < 2 * n; ++j) W[c][j] /= piv;
    for (int r = 0; r < n; ++r)
      if (r != c) {
        const double f = W[r][c];
        for (int j = 0; j < 2 * n; ++j) W[r][j] -= f * W[c][j];
      }
  }
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) X[i][j] = W[i][n + j];
}

// symmetric eigenproblem by cyclic Jacobi rotations: A = Q diag(e) Q^T
void sym_eig(int n, double (&A)[kMaxN][kMaxN], double (&Q)[kMaxN][kMaxN], double* e) {
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) Q[i][j] = i == j ? 1.0 : 0.0;
  for (int sweep = 0; sweep < 100; ++sweep) {
    double off = 0.0;
    for (int p = 0; p < n; ++p)
      for (int q = p + 1; q < n; ++q) off += A[p][q] * A[p][q];
    if (off < 1e-300) break;
    for (int p = 0; p < n; ++p)
      for (int q = p + 1; q < n; ++q) {
        if (A[p][q] == 0.0) continue;
        const double th = (A[q][q] - A[p][p]) / (2.0 * A[p][q]);
        const double tt = (th >= 0 ? 1.0 : -1.0) / (std::fabs(th) + std::sqrt(th * th + 1.0));
        const double c = 1.0 / std::sqrt(tt * tt + 1.0), s = tt * c;
        for (int k = 0; k < n; ++k) {
          const double akp = A[k][p], akq = A[k][q];
          A[k][p] = c * akp - s * akq;
          A[k][q] = s * akp + c * akq;
        }
        for (int k = 0; k < n; ++k) {
          const double apk = A[p][k], aqk = A[q][k];
          A[p][k] = c * apk - s * aqk;
          A[q][k] = s * apk + c * aqk;
        }
        for (int k = 0; k < n; ++k) {
          const double qkp = Q[k][p], qkq = Q[k][q];
          Q[k][p] = c * qkp - s * qkq;
          Q[k][q] = s * qkp + c * qkq;
        }
      }
  }
  for (int i = 0; i < n; ++i) e[i] = A[i][i];
}

void build_hdg_tab(int k, const double h[3], double tau, HdgTab& T) {
  Tables1D t1;
  build_tables(k, t1);
  const int n = k + 1;
  T = HdgTab{};
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) {
      double m = 0.0, dm = 0.0;
      for (int q = 0; q < n; ++q) {
        m += t1.qw[q] * t1.val[q][i] * t1.val[q][j];
        dm += t1.qw[q] * t1.val[q][i] * t1.der[q][j];
      }
      T.M[i][j] = m;
      T.Dm[i][j] = dm;
    }
  invert(n, T.M, T.Minv);
  double DMi[kMaxN][kMaxN] = {};   // Dm M^-1
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) {
      double p = 0.0, dmi = 0.0;
      for (int m = 0; m < n; ++m) {
        p += T.Minv[i][m] * T.Dm[j][m];
        dmi += T.Dm[i][m] * T.Minv[m][j];
      }
      T.P[i][j] = p;
      DMi[i][j] = dmi;
    }
  T.J = h[0] * h[1] * h[2] / 8.0;
  T.tau = tau;
  // M = R R^T (Cholesky, lower R), R^-1
  double R[kMaxN][kMaxN] = {}, Ri[kMaxN][kMaxN] = {};
  for (int i = 0; i < n; ++i)
    for (int j = 0; j <= i; ++j) {
      double s = T.M[i][j];
      for (int m = 0; m < j; ++m) s -= R[i][m] * R[j][m];
      R[i][j] = i == j ? std::sqrt(s) : s / R[j][j];
    }
  invert(n, R, Ri);
  for (int d = 0; d < 3; ++d) {
    const double ad = 2.0 / h[d];
    T.a[d] = ad;
    double L[kMaxN][kMaxN] = {}, Cm[kMaxN][kMaxN] = {}, Q[kMaxN][kMaxN] = {};
    for (int i = 0; i < n; ++i)
      for (int j = 0; j < n; ++j) {
        double s = 0.0;
        for (int m = 0; m < n; ++m) s += DMi[i][m] * T.Dm[j][m];
        L[i][j] = ad * ad * s + ((i == j && (i == 0 || i == k)) ? tau * ad : 0.0);
      }
    for (int i = 0; i < n; ++i)   // Cm = R^-1 L R^-T
      for (int j = 0; j < n; ++j) {
        double s = 0.0;
        for (int p = 0; p < n; ++p)
          for (int q = 0; q < n; ++q) s += Ri[i][p] * L[p][q] * Ri[j][q];
        Cm[i][j] = s;
      }
    for (int i = 0; i < n; ++i)
      for (int j = i + 1; j < n; ++j) Cm[i][j] = Cm[j][i] = 0.5 * (Cm[i][j] + Cm[j][i]);
    sym_eig(n, Cm, Q, T.lam[d]);
    for (int i = 0; i < n; ++i)   // V = R^-T Q
      for (int j = 0; j < n; ++j) {
        double s = 0.0;
        for (int p = 0; p < n; ++p) s += Ri[p][i] * Q[p][j];
        T.V[d][i][j] = s;
      }
    for (int hi = 0; hi < 2; ++hi) {
      const int l = hi ? k : 0;
      const double sg = hi ? 1.0 : -1.0;
      for (int i = 0; i < n; ++i)
        T.w[2 * d + hi][i] = T.J * ((i == l ? tau * ad : 0.0) + sg * ad * ad * DMi[i][l]);
    }
  }
}


// ================================================================ curved cells (the paper's design)
// "HDG trace matrix-free" with the inner Schur complement's inverse STORED per cell (P:L449-460:
// "Only the (k+1)^d x (k+1)^d matrix (D - B A^-1 B^T)^-1 needs to be explicitly stored"), on the
// deformed box map x = xhat + eps s(xhat) (1,1,1) (reading R2), k <= 4 (the per-cell inversion
// runs in shared memory).  With the GLL basis and the (k+1)-point Gauss rule the interpolation
// B3 = val (x) val (x) val is square and invertible, so on every cell
//   A^-1 = B3^-1 W^-1 B3^-T  (W = w det J at the Gauss points),   E_i = B3^T W sum_e Jinv_ei D_e,
//   D_e B3^-1 = Dco_e (collocation derivative at the Gauss points, slot e),
// and the inner Schur complement S = D + E A^-1 E^T = K_e + D: the cell's Laplace stiffness plus
// tau times the face masses of its face layers (built by quadrature, inverted at setup).
// Per cell and apply (R_q, R_u of step (1) are supported on the face layers):
//   r_i(q) = sum_s (val^-T e_l)(q_d) g_si(q_t) / W(q),  g_si = -(w_F det J m_i) lambda_s(q_t)
//   t = R_u - B3^T W sum_i sum_e Jinv_ei (Dco_e r_i)       (W^-1 B3^-T R_q,i = r_i)
//   u = S^-1 t;  u_q = B3 u;  z_i = W^-1 sum_e Dco_e^T (Jinv_ei W u_q)
//   at face points: q_i = sum_qd val^-1[l][qd] (r_i + z_i),  u = sum_qd val^-1[l][qd] u_q
//   y_s = B_F^T [tau JxW (lambda - u) - sum_i (w_F det J m_i) q_i],
// m = J^-T nhat (Nanson: JxW n = w_F det J m, JxW = w_F det J |m|).
struct CurvTab {
  double val[kMaxN][kMaxN];    // [q][i] GLL basis at the Gauss points
  double vinv[kMaxN][kMaxN];   // [i][q] val^-1
  double der[kMaxN][kMaxN];    // [q][i]
  double dco[kMaxN][kMaxN];    // [q][p] collocation derivative at the Gauss points
  double qw[kMaxN], qp[kMaxN];
  double lo[3], len[3], h[3], eps, tau;
};
constexpr int kCurvDoubles = sizeof(CurvTab) / sizeof(double);

template <int N>
struct CurvCellGeo {                 // sin / cos of pi t_d at the Gauss points and the two faces
  double sn[3][N], cs[3][N], sb[3][2], cb[3][2];
};

template <int N>
__device__ void curv_cell_geo(const CurvTab& T, int cx, int cy, int cz, int t, CurvCellGeo<N>& G) {
  const int c3[3] = {cx, cy, cz};
  for (int i = t; i < 3 * (N + 2); i += N * N) {
    const int d = i / (N + 2), j = i % (N + 2);
    const double xr = j < N ? T.h[d] * (c3[d] + 0.5 * (T.qp[j] + 1.0)) : T.h[d] * (c3[d] + (j - N));
    double sv, cv;
    sincospi(xr / T.len[d], &sv, &cv);
    if (j < N) {
      G.sn[d][j] = sv;
      G.cs[d][j] = cv;
    } else {
      G.sb[d][j - N] = sv;
      G.cb[d][j - N] = cv;
    }
  }
}

// grad s at a point given sin / cos per direction; returns beta = eps / (1 + eps sum g), det J
__device__ __forceinline__ void curv_point(const CurvTab& T, const double s[3], const double c[3], double g[3],
                                           double& beta, double& detJ) {
  g[0] = M_PI / T.len[0] * c[0] * s[1] * s[2];
  g[1] = M_PI / T.len[1] * s[0] * c[1] * s[2];
  g[2] = M_PI / T.len[2] * s[0] * s[1] * c[2];
  const double sg = 1.0 + T.eps * (g[0] + g[1] + g[2]);
  beta = T.eps / sg;
  detJ = 0.125 * T.h[0] * T.h[1] * T.h[2] * sg;
}
// Jinv[e][d] = (2/h_e)(delta_ed - beta g_d)
__device__ __forceinline__ double curv_jinv(const CurvTab& T, const double g[3], double beta, int e, int d) {
  return (2.0 / T.h[e]) * ((e == d ? 1.0 : 0.0) - beta * g[d]);
}

template <int N>
__device__ __forceinline__ int cidx(int e, int i, int ta, int tb) {   // node i on the e-line at (ta, tb)
  return e == 0 ? i + N * ta + N * N * tb : e == 1 ? ta + N * i + N * N * tb : ta + N * tb + N * N * i;
}

// S_cell = D + E A^-1 E^T = D + sum_c P_c^T W P_c, P_c = W^-1 sum_e Dco_e^T (Jinv_ec W) B3, built
// column by column with the apply's sum-factorized sweeps, then S^-1 by Gauss-Jordan in shared
// memory (SPD: no pivoting); one block per cell, the first (k+1)^2 threads own the sweep lines.
template <int K>
__global__ void __launch_bounds__(128) hdg_curved_setup_kernel(const CurvTab* tab, double* __restrict__ Sinv,
                                                               int nx, int ny, int64_t ncells) {
  constexpr int N = K + 1, NF = N * N, M = N * N * N;
  extern __shared__ double sm[];
  CurvTab& T = *reinterpret_cast<CurvTab*>(sm);
  double* A = sm + kCurvDoubles;   // [M][M]
  double* Uq = A + M * M;          // [M]
  double* P = Uq + M;              // [M]
  double* T1 = P + M;              // [M]
  double* T2 = T1 + M;             // [M]
  double* Y = T2 + M;              // [M]
  double* row = Y + M;             // [M]
  __shared__ CurvCellGeo<N> geo;
  const int tid = threadIdx.x, nt = blockDim.x;
  const int t = tid < NF ? tid : 0, ta = t % N, tb = t / N;
  const bool ln = tid < NF;
  for (int i = tid; i < kCurvDoubles; i += nt) sm[i] = reinterpret_cast<const double*>(tab)[i];
  const int64_t cell = blockIdx.x;
  const int cx = (int)(cell % nx), cy = (int)((cell / nx) % ny), cz = (int)(cell / ((int64_t)nx * ny));
  __syncthreads();
  if (ln) curv_cell_geo<N>(T, cx, cy, cz, t, geo);
  __syncthreads();
  auto cell_geo = [&](int q, double& W, double Ji[3][3]) {
    const int q0 = q % N, q1 = (q / N) % N, q2 = q / NF;
    const double s[3] = {geo.sn[0][q0], geo.sn[1][q1], geo.sn[2][q2]}, c[3] = {geo.cs[0][q0], geo.cs[1][q1], geo.cs[2][q2]};
    double g[3], beta, detJ;
    curv_point(T, s, c, g, beta, detJ);
    W = T.qw[q0] * T.qw[q1] * T.qw[q2] * detJ;
    for (int e = 0; e < 3; ++e)
      for (int d = 0; d < 3; ++d) Ji[e][d] = curv_jinv(T, g, beta, e, d);
  };
  auto sweep = [&](int e, const double* src, double* dst, auto Mt) {   // lines of the first NF threads
    if (!ln) return;
    double g[N];
#pragma unroll
    for (int i = 0; i < N; ++i) g[i] = src[cidx<N>(e, i, ta, tb)];
#pragma unroll
    for (int o = 0; o < N; ++o) {
      double v = 0.0;
#pragma unroll
      for (int i = 0; i < N; ++i) v = fma(Mt(o, i), g[i], v);
      dst[cidx<N>(e, o, ta, tb)] = v;
    }
  };
  for (int jc = 0; jc < M; ++jc) {
    const int j0 = jc % N, j1 = (jc / N) % N, j2 = jc / NF;
    for (int q = tid; q < M; q += nt) {   // u_q = B3 e_j (a tensor product of basis columns)
      Uq[q] = T.val[q % N][j0] * T.val[(q / N) % N][j1] * T.val[q / NF][j2];
      Y[q] = 0.0;
    }
    __syncthreads();
    for (int c = 0; c < 3; ++c) {
      // P_c e_j = W^-1 sum_e Dco_e^T (Jinv_ec W u_q)
      for (int q = tid; q < M; q += nt) P[q] = 0.0;
      __syncthreads();
      for (int e = 0; e < 3; ++e) {
        for (int q = tid; q < M; q += nt) {
          double W, Ji[3][3];
          cell_geo(q, W, Ji);
          T1[q] = Ji[e][c] * W * Uq[q];
        }
        __syncthreads();
        sweep(e, T1, T2, [&](int o, int i) { return T.dco[i][o]; });
        __syncthreads();
        for (int q = tid; q < M; q += nt) P[q] += T2[q];
        __syncthreads();
      }
      // p_c = P_c e_j = W^-1 X;  P_c^T W p_c = B3^T sum_e (Jinv_ec W) Dco_e p_c
      for (int q = tid; q < M; q += nt) {
        double W, Ji[3][3];
        cell_geo(q, W, Ji);
        P[q] /= W;
      }
      __syncthreads();
      for (int e = 0; e < 3; ++e) {
        sweep(e, P, T2, [&](int o, int i) { return T.dco[o][i]; });
        __syncthreads();
        for (int q = tid; q < M; q += nt) {
          double W, Ji[3][3];
          cell_geo(q, W, Ji);
          Y[q] += Ji[e][c] * W * T2[q];
        }
        __syncthreads();
      }
    }
    // the column of sum_c P_c^T W P_c is B3^T Y
    sweep(0, Y, T1, [&](int o, int i) { return T.val[i][o]; });
    __syncthreads();
    sweep(1, T1, T2, [&](int o, int i) { return T.val[i][o]; });
    __syncthreads();
    sweep(2, T2, T1, [&](int o, int i) { return T.val[i][o]; });
    __syncthreads();
    for (int i = tid; i < M; i += nt) A[i * M + jc] = T1[i];
    __syncthreads();
  }
  // + D: tau face masses on the face layers
  for (int p = tid; p < M * M; p += nt) {
    const int i = p / M, j = p % M;
    const int ic[3] = {i % N, (i / N) % N, i / NF}, jcc[3] = {j % N, (j / N) % N, j / NF};
    double add = 0.0;
    for (int sd = 0; sd < 6; ++sd) {
      const int d = sd / 2, hi = sd & 1, l = hi ? K : 0;
      if (ic[d] != l || jcc[d] != l) continue;
      const int t1 = d == 0 ? 1 : 0, t2 = d == 2 ? 1 : 2;
      for (int b = 0; b < N; ++b)
        for (int a2 = 0; a2 < N; ++a2) {
          double sv[3], cv[3];
          sv[d] = geo.sb[d][hi];
          cv[d] = geo.cb[d][hi];
          sv[t1] = geo.sn[t1][a2];
          cv[t1] = geo.cs[t1][a2];
          sv[t2] = geo.sn[t2][b];
          cv[t2] = geo.cs[t2][b];
          double g[3], beta, detJ;
          curv_point(T, sv, cv, g, beta, detJ);
          double m2 = 0.0;
          for (int e = 0; e < 3; ++e) {
            const double me = curv_jinv(T, g, beta, d, e);
            m2 += me * me;
          }
          add += T.tau * T.qw[a2] * T.qw[b] * detJ * sqrt(m2) * T.val[a2][ic[t1]] * T.val[b][ic[t2]] *
                 T.val[a2][jcc[t1]] * T.val[b][jcc[t2]];
        }
    }
    A[p] += add;
  }
  __syncthreads();
  for (int p = tid; p < M * M; p += nt) {   // symmetrize (rounding)
    const int i = p / M, j = p % M;
    if (i < j) {
      const double v = 0.5 * (A[i * M + j] + A[j * M + i]);
      A[i * M + j] = v;
      A[j * M + i] = v;
    }
  }
  __syncthreads();
  // in-place Gauss-Jordan inverse (SPD: no pivoting)
  for (int k = 0; k < M; ++k) {
    const double piv = A[k * M + k];
    for (int j = tid; j < M; j += nt) {
      row[j] = (j == k ? 1.0 : A[k * M + j]) / piv;
      P[j] = A[j * M + k];   // the pivot column, read before any thread overwrites it
    }
    __syncthreads();
    for (int p = tid; p < M * M; p += nt) {
      const int i = p / M, j = p % M;
      if (i == k) continue;
      A[p] = (j == k ? 0.0 : A[p]) - P[i] * row[j];
    }
    __syncthreads();
    for (int j = tid; j < M; j += nt) A[k * M + j] = row[j];
    __syncthreads();
  }
  double* out = Sinv + cell * (int64_t)M * M;
  for (int p = tid; p < M * M; p += nt) out[p] = A[p];
}

template <int N>
struct CurvCfg {
  static constexpr int NF = N * N, M = N * N * N;
  static constexpr int PER_CELL = 10 * M + 3 * 6 * NF;   // r[3], z[3], T1, T2, U, Uq; lam, lq, fo
  static constexpr int SMEM = kCurvDoubles + PER_CELL;
};

// MODE kApply / kRhs / kRecover (see hdg_cell_kernel), one cell per block of (k+1)^2 threads.
// kDiag here: blockIdx = cell; the 6 (k+1)^2 unit traces of that cell in turn, output the
// diagonal entry of the cell's trace matrix (a.y[cell * 6 NF + s NF + a]).
template <int K, int MODE>
__global__ void __launch_bounds__((K + 1) * (K + 1)) hdg_curved_kernel(HdgArgs a, const CurvTab* tab,
                                                                      const double* __restrict__ Sinv) {
  constexpr int N = K + 1, NF = N * N, M = N * N * N;
  extern __shared__ double sm[];
  CurvTab& T = *reinterpret_cast<CurvTab*>(sm);
  __shared__ CurvCellGeo<N> geo;
  const int t = threadIdx.x, ta = t % N, tb = t / N;
  for (int i = t; i < kCurvDoubles; i += NF) sm[i] = reinterpret_cast<const double*>(tab)[i];
  double* R = sm + kCurvDoubles;   // [3][M]
  double* Z = R + 3 * M;           // [3][M]
  double* T1 = Z + 3 * M;
  double* T2 = T1 + M;
  double* U = T2 + M;
  double* Uq = U + M;
  double* lam = Uq + M;            // [6][NF]
  double* lq = lam + 6 * NF;       // [6][NF] lambda at the face points
  double* fo = lq + 6 * NF;        // [6][NF]
  const int64_t j = blockIdx.x;
  int cx, cy, cz;
  bool active = true;
  if (MODE != kDiag && a.color >= 0) {
    const int cpr = (a.nx + 1) / 2;
    const int64_t rowi = j / cpr;
    cy = (int)(rowi % a.ny);
    cz = (int)(rowi / a.ny);
    cx = 2 * (int)(j % cpr) + ((cy + cz + a.color) & 1);
    active = cz < a.nz && cx < a.nx;
    if (!active) return;   // block-uniform
  } else {
    cx = (int)(j % a.nx);
    cy = (int)((j / a.nx) % a.ny);
    cz = (int)(j / ((int64_t)a.nx * a.ny));
  }
  const int64_t cell = cx + (int64_t)a.nx * (cy + (int64_t)a.ny * cz);
  int64_t fid[6];
  bool inter[6], dir[6];
  {
    const int c3[3] = {cx, cy, cz}, n3[3] = {a.nx, a.ny, a.nz};
    for (int s = 0; s < 6; ++s) {
      const int d = s / 2, hi = s & 1;
      fid[s] = d == 0 ? (cx + hi) + (int64_t)(a.nx + 1) * (cy + (int64_t)a.ny * cz)
             : d == 1 ? a.fx + cx + (int64_t)a.nx * ((cy + hi) + (int64_t)(a.ny + 1) * cz)
                      : a.fx + a.fy + cx + (int64_t)a.nx * (cy + (int64_t)a.ny * (cz + hi));
      inter[s] = hi ? c3[d] < n3[d] - 1 : c3[d] > 0;
      dir[s] = !inter[s] && ((a.bc >> s) & 1);
    }
  }
  __syncthreads();
  curv_cell_geo<N>(T, cx, cy, cz, t, geo);
  __syncthreads();
  const double* Sc = Sinv + cell * (int64_t)M * M;

  // face-point geometry of face s at the thread's face point (a, b) = (ta, tb)
  auto face_geo = [&](int s, double wm[3], double& jxw) {
    const int d = s / 2, hi = s & 1, t1 = d == 0 ? 1 : 0, t2 = d == 2 ? 1 : 2;
    double sv[3], cv[3];
    sv[d] = geo.sb[d][hi];
    cv[d] = geo.cb[d][hi];
    sv[t1] = geo.sn[t1][ta];
    cv[t1] = geo.cs[t1][ta];
    sv[t2] = geo.sn[t2][tb];
    cv[t2] = geo.cs[t2][tb];
    double g[3], beta, detJ;
    curv_point(T, sv, cv, g, beta, detJ);
    const double sg = hi ? 1.0 : -1.0, wf = T.qw[ta] * T.qw[tb] * detJ;
    double m2 = 0.0;
    for (int e = 0; e < 3; ++e) {
      const double me = sg * curv_jinv(T, g, beta, d, e);
      wm[e] = wf * me;
      m2 += me * me;
    }
    jxw = wf * sqrt(m2);
  };
  // the cell's q-point metric at q-point (q0, q1, q2)
  auto cell_geo = [&](int q0, int q1, int q2, double& W, double Ji[3][3]) {
    const double s[3] = {geo.sn[0][q0], geo.sn[1][q1], geo.sn[2][q2]}, c[3] = {geo.cs[0][q0], geo.cs[1][q1], geo.cs[2][q2]};
    double g[3], beta, detJ;
    curv_point(T, s, c, g, beta, detJ);
    W = T.qw[q0] * T.qw[q1] * T.qw[q2] * detJ;
    for (int e = 0; e < 3; ++e)
      for (int d = 0; d < 3; ++d) Ji[e][d] = curv_jinv(T, g, beta, e, d);
  };
  // sweep along direction e with the 1-D matrix Mt (out[o] = sum_i Mt(o, i) in[i])
  auto sweep = [&](int e, const double* src, double* dst, auto Mt) {
    double g[N];
#pragma unroll
    for (int i = 0; i < N; ++i) g[i] = src[cidx<N>(e, i, ta, tb)];
#pragma unroll
    for (int o = 0; o < N; ++o) {
      double v = 0.0;
#pragma unroll
      for (int i = 0; i < N; ++i) v = fma(Mt(o, i), g[i], v);
      dst[cidx<N>(e, o, ta, tb)] = v;
    }
  };

  const int nrep = MODE == kDiag ? 6 * NF : 1;
  for (int rep = 0; rep < nrep; ++rep) {
    // ---- inputs
    for (int s = 0; s < 6; ++s) {
      double v = 0.0;
      if (MODE == kDiag) v = (rep == s * NF + t) ? 1.0 : 0.0;
      else if ((MODE == kApply || MODE == kRecover) && !dir[s]) v = a.lam[fid[s] * NF + t];
      lam[s * NF + t] = v;
    }
    __syncthreads();
    // lambda at the face points (B_F: val in both tangential directions)
    for (int s = 0; s < 6; ++s) {
      double v = 0.0;
#pragma unroll
      for (int i = 0; i < N; ++i) v = fma(T.val[ta][i], lam[s * NF + i + N * tb], v);
      fo[s * NF + t] = v;
    }
    __syncthreads();
    for (int s = 0; s < 6; ++s) {
      double v = 0.0;
#pragma unroll
      for (int i = 0; i < N; ++i) v = fma(T.val[tb][i], fo[s * NF + ta + N * i], v);
      lq[s * NF + t] = v;
    }
    __syncthreads();
    // ---- r_i(q) = sum_s vinv[l][q_d] g_si(q_t) / W(q), g_si = -wm_i lambda_q; R_u on the face layers
    for (int i = t; i < 3 * M + M; i += NF) (i < 3 * M ? R : T1)[i < 3 * M ? i : i - 3 * M] = 0.0;
    __syncthreads();
    for (int s = 0; s < 6; ++s) {   // thread = face point (ta, tb) of face s: its normal line
      const int d = s / 2, l = (s & 1) ? K : 0;
      double wm[3], jxw;
      face_geo(s, wm, jxw);
      const double lv = lq[s * NF + t];
      fo[s * NF + t] = T.tau * jxw * lv;   // gu_s at the face point
#pragma unroll
      for (int qd = 0; qd < N; ++qd) {
        const int q = cidx<N>(d, qd, ta, tb);
        const double vl = T.vinv[l][qd];
        for (int c = 0; c < 3; ++c) R[c * M + q] += vl * (-wm[c] * lv);   // / W below
      }
      __syncthreads();   // faces of the same direction touch the same lines
    }
    for (int q = t; q < M; q += NF) {
      double W, Ji[3][3];
      cell_geo(q % N, (q / N) % N, q / NF, W, Ji);
      for (int c = 0; c < 3; ++c) R[c * M + q] /= W;
    }
    // R_u = sum_s e_l (x) B_F^T gu_s  (two tangential sweeps, then onto the layer)
    for (int s = 0; s < 6; ++s) {
      double v = 0.0;
#pragma unroll
      for (int i = 0; i < N; ++i) v = fma(T.val[i][ta], fo[s * NF + i + N * tb], v);
      lq[s * NF + t] = lq[s * NF + t];   // keep lambda_q
      Z[s * NF + t] = v;                 // scratch (Z is free until step z)
    }
    __syncthreads();
    for (int s = 0; s < 6; ++s) {
      const int d = s / 2, l = (s & 1) ? K : 0;
      double v = 0.0;
#pragma unroll
      for (int i = 0; i < N; ++i) v = fma(T.val[i][tb], Z[s * NF + ta + N * i], v);
      __syncthreads();
      T1[cidx<N>(d, l, ta, tb)] += v;
      __syncthreads();
    }
    if (MODE != kDiag && a.F && (MODE == kRhs || MODE == kRecover))
      for (int i = t; i < M; i += NF) T1[i] += a.F[cell * M + i];
    __syncthreads();
    // ---- h = sum_i sum_e Jinv_ei Dco_e r_i at the q-points -> U (scratch), then t = R_u - B3^T W h
    for (int q = t; q < M; q += NF) U[q] = 0.0;
    __syncthreads();
    for (int e = 0; e < 3; ++e) {
      for (int c = 0; c < 3; ++c) {
        sweep(e, R + c * M, T2, [&](int o, int i) { return T.dco[o][i]; });
        __syncthreads();
        for (int q = t; q < M; q += NF) {
          double W, Ji[3][3];
          cell_geo(q % N, (q / N) % N, q / NF, W, Ji);
          U[q] += Ji[e][c] * T2[q];
        }
        __syncthreads();
      }
    }
    for (int q = t; q < M; q += NF) {
      double W, Ji[3][3];
      cell_geo(q % N, (q / N) % N, q / NF, W, Ji);
      U[q] *= W;
    }
    __syncthreads();
    sweep(0, U, T2, [&](int o, int i) { return T.val[i][o]; });   // B3^T = val^T per direction
    __syncthreads();
    sweep(1, T2, U, [&](int o, int i) { return T.val[i][o]; });
    __syncthreads();
    sweep(2, U, T2, [&](int o, int i) { return T.val[i][o]; });
    __syncthreads();
    for (int i = t; i < M; i += NF) T1[i] -= T2[i];   // t
    __syncthreads();
    // ---- u = S^-1 t (dense, the stored inverse)
    for (int i = t; i < M; i += NF) {
      double v = 0.0;
      for (int jj = 0; jj < M; ++jj) v = fma(Sc[(int64_t)jj * M + i], T1[jj], v);
      U[i] = v;
    }
    __syncthreads();
    if (MODE == kRecover)
      for (int i = t; i < M; i += NF) a.u[cell * M + i] = U[i];
    // ---- u_q = B3 u
    sweep(0, U, T2, [&](int o, int i) { return T.val[o][i]; });
    __syncthreads();
    sweep(1, T2, Uq, [&](int o, int i) { return T.val[o][i]; });
    __syncthreads();
    sweep(2, Uq, T2, [&](int o, int i) { return T.val[o][i]; });
    __syncthreads();
    for (int i = t; i < M; i += NF) Uq[i] = T2[i];
    __syncthreads();
    // ---- z_i = W^-1 sum_e Dco_e^T (Jinv_ei W u_q)
    for (int i = t; i < 3 * M; i += NF) Z[i] = 0.0;
    __syncthreads();
    for (int e = 0; e < 3; ++e) {
      for (int c = 0; c < 3; ++c) {
        for (int q = t; q < M; q += NF) {
          double W, Ji[3][3];
          cell_geo(q % N, (q / N) % N, q / NF, W, Ji);
          T2[q] = Ji[e][c] * W * Uq[q];
        }
        __syncthreads();
        sweep(e, T2, T1, [&](int o, int i) { return T.dco[i][o]; });
        __syncthreads();
        for (int q = t; q < M; q += NF) Z[c * M + q] += T1[q];
        __syncthreads();
      }
    }
    for (int q = t; q < M; q += NF) {
      double W, Ji[3][3];
      cell_geo(q % N, (q / N) % N, q / NF, W, Ji);
      for (int c = 0; c < 3; ++c) Z[c * M + q] = Z[c * M + q] / W + R[c * M + q];   // r_i + z_i
    }
    __syncthreads();
    if (MODE == kRecover) {
      if (a.q) {   // q_i nodal = B3^-1 (r_i + z_i)
        for (int c = 0; c < 3; ++c) {
          sweep(0, Z + c * M, T1, [&](int o, int i) { return T.vinv[o][i]; });
          __syncthreads();
          sweep(1, T1, T2, [&](int o, int i) { return T.vinv[o][i]; });
          __syncthreads();
          sweep(2, T2, T1, [&](int o, int i) { return T.vinv[o][i]; });
          __syncthreads();
          for (int i = t; i < M; i += NF) a.q[(int64_t)c * a.n_work * M + cell * M + i] = T1[i];
          __syncthreads();
        }
      }
      return;
    }
    // ---- face outputs: out = tau JxW (lambda - u) - sum_i wm_i q_i at the face points, then B_F^T
    for (int s = 0; s < 6; ++s) {
      const int d = s / 2, l = (s & 1) ? K : 0;
      double wm[3], jxw;
      face_geo(s, wm, jxw);
      double qv[3] = {0, 0, 0}, uv = 0.0;
#pragma unroll
      for (int qd = 0; qd < N; ++qd) {
        const int q = cidx<N>(d, qd, ta, tb);
        const double vl = T.vinv[l][qd];
        uv = fma(vl, Uq[q], uv);
        for (int c = 0; c < 3; ++c) qv[c] = fma(vl, Z[c * M + q], qv[c]);
      }
      fo[s * NF + t] = T.tau * jxw * (lq[s * NF + t] - uv) - (wm[0] * qv[0] + wm[1] * qv[1] + wm[2] * qv[2]);
    }
    __syncthreads();
    for (int s = 0; s < 6; ++s) {
      double v = 0.0;
#pragma unroll
      for (int i = 0; i < N; ++i) v = fma(T.val[i][ta], fo[s * NF + i + N * tb], v);
      lq[s * NF + t] = v;
    }
    __syncthreads();
    for (int s = 0; s < 6; ++s) {
      double v = 0.0;
#pragma unroll
      for (int i = 0; i < N; ++i) v = fma(T.val[i][tb], lq[s * NF + ta + N * i], v);
      if (MODE == kDiag) {
        if (rep == s * NF + t) a.y[cell * 6 * NF + rep] = v;
        continue;
      }
      double* yp = a.y + fid[s] * NF + t;
      if (dir[s]) {
        *yp = MODE == kApply ? a.lam[fid[s] * NF + t] : 0.0;
      } else {
        if (MODE == kRhs) v = -v;
        if (a.color == 1 && inter[s]) *yp += v;
        else *yp = v;
      }
    }
    __syncthreads();
  }
}

// diag(K) from the per-cell element diagonals dc[cell][6][NF] (curved meshes)
__global__ void hdg_curved_diag_kernel(double* d, const double* dc, int N, int nx, int ny, int nz, int64_t fx,
                                       int64_t fy, int bc, int64_t n) {
  const int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (g >= n) return;
  const int NF = N * N;
  const int64_t f = g / NF;
  const int t = (int)(g % NF);
  int dd, i, nn;
  int64_t c_above;   // the cell whose lo side the face is (index with i)
  int64_t step;
  if (f < fx) {
    dd = 0;
    i = (int)(f % (nx + 1));
    const int64_t r = f / (nx + 1);
    c_above = i + (int64_t)nx * r;
    step = 1;
    nn = nx;
  } else if (f < fx + fy) {
    const int64_t ff = f - fx;
    dd = 1;
    const int cx = (int)(ff % nx);
    i = (int)((ff / nx) % (ny + 1));
    const int cz = (int)(ff / ((int64_t)nx * (ny + 1)));
    c_above = cx + (int64_t)nx * (i + (int64_t)ny * cz);
    step = nx;
    nn = ny;
  } else {
    const int64_t ff = f - fx - fy;
    dd = 2;
    i = (int)(ff / ((int64_t)nx * ny));
    c_above = ff % ((int64_t)nx * ny) + (int64_t)nx * ny * i;
    step = (int64_t)nx * ny;
    nn = nz;
  }
  const bool has_hi = i < nn, has_lo = i > 0;
  if ((!has_lo && ((bc >> (2 * dd)) & 1)) || (!has_hi && ((bc >> (2 * dd + 1)) & 1))) {
    d[g] = 1.0;
    return;
  }
  double v = 0.0;
  if (has_hi) v += dc[c_above * 6 * NF + (2 * dd) * NF + t];
  if (has_lo) v += dc[(c_above - step) * 6 * NF + (2 * dd + 1) * NF + t];
  d[g] = v;
}

// manufactured load on the deformed map: F_v = sum_q f(x(q)) phi_v(q) w det J(q)
__global__ void hdg_curved_load_kernel(double* F, const CurvTab* tab, int N, int nx, int ny, int64_t total) {
  const int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (g >= total) return;
  const CurvTab& T = *tab;
  const int M = N * N * N;
  const int64_t cell = g / M;
  const int v = (int)(g % M);
  const int v0 = v % N, v1 = (v / N) % N, v2 = v / (N * N);
  const int c3[3] = {(int)(cell % nx), (int)((cell / nx) % ny), (int)(cell / ((int64_t)nx * ny))};
  const double cf = M_PI * M_PI * (1.0 / (T.len[0] * T.len[0]) + 1.0 / (T.len[1] * T.len[1]) + 1.0 / (T.len[2] * T.len[2]));
  double acc = 0.0;
  for (int q2 = 0; q2 < N; ++q2)
    for (int q1 = 0; q1 < N; ++q1)
      for (int q0 = 0; q0 < N; ++q0) {
        const int qq[3] = {q0, q1, q2};
        double s[3], c[3], xh[3];
        for (int d = 0; d < 3; ++d) {
          xh[d] = T.h[d] * (c3[d] + 0.5 * (T.qp[qq[d]] + 1.0));
          sincospi(xh[d] / T.len[d], &s[d], &c[d]);
        }
        double g3[3], beta, detJ;
        curv_point(T, s, c, g3, beta, detJ);
        const double sx = s[0] * s[1] * s[2];
        double f = cf;
        for (int d = 0; d < 3; ++d) f *= sinpi((xh[d] + T.eps * sx) / T.len[d]);
        acc += f * T.val[q0][v0] * T.val[q1][v1] * T.val[q2][v2] * T.qw[q0] * T.qw[q1] * T.qw[q2] * detJ;
      }
  F[g] = acc;
}

}  // namespace
}  // namespace fem

struct hdg_ctx {
  fem_mesh mesh{};
  int k = 0, n = 0;
  double tau = 5.0;
  double h[3] = {0, 0, 0};
  cudaStream_t stream = nullptr;
  int64_t fx = 0, fy = 0, fz = 0, n_trace = 0, n_cells = 0;
  int bc = 0;
  fem::HdgTab tab_host{};
  fem::HdgTab* tab = nullptr;      // device
  double* de = nullptr;            // element diagonal [6][NF]
  double* diag = nullptr;          // diag(K)
  double* dinv = nullptr;
  double* F = nullptr;             // load vector (lazily)
  double* ydiag = nullptr;         // scratch
  double *r = nullptr, *p = nullptr, *q = nullptr, *z = nullptr, *part = nullptr, *scal = nullptr;
  double* d1d = nullptr;           // qp, qw, val for the load kernel
  // curved meshes (deform_eps != 0) or FEM_HDG_DENSE=1: the paper's design, S^-1 stored per cell
  bool curved = false;
  fem::CurvTab* ctab = nullptr;    // device
  double* Sinv = nullptr;          // [n_cells][M][M]
  double* dc = nullptr;            // [n_cells][6][NF] element diagonals
};

namespace fem {
namespace {

template <typename F>
int hdg_guard(F&& f) {
  try {
    f();
    return FEM_OK;
  } catch (const Error& e) {
    set_error(e.msg);
    return e.code;
  } catch (const std::exception& e) {
    set_error(e.what());
    return FEM_E_ARG;
  }
}

double* hdg_alloc(int64_t n) {
  void* p = nullptr;
  FEM_CUDA_TRY(cudaMalloc(&p, sizeof(double) * std::max<int64_t>(n, 1)));
  return static_cast<double*>(p);
}

void check_dev(const void* p, const char* what) {
  if (!p) throw Error{FEM_E_ARG, std::string("null ") + what};
  cudaPointerAttributes at{};
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess || at.type != cudaMemoryTypeDevice) {
    cudaGetLastError();
    throw Error{FEM_E_ARG, std::string(what) + ": the HDG entry points take device pointers"};
  }
}

template <int K, int MODE>
void launch_cells_k(hdg_ctx* h, HdgArgs a) {
  constexpr int N = K + 1;
  using Cfg = HdgCfg<N>;
  const size_t sm = sizeof(double) * Cfg::SMEM;
  auto kern = hdg_cell_kernel<K, MODE>;
  smem_attr(reinterpret_cast<const void*>(kern), sm);
  FEM_CUDA_TRY(cudaFuncSetAttribute(reinterpret_cast<const void*>(kern),
                                    cudaFuncAttributePreferredSharedMemoryCarveout, 100));
  a.tab = h->tab;
  a.nx = h->mesh.n[0];
  a.ny = h->mesh.n[1];
  a.nz = h->mesh.n[2];
  a.fx = h->fx;
  a.fy = h->fy;
  a.bc = h->bc;
  auto go = [&](int color) {
    a.color = color;
    if (MODE == kDiag) a.n_work = 6 * N * N;
    else if (color >= 0) a.n_work = (int64_t)((a.nx + 1) / 2) * a.ny * a.nz;
    else a.n_work = h->n_cells;
    const int64_t blocks = (a.n_work + Cfg::CPB - 1) / Cfg::CPB;
    kern<<<(unsigned)blocks, dim3(N * N, Cfg::CPB), sm, h->stream>>>(a, h->tab_host);
    count_launch();
    check_launch("hdg_cell_kernel");
  };
  if (MODE == kApply || MODE == kRhs) {
    go(0);
    go(1);
  } else {
    go(-1);
  }
}

template <int MODE>
void launch_cells(hdg_ctx* h, const HdgArgs& a) {
  switch (h->k) {
    case 1: launch_cells_k<1, MODE>(h, a); break;
    case 2: launch_cells_k<2, MODE>(h, a); break;
    case 3: launch_cells_k<3, MODE>(h, a); break;
    case 4: launch_cells_k<4, MODE>(h, a); break;
    case 5: launch_cells_k<5, MODE>(h, a); break;
    case 6: launch_cells_k<6, MODE>(h, a); break;
    case 7: launch_cells_k<7, MODE>(h, a); break;
    case 8: launch_cells_k<8, MODE>(h, a); break;
    default: throw Error{FEM_E_ARG, "degree must be 1..8"};
  }
}

template <int K>
void launch_mixed_k(hdg_ctx* h, const double* qu, double* y) {
  constexpr int N = K + 1;
  using Cfg = MixCfg<N>;
  const size_t sm = sizeof(double) * Cfg::SMEM;
  auto kern = hdg_mixed_kernel<K>;
  smem_attr(reinterpret_cast<const void*>(kern), sm);
  FEM_CUDA_TRY(cudaFuncSetAttribute(reinterpret_cast<const void*>(kern),
                                    cudaFuncAttributePreferredSharedMemoryCarveout, 100));
  const int64_t blocks = (h->n_cells + Cfg::CPB - 1) / Cfg::CPB;
  kern<<<(unsigned)blocks, dim3(N * N, Cfg::CPB), sm, h->stream>>>(qu, y, h->tab_host, h->mesh.n[0], h->mesh.n[1],
                                                                    h->mesh.n[2], h->bc, h->n_cells);
  count_launch();
  check_launch("hdg_mixed_kernel");
}

void launch_mixed(hdg_ctx* h, const double* qu, double* y) {
  switch (h->k) {
    case 1: launch_mixed_k<1>(h, qu, y); break;
    case 2: launch_mixed_k<2>(h, qu, y); break;
    case 3: launch_mixed_k<3>(h, qu, y); break;
    case 4: launch_mixed_k<4>(h, qu, y); break;
    case 5: launch_mixed_k<5>(h, qu, y); break;
    case 6: launch_mixed_k<6>(h, qu, y); break;
    case 7: launch_mixed_k<7>(h, qu, y); break;
    case 8: launch_mixed_k<8>(h, qu, y); break;
    default: throw Error{FEM_E_ARG, "degree must be 1..8"};
  }
}

template <int K, int MODE>
void launch_curved_k(hdg_ctx* h, HdgArgs a) {
  constexpr int N = K + 1;
  using Cfg = CurvCfg<N>;
  const size_t sm = sizeof(double) * Cfg::SMEM;
  auto kern = hdg_curved_kernel<K, MODE>;
  smem_attr(reinterpret_cast<const void*>(kern), sm);
  a.tab = h->tab;
  a.nx = h->mesh.n[0];
  a.ny = h->mesh.n[1];
  a.nz = h->mesh.n[2];
  a.fx = h->fx;
  a.fy = h->fy;
  a.bc = h->bc;
  auto go = [&](int color) {
    a.color = color;
    const int64_t blocks = color >= 0 ? (int64_t)((a.nx + 1) / 2) * a.ny * a.nz : h->n_cells;
    a.n_work = h->n_cells;
    kern<<<(unsigned)blocks, N * N, sm, h->stream>>>(a, h->ctab, h->Sinv);
    count_launch();
    check_launch("hdg_curved_kernel");
  };
  if (MODE == kApply || MODE == kRhs) {
    go(0);
    go(1);
  } else {
    go(-1);
  }
}

template <int MODE>
void launch_curved(hdg_ctx* h, const HdgArgs& a) {
  switch (h->k) {
    case 1: launch_curved_k<1, MODE>(h, a); break;
    case 2: launch_curved_k<2, MODE>(h, a); break;
    case 3: launch_curved_k<3, MODE>(h, a); break;
    case 4: launch_curved_k<4, MODE>(h, a); break;
    default: throw Error{FEM_E_ARG, "curved HDG: degree 1..4"};
  }
}

template <int K>
void curved_setup_k(hdg_ctx* h) {
  constexpr int N = K + 1, M = N * N * N;
  const size_t sm = sizeof(double) * (kCurvDoubles + M * M + 6 * M);
  auto kern = hdg_curved_setup_kernel<K>;
  smem_attr(reinterpret_cast<const void*>(kern), sm);
  kern<<<(unsigned)h->n_cells, 128, sm, h->stream>>>(h->ctab, h->Sinv, h->mesh.n[0], h->mesh.n[1], h->n_cells);
  count_launch();
  check_launch("hdg_curved_setup_kernel");
}

// dispatch: the fast-diagonalization kernels on Cartesian meshes, the stored-inverse ones otherwise
template <int MODE>
void launch_any(hdg_ctx* h, const HdgArgs& a) {
  if (h->curved) launch_curved<MODE>(h, a);
  else launch_cells<MODE>(h, a);
}

double lagr1(const double* nodes, int n, int i, double z) {
  double v = 1.0;
  for (int j = 0; j < n; ++j)
    if (j != i) v *= (z - nodes[j]) / (nodes[i] - nodes[j]);
  return v;
}
void build_post_tab(int k, const double h[3], PostTab& T) {
  Tables1D tk, tp;
  build_tables(k, tk);
  build_tables(k + 1, tp);   // degree k+1 basis, (k+2)-point Gauss rule
  const int n = k + 1, p = k + 2;
  T = PostTab{};
  double Ms[kMaxN][kMaxN] = {}, Ss[kMaxN][kMaxN] = {};
  for (int i = 0; i < p; ++i)
    for (int j = 0; j < p; ++j) {
      double m = 0.0, st = 0.0;
      for (int q = 0; q < p; ++q) {
        m += tp.qw[q] * tp.val[q][i] * tp.val[q][j];
        st += tp.qw[q] * tp.der[q][i] * tp.der[q][j];
      }
      Ms[i][j] = m;
      Ss[i][j] = st;
    }
  for (int i = 0; i < p; ++i)
    for (int j = 0; j < n; ++j) {
      double c = 0.0, x = 0.0;
      for (int q = 0; q < p; ++q) {
        const double pk = lagr1(tk.gll, n, j, tp.qp[q]);
        c += tp.qw[q] * tp.der[q][i] * pk;
        x += tp.qw[q] * tp.val[q][i] * pk;
      }
      T.C[i][j] = c;
      T.X[i][j] = x;
    }
  for (int j = 0; j < n; ++j) {
    double m = 0.0;
    for (int q = 0; q < n; ++q) m += tk.qw[q] * tk.val[q][j];
    T.mk[j] = m;
  }
  // S* V = M* V Lambda: Cholesky M* = R R^T, eig of R^-1 S* R^-T
  double R[kMaxN][kMaxN] = {}, Ri[kMaxN][kMaxN] = {}, Cm[kMaxN][kMaxN] = {}, Q[kMaxN][kMaxN] = {};
  for (int i = 0; i < p; ++i)
    for (int j = 0; j <= i; ++j) {
      double s = Ms[i][j];
      for (int m = 0; m < j; ++m) s -= R[i][m] * R[j][m];
      R[i][j] = i == j ? std::sqrt(s) : s / R[j][j];
    }
  invert(p, R, Ri);
  for (int i = 0; i < p; ++i)
    for (int j = 0; j < p; ++j) {
      double s = 0.0;
      for (int a2 = 0; a2 < p; ++a2)
        for (int b = 0; b < p; ++b) s += Ri[i][a2] * Ss[a2][b] * Ri[j][b];
      Cm[i][j] = s;
    }
  for (int i = 0; i < p; ++i)
    for (int j = i + 1; j < p; ++j) Cm[i][j] = Cm[j][i] = 0.5 * (Cm[i][j] + Cm[j][i]);
  double lam[kMaxN];
  sym_eig(p, Cm, Q, lam);
  int z = 0;
  for (int i = 1; i < p; ++i)
    if (std::fabs(lam[i]) < std::fabs(lam[z])) z = i;
  for (int i = 0; i < p; ++i) {
    T.lam[i] = i == z ? 0.0 : lam[i];
    for (int j = 0; j < p; ++j) {
      double s = 0.0;
      for (int m = 0; m < p; ++m) s += Ri[m][i] * Q[m][j];
      T.V[i][j] = s;
    }
  }
  T.z = z;
  double vs = 0.0;   // 1^T M* v_z
  for (int i = 0; i < p; ++i)
    for (int j = 0; j < p; ++j) vs += Ms[i][j] * T.V[j][z];
  T.vzsum = vs;
  T.J = h[0] * h[1] * h[2] / 8.0;
  for (int d = 0; d < 3; ++d) {
    T.a[d] = 2.0 / h[d];
    T.a2[d] = T.a[d] * T.a[d];
  }
}

template <int K>
void post_k(hdg_ctx* h, const double* q, const double* u, double* us) {
  PostTab T;
  build_post_tab(K, h->h, T);
  hdg_post_kernel<K><<<(unsigned)h->n_cells, (K + 2) * (K + 2), 0, h->stream>>>(q, u, us, T, h->n_cells);
  count_launch();
  check_launch("hdg_post_kernel");
}

unsigned grid_for(int64_t n) { return (unsigned)std::min<int64_t>((n + 255) / 256, 148 * 8); }

void ensure_load(hdg_ctx* h) {
  if (h->F) return;
  const int N = h->n;
  h->F = hdg_alloc(h->n_cells * N * N * N);
  if (h->curved) {
    const int64_t tot = h->n_cells * N * N * N;
    hdg_curved_load_kernel<<<(unsigned)((tot + 127) / 128), 128, 0, h->stream>>>(h->F, h->ctab, N, h->mesh.n[0],
                                                                               h->mesh.n[1], tot);
    count_launch();
    check_launch("hdg_curved_load_kernel");
    return;
  }
  const double len[3] = {h->mesh.hi[0] - h->mesh.lo[0], h->mesh.hi[1] - h->mesh.lo[1], h->mesh.hi[2] - h->mesh.lo[2]};
  const double c = M_PI * M_PI * (1.0 / (len[0] * len[0]) + 1.0 / (len[1] * len[1]) + 1.0 / (len[2] * len[2]));
  const int64_t total = h->n_cells * N * N * N;
  hdg_load_kernel<<<(unsigned)((total + 255) / 256), 256, 0, h->stream>>>(
      h->F, h->d1d, h->d1d + kMaxN, h->d1d + 2 * kMaxN, N, h->mesh.n[0], h->mesh.n[1], h->mesh.n[2], h->mesh.lo[0],
      h->mesh.lo[1], h->mesh.lo[2], h->h[0], h->h[1], h->h[2], c, total);
  count_launch();
  check_launch("hdg_load_kernel");
}

double dot(hdg_ctx* h, const double* x, const double* y) {
  const unsigned g = grid_for(h->n_trace);
  hdg_dot_kernel<<<g, 256, 0, h->stream>>>(x, y, h->n_trace, h->part);
  hdg_sum_kernel<<<1, 256, 0, h->stream>>>(h->part, (int)g, h->scal);
  count_launch(2);
  check_launch("hdg_dot");
  double v = 0.0;
  FEM_CUDA_TRY(cudaMemcpyAsync(&v, h->scal, sizeof(double), cudaMemcpyDeviceToHost, h->stream));
  FEM_CUDA_TRY(cudaStreamSynchronize(h->stream));
  return v;
}

}  // namespace
}  // namespace fem

using namespace fem;

extern "C" {

int hdg_setup(const fem_mesh* mesh, int32_t degree, double tau, void* stream, hdg_handle* out) {
  return hdg_guard([&] {
    if (!mesh || !out) throw Error{FEM_E_ARG, "null argument"};
    *out = nullptr;
    if (degree < 1 || degree > kMaxDeg) throw Error{FEM_E_ARG, "degree must be 1..8"};
    if (!(tau > 0.0)) throw Error{FEM_E_ARG, "tau must be positive"};
    if (mesh->geometry != FEM_GEOM_BOX || mesh->mapping_degree != 0 || mesh->kappa_amplitude != 0.0)
      throw Error{FEM_E_ARG, "HDG: box meshes (Cartesian or the deformed map) only"};
    if (mesh->nranks > 1) throw Error{FEM_E_ARG, "HDG: single rank"};
    for (int d = 0; d < 3; ++d)
      if (mesh->n[d] < 1 || !(mesh->hi[d] > mesh->lo[d])) throw Error{FEM_E_ARG, "bad mesh"};
    auto h = std::make_unique<hdg_ctx>();
    h->mesh = *mesh;
    h->k = degree;
    h->n = degree + 1;
    h->tau = tau;
    h->stream = static_cast<cudaStream_t>(stream);
    for (int d = 0; d < 3; ++d) h->h[d] = (mesh->hi[d] - mesh->lo[d]) / mesh->n[d];
    const int64_t nx = mesh->n[0], ny = mesh->n[1], nz = mesh->n[2];
    h->fx = (nx + 1) * ny * nz;
    h->fy = nx * (ny + 1) * nz;
    h->fz = nx * ny * (nz + 1);
    h->n_cells = nx * ny * nz;
    h->n_trace = (h->fx + h->fy + h->fz) * h->n * h->n;
    for (int s = 0; s < 6; ++s)
      if (mesh->bc[s] == FEM_BC_DIRICHLET) h->bc |= 1 << s;
    build_hdg_tab(degree, h->h, tau, h->tab_host);
    Tables1D t1;
    build_tables(degree, t1);
    h->tab = reinterpret_cast<HdgTab*>(hdg_alloc(kTabDoubles));
    FEM_CUDA_TRY(cudaMemcpyAsync(h->tab, &h->tab_host, sizeof(HdgTab), cudaMemcpyHostToDevice, h->stream));
    std::vector<double> d1(3 * kMaxN + kMaxN * kMaxN, 0.0);
    for (int q = 0; q < h->n; ++q) {
      d1[q] = t1.qp[q];
      d1[kMaxN + q] = t1.qw[q];
      for (int i = 0; i < h->n; ++i) d1[2 * kMaxN + q * h->n + i] = t1.val[q][i];
    }
    h->d1d = hdg_alloc((int64_t)d1.size());
    FEM_CUDA_TRY(cudaMemcpyAsync(h->d1d, d1.data(), sizeof(double) * d1.size(), cudaMemcpyHostToDevice, h->stream));
    // element diagonal by the cell kernel on unit traces, then diag(K) and its inverse
    const int NF = h->n * h->n;
    const char* dense = std::getenv("FEM_HDG_DENSE");
    h->curved = mesh->deform_eps != 0.0 || (dense && std::atoi(dense) != 0);
    h->diag = hdg_alloc(h->n_trace);
    h->dinv = hdg_alloc(h->n_trace);
    if (h->curved) {
      if (degree > 4) throw Error{FEM_E_ARG, "HDG on deformed meshes (stored local inverses): degree 1..4"};
      CurvTab ct{};
      const int n = h->n;
      for (int q = 0; q < n; ++q) {
        ct.qw[q] = t1.qw[q];
        ct.qp[q] = t1.qp[q];
        for (int i = 0; i < n; ++i) {
          ct.val[q][i] = t1.val[q][i];
          ct.der[q][i] = t1.der[q][i];
          ct.dco[q][i] = t1.colloc[q][i];
        }
      }
      invert(n, ct.val, ct.vinv);
      for (int d = 0; d < 3; ++d) {
        ct.lo[d] = mesh->lo[d];
        ct.len[d] = mesh->hi[d] - mesh->lo[d];
        ct.h[d] = h->h[d];
      }
      ct.eps = mesh->deform_eps;
      ct.tau = tau;
      h->ctab = reinterpret_cast<CurvTab*>(hdg_alloc(kCurvDoubles));
      FEM_CUDA_TRY(cudaMemcpyAsync(h->ctab, &ct, sizeof(CurvTab), cudaMemcpyHostToDevice, h->stream));
      const int64_t M = (int64_t)n * n * n;
      h->Sinv = hdg_alloc(h->n_cells * M * M);
      switch (degree) {
        case 1: curved_setup_k<1>(h.get()); break;
        case 2: curved_setup_k<2>(h.get()); break;
        case 3: curved_setup_k<3>(h.get()); break;
        default: curved_setup_k<4>(h.get()); break;
      }
      h->dc = hdg_alloc(h->n_cells * 6 * NF);
      HdgArgs a{};
      a.y = h->dc;
      launch_curved<kDiag>(h.get(), a);
      hdg_curved_diag_kernel<<<(unsigned)((h->n_trace + 255) / 256), 256, 0, h->stream>>>(
          h->diag, h->dc, h->n, mesh->n[0], mesh->n[1], mesh->n[2], h->fx, h->fy, h->bc, h->n_trace);
    } else {
      h->de = hdg_alloc(6 * NF);
      HdgArgs a{};
      a.y = h->de;
      launch_cells<kDiag>(h.get(), a);
      hdg_diag_kernel<<<(unsigned)((h->n_trace + 255) / 256), 256, 0, h->stream>>>(
          h->diag, h->de, h->n, mesh->n[0], mesh->n[1], mesh->n[2], h->fx, h->fy, h->bc, h->n_trace);
    }
    hdg_inv_kernel<<<grid_for(h->n_trace), 256, 0, h->stream>>>(h->dinv, h->diag, h->n_trace);
    count_launch(2);
    check_launch("hdg_diag");
    FEM_CUDA_TRY(cudaStreamSynchronize(h->stream));
    *out = h.release();
  });
}

int hdg_info(hdg_handle h, int64_t* n_trace, int64_t* n_cells) {
  return hdg_guard([&] {
    if (!h) throw Error{FEM_E_ARG, "null handle"};
    if (n_trace) *n_trace = h->n_trace;
    if (n_cells) *n_cells = h->n_cells;
  });
}

int hdg_apply(hdg_handle h, const double* lambda, int64_t n, double* y, int64_t ny) {
  return hdg_guard([&] {
    if (!h) throw Error{FEM_E_ARG, "null handle"};
    if (n != h->n_trace || ny != h->n_trace) throw Error{FEM_E_SIZE, "trace vectors must have n_trace entries"};
    check_dev(lambda, "lambda");
    check_dev(y, "y");
    if (lambda == y) throw Error{FEM_E_ARG, "hdg_apply: y must not alias lambda"};
    HdgArgs a{};
    a.lam = lambda;
    a.y = y;
    launch_any<kApply>(h, a);
  });
}

int hdg_diagonal(hdg_handle h, double* d, int64_t nd) {
  return hdg_guard([&] {
    if (!h) throw Error{FEM_E_ARG, "null handle"};
    if (nd != h->n_trace) throw Error{FEM_E_SIZE, "diagonal length"};
    check_dev(d, "d");
    FEM_CUDA_TRY(cudaMemcpyAsync(d, h->diag, sizeof(double) * nd, cudaMemcpyDeviceToDevice, h->stream));
  });
}

int hdg_rhs(hdg_handle h, double* r, int64_t nr) {
  return hdg_guard([&] {
    if (!h) throw Error{FEM_E_ARG, "null handle"};
    if (nr != h->n_trace) throw Error{FEM_E_SIZE, "rhs length"};
    check_dev(r, "r");
    ensure_load(h);
    HdgArgs a{};
    a.F = h->F;
    a.y = r;
    launch_any<kRhs>(h, a);
  });
}

int hdg_local_solve(hdg_handle h, const double* lambda, int64_t n, int32_t with_f, double* u, int64_t nu,
                    double* q, int64_t nq) {
  return hdg_guard([&] {
    if (!h) throw Error{FEM_E_ARG, "null handle"};
    const int64_t nc = h->n_cells * h->n * h->n * h->n;
    if (n != h->n_trace || nu != nc || (q && nq != 3 * nc)) throw Error{FEM_E_SIZE, "local solve lengths"};
    check_dev(lambda, "lambda");
    check_dev(u, "u");
    if (q) check_dev(q, "q");
    if (with_f) ensure_load(h);
    HdgArgs a{};
    a.lam = lambda;
    a.F = with_f ? h->F : nullptr;
    a.u = u;
    a.q = q;
    launch_any<kRecover>(h, a);
  });
}

int hdg_mixed_apply(hdg_handle h, const double* qu, int64_t n, double* y, int64_t ny) {
  return hdg_guard([&] {
    if (!h) throw Error{FEM_E_ARG, "null handle"};
    const int64_t nc = 4 * h->n_cells * h->n * h->n * h->n;
    if (n != nc || ny != nc) throw Error{FEM_E_SIZE, "mixed vectors must have 4 n_cells (k+1)^3 entries"};
    check_dev(qu, "qu");
    check_dev(y, "y");
    if (qu == y) throw Error{FEM_E_ARG, "hdg_mixed_apply: y must not alias qu"};
    if (h->mesh.deform_eps != 0.0) throw Error{FEM_E_ARG, "hdg_mixed_apply: Cartesian meshes only"};
    launch_mixed(h, qu, y);
  });
}

int hdg_postprocess(hdg_handle h, const double* q, int64_t nq, const double* u, int64_t nu, double* ustar,
                    int64_t nus) {
  return hdg_guard([&] {
    if (!h) throw Error{FEM_E_ARG, "null handle"};
    if (h->mesh.deform_eps != 0.0) throw Error{FEM_E_ARG, "hdg_postprocess: Cartesian meshes only"};
    if (h->k > kMaxDeg - 1) throw Error{FEM_E_ARG, "hdg_postprocess: degree 1..7 (u* has degree k+1)"};
    const int64_t n3 = (int64_t)h->n * h->n * h->n, p3 = (int64_t)(h->n + 1) * (h->n + 1) * (h->n + 1);
    if (nq != 3 * h->n_cells * n3 || nu != h->n_cells * n3 || nus != h->n_cells * p3)
      throw Error{FEM_E_SIZE, "postprocess lengths"};
    check_dev(q, "q");
    check_dev(u, "u");
    check_dev(ustar, "ustar");
    switch (h->k) {
      case 1: post_k<1>(h, q, u, ustar); break;
      case 2: post_k<2>(h, q, u, ustar); break;
      case 3: post_k<3>(h, q, u, ustar); break;
      case 4: post_k<4>(h, q, u, ustar); break;
      case 5: post_k<5>(h, q, u, ustar); break;
      case 6: post_k<6>(h, q, u, ustar); break;
      default: post_k<7>(h, q, u, ustar); break;
    }
  });
}

int hdg_cg_solve(hdg_handle h, const double* b, int64_t nb, double* x, int64_t nx, double rtol, int32_t maxit,
                 int32_t* iters, double* relres) {
  int code = FEM_OK;
  const int rc = hdg_guard([&] {
    if (!h) throw Error{FEM_E_ARG, "null handle"};
    if (nb != h->n_trace || nx != h->n_trace) throw Error{FEM_E_SIZE, "solve lengths"};
    check_dev(b, "b");
    check_dev(x, "x");
    const int64_t n = h->n_trace;
    if (!h->r) {
      h->r = hdg_alloc(n);
      h->p = hdg_alloc(n);
      h->q = hdg_alloc(n);
      h->z = hdg_alloc(n);
      h->part = hdg_alloc(148 * 8);
      h->scal = hdg_alloc(4);
    }
    const unsigned g = grid_for(n);
    HdgArgs a{};
    a.lam = x;
    a.y = h->q;
    launch_any<kApply>(h, a);   // q = K x0
    hdg_res_kernel<<<g, 256, 0, h->stream>>>(h->r, h->z, b, h->q, h->dinv, n);
    hdg_axpy_kernel<<<g, 256, 0, h->stream>>>(h->p, h->z, 0.0, n);
    count_launch(2);
    const double nb2 = std::sqrt(dot(h, b, b));
    double rz = dot(h, h->r, h->z);
    double rel = nb2 > 0 ? std::sqrt(dot(h, h->r, h->r)) / nb2 : 0.0;
    int it = 0;
    while (rel > rtol && it < maxit) {
      a.lam = h->p;
      a.y = h->q;
      launch_any<kApply>(h, a);
      const double pq = dot(h, h->p, h->q);
      if (!(pq > 0.0)) throw Error{FEM_E_BREAKDOWN, "hdg_cg_solve: p^T K p <= 0 at iteration " + std::to_string(it)};
      const double alpha = rz / pq;
      hdg_upd_kernel<<<g, 256, 0, h->stream>>>(x, h->r, h->z, h->p, h->q, h->dinv, alpha, n);
      count_launch();
      ++it;
      rel = std::sqrt(dot(h, h->r, h->r)) / nb2;
      if (rel <= rtol) break;
      const double rzn = dot(h, h->r, h->z);
      hdg_axpy_kernel<<<g, 256, 0, h->stream>>>(h->p, h->z, rzn / rz, n);
      count_launch();
      rz = rzn;
    }
    check_launch("hdg_cg_solve");
    if (iters) *iters = it;
    if (relres) *relres = rel;
    if (rel > rtol) code = FEM_NOT_CONVERGED;
  });
  return rc != FEM_OK ? rc : code;
}

void hdg_destroy(hdg_handle h) {
  if (!h) return;
  for (double* p : {reinterpret_cast<double*>(h->tab), h->de, h->diag, h->dinv, h->F, h->ydiag, h->r, h->p, h->q,
                    h->z, h->part, h->scal, h->d1d, reinterpret_cast<double*>(h->ctab), h->Sinv, h->dc})
    if (p) cudaFree(p);
  delete h;
}

}  // extern "C"
