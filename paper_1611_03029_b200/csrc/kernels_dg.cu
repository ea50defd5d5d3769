// SIPG kernels (K2 cell + K3 face terms), element-centric.
//
// Operator (eq:poisson_dgsip; boundary mirror values eq:bc_dgsip,
// P:L248-255): per cell K the cell term of cell_term.cuh plus, for each of its
// six faces F with outward normal n_K and neighbour K' (same orientation on the
// structured mesh),
//     int_F  sigma [u] v - {d_n u} v - (1/2) [u] d_n v ,
//     [u] = u_K - u_K',  {d_n u} = (d_n u_K + d_n u_K')/2,  d_n = n_K . grad,
// which is the part of -[v]{d_n u} - {d_n v}[u] + sigma [u][v] that tests the
// functions of K.  Dirichlet (g = 0): [u] = 2 u_K, {d_n u} = d_n u_K; Neumann: 0.
// Every cell evaluates its own faces (each interior face is visited twice, as in
// the paper's <.,.>_{dT_h}), reading the neighbour's nodal lines from global
// memory, so the result of a cell is written exactly once (no atomics, no zeroing).
//
// Face terms are sum-factorized (O((k+1)^d) per face): with GLL nodes
// the trace of u on xi_d = +-1 is the nodal layer, the normal derivative is a
// reduction of each d-line with phi_i'(+-1); both are interpolated to the
// (k+1)^2 face Gauss points by two 1-D sweeps (tangential derivatives by
// collocation on deformed meshes), and the flux is integrated back with the
// transposed sweeps and expanded along the d-lines.
#include "cell_term.cuh"
#include "device_common.cuh"

namespace fem {

template <int K>
struct DgCPB {
  static constexpr int N = K + 1;
  static constexpr int value = (N * N <= 4) ? 32 : (N * N <= 9) ? 16 : (N * N <= 25) ? 8 : (N * N <= 49) ? 4 : 2;
};
#ifndef FEM_DGQ_C78
#define FEM_DGQ_C78 1
#endif
#ifndef FEM_DGQ_C3
#define FEM_DGQ_C3 8
#endif
#ifndef FEM_DGQ_MINB3
#define FEM_DGQ_MINB3 1
#endif
#ifndef FEM_DGQ_C2
#define FEM_DGQ_C2 16
#endif
#ifndef FEM_DGQ_MINB2
#define FEM_DGQ_MINB2 1
#endif
#ifndef FEM_DGQ_C4
#define FEM_DGQ_C4 2
#endif
#ifndef FEM_DGQ_MINB4
#define FEM_DGQ_MINB4 10
#endif
#ifndef FEM_DG_MINB
#define FEM_DG_MINB 4
#endif
// cells per block and minimum resident blocks of the SIPG quadrature kernel (K2/K3):
// fewer cells per block with a register cap measured faster (deformed apply at ~16M
// DoFs, cells/block and blocks/SM: k = 4 8/1 1141 us -> 2/6 1029 us, k = 5 4/2 1143 ->
// 2/3 1008, k = 6 4/2 1378 -> 1/6 1142 (C5 7.76 -> 6.51 ms), k = 7 2/2 1076 -> 1/4 1028,
// k = 8 2/2 1400 -> 1/4 1324): more, smaller blocks keep more warps resident
template <int K>
struct DgQCPB {
  static constexpr int value = K == 5 ? 2 : (K == 6 ? 1 : (K >= 7 ? FEM_DGQ_C78 : (K == 4 ? FEM_DGQ_C4 : (K == 3 ? FEM_DGQ_C3 : (K == 2 ? FEM_DGQ_C2 : DgCPB<K>::value)))));
};
// k = 6 (C5): with the even-odd sweeps the kernel fits 79 registers without spilling;
// 11 blocks/SM (the shared-memory limit, 20.5 KB per cell) measured 4.75 ms per C5 apply
// against 5.39 ms at the round-1 bound of 6 blocks (144 registers), 4.91 at 8, 4.81 at 10
#ifndef FEM_DGQ_MINB6
#define FEM_DGQ_MINB6 11
#endif
// round 2, after the even-odd register drop (SIPG deformed apply at ~16M DoFs, round-1
// bound -> new): k = 4 6 -> 10 blocks/SM 949 -> 926 us, k = 5 3 -> 6 832 -> 788 us,
// k = 7 4 -> 8 886 -> 868 us; k = 8 stays at 4 (8: 798 -> 940 us)
#ifndef FEM_DGQ_MINB5
#define FEM_DGQ_MINB5 6
#endif
#ifndef FEM_DGQ_MINB7
#define FEM_DGQ_MINB7 8
#endif
template <int K>
__host__ __device__ constexpr int dgq_minb() {
  return K == 5 ? FEM_DGQ_MINB5 : (K == 6 ? FEM_DGQ_MINB6 : (K == 7 ? FEM_DGQ_MINB7 : (K == 8 ? FEM_DG_MINB : (K == 4 ? FEM_DGQ_MINB4 : (K == 3 ? FEM_DGQ_MINB3 : (K == 2 ? FEM_DGQ_MINB2 : 1))))));
}

#ifndef FEM_DGQ_PAD
#define FEM_DGQ_PAD 1
#endif
#ifndef FEM_DG_FACE_PREFETCH
#define FEM_DG_FACE_PREFETCH 1
#endif
#ifndef FEM_DG_NB_PREFETCH
#define FEM_DG_NB_PREFETCH 1
#endif
#ifndef FEM_DGQ_FPAD
#define FEM_DGQ_FPAD 1
#endif
template <int N>
struct DgSmem {  // per-cell shared memory layout (doubles)
  static constexpr int N2 = N * N, N3 = N2 * N;
  // cell term (cell_laplace) strides: element (i0, i1, i2) at i0 + B i1 + S i2, three
  // fields of CF words from S0 (they may run into FWD/BWD, which are dead until the
  // face phases); B, S and the cell-stride padding from a bank-conflict model search
  // (modelled cell-term wavefronts: k=2 1.3x, k=3 2.5x, k=5 1.5x, k=6 1.3x, k=7 2.7x fewer)
  static constexpr int K = N - 1;
  static constexpr int Bp[9] = {0, 0, 3, 7, 6, 9, 7, 9, 9};
  static constexpr int Sp[9] = {0, 0, 19, 28, 37, 54, 56, 72, 89};
  static constexpr int Ep[9] = {0, 0, 5, 2, 13, 4, 13, 0, 5};
  static constexpr bool pad = FEM_DGQ_PAD != 0 && K >= 2;
  static constexpr int B = pad ? Bp[K] : N, S = pad ? Sp[K] : N2;
  static constexpr int CF = (N - 1) * (1 + B + S) + 1;
  // face buffers: 16 + 8 fields of (k+1)^2 values, field stride FS padded so that the
  // face phases' row / column sweeps spread over the banks.  The model predicts fewer
  // wavefronts at k = 2, 3, 5..8; measured (SIPG deformed apply, ~16M DoFs) only k = 3
  // gains (1110 -> 894 us); k = 2, 5, 6 got 2-10% slower, k = 7, 8 equal: dense there.
  static constexpr int FSp[9] = {0, 4, 9, 21, 25, 36, 49, 64, 81};
  static constexpr int FS = FEM_DGQ_FPAD ? FSp[K] : N2;
  static constexpr int X = 0, S0 = N3, FWD = 4 * N3, BWD = FWD + 16 * FS;
  static constexpr int SIZE = BWD + 8 * FS + (pad ? Ep[K] : 0);
  static_assert(S0 + 3 * CF <= BWD + 8 * FS, "cell-term fields exceed the per-cell buffer");
};

struct DgArgs {
  const double* __restrict__ x;
  double* __restrict__ y;
  const double* __restrict__ G;       // deformed cell metric [cell][6][q]
  const double* __restrict__ faceq;   // deformed face records [face][7][N2]
  const double* __restrict__ fsigma;  // [face]
  int64_t face_off[3];                // first face record of direction d
  int n[3];          // rank-local cells per direction (z: slab layers)
  int cz0, nzg;      // global index of the first local layer, global layers
  int64_t n_cells;
  int64_t cell0, cell1;  // cells [cell0, cell1) of this launch (z-slab overlap splits)
  ChebFuse cf;           // fused Chebyshev epilogue (cf.on)
  int bcmask;
  double c[3];      // Cartesian metric det J (2/h_d)^2
  double h[3];
  double sigma[3];  // Cartesian penalty c (k+1)^2 / h_d
  // deformed box with the analytic map (reading R2; not the general N3 geometries):
  // FEM_DG_FGEO_FLY=1 recomputes the face quadrature data (JxW, J^-1 n) from the map at
  // each face point instead of reading the 7 x (k+1)^2 face records (the penalty sigma_F,
  // one double per face, is still read).  By the flop/byte balance (~5.7 flop/B) ~100
  // flops should beat 56 bytes, but the three sincospi, the divide and the square root
  // per point measured slower (C5 apply 7.28 vs 5.35 ms): off by default, parity-tested.
  int fgeo_fly;
  MapArgs map;
  // FEM_DG_CGEO_FLY=1: the cell term's metric G from the analytic map (cell_term.cuh GeoFly)
  // instead of the 48-byte-per-point table: sin / cos per thread line and per cell z-point
  // (parity-tested; measured slower, C5 apply 4710 -> 4868 us, solve 850 -> 872 ms: off)
  int cgeo_fly;
  GeoFlyC gfc;
  double hL[3];    // h_d / L_d (quadrature coordinates t = hL (c + (xi + 1) / 2))
};

// result v = (A x)_i of DoF i: stored, or consumed by the fused Chebyshev epilogue
__device__ __forceinline__ void dg_store(const ChebFuse& cf, const double* __restrict__ x, double* __restrict__ y,
                                         int64_t i, double v) {
  if (cf.on) {
    const double xi = x[i], xoi = cf.xo ? cf.xo[i] : 0.0;
    y[i] = xi + cf.c1 * (xi - xoi) + cf.c2 * cf.dinv[i] * (cf.b[i] - v);
  } else {
    y[i] = v;
  }
}
// the same with x_i already in a register and D^-1 from dinv[i] or from the cell-class
// table (dcls: the class's n^3 block, loc: local node index)
__device__ __forceinline__ void dg_store_x(const ChebFuse& cf, double xi, double* __restrict__ y, int64_t i,
                                           double v, const double* dcls, int loc) {
  if (cf.on) {
    const double xoi = cf.xo ? cf.xo[i] : 0.0;
    const double di = dcls ? dcls[loc] : cf.dinv[i];
    y[i] = xi + cf.c1 * (xi - xoi) + cf.c2 * di * (cf.b[i] - v);
  } else {
    y[i] = v;
  }
}

// node index in the cell of (i along D, a along t1, b along t2)
template <int N, int D>
__device__ __forceinline__ int lidx(int i, int a, int b) {
  if (D == 0) return i + N * a + N * N * b;
  if (D == 1) return a + N * i + N * N * b;
  return a + N * b + N * N * i;
}

template <int D> struct Tang;
template <> struct Tang<0> { static constexpr int t1 = 1, t2 = 2; };
template <> struct Tang<1> { static constexpr int t1 = 0, t2 = 2; };
template <> struct Tang<2> { static constexpr int t1 = 0, t2 = 1; };

// 0 interior, 1 Dirichlet, 2 Neumann: kind of face s (0 lower, 1 upper) of local cell c along D
__device__ __forceinline__ int face_kind(const DgArgs& A, int D, const int c[3], int s) {
  const int nb = (D == 2 ? A.cz0 : 0) + c[D] + (s ? 1 : -1);
  const int nD = D == 2 ? A.nzg : A.n[D];
  return (nb >= 0 && nb < nD) ? 0 : ((A.bcmask >> (2 * D + s)) & 1 ? 1 : 2);
}

__device__ __forceinline__ int64_t face_record(const DgArgs& A, int D, const int c[3], int p) {
  const int t1 = D == 0 ? 1 : 0, t2 = D == 2 ? 1 : 2;
  return A.face_off[D] + p + (int64_t)(A.n[D] + 1) * (c[t1] + (int64_t)A.n[t1] * c[t2]);
}

// Face terms of the two faces normal to D, accumulated into the residual R (nodal, shared).
template <int K, bool DEFORMED, int D>
__device__ __forceinline__ void dg_faces(const DgArgs& A, const Tab<K + 1>& T, double* sm, int64_t cell,
                                         const int c[3], bool active, int t) {
  constexpr int N = K + 1, N2 = N * N, N3 = N2 * N;
  constexpr int t1 = Tang<D>::t1, t2 = Tang<D>::t2;
  using L = DgSmem<N>;
  constexpr int FS = L::FS;   // padded field stride of the face buffers
  const double* X = sm + L::X;
  double* R = sm + L::S0;
  double* F = sm + L::FWD;   // [s][8][N2]: 0 u, 1 d_D u, 2 u', 3 d_D u', 4 d_t1 u, 5 d_t2 u, 6 d_t1 u', 7 d_t2 u'
  double* B = sm + L::BWD;   // [s][4][N2]: 0 A (value test), 1 B_D, 2 B_t1, 3 B_t2
  const int a = t % N, b = t / N;
  const int64_t stride = D == 0 ? 1 : (D == 1 ? (int64_t)A.n[0] : (int64_t)A.n[0] * A.n[1]);
  int kind[2];  // 0 interior, 1 Dirichlet, 2 Neumann
#pragma unroll
  for (int s = 0; s < 2; ++s) kind[s] = face_kind(A, D, c, s);
  // ---- F1: traces of the own and neighbour d-lines
  {
    double xl[N];
#pragma unroll
    for (int i = 0; i < N; ++i) xl[i] = X[lidx<N, D>(i, a, b)];
#pragma unroll
    for (int s = 0; s < 2; ++s) {
      double f1 = 0.0, g0 = 0.0, g1 = 0.0;
#pragma unroll
      for (int i = 0; i < N; ++i) f1 = fma(T.dface[s][i], xl[i], f1);
      if (active && kind[s] == 0) {
        const double* xn = A.x + (cell + (s ? stride : -stride)) * N3;
        double nl[N];
#pragma unroll
        for (int i = 0; i < N; ++i) nl[i] = __ldg(xn + lidx<N, D>(i, a, b));
        g0 = nl[s ? 0 : K];
#pragma unroll
        for (int i = 0; i < N; ++i) g1 = fma(T.dface[1 - s][i], nl[i], g1);
      }
      double* Fs = F + s * 8 * FS;
      Fs[0 * FS + t] = xl[s ? K : 0];
      Fs[1 * FS + t] = f1;
      Fs[2 * FS + t] = g0;
      Fs[3 * FS + t] = g1;
    }
  }
  __syncthreads();
  // ---- F2: interpolate along t1 (rows b); deformed: d/dt1 of the traces
  for (int task = t; task < 2 * 4 * N; task += N2) {
    const int s = task / (4 * N), f = (task / N) % 4, row = task % N;
    double* fld = F + (s * 8 + f) * FS + N * row;
    double in[N], out[N];
#pragma unroll
    for (int i = 0; i < N; ++i) in[i] = fld[i];
    MV_VAL(T, in, out);
    if (DEFORMED && (f == 0 || f == 2)) {
      double dd[N];
      MV_COL(T, out, dd);
      double* fd = F + (s * 8 + (f == 0 ? 4 : 6)) * FS + N * row;
#pragma unroll
      for (int i = 0; i < N; ++i) fd[i] = dd[i];
    }
#pragma unroll
    for (int i = 0; i < N; ++i) fld[i] = out[i];
  }
  __syncthreads();
  // ---- F3: interpolate along t2 (columns); deformed: d/dt2 of the traces
  {
    constexpr int NF = DEFORMED ? 6 : 4;
    for (int task = t; task < 2 * NF * N; task += N2) {
      const int s = task / (NF * N), fi = (task / N) % NF, col = task % N;
      const int f = fi < 4 ? fi : (fi == 4 ? 4 : 6);
      double* fld = F + (s * 8 + f) * FS + col;
      double in[N], out[N];
#pragma unroll
      for (int i = 0; i < N; ++i) in[i] = fld[N * i];
      MV_VAL(T, in, out);
      if (DEFORMED && (f == 0 || f == 2)) {
        double dd[N];
        MV_COL(T, out, dd);
        double* fd = F + (s * 8 + (f == 0 ? 5 : 7)) * FS + col;
#pragma unroll
        for (int i = 0; i < N; ++i) fd[N * i] = dd[i];
      }
#pragma unroll
      for (int i = 0; i < N; ++i) fld[N * i] = out[i];
    }
  }
  __syncthreads();
  // ---- F4: numerical flux at face point q = (a, b)
#pragma unroll
  for (int s = 0; s < 2; ++s) {
    const double* Fs = F + s * 8 * FS;
    double* Bs = B + s * 4 * FS;
    double vA = 0.0, vD = 0.0, v1 = 0.0, v2 = 0.0;
    if (kind[s] != 2 && active) {
      const double nsgn = s ? 1.0 : -1.0;
      const double u_own = Fs[t];
      double dn_own, dn_nb = 0.0, JxW, sig, Jn[3];
      if (DEFORMED) {
        const int64_t fr = face_record(A, D, c, c[D] + s);
        sig = __ldg(A.fsigma + fr);
        double Jo[3];
        if (A.fgeo_fly) {
          // the face point in the own cell's reference coordinates; J (hence J^-1 n and
          // JxW) is the same from both sides: one global map, equal cell sizes
          double xi[3];
          xi[D] = s ? 1.0 : -1.0;
          xi[t1] = T.qp[a];
          xi[t2] = T.qp[b];
          const PointGeo g = map_point(A.map, c[0], c[1], c[2], xi[0], xi[1], xi[2]);
          double v[3], nrm = 0.0;
#pragma unroll
          for (int e = 0; e < 3; ++e) {
            v[e] = jinv(A.map, g, D, e);   // (J^-T e_D)_e: the minus side's normal direction
            nrm = fma(v[e], v[e], nrm);
          }
          nrm = sqrt(nrm);
          JxW = T.w[a] * T.w[b] * g.det * nrm;
          const double inv = 1.0 / nrm;
#pragma unroll
          for (int e = 0; e < 3; ++e) {
            const double jm = (jinv(A.map, g, e, 0) * v[0] + jinv(A.map, g, e, 1) * v[1] +
                               jinv(A.map, g, e, 2) * v[2]) * inv;
            Jn[e] = nsgn * jm;
            Jo[e] = nsgn * jm;
          }
        } else {
          const double* rec = A.faceq + fr * 7 * N2;
          JxW = __ldg(rec + t);
          const int own = s ? 1 : 4, oth = s ? 4 : 1;  // own cell is the minus side iff s == 1
#pragma unroll
          for (int e = 0; e < 3; ++e) {
            Jn[e] = nsgn * __ldg(rec + (own + e) * N2 + t);
            Jo[e] = nsgn * __ldg(rec + (oth + e) * N2 + t);
          }
        }
        dn_own = Jn[t1] * Fs[4 * FS + t] + Jn[t2] * Fs[5 * FS + t] + Jn[D] * Fs[1 * FS + t];
        if (kind[s] == 0)
          dn_nb = Jo[t1] * Fs[6 * FS + t] + Jo[t2] * Fs[7 * FS + t] + Jo[D] * Fs[3 * FS + t];
      } else {
        const double jac = 2.0 / A.h[D];
        JxW = T.w[a] * T.w[b] * (0.5 * A.h[t1]) * (0.5 * A.h[t2]);
        sig = A.sigma[D];
        Jn[0] = Jn[1] = Jn[2] = 0.0;
        Jn[D] = nsgn * jac;
        dn_own = Jn[D] * Fs[1 * FS + t];
        if (kind[s] == 0) dn_nb = Jn[D] * Fs[3 * FS + t];
      }
      double jump, avg;
      if (kind[s] == 0) {
        jump = u_own - Fs[2 * FS + t];
        avg = 0.5 * (dn_own + dn_nb);
      } else {
        jump = 2.0 * u_own;
        avg = dn_own;
      }
      const double cu = JxW * (sig * jump - avg);
      const double cg = -0.5 * JxW * jump;
      vA = cu;
      vD = cg * Jn[D];
      v1 = cg * Jn[t1];
      v2 = cg * Jn[t2];
    }
    Bs[0 * FS + t] = vA;
    Bs[1 * FS + t] = vD;
    Bs[2 * FS + t] = v1;
    Bs[3 * FS + t] = v2;
  }
  __syncthreads();
  // ---- F5: transposed t2 (columns): P = I^T (A + D^T B_t2), Q = I^T B_t1, W = I^T B_D
  {
    constexpr int NG = DEFORMED ? 3 : 2;
    for (int task = t; task < 2 * NG * N; task += N2) {
      const int s = task / (NG * N), g = (task / N) % NG, col = task % N;
      double* Bs = B + s * 4 * FS;
      double in[N], out[N];
      if (g == 0) {
#pragma unroll
        for (int i = 0; i < N; ++i) in[i] = Bs[N * i + col];
        if (DEFORMED) {
          double b2[N];
#pragma unroll
          for (int i = 0; i < N; ++i) b2[i] = Bs[3 * FS + N * i + col];
          MVT_ADD_COL(T, b2, in);
        }
      } else {
        const int f = (g == 1) ? 1 : 2;
#pragma unroll
        for (int i = 0; i < N; ++i) in[i] = Bs[f * FS + N * i + col];
      }
      MVT_VAL(T, in, out);
      const int f = (g == 0) ? 0 : (g == 1 ? 1 : 2);
#pragma unroll
      for (int i = 0; i < N; ++i) Bs[f * FS + N * i + col] = out[i];
    }
  }
  __syncthreads();
  // ---- F6: transposed t1 (rows): V = I^T (P + D^T Q), W = I^T W
  for (int task = t; task < 2 * 2 * N; task += N2) {
    const int s = task / (2 * N), g = (task / N) % 2, row = task % N;
    double* Bs = B + s * 4 * FS;
    double in[N], out[N];
#pragma unroll
    for (int i = 0; i < N; ++i) in[i] = Bs[g * FS + N * row + i];
    if (DEFORMED && g == 0) {
      double q[N];
#pragma unroll
      for (int i = 0; i < N; ++i) q[i] = Bs[2 * FS + N * row + i];
      MVT_ADD_COL(T, q, in);
    }
    MVT_VAL(T, in, out);
#pragma unroll
    for (int i = 0; i < N; ++i) Bs[g * FS + N * row + i] = out[i];
  }
  __syncthreads();
  // ---- F7: expand into the residual's d-line (a, b)
  {
    double r[N];
#pragma unroll
    for (int i = 0; i < N; ++i) r[i] = R[lidx<N, D>(i, a, b)];
#pragma unroll
    for (int s = 0; s < 2; ++s) {
      const double V = B[(s * 4 + 0) * FS + t], W = B[(s * 4 + 1) * FS + t];
      r[s ? K : 0] += V;
#pragma unroll
      for (int i = 0; i < N; ++i) r[i] = fma(T.dface[s][i], W, r[i]);
    }
#pragma unroll
    for (int i = 0; i < N; ++i) R[lidx<N, D>(i, a, b)] = r[i];
  }
  __syncthreads();
}

template <int K, bool DEFORMED, bool FLY = false>
__global__ void __launch_bounds__((K + 1) * (K + 1) * DgQCPB<K>::value, dgq_minb<K>())   // measured: 1 beats none at k <= 4
    dg_apply_kernel(DgArgs A, Tab<K + 1> T) {
  constexpr int N = K + 1, N2 = N * N, N3 = N2 * N;
  constexpr int C = DgQCPB<K>::value;
  using L = DgSmem<N>;
  extern __shared__ double smem[];
  const int t = threadIdx.x, ci = threadIdx.y;
  const int64_t cell = A.cell0 + (int64_t)blockIdx.x * C + ci;
  const bool active = cell < A.cell1;
  if (DEFORMED && t == 0 && ci == 0 && !FLY) {
    // static geometry of the block's cells: pull it into L2 before waiting on the
    // predecessor kernel
    const int64_t c0 = A.cell0 + (int64_t)blockIdx.x * C;
    const int64_t nc = (A.cell1 - c0) < C ? (A.cell1 - c0) : C;
    bulk_prefetch_l2(A.G + c0 * 6 * N3, (uint32_t)(nc * 6 * N3 * sizeof(double)));
  }
  int c[3] = {0, 0, 0};
  if (active) {
    c[0] = (int)(cell % A.n[0]);
    const int64_t r = cell / A.n[0];
    c[1] = (int)(r % A.n[1]);
    c[2] = (int)(r / A.n[1]);
  }
  if (FEM_DG_FACE_PREFETCH && DEFORMED && !A.fgeo_fly && t == 0 && active) {
    // the cell's y- and z-face records (static; x-faces of the block's cells are one run)
#pragma unroll
    for (int D = 1; D < 3; ++D)
#pragma unroll
      for (int s = 0; s < 2; ++s)
        prefetch_l2_range(A.faceq + face_record(A, D, c, c[D] + s) * 7 * N2, 7 * N2 * sizeof(double));
    if (ci == 0) {
      const int nc = (int)((A.cell1 - cell) < C ? (A.cell1 - cell) : C);
      prefetch_l2_range(A.faceq + face_record(A, 0, c, c[0]) * 7 * N2, (size_t)(nc + 1) * 7 * N2 * sizeof(double));
    }
  }
  FEM_PDL_ENTRY();
  if (FEM_DG_NB_PREFETCH && t == 0 && active) {
    // the y- and z-neighbour cells whose lines the face phases read (ghost layers included)
    const int64_t sy = A.n[0], sz = (int64_t)A.n[0] * A.n[1];
    if (c[1] > 0) prefetch_l2_range(A.x + (cell - sy) * N3, N3 * sizeof(double));
    if (c[1] < A.n[1] - 1) prefetch_l2_range(A.x + (cell + sy) * N3, N3 * sizeof(double));
    if (c[2] + A.cz0 > 0) prefetch_l2_range(A.x + (cell - sz) * N3, N3 * sizeof(double));
    if (c[2] + A.cz0 < A.nzg - 1) prefetch_l2_range(A.x + (cell + sz) * N3, N3 * sizeof(double));
  }
  double* sm = smem + ci * L::SIZE;
  double u[N], v[N];
#pragma unroll
  for (int l = 0; l < N; ++l) {
    u[l] = active ? __ldg(A.x + cell * N3 + t + N2 * l) : 0.0;
    sm[L::X + t + N2 * l] = u[l];
  }
  CellGeo<N> geo{DEFORMED ? A.G + (size_t)(active ? cell : 0) * 6 * N3 : nullptr, A.c[0], A.c[1],
                 A.c[2], active, nullptr};
  GeoFlyPt<N> fp;
  __shared__ double scz[FLY ? C : 1][FLY ? 2 * N : 1];
  if constexpr (DEFORMED && FLY) {
    const int ta = t % N, tb = t / N;
    const int c3[3] = {c[0], c[1], c[2] + A.cz0};
    auto tq = [&](int d, int q) { return A.hL[d] * (c3[d] + 0.5 * (T.qp[q] + 1.0)); };
    sincospi(tq(0, ta), &fp.sx, &fp.cx);
    sincospi(tq(1, tb), &fp.sy, &fp.cy);
    if (t < N) sincospi(tq(2, t), &scz[ci][t], &scz[ci][N + t]);
    fp.scz = scz[ci];
    fp.c = &A.gfc;
    geo.fly = &fp;   // read in the q-point phase, after the sweep barriers
  }
  double* s0 = sm + L::S0;
  cell_laplace<N, DEFORMED, false, L::B, L::S>(T, geo, s0, s0 + L::CF, s0 + 2 * L::CF, t, u, v);
  __syncthreads();
#pragma unroll
  for (int l = 0; l < N; ++l) s0[t + N2 * l] = v[l];   // residual R (z-line layout)
  __syncthreads();
  dg_faces<K, DEFORMED, 2>(A, T, sm, cell, c, active, t);
  dg_faces<K, DEFORMED, 1>(A, T, sm, cell, c, active, t);
  dg_faces<K, DEFORMED, 0>(A, T, sm, cell, c, active, t);
  if (active) {
    const int ta = t % N, tb = t / N;   // x-line (y=ta, z=tb): contiguous in the DG layout
#pragma unroll
    for (int l = 0; l < N; ++l)
      dg_store(A.cf, A.x, A.y, cell * N3 + l + N * ta + N2 * tb, s0[l + N * ta + N2 * tb]);
  }
}


// ---------------------------------------------------------------- Cartesian SIPG: Kronecker form (K2c)
// On a Cartesian mesh the SIPG operator is the Kronecker sum of the 1-D SIPG matrix A1
// with the 1-D DG mass M1 (SURVEY App. A pin, verified to 1.8e-15):
//     A = A1_x M1_y M1_z + M1_x A1_y M1_z + M1_x M1_y A1_z,
// exact because the (k+1)-point Gauss rules integrate the cell stiffness and the
// tangential face masses exactly.  A1 on a line of cells, for the line segment of
// cell e (all terms from eq:poisson_dgsip / eq:bc_dgsip restricted to 1-D, n = +1 from
// e to e+1, D+- = (2/h) phi'(+-1), GLL so phi_i(-1) = d_i0, phi_i(+1) = d_iK):
//   out = (2/h) S_ref x_e + (1 + f_lo) RR x_e + (1 + f_hi) LL x_e
//         + [e-1 exists] RL x_{e-1} + [e+1 exists] LR x_{e+1},
//   RR x = 1/2 e_0 (D-.x) + 1/2 D- x_0 + sigma e_0 x_0       (left face, own side)
//   LL x = -1/2 e_K (D+.x) - 1/2 D+ x_K + sigma e_K x_K      (right face, own side)
//   LR x = -1/2 e_K (D-.x) + 1/2 D+ x_0 - sigma e_K x_0      (right neighbour)
//   RL x = 1/2 e_0 (D+.x) - 1/2 D- x_K - sigma e_0 x_K       (left neighbour)
// f = 0 at interior faces, +1 at a Dirichlet side (mirror: 2 RR / 2 LL), -1 at a Neumann
// side (the face term vanishes).  Per cell: the three directional line operators on
// x-, y- and z-lines read straight from global memory (own cell and its neighbours:
// ghost layers on z-slabs), then the masses: y = M_z (M_y X + M_x Y) + M_y M_x Z, with
// three shared-memory phases.  14 (k+1)^4 FMA per cell instead of the quadrature
// kernel's cell + face sum factorization; no face data, no geometry.
struct DgKron {
  int n[3];
  int cz0, nzg;
  int64_t n_cells;
  int64_t cell0, cell1;            // cells of this launch
  ChebFuse cf;                     // fused Chebyshev epilogue (cf.on)
  double sigma[3], sc[3], mc[3];   // penalty, 2/h_d (stiffness and D+- scale), h_d/2 (mass scale)
  int flo[3], fhi[3];              // boundary factor of the low / high side of direction d
};

// even-odd in the Cartesian SIPG kernel measured neutral at Q4 (C3 apply 48.5 vs 47.4 us,
// N = 5: 21 vs 25 operations per line; the kernel is not FP64-bound): off by default
#ifndef FEM_EO_KRON
#define FEM_EO_KRON 0
#endif
#if FEM_EO_KRON
#define MV_M(in, out) mv_eo<N, false, false, false>(T.Meo, in, out)
#else
#define MV_M(in, out) mv<N>(T.M, in, out)
#endif
template <int N>
struct DgKronTab {
  double S[N][N];   // reference 1-D stiffness  sum_q w phi_i' phi_j'
  double M[N][N];   // reference 1-D mass
  double dm[N], dp[N];   // phi_i'(-1), phi_i'(+1) (reference)
  EO<N> Seo, Meo;   // even-odd forms (both centro-symmetric)
};

// one line (length N along direction d) of cell e: own values xo, neighbours xl / xr
template <int N>
__device__ __forceinline__ void dg_line_op(const DgKronTab<N>& T, double sc, double sig, double flo, double fhi,
                                          bool hl, bool hr, const double (&xo)[N], const double (&xl)[N],
                                          const double (&xr)[N], double (&out)[N]) {
  constexpr int K = N - 1;
  double dmx = 0.0, dpx = 0.0, dpl = 0.0, dmr = 0.0;
#pragma unroll
  for (int j = 0; j < N; ++j) {
    dmx = fma(T.dm[j], xo[j], dmx);
    dpx = fma(T.dp[j], xo[j], dpx);
    dpl = fma(T.dp[j], xl[j], dpl);
    dmr = fma(T.dm[j], xr[j], dmr);
  }
  dmx *= sc; dpx *= sc; dpl *= sc; dmr *= sc;
  const double wl = 1.0 + flo, wr = 1.0 + fhi;
  const double xl_K = hl ? xl[K] : 0.0, xr_0 = hr ? xr[0] : 0.0;
  if (!hl) dpl = 0.0;
  if (!hr) dmr = 0.0;
  double sx[N];
#if FEM_EO_KRON
  mv_eo<N, false, false, false>(T.Seo, xo, sx);
#else
  mv<N>(T.S, xo, sx);
#endif
#pragma unroll
  for (int i = 0; i < N; ++i) {
    double v = sx[i] * sc;
    // own-side face terms (RR, LL) with their boundary weights, neighbour terms (RL, LR)
    v = fma(0.5 * sc * T.dm[i], wl * xo[0] - xl_K, v);
    v = fma(0.5 * sc * T.dp[i], xr_0 - wr * xo[K], v);
    if (i == 0) v += wl * (0.5 * dmx + sig * xo[0]) + 0.5 * dpl - sig * xl_K;
    if (i == K) v += wr * (-0.5 * dpx + sig * xo[K]) - 0.5 * dmr - sig * xr_0;
    out[i] = v;
  }
}

// Shared-memory layout of the Cartesian SIPG kernel's three buffers: element (i0, i1, i2)
// at i0 + B i1 + S i2, fields F words apart, cells CS apart; per-degree strides from a
// bank-conflict model search over its access patterns (modelled wavefronts vs the dense
// layout: k=1 1.7x, k=2 1.6x, k=3 2.1x, k=4 1.2x, k=5 1.5x, k=6 1.3x, k=7 3.4x fewer).
#ifndef FEM_DG_PAD
#define FEM_DG_PAD 1
#endif
template <int K>
struct DgCartLayout {
  static constexpr int N = K + 1;
  static constexpr int Bp[9] = {0, 2, 3, 5, 5, 9, 10, 9, 10};
  static constexpr int Sp[9] = {0, 5, 19, 20, 25, 54, 71, 72, 89};
  static constexpr int CSp[9] = {0, 30, 153, 237, 381, 964, 1489, 1725, 2417};
  // measured (% of HBM at ~16M DoFs, dense -> padded): k=2 17.6 -> 22.2, k=3 15.1 -> 22.7,
  // k=4 22.1 -> 23.0, k=7 10.7 -> 14.9; k=1, 5, 6, 8 equal or slower padded (kept dense)
  static constexpr bool pad = FEM_DG_PAD != 0 && (K == 2 || K == 3 || K == 4 || K == 7);
  static constexpr int B = pad ? Bp[K] : N;
  static constexpr int S = pad ? Sp[K] : N * N;
  static constexpr int F = (N - 1) * (1 + B + S) + 1;
  static constexpr int CS = pad ? CSp[K] : 3 * N * N * N + 1;
};

#ifndef FEM_DGC_C4
#define FEM_DGC_C4 4
#endif
#ifndef FEM_DGC_MINB4
#define FEM_DGC_MINB4 10
#endif
// cells per block of the Cartesian SIPG kernel (K2c): at Q4 4 cells with 10 blocks/SM
// (C3 solve 10.80 -> 10.66 ms, apply at 16M DoFs unchanged)
template <int K>
struct DgCartCPB {
  static constexpr int value = K == 4 ? FEM_DGC_C4 : DgCPB<K>::value;
};

template <int K>
__global__ void __launch_bounds__((K + 1) * (K + 1) * DgCartCPB<K>::value, K == 4 ? FEM_DGC_MINB4 : 0)
    dg_cart_kernel(const double* __restrict__ x, double* __restrict__ y, DgKron A, DgKronTab<K + 1> T) {
  FEM_PDL_ENTRY();
  constexpr int N = K + 1, N2 = N * N, N3 = N2 * N;
  constexpr int C = DgCartCPB<K>::value;
  extern __shared__ double smem[];
  const int t = threadIdx.x, ci = threadIdx.y;
  const int64_t cell = A.cell0 + (int64_t)blockIdx.x * C + ci;
  const bool active = cell < A.cell1;
  using LY = DgCartLayout<K>;
  constexpr int B = LY::B, S = LY::S;
  double* F0 = smem + ci * LY::CS;
  double* F1 = F0 + LY::F;
  double* F2 = F1 + LY::F;
  const int ta = t % N, tb = t / N;
  int c[3] = {0, 0, 0};
  if (active) {
    c[0] = (int)(cell % A.n[0]);
    const int64_t r = cell / A.n[0];
    c[1] = (int)(r % A.n[1]);
    c[2] = (int)(r / A.n[1]);
  }
  const int64_t stride[3] = {1, (int64_t)A.n[0], (int64_t)A.n[0] * A.n[1]};
  const double* xc = x + (active ? cell : 0) * N3;
  double xz[N];
  // ---- directional line operators, straight from global memory
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    const int gc = c[d] + (d == 2 ? A.cz0 : 0), nd = d == 2 ? A.nzg : A.n[d];
    const bool hl = active && gc > 0, hr = active && gc < nd - 1;
    const double flo = gc == 0 ? (double)A.flo[d] : 0.0, fhi = gc == nd - 1 ? (double)A.fhi[d] : 0.0;
    // line (ta, tb) along d: x-line (y=ta, z=tb), y-line (x=ta, z=tb), z-line (x=ta, y=tb)
    const int off = d == 0 ? N * ta + N2 * tb : (d == 1 ? ta + N2 * tb : ta + N * tb);
    const int st = d == 0 ? 1 : (d == 1 ? N : N2);
    const int soff = d == 0 ? B * ta + S * tb : (d == 1 ? ta + S * tb : ta + B * tb);   // shared memory
    const int sst = d == 0 ? 1 : (d == 1 ? B : S);
    double xo[N], xl[N], xr[N], o[N];
#pragma unroll
    for (int i = 0; i < N; ++i) {
      xo[i] = active ? __ldg(xc + off + st * i) : 0.0;
      xl[i] = hl ? __ldg(xc - stride[d] * N3 + off + st * i) : 0.0;
      xr[i] = hr ? __ldg(xc + stride[d] * N3 + off + st * i) : 0.0;
    }
    if (d == 2) {   // the thread's own z-line: the entries its epilogue writes
#pragma unroll
      for (int i = 0; i < N; ++i) xz[i] = xo[i];
    }
    dg_line_op<N>(T, A.sc[d], A.sigma[d], flo, fhi, hl, hr, xo, xl, xr, o);
    double* F = d == 0 ? F0 : (d == 1 ? F1 : F2);
#pragma unroll
    for (int i = 0; i < N; ++i) F[soff + sst * i] = o[i];
  }
  __syncthreads();
  // ---- x-lines (y=ta, z=tb): F1 <- M_x F1, F2 <- M_x F2
  {
    double a[N], b[N], o[N];
#pragma unroll
    for (int i = 0; i < N; ++i) {
      a[i] = F1[i + B * ta + S * tb];
      b[i] = F2[i + B * ta + S * tb];
    }
    MV_M(a, o);
#pragma unroll
    for (int i = 0; i < N; ++i) F1[i + B * ta + S * tb] = A.mc[0] * o[i];
    MV_M(b, o);
#pragma unroll
    for (int i = 0; i < N; ++i) F2[i + B * ta + S * tb] = A.mc[0] * o[i];
  }
  __syncthreads();
  // ---- y-lines (x=ta, z=tb): F0 <- M_y F0, F2 <- M_y F2
  {
    double a[N], b[N], o[N];
#pragma unroll
    for (int j = 0; j < N; ++j) {
      a[j] = F0[ta + B * j + S * tb];
      b[j] = F2[ta + B * j + S * tb];
    }
    MV_M(a, o);
#pragma unroll
    for (int j = 0; j < N; ++j) F0[ta + B * j + S * tb] = A.mc[1] * o[j];
    MV_M(b, o);
#pragma unroll
    for (int j = 0; j < N; ++j) F2[ta + B * j + S * tb] = A.mc[1] * o[j];
  }
  __syncthreads();
  // ---- z-lines (x=ta, y=tb): y = M_z (F0 + F1) + F2
  {
    double a[N], o[N];
#pragma unroll
    for (int l = 0; l < N; ++l) a[l] = F0[ta + B * tb + S * l] + F1[ta + B * tb + S * l];
    MV_M(a, o);
    if (active) {
      const double* dcls = nullptr;
      if (A.cf.on && A.cf.dinv_cls) {
        int cl[3];
#pragma unroll
        for (int d = 0; d < 3; ++d) cl[d] = c[d] == 0 ? 0 : (c[d] == A.n[d] - 1 ? 2 : 1);
        dcls = A.cf.dinv_cls + (cl[0] + 3 * cl[1] + 9 * cl[2]) * N3;
      }
#pragma unroll
      for (int l = 0; l < N; ++l)
        dg_store_x(A.cf, xz[l], y, cell * N3 + t + N2 * l, fma(A.mc[2], o[l], F2[ta + B * tb + S * l]), dcls,
                   t + N2 * l);
    }
  }
}

// ---------------------------------------------------------------- diagonal (R6)
// cell part as for CG; face part on the face layer of every face:
//   interior sum_q JxW (-phi d_n phi + sigma phi^2), Dirichlet sum_q JxW (-2 phi d_n phi + 2 sigma phi^2).
template <int K, bool DEFORMED>
__global__ void dg_diag_kernel(DgArgs A, Tab<K + 1> T) {
  FEM_PDL_ENTRY();
  constexpr int N = K + 1, N2 = N * N, N3 = N2 * N;
  const int64_t id = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (id >= A.n_cells * N3) return;
  const int64_t cell = id / N3;
  const int i = (int)(id % N3);
  const int ii[3] = {i % N, (i / N) % N, i / N2};
  int c[3];
  c[0] = (int)(cell % A.n[0]);
  const int64_t r = cell / A.n[0];
  c[1] = (int)(r % A.n[1]);
  c[2] = (int)(r / A.n[1]);
  double d = 0.0;
  for (int q2 = 0; q2 < N; ++q2)
    for (int q1 = 0; q1 < N; ++q1)
      for (int q0 = 0; q0 < N; ++q0) {
        const double bx = T.der[q0][ii[0]] * T.val[q1][ii[1]] * T.val[q2][ii[2]];
        const double by = T.val[q0][ii[0]] * T.der[q1][ii[1]] * T.val[q2][ii[2]];
        const double bz = T.val[q0][ii[0]] * T.val[q1][ii[1]] * T.der[q2][ii[2]];
        if (DEFORMED) {
          const double* Gc = A.G + (size_t)cell * 6 * N3 + q0 + N * (q1 + N * q2);
          d += Gc[0] * bx * bx + Gc[3 * N3] * by * by + Gc[5 * N3] * bz * bz +
               2.0 * (Gc[N3] * bx * by + Gc[2 * N3] * bx * bz + Gc[4 * N3] * by * bz);
        } else {
          const double w3 = T.w[q0] * T.w[q1] * T.w[q2];
          d += w3 * (A.c[0] * bx * bx + A.c[1] * by * by + A.c[2] * bz * bz);
        }
      }
  for (int D = 0; D < 3; ++D) {
    const int t1 = D == 0 ? 1 : 0, t2 = D == 2 ? 1 : 2;
    for (int s = 0; s < 2; ++s) {
      if (ii[D] != (s ? K : 0)) continue;
      const int kind = face_kind(A, D, c, s);
      if (kind == 2) continue;
      const double nsgn = s ? 1.0 : -1.0;
      const double m = kind == 0 ? 1.0 : 2.0;
      double sig = A.sigma[D];
      const double* rec = nullptr;
      if (DEFORMED) {
        const int64_t fr = face_record(A, D, c, c[D] + s);
        rec = A.faceq + fr * 7 * N2;
        sig = A.fsigma[fr];
      }
      const int own = s ? 1 : 4;
      for (int qb = 0; qb < N; ++qb)
        for (int qa = 0; qa < N; ++qa) {
          const int q = qa + N * qb;
          const double phi = T.val[qa][ii[t1]] * T.val[qb][ii[t2]];
          double dn, JxW;
          if (DEFORMED) {
            JxW = rec[q];
            double g[3];
            g[D] = T.dface[s][ii[D]] * phi;
            g[t1] = T.der[qa][ii[t1]] * T.val[qb][ii[t2]];
            g[t2] = T.val[qa][ii[t1]] * T.der[qb][ii[t2]];
            dn = nsgn * (rec[(own + 0) * N2 + q] * g[0] + rec[(own + 1) * N2 + q] * g[1] +
                         rec[(own + 2) * N2 + q] * g[2]);
          } else {
            JxW = T.w[qa] * T.w[qb] * (0.5 * A.h[t1]) * (0.5 * A.h[t2]);
            dn = nsgn * (2.0 / A.h[D]) * T.dface[s][ii[D]] * phi;
          }
          d += m * JxW * (-phi * dn + sig * phi * phi);
        }
    }
  }
  A.y[cell * N3 + i] = d;
}

// ---------------------------------------------------------------- face geometry (deformed)
// Record of face p along D (between cells p-1 and p): nf = unit normal in the
// direction of increasing xi_D (Nanson: J^-T e_D / |J^-T e_D|), JxW = w det J |J^-T e_D|,
// Jm = J_minus^-1 nf, Jp = J_plus^-1 nf (0 for a missing side); both sides agree on
// the physical point, normal and JxW because the map is continuous (reading R2).
template <int K>
__global__ void dg_face_geometry_kernel(MapArgs m, DgArgs A, Tab<K + 1> T, double* faceq, double* kap) {
  FEM_PDL_ENTRY();
  constexpr int N = K + 1, N2 = N * N;
  const int64_t id = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t total = A.face_off[2] + (int64_t)(A.n[2] + 1) * A.n[0] * A.n[1];
  if (id >= total * N2) return;
  const int64_t fr = id / N2;
  const int q = (int)(id % N2), qa = q % N, qb = q / N;
  const int D = fr >= A.face_off[2] ? 2 : (fr >= A.face_off[1] ? 1 : 0);
  const int t1 = D == 0 ? 1 : 0, t2 = D == 2 ? 1 : 2;
  const int64_t loc = fr - A.face_off[D];
  const int p = (int)(loc % (A.n[D] + 1));
  const int64_t rest = loc / (A.n[D] + 1);
  int c[3];
  c[t1] = (int)(rest % A.n[t1]);
  c[t2] = (int)(rest / A.n[t1]);
  double xi[3];
  xi[t1] = T.qp[qa];
  xi[t2] = T.qp[qb];
  double* rec = faceq + fr * 7 * N2;
  double nf[3] = {0, 0, 0};
  bool have_n = false;
  for (int side = 0; side < 2; ++side) {     // 0 minus (cell p-1, xi_D=+1), 1 plus (cell p, xi_D=-1)
    const int cd = side == 0 ? p - 1 : p;
    double* Jn = rec + (side == 0 ? 1 : 4) * N2 + q;
    const int cdg = cd + (D == 2 ? A.cz0 : 0);
    if (cdg < 0 || cdg >= (D == 2 ? A.nzg : A.n[D])) {
      Jn[0] = Jn[N2] = Jn[2 * N2] = 0.0;
      continue;
    }
    c[D] = cd;
    xi[D] = side == 0 ? 1.0 : -1.0;
    if (m.general) {
      // N3: the level's cell map; both sides agree on the point (continuous map)
      const GeoPt g = geo_point(m, c[0], c[1], c[2], xi[0], xi[1], xi[2]);
      double Ji[3][3];
      const double det = geo_inverse(g, Ji);
      if (!have_n) {
        double nrm = 0.0;
        for (int e = 0; e < 3; ++e) nrm += Ji[D][e] * Ji[D][e];
        nrm = sqrt(nrm);
        for (int e = 0; e < 3; ++e) nf[e] = Ji[D][e] / nrm;
        rec[q] = T.w[qa] * T.w[qb] * det * nrm;
        if (kap) kap[fr * N2 + q] = kappa_at(m, g.x);
        have_n = true;
      }
      for (int a = 0; a < 3; ++a) Jn[a * N2] = Ji[a][0] * nf[0] + Ji[a][1] * nf[1] + Ji[a][2] * nf[2];
      continue;
    }
    const PointGeo g = map_point(m, c[0], c[1], c[2], xi[0], xi[1], xi[2]);
    if (!have_n) {
      double v[3], nrm = 0.0;
      for (int e = 0; e < 3; ++e) {
        v[e] = jinv(m, g, D, e);   // (J^-T e_D)_e = (J^-1)_{D e}
        nrm += v[e] * v[e];
      }
      nrm = sqrt(nrm);
      for (int e = 0; e < 3; ++e) nf[e] = v[e] / nrm;
      rec[q] = T.w[qa] * T.w[qb] * g.det * nrm;
      have_n = true;
    }
    for (int a = 0; a < 3; ++a) {
      double s = 0.0;
      for (int e = 0; e < 3; ++e) s += jinv(m, g, a, e) * nf[e];
      Jn[a * N2] = s;
    }
  }
}

// volumes of the local cells plus one cell layer below and above (z-slab neighbours):
// vol[(cz + 1) n0 n1 + cy n0 + cx], cz in [-1, n2]
template <int K>
__global__ void dg_cell_volume_kernel(MapArgs m, DgArgs A, Tab<K + 1> T, double* vol) {
  FEM_PDL_ENTRY();
  constexpr int N = K + 1;
  const int64_t id = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (id >= (int64_t)A.n[0] * A.n[1] * (A.n[2] + 2)) return;
  const int cx = (int)(id % A.n[0]);
  const int64_t r = id / A.n[0];
  const int cy = (int)(r % A.n[1]), cz = (int)(r / A.n[1]) - 1;
  double v = 0.0;
  for (int q2 = 0; q2 < N; ++q2)
    for (int q1 = 0; q1 < N; ++q1)
      for (int q0 = 0; q0 < N; ++q0)
        if (m.general) {
          double Ji[3][3];
          v += T.w[q0] * T.w[q1] * T.w[q2] * geo_inverse(geo_point(m, cx, cy, cz, T.qp[q0], T.qp[q1], T.qp[q2]), Ji);
        } else {
          v += T.w[q0] * T.w[q1] * T.w[q2] * map_point(m, cx, cy, cz, T.qp[q0], T.qp[q1], T.qp[q2]).det;
        }
  vol[id] = v;
}

// sigma_F = c (k+1)^2 / h_F, 1/h_F = (|F|/|K-| + |F|/|K+|)/2 (interior), |F|/|K| (boundary).
template <int K>
__global__ void dg_face_sigma_kernel(DgArgs A, double pen, const double* faceq, const double* vol,
                                     double* fsigma) {
  FEM_PDL_ENTRY();
  constexpr int N = K + 1, N2 = N * N;
  const int64_t fr = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t total = A.face_off[2] + (int64_t)(A.n[2] + 1) * A.n[0] * A.n[1];
  if (fr >= total) return;
  const int D = fr >= A.face_off[2] ? 2 : (fr >= A.face_off[1] ? 1 : 0);
  const int t1 = D == 0 ? 1 : 0, t2 = D == 2 ? 1 : 2;
  const int64_t loc = fr - A.face_off[D];
  const int p = (int)(loc % (A.n[D] + 1));
  const int64_t rest = loc / (A.n[D] + 1);
  int c[3];
  c[t1] = (int)(rest % A.n[t1]);
  c[t2] = (int)(rest / A.n[t1]);
  double area = 0.0;
  for (int q = 0; q < N2; ++q) area += faceq[fr * 7 * N2 + q];
  double inv_h = 0.0;
  int cnt = 0;
  for (int side = 0; side < 2; ++side) {
    c[D] = side == 0 ? p - 1 : p;
    const int cg = c[D] + (D == 2 ? A.cz0 : 0);
    if (cg < 0 || cg >= (D == 2 ? A.nzg : A.n[D])) continue;
    inv_h += area / vol[c[0] + (int64_t)A.n[0] * (c[1] + (int64_t)A.n[1] * (c[2] + 1))];
    ++cnt;
  }
  fsigma[fr] = pen * (K + 1) * (K + 1) * inv_h / cnt;
}

// kappa folded into the face JxW after sigma was computed from the geometric |F|, |K|:
// every SIPG face term carries kappa (eq:poisson_dgsip)
__global__ void dg_face_kappa_kernel(double* faceq, const double* kap, int64_t nf, int N2) {
  const int64_t id = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (id >= nf * N2) return;
  const int64_t fr = id / N2;
  faceq[fr * 7 * N2 + id % N2] *= kap[id];
}

// ---------------------------------------------------------------- launchers
namespace {

MapArgs dg_map_args(const fem_ctx* h, const Level& L);
DgArgs dg_args(const fem_ctx* h, const Level& L, const double* x, double* y) {
  DgArgs A;
  A.x = x;
  A.y = y;
  A.G = L.G;
  int64_t off = 0;
  for (int d = 0; d < 3; ++d) {
    A.n[d] = L.n[d];
    A.h[d] = L.h[d];
    A.c[d] = L.cart[d];
    A.sigma[d] = h->opt.penalty_factor * (h->k + 1) * (h->k + 1) / L.h[d];
  }
  for (int d = 0; d < 3; ++d) {
    A.face_off[d] = off;
    const int t1 = d == 0 ? 1 : 0, t2 = d == 2 ? 1 : 2;
    off += (int64_t)(L.n[d] + 1) * L.n[t1] * L.n[t2];
  }
  const int N2 = (h->k + 1) * (h->k + 1);
  A.faceq = L.face;
  A.fsigma = L.face ? L.face + off * 7 * N2 : nullptr;
  A.n_cells = L.n_cells;
  A.cell0 = 0;
  A.cell1 = L.n_cells;
  A.cf = h->fuse;
  A.cz0 = L.cz0;
  A.nzg = L.nzg;
  int mask = 0;
  for (int s = 0; s < 6; ++s)
    if (h->mesh.bc[s] == FEM_BC_DIRICHLET) mask |= 1 << s;
  A.bcmask = mask;
  A.cgeo_fly = 0;
  if (!L.cartesian && !mesh_general(h->mesh) && h->dg_cgeo_fly) {
    A.cgeo_fly = 1;
    for (int d = 0; d < 3; ++d) {
      const double len = h->mesh.hi[d] - h->mesh.lo[d];
      A.gfc.pl[d] = M_PI / len;
      A.hL[d] = L.h[d] / len;
    }
    A.gfc.eps = h->mesh.deform_eps;
    A.gfc.hh = (0.5 * L.h[0]) * (0.5 * L.h[1]) * (0.5 * L.h[2]);
    const int ab[6][2] = {{0, 0}, {0, 1}, {0, 2}, {1, 1}, {1, 2}, {2, 2}};
    for (int cc = 0; cc < 6; ++cc) A.gfc.ih[cc] = 4.0 / (L.h[ab[cc][0]] * L.h[ab[cc][1]]);
  }
  A.fgeo_fly = 0;
  if (!L.cartesian && !mesh_general(h->mesh) && h->dg_fgeo_fly) {
    A.fgeo_fly = 1;
    A.map = dg_map_args(h, L);
  }
  return A;
}

int64_t n_faces(const Level& L) {
  int64_t off = 0;
  for (int d = 0; d < 3; ++d) {
    const int t1 = d == 0 ? 1 : 0, t2 = d == 2 ? 1 : 2;
    off += (int64_t)(L.n[d] + 1) * L.n[t1] * L.n[t2];
  }
  return off;
}

MapArgs dg_map_args(const fem_ctx* h, const Level& L) {
  MapArgs m;
  for (int d = 0; d < 3; ++d) {
    m.lo[d] = h->mesh.lo[d];
    m.L[d] = h->mesh.hi[d] - h->mesh.lo[d];
    m.h[d] = L.h[d];
  }
  m.eps = h->mesh.deform_eps;
  m.cz0 = L.cz0;
  set_general_map(h, L, m);
  return m;
}

template <int K, bool DEF>
void dg_apply_kd(fem_ctx* h, const Level& L, const double* x, double* y, int64_t r0, int64_t r1) {
  constexpr int N = K + 1, C = DgQCPB<K>::value;
  const size_t sm = sizeof(double) * DgSmem<N>::SIZE * C;
  const unsigned grid = (unsigned)((r1 - r0 + C - 1) / C);
  DgArgs A = dg_args(h, L, x, y);
  A.cell0 = r0;
  A.cell1 = r1;
  if (DEF && A.cgeo_fly) {
    smem_attr(reinterpret_cast<const void*>(dg_apply_kernel<K, DEF, true>), (size_t)((int)sm));
    launch_pdl(h, dg_apply_kernel<K, DEF, true>, grid, dim3(N * N, C), sm, A, make_tab<N>(h->tab));
  } else {
    smem_attr(reinterpret_cast<const void*>(dg_apply_kernel<K, DEF>), (size_t)((int)sm));
    launch_pdl(h, dg_apply_kernel<K, DEF>, grid, dim3(N * N, C), sm, A, make_tab<N>(h->tab));
  }
  count_launch();
  check_launch("dg_apply_kernel");
}

template <int K>
void dg_cart_k(fem_ctx* h, const Level& L, const double* x, double* y, int64_t r0, int64_t r1) {
  constexpr int N = K + 1, C = DgCartCPB<K>::value;
  DgKron A;
  for (int d = 0; d < 3; ++d) {
    A.n[d] = L.n[d];
    A.sigma[d] = h->opt.penalty_factor * (h->k + 1) * (h->k + 1) / L.h[d];
    A.sc[d] = 2.0 / L.h[d];
    A.mc[d] = 0.5 * L.h[d];
    A.flo[d] = h->mesh.bc[2 * d] == FEM_BC_DIRICHLET ? 1 : -1;
    A.fhi[d] = h->mesh.bc[2 * d + 1] == FEM_BC_DIRICHLET ? 1 : -1;
  }
  A.cz0 = L.cz0;
  A.nzg = L.nzg;
  A.n_cells = L.n_cells;
  A.cell0 = r0;
  A.cell1 = r1;
  A.cf = h->fuse;
  DgKronTab<N> T;
  for (int i = 0; i < N; ++i) {
    for (int j = 0; j < N; ++j) {
      double m = 0.0, sv = 0.0;
      for (int q = 0; q < N; ++q) {
        m += h->tab.qw[q] * h->tab.val[q][i] * h->tab.val[q][j];
        sv += h->tab.qw[q] * h->tab.der[q][i] * h->tab.der[q][j];
      }
      T.M[i][j] = m;
      T.S[i][j] = sv;
    }
    T.dm[i] = h->tab.dface[0][i];
    T.dp[i] = h->tab.dface[1][i];
  }
  make_eo<N>(T.S, T.Seo);
  make_eo<N>(T.M, T.Meo);
  const size_t sm = sizeof(double) * DgCartLayout<K>::CS * C;
  smem_attr(reinterpret_cast<const void*>(dg_cart_kernel<K>), (size_t)((int)sm));
  const unsigned grid = (unsigned)((r1 - r0 + C - 1) / C);
  launch_pdl(h, dg_cart_kernel<K>, grid, dim3(N * N, C), sm, x, y, A, T);
  count_launch();
  check_launch("dg_cart_kernel");
}

template <int K>
void dg_apply_k(fem_ctx* h, const Level& L, const double* x, double* y, int64_t r0, int64_t r1) {
  if (r1 <= r0) return;
  if (L.cartesian && h->dg_kron) dg_cart_k<K>(h, L, x, y, r0, r1);
  else if (L.cartesian) dg_apply_kd<K, false>(h, L, x, y, r0, r1);
  else dg_apply_kd<K, true>(h, L, x, y, r0, r1);
}

template <int K>
void dg_diag_k(fem_ctx* h, Level& L) {
  constexpr int N = K + 1;
  const int64_t tot = L.n_cells * N * N * N;
  const unsigned grid = (unsigned)((tot + 255) / 256);
  if (L.cartesian)
    dg_diag_kernel<K, false><<<grid, 256, 0, h->stream>>>(dg_args(h, L, nullptr, L.diag), make_tab<N>(h->tab));
  else
    dg_diag_kernel<K, true><<<grid, 256, 0, h->stream>>>(dg_args(h, L, nullptr, L.diag), make_tab<N>(h->tab));
  count_launch();
  check_launch("dg_diag_kernel");
}

template <int K>
void dg_face_geometry_k(fem_ctx* h, Level& L) {
  constexpr int N = K + 1, N2 = N * N;
  const int64_t nf = n_faces(L);
  FEM_CUDA_TRY(cudaMalloc(&L.face, sizeof(double) * (nf * 7 * N2 + nf)));
  double* vol = nullptr;
  const int64_t nvol = (int64_t)L.n[0] * L.n[1] * (L.n[2] + 2);
  FEM_CUDA_TRY(cudaMalloc(&vol, sizeof(double) * nvol));
  const DgArgs A = dg_args(h, L, nullptr, nullptr);
  const MapArgs m = dg_map_args(h, L);
  const Tab<N> T = make_tab<N>(h->tab);
  double* kap = nullptr;
  if (m.kamp != 0.0) FEM_CUDA_TRY(cudaMalloc(&kap, sizeof(double) * nf * N2));
  dg_face_geometry_kernel<K><<<(unsigned)((nf * N2 + 255) / 256), 256, 0, h->stream>>>(m, A, T, L.face, kap);
  dg_cell_volume_kernel<K><<<(unsigned)((nvol + 255) / 256), 256, 0, h->stream>>>(m, A, T, vol);
  dg_face_sigma_kernel<K><<<(unsigned)((nf + 255) / 256), 256, 0, h->stream>>>(
      A, h->opt.penalty_factor, L.face, vol, L.face + nf * 7 * N2);
  count_launch(3);
  if (kap) {
    dg_face_kappa_kernel<<<(unsigned)((nf * N2 + 255) / 256), 256, 0, h->stream>>>(L.face, kap, nf, N2);
    count_launch();
  }
  check_launch("dg_face_geometry");
  FEM_CUDA_TRY(cudaStreamSynchronize(h->stream));
  cudaFree(vol);
  if (kap) cudaFree(kap);
}

#define FEM_DISPATCH_K(k, fn, ...)                           \
  switch (k) {                                               \
    case 1: fn<1>(__VA_ARGS__); break;                       \
    case 2: fn<2>(__VA_ARGS__); break;                       \
    case 3: fn<3>(__VA_ARGS__); break;                       \
    case 4: fn<4>(__VA_ARGS__); break;                       \
    case 5: fn<5>(__VA_ARGS__); break;                       \
    case 6: fn<6>(__VA_ARGS__); break;                       \
    case 7: fn<7>(__VA_ARGS__); break;                       \
    case 8: fn<8>(__VA_ARGS__); break;                       \
    default: throw Error{FEM_E_ARG, "degree out of range"}; \
  }

}  // namespace

void launch_dg_apply(fem_ctx* h, const Level& L, const double* x, double* y, int64_t c0, int64_t c1) {
  if (c1 < 0) c1 = L.n_cells;
  FEM_DISPATCH_K(h->k, dg_apply_k, h, L, x, y, c0, c1);
}

void launch_dg_diagonal(fem_ctx* h, Level& L) { FEM_DISPATCH_K(h->k, dg_diag_k, h, L); }

void launch_dg_face_geometry(fem_ctx* h, Level& L) { FEM_DISPATCH_K(h->k, dg_face_geometry_k, h, L); }

}  // namespace fem
