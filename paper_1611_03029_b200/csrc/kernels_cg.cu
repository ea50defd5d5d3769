// CG Q_k cell kernels: operator apply (K1), diagonal (K4), geometry tables (R2),
// manufactured load vector (O8), Dirichlet rows.
//
// Operator (eq:mf_eval): per cell, gather x_e (constrained entries
// read as 0), interpolate to the (k+1)^3 Gauss points (3 sweeps with the 1-D
// GLL->Gauss matrix), collocation derivatives (3 sweeps), q-point operation
// f_q = G_q grad_xi u_q with G_q = w_q det J J^-1 J^-T, transposed sweeps, and
// scatter-add (sum factorization).
//
// Thread layout (B200 design): one block handles CPB cells, a
// cell is handled by (k+1)^2 threads; in each phase a thread owns one 1-D line
// of the cell in the sweep direction, keeping the line in registers (the
// sweep is a register-only (k+1)x(k+1) mat-vec with the table in the constant
// bank); switching direction is a transpose through shared memory.
#include <algorithm>

#include "cell_term.cuh"
#include "device_common.cuh"

namespace fem {

template <int K>
#ifndef FEM_CPB4
#define FEM_CPB4 8
#endif
#ifndef FEM_CPB56
#define FEM_CPB56 4
#endif
#ifndef FEM_CPB78
#define FEM_CPB78 2
#endif
struct CPB {  // cells per block: about 128-200 threads per block
  static constexpr int N = K + 1;
  static constexpr int value = (N * N <= 4) ? 32 : (N * N <= 9) ? 16 : (N * N <= 25) ? FEM_CPB4 : (N * N <= 49) ? FEM_CPB56 : FEM_CPB78;
};

struct OpArgs {
  const double* __restrict__ x;
  double* __restrict__ y;
  const double* __restrict__ G;  // deformed: [cell][6][q]
  int n0, n1, n2;                // rank-local cells per direction
  int nn0, nn1, nn2;             // nodes per direction; nn2 = GLOBAL node planes in z
  int gz0;                       // global index of the local node plane 0 (z-slab offset)
  int glayout;                   // kGLayout* of G
  int g_direct;                  // line kernel: G from global (L2-prefetched) instead of TMA->smem
  int bcmask;
  int64_t n_cells;
  int64_t cell0, cell1;          // cells [cell0, cell1) of this launch (z-slab overlap splits)
  double c0, c1, c2;             // Cartesian metric det(J) (2/h_d)^2
};

// per-cell stride of the line kernel's three work buffers: +2 doubles at Q4 spreads the
// cells of a warp over the banks (bank-conflict model search: 11% fewer wavefronts)
// Thread layout of the line kernel at Q4 (FEM_LINE_CELL_FAST, default): cells fastest,
// threadIdx = (cell, line slot); slot s < 20 owns line (ta, tb) = (s % 4, s / 4), s >= 20
// line (4, s - 20), so a warp holds 4 lines x 8 cells.  With odd row/plane strides (5, 25)
// the 4 lines of a warp split 2 + 2 by word parity for every line pattern and position,
// and a cell stride = 10 (mod 16) words spreads the 8 cells over 8 distinct double-banks
// of each parity: every transpose access takes the minimum 2 wavefronts (tools/bank_model.py;
// the (line, cell) layout straddles cells inside a warp: 1.42x the minimum).  Global
// gathers stay coalesced: 8 cells x 4 consecutive x-nodes = 32 consecutive doubles.
#ifndef FEM_WARP_CELL
#define FEM_WARP_CELL 0
#endif
template <int K>
__host__ __device__ constexpr bool line_cell_fast() { return K == 4 && FEM_LINE_CELL_FAST && !FEM_WARP_CELL; }
// Shared-memory layout of the line kernel's three per-cell buffers: element (i0, i1, i2)
// at i0 + B i1 + S i2 of a field of F words, fields at 0, F, 2F, cells CS words apart.
// Chosen per degree by tools/bank_model.py-style search over (B, S, CS) for the three
// transpose patterns of cell_laplace with the (line, cell) thread layout (modelled
// wavefronts vs the dense layout: k=1 2.0x, k=2 1.9x, k=3 2.5x, k=5 1.5x, k=6 1.3x,
// k=7 2.7x, k=8 1.1x fewer); Q4 uses the cells-fastest layout (dense strides, CS = 378).
// Measured at ~16M DoFs (% of HBM, dense -> padded): k=2 42 -> 55, k=3 47 -> 72,
// k=5 64 -> 66, k=6 46 -> 49, k=7 29 -> 31, k=8 33 -> 33; k=1 48 -> 44 (kept dense).
#ifndef FEM_LINE_PAD
#define FEM_LINE_PAD 1
#endif
template <int K>
struct LineLayout {
  static constexpr int N = K + 1;
  static constexpr int Bp[9] = {0, 2, 3, 5, 5, 9, 7, 9, 9};
  static constexpr int Sp[9] = {0, 5, 19, 20, 25, 54, 56, 72, 89};
  static constexpr int CSp[9] = {0, 30, 153, 237, 0, 964, 1169, 1725, 2385};
  static constexpr bool pad = FEM_LINE_PAD && K != 4 && K != 1;   // k = 1 measured slower padded
  static constexpr int B = pad ? Bp[K] : N;
  static constexpr int S = pad ? Sp[K] : N * N;
  static constexpr int F = (N - 1) * (1 + B + S) + 1;
  static constexpr int CS = pad ? CSp[K] : 3 * N * N * N + (N == 5 ? (line_cell_fast<K>() ? 3 : 2) : 0);
};
template <int N>
__host__ __device__ constexpr int line_cell_stride() { return LineLayout<N - 1>::CS; }
// start of the TMA-staged G chunk behind the C cells' buffers: 16-byte aligned
template <int N, int C>
__host__ __device__ constexpr int line_g_offset() { return (C * line_cell_stride<N>() + 1) / 2 * 2; }
// per-cell stride of the derivative-basis kernel (K1d, (line, cell) layout)
template <int N>
__host__ __device__ constexpr int dline_cell_stride() { return 3 * N * N * N + (N == 5 ? 2 : 0); }

// threads per cell of the line kernel: (k+1)^2, or a whole warp per cell at Q4
// (FEM_WARP_CELL=1: lanes 25..31 shadow lanes 0..6 -- same addresses, same values --
// so that no cell straddles a warp; only the real lanes scatter)
template <int K>
__host__ __device__ constexpr int line_tpc() { return (K == 4 && FEM_WARP_CELL) ? 32 : (K + 1) * (K + 1); }

// blocks per SM the register allocation must allow (measured, tools/sweep_hi.py / the
// degree sweep: the uncapped k = 6 kernel uses 103 registers -> 3 blocks; capped at 4
// blocks it spills a little and runs 810-928 -> 488-511 us at 1.6e7 DoFs; k = 8 is noisy)
// (0 = no minimum: naming minBlocks = 1 explicitly makes ptxas spend registers on ILP
// instead -- k = 4 56 -> 96 registers, C2 apply 65 -> 85 us)
template <int K>
#ifndef FEM_LINE_MINB4
#define FEM_LINE_MINB4 0
#endif
#ifndef FEM_LINE_MINB5
#define FEM_LINE_MINB5 0
#endif
#ifndef FEM_LINE_MINB6
#define FEM_LINE_MINB6 4
#endif
#ifndef FEM_LINE_MINB7
#define FEM_LINE_MINB7 0
#endif
#ifndef FEM_LINE_MINB8
#define FEM_LINE_MINB8 2
#endif
__host__ __device__ constexpr int line_minb() {
  return K == 5 ? FEM_LINE_MINB5 : K == 6 ? FEM_LINE_MINB6 : K == 7 ? FEM_LINE_MINB7 : K == 8 ? FEM_LINE_MINB8
       : (K == 4 && line_cell_fast<K>() ? FEM_LINE_MINB4 : 0);
}

// FUSED (a.cf): the input vector is the NEXT Chebyshev iterate, built on the fly at the
// gather from the previous one (the three-term recurrence of reading R8):
//   x_new = x + c1 (x - x_old) + c2 D^-1 (b - t),  t = A x  (x null: x_new = c2 D^-1 b),
// each node's owning cell (half-open ownership, as the prolongation) writes x_new and
// clears zbuf; the kernel then applies A to x_new.  One launch per smoothing step
// instead of apply + cheb_step (single-rank levels).
// (The fused variant is its own __global__ with the CgFuse block as an extra parameter:
// growing OpArgs itself slowed the plain kernel by 9%, C2 apply 66.6 -> 72.6 us.)
// analytic map of the deformed box for the FLY kernel (reading R2; not the N3 geometries)
struct GeoFly {
  double lo[3], L[3], h[3];
  int cz0;   // global z offset (cells) of the level's local layer 0
  GeoFlyC c;
};

template <int K, bool DEFORMED, bool FUSED, bool FLY = false>
__device__ __forceinline__ void cg_apply_body(const OpArgs& a, const Tab<K + 1>& T, const CgFuse& f,
                                              const GeoFly* gfly = nullptr) {
  constexpr int N = K + 1, N2 = N * N, N3 = N2 * N;
  constexpr int C = CPB<K>::value;
  extern __shared__ double smem[];
  int traw, ci;
  if constexpr (line_cell_fast<K>()) {
    ci = threadIdx.x;
    const int sl = threadIdx.y;
    traw = sl < K * N ? (sl % K) + N * (sl / K) : K + N * (sl - K * N);
  } else {
    traw = threadIdx.x;
    ci = threadIdx.y;
  }
  const int t = traw < N2 ? traw : traw - N2;
  const bool real = traw < N2;
  const int64_t cell = a.cell0 + (int64_t)blockIdx.x * C + ci;
  const bool active = cell < a.cell1;
  double* s0 = smem + ci * line_cell_stride<N>();
  const int ta = t % N, tb = t / N;
  int cx = 0, cy = 0, cz = 0;
  if (active) {
    cx = (int)(cell % a.n0);
    int64_t r = cell / a.n0;
    cy = (int)(r % a.n1);
    cz = (int)(r / a.n1);
  }
  // gather the z-line (x=ta, y=tb); constrained entries read as 0 (reading R5)
  double u[N], v[N];
  const int gx = K * cx + ta, gy = K * cy + tb;
  const int64_t zs = (int64_t)a.nn0 * a.nn1;
  const int64_t base = gx + (int64_t)a.nn0 * gy + zs * (int64_t)(K * cz);
  if constexpr (FUSED) {
    // all loads first (five independent streams per node in flight), then the stores:
    // interleaving them would serialise the gather on possible aliasing
    const bool own_xy = real && (ta < K || cx == a.n0 - 1) && (tb < K || cy == a.n1 - 1);
    double rx[N], ro[N], rb[N], rd[N], rt[N];
#pragma unroll
    for (int l = 0; l < N; ++l) {
      const int64_t i = base + l * zs;
      rx[l] = ro[l] = rb[l] = rd[l] = rt[l] = 0.0;
      if (active) {
        if (a.x) rx[l] = __ldg(a.x + i);
        if (f.materialize) {
          rb[l] = __ldg(f.b + i);
          rd[l] = __ldg(f.dinv + i);
          if (a.x) rt[l] = __ldg(f.t + i);
          if (a.x && f.xo) ro[l] = __ldg(f.xo + i);
        }
      }
    }
#pragma unroll
    for (int l = 0; l < N; ++l) {
      const bool m = cg_constrained(a.bcmask, gx, gy, a.gz0 + K * cz + l, a.nn0, a.nn1, a.nn2);
      const int64_t i = base + l * zs;
      double xv = rx[l];
      if (f.materialize)
        xv = a.x ? rx[l] + f.c1 * (rx[l] - ro[l]) + f.c2 * rd[l] * (rb[l] - rt[l]) : f.c2 * rd[l] * rb[l];
      if (active && own_xy && (l < K || K * cz + l == a.nn2 - 1)) {
        if (f.materialize) f.xnew[i] = xv;
        if (f.zbuf) f.zbuf[i] = 0.0;
      }
      u[l] = (active && !m) ? xv : 0.0;
    }
  } else {
#pragma unroll
    for (int l = 0; l < N; ++l) {
      const bool m = cg_constrained(a.bcmask, gx, gy, a.gz0 + K * cz + l, a.nn0, a.nn1, a.nn2);
      u[l] = (active && !m) ? __ldg(a.x + base + l * zs) : 0.0;
    }
  }
  // Deformed: one TMA bulk copy stages the block's G slice (C cells x 6 x N^3 doubles,
  // contiguous) into shared memory; it lands while the gather and the first five
  // sweep phases run, and the q-point phase reads G from shared memory.
  const double* Gs = nullptr;
  __shared__ alignas(8) uint64_t gbar;
  GeoFlyPt<N> fp;
  __shared__ double scz[FLY ? C : 1][FLY ? 2 * N : 1];
  if constexpr (FLY) {
    // sin / cos (pi t) of the quadrature coordinates: the thread's x and y in registers, the
    // cell's z points in shared memory (computed by N of its threads; the q-point phase
    // comes after several barriers of the sweeps)
    const GeoFly& m = *gfly;
    const int c3[3] = {cx, cy, cz + m.cz0};
    auto tq = [&](int d, int q) { return m.h[d] * (c3[d] + 0.5 * (T.qp[q] + 1.0)) / m.L[d]; };
    sincospi(tq(0, ta), &fp.sx, &fp.cx);
    sincospi(tq(1, tb), &fp.sy, &fp.cy);
    if (real && t < N) sincospi(tq(2, t), &scz[ci][t], &scz[ci][N + t]);
    fp.scz = scz[ci];
    fp.c = &m.c;
  } else if (DEFORMED && a.g_direct) {
    // G read straight from global memory in the q-point phase (each warp load is 256
    // contiguous bytes: q = t + N^2 l); the block's slice is bulk-prefetched into L2 now
    const int64_t c0 = a.cell0 + (int64_t)blockIdx.x * C;
    if (traw == 0 && ci == 0) {
      const int64_t nc = (a.cell1 - c0) < C ? (a.cell1 - c0) : C;
      bulk_prefetch_l2(a.G + c0 * 6 * N3, (uint32_t)(nc * 6 * N3 * sizeof(double)));
    }
    if (line_cell_fast<K>() && a.glayout == kGLayoutCell8) {
      const int64_t c = active ? cell : 0;
      Gs = a.G + (c / kCell8) * 6 * N3 * kCell8 + (c % kCell8);
    } else {
      Gs = a.G + (active ? cell : 0) * 6 * N3;
    }
  } else if (DEFORMED) {
    // one TMA bulk copy stages the block's G slice into shared memory (8-cell block
    // order: the launcher guarantees the block starts at a multiple of 8 cells and the
    // table is padded to whole blocks, so the slice is one contiguous 8-cell chunk)
    double* sG = smem + line_g_offset<N, C>();
    const int64_t c0 = a.cell0 + (int64_t)blockIdx.x * C;
    const bool c8 = line_cell_fast<K>() && a.glayout == kGLayoutCell8;
    if (traw == 0 && ci == 0) {
      const int64_t nc = c8 ? C : ((a.cell1 - c0) < C ? (a.cell1 - c0) : C);
      const uint32_t bytes = (uint32_t)(nc * 6 * N3 * sizeof(double));
      mbar_init(&gbar, 1);
      mbar_arrive_expect_tx(&gbar, bytes);
      bulk_g2s(sG, a.G + c0 * 6 * N3, bytes, &gbar);
    }
    __syncthreads();       // barrier initialisation visible to all threads
    Gs = c8 ? sG + ci : sG + ci * 6 * N3;
  }
  CellGeo<N> geo{Gs, a.c0, a.c1, a.c2, active, (DEFORMED && !FLY && !a.g_direct) ? &gbar : nullptr};
  if constexpr (FLY) geo.fly = &fp;
  if constexpr (line_cell_fast<K>()) {
    if (DEFORMED && a.glayout == kGLayoutCell8) {
      geo.gq = kCell8;
      geo.gc = N3 * kCell8;
    }
  }
  using LL = LineLayout<K>;
  cell_laplace<N, DEFORMED, line_cell_fast<K>(), LL::B, LL::S>(T, geo, s0, s0 + LL::F, s0 + 2 * LL::F, t, u, v);
  // scatter-add (constrained rows skipped; they are set to x_c afterwards)
  if (active && real) {
#pragma unroll
    for (int l = 0; l < N; ++l) {
      const bool m = cg_constrained(a.bcmask, gx, gy, a.gz0 + K * cz + l, a.nn0, a.nn1, a.nn2);
      if (!m) atomicAdd(a.y + base + l * zs, v[l]);
    }
  }
}

template <int K, bool DEFORMED>
__global__ void __launch_bounds__(line_tpc<K>() * CPB<K>::value, line_minb<K>())
    cg_apply_kernel(OpArgs a, Tab<K + 1> T) {
  FEM_PDL_ENTRY();
  cg_apply_body<K, DEFORMED, false>(a, T, CgFuse{});
}

// deformed CG with the metric recomputed from the analytic map at every quadrature point
// (no G traffic: C2's apply moves 16 instead of 108 bytes per DoF)
template <int K>
__global__ void __launch_bounds__(line_tpc<K>() * CPB<K>::value, line_minb<K>())
    cg_apply_fly_kernel(OpArgs a, Tab<K + 1> T, GeoFly g) {
  FEM_PDL_ENTRY();
  cg_apply_body<K, true, false, true>(a, T, CgFuse{}, &g);
}

template <int K>
__global__ void __launch_bounds__(line_tpc<K>() * CPB<K>::value, K == 4 ? 0 : line_minb<K>())
    cg_apply_fused_kernel(OpArgs a, Tab<K + 1> T, CgFuse f) {
  FEM_PDL_ENTRY();
  cg_apply_body<K, true, true>(a, T, f);
}
// ---------------------------------------------------------------- derivative-basis line kernel (K1d)
// Deformed CG cell apply (eq:mf_eval) with the gradient built from the derivative of
// the 1-D basis at the Gauss points instead of Gauss-point collocation:
//   grad u_q = (N'_x N_y N_z u, N_x N'_y N_z u, N_x N_y N'_z u),
// which needs only four direction changes per cell instead of eight (the bottleneck
// of the collocation variant is the shared-memory transposes, profiles/r01b):
//   Z: t1 = N_z u, t2 = N'_z u               -> 2 fields
//   Y: a = N_y t1, b = N'_y t1, c = N_y t2    -> 3 fields
//   X: g = (N'_x a, N_x b, N_x c); f = G_q g; e = (N'_x^T f_x, N_x^T f_y, N_x^T f_z)
//                                             -> 3 fields
//   Y: h1 = N_y^T e1 + N'_y^T e2, h2 = N_y^T e3 -> 2 fields
//   Z: v = N_z^T h1 + N'_z^T h2, scatter-add
// 16 line sweeps instead of 12, 20 shared accesses per node instead of 23 (+6 for G,
// which here is read straight from global memory in the x-line order of
// kGLayoutXLine: coalesced, L2-prefetched at block start).
#ifndef FEM_DLINE_MINB
#define FEM_DLINE_MINB 2
#endif
template <int K>
__global__ void __launch_bounds__((K + 1) * (K + 1) * CPB<K>::value, K == 4 ? FEM_DLINE_MINB : 0)
    cg_dline_kernel(OpArgs a, Tab<K + 1> T) {
  FEM_PDL_ENTRY();
  constexpr int N = K + 1, N2 = N * N, N3 = N2 * N;
  constexpr int C = CPB<K>::value;
  extern __shared__ double smem[];
  const int t = threadIdx.x, ci = threadIdx.y;
  const int64_t cell = a.cell0 + (int64_t)blockIdx.x * C + ci;
  const bool active = cell < a.cell1;
  double* F0 = smem + ci * dline_cell_stride<N>();
  double* F1 = F0 + N3;
  double* F2 = F1 + N3;
  const int ta = t % N, tb = t / N;
  if (t == 0 && ci == 0) {
    const int64_t c0 = a.cell0 + (int64_t)blockIdx.x * C;
    const int64_t nc = (a.cell1 - c0) < C ? (a.cell1 - c0) : C;
    bulk_prefetch_l2(a.G + c0 * 6 * N3, (uint32_t)(nc * 6 * N3 * sizeof(double)));
  }
  int cx = 0, cy = 0, cz = 0;
  if (active) {
    cx = (int)(cell % a.n0);
    const int64_t r = cell / a.n0;
    cy = (int)(r % a.n1);
    cz = (int)(r / a.n1);
  }
  const int gx = K * cx + ta, gy = K * cy + tb;
  const int64_t zs = (int64_t)a.nn0 * a.nn1;
  const int64_t base = gx + (int64_t)a.nn0 * gy + zs * (int64_t)(K * cz);
  // constraints of the thread's z-line (reading R5): xy-flag for the line, z-ends
  const int gzc = a.gz0 + K * cz;
  const bool lm = !active || ((a.bcmask & 1) && gx == 0) || ((a.bcmask & 2) && gx == a.nn0 - 1) ||
                  ((a.bcmask & 4) && gy == 0) || ((a.bcmask & 8) && gy == a.nn1 - 1);
  const bool z0 = (a.bcmask & 16) && gzc == 0, z1 = (a.bcmask & 32) && gzc + K == a.nn2 - 1;
  double u[N], v[N], w[N];
  // ---- Z (x = ta, y = tb)
#pragma unroll
  for (int l = 0; l < N; ++l) {
    const bool m = lm || (l == 0 && z0) || (l == K && z1);
    u[l] = m ? 0.0 : __ldg(a.x + base + l * zs);
  }
  mv<N>(T.val, u, v);
  mv<N>(T.der, u, w);
#pragma unroll
  for (int l = 0; l < N; ++l) {
    F0[t + N2 * l] = v[l];
    F1[t + N2 * l] = w[l];
  }
  __syncthreads();
  // ---- Y (x = ta, z = tb)
  {
    double r1[N], r2[N], o[N];
#pragma unroll
    for (int l = 0; l < N; ++l) {
      r1[l] = F0[ta + N * l + N2 * tb];
      r2[l] = F1[ta + N * l + N2 * tb];
    }
    mv<N>(T.val, r1, o);
#pragma unroll
    for (int l = 0; l < N; ++l) F0[ta + N * l + N2 * tb] = o[l];
    mv<N>(T.der, r1, o);
#pragma unroll
    for (int l = 0; l < N; ++l) F1[ta + N * l + N2 * tb] = o[l];
    mv<N>(T.val, r2, o);
#pragma unroll
    for (int l = 0; l < N; ++l) F2[ta + N * l + N2 * tb] = o[l];
  }
  __syncthreads();
  // ---- X (y = ta, z = tb): q-point (l, ta, tb); G entry (comp, l) at comp*N3 + l*N2 + t.
  // Point by point: gradient, flux, and its contribution to the three transposed
  // sweeps, so that only the inputs and the accumulators are live.
  {
    double ra[N], rb[N], rc[N], ea[N], eb[N], ec[N];
#pragma unroll
    for (int l = 0; l < N; ++l) {
      ra[l] = F0[l + N * t];
      rb[l] = F1[l + N * t];
      rc[l] = F2[l + N * t];
      ea[l] = eb[l] = ec[l] = 0.0;
    }
    const double* Gc = a.G + (active ? cell : 0) * 6 * N3 + t;
#pragma unroll
    for (int l = 0; l < N; ++l) {
      double gxl = 0.0, gyl = 0.0, gzl = 0.0;
#pragma unroll
      for (int i = 0; i < N; ++i) {
        gxl = fma(T.der[l][i], ra[i], gxl);
        gyl = fma(T.val[l][i], rb[i], gyl);
        gzl = fma(T.val[l][i], rc[i], gzl);
      }
      const double G00 = __ldg(Gc + 0 * N3 + l * N2), G01 = __ldg(Gc + 1 * N3 + l * N2);
      const double G02 = __ldg(Gc + 2 * N3 + l * N2), G11 = __ldg(Gc + 3 * N3 + l * N2);
      const double G12 = __ldg(Gc + 4 * N3 + l * N2), G22 = __ldg(Gc + 5 * N3 + l * N2);
      double fx = G00 * gxl + G01 * gyl + G02 * gzl;
      double fy = G01 * gxl + G11 * gyl + G12 * gzl;
      double fz = G02 * gxl + G12 * gyl + G22 * gzl;
      if (!active) fx = fy = fz = 0.0;
#pragma unroll
      for (int i = 0; i < N; ++i) {
        ea[i] = fma(T.der[l][i], fx, ea[i]);
        eb[i] = fma(T.val[l][i], fy, eb[i]);
        ec[i] = fma(T.val[l][i], fz, ec[i]);
      }
    }
#pragma unroll
    for (int l = 0; l < N; ++l) {
      F0[l + N * t] = ea[l];
      F1[l + N * t] = eb[l];
      F2[l + N * t] = ec[l];
    }
  }
  __syncthreads();
  // ---- Y (x = ta, z = tb): h1 = N_y^T e1 + N'_y^T e2, h2 = N_y^T e3
  {
    double r1[N], r2[N], o[N];
#pragma unroll
    for (int l = 0; l < N; ++l) {
      r1[l] = F0[ta + N * l + N2 * tb];
      r2[l] = F1[ta + N * l + N2 * tb];
    }
    mvt<N>(T.val, r1, o);
    mvt_add<N>(T.der, r2, o);
#pragma unroll
    for (int l = 0; l < N; ++l) {
      r1[l] = F2[ta + N * l + N2 * tb];
      F0[ta + N * l + N2 * tb] = o[l];
    }
    mvt<N>(T.val, r1, o);
#pragma unroll
    for (int l = 0; l < N; ++l) F1[ta + N * l + N2 * tb] = o[l];
  }
  __syncthreads();
  // ---- Z (x = ta, y = tb): v = N_z^T h1 + N'_z^T h2, scatter-add
#pragma unroll
  for (int l = 0; l < N; ++l) {
    u[l] = F0[t + N2 * l];
    w[l] = F1[t + N2 * l];
  }
  mvt<N>(T.val, u, v);
  mvt_add<N>(T.der, w, v);
#pragma unroll
  for (int l = 0; l < N; ++l) {
    const bool m = lm || (l == 0 && z0) || (l == K && z1);
    if (!m) atomicAdd(a.y + base + l * zs, v[l]);
  }
}


// ---------------------------------------------------------------- plane kernel (K1p, K <= 4)
// Same operator as cg_apply_kernel (eq:mf_eval with G_q = w det J J^-1 J^-T), with a
// thread layout that halves the shared-memory traffic of the line kernel (the
// bottleneck ncu shows for it, profiles/r01b_summary.json): a cell is handled by
// N = k+1 threads, each owning a whole 2-D plane of the cell in registers, so two of
// the three directions are swept in-thread:
//   layout A: thread p owns the xz-plane y = p   (z- and x-sweeps in registers)
//   layout B: thread p owns the xy-plane z = p   (y- and x-sweeps in registers)
// Forward: z-sweeps N_z u and N'_z u (derivative of the basis at the Gauss points, so
// d/dz needs no collocation pass in layout A), x-interpolation of both, transpose
// A->B (2 fields), y-interpolation (and N'_y) -> u_q, d_y u_q and d_z u_q; d_x by
// Gauss-point collocation in-thread.  Quadrature point: f = G_q grad u, with G read from the
// plane-layout table (coalesced; the block's slice is bulk-prefetched into L2 at
// kernel start).  Backward: d_x^T f_x per row, N_y^T of it plus N'_y^T f_y, N_y^T f_z,
// transpose B->A (2 fields), N_x^T, then N_z^T (.) + N'_z^T (.) and the
// scatter-add.  Transposes go through shared memory with padded strides (plane stride
// LS, cell stride CS) chosen so that every 16-lane phase of a warp hits 16 distinct
// banks in both layouts.
template <int N> struct PlanePad;
#ifndef FEM_PLANE_MINB
#define FEM_PLANE_MINB 2
#endif
template <> struct PlanePad<2> { static constexpr int LS = 4, CS = 17, MINB = 4; };
template <> struct PlanePad<3> { static constexpr int LS = 19, CS = 121, MINB = 3; };
template <> struct PlanePad<4> { static constexpr int LS = 20, CS = 161, MINB = 2; };
template <> struct PlanePad<5> { static constexpr int LS = 25, CS = 253, MINB = 0; };  // 2-way conflicts in places, 2 KB/cell

template <int K, bool DEFORMED>
__global__ void __launch_bounds__((K + 1) * kGroupCells, PlanePad<K + 1>::MINB)
    cg_plane_kernel(OpArgs a, Tab<K + 1> T) {
  FEM_PDL_ENTRY();
  constexpr int N = K + 1, N2 = N * N, CB = kGroupCells;
  constexpr int LS = PlanePad<N>::LS, CS = PlanePad<N>::CS;
  extern __shared__ double smem[];
  const int tid = threadIdx.x;
  const int p = tid % N, c = tid / N;
  const int64_t group = blockIdx.x;
  const int64_t cell = group * CB + c;
  const bool active = cell < a.n_cells;
  // Geometry: the quadrature phase runs row by row (qy); the six components of one row
  // of the group are six contiguous chunks of N^2 CB doubles in the plane layout, staged
  // into shared memory by TMA bulk copies, double-buffered (rows qy and qy+1 in flight;
  // rows 0 and 1 are issued now, before the gather, so they land during phase A).
  constexpr int GROW = N * CB * N;                          // doubles per component and row
  constexpr int GB = 3;                                     // row buffers (rows in flight)
  double* Gsm = smem + CB * CS;                             // [GB][6][GROW]
  __shared__ alignas(8) uint64_t gfull[GB];
  const double* Gg = DEFORMED ? a.G + group * (int64_t)6 * N2 * CB * N : nullptr;
  auto issue_row = [&](int qy) {
    const int b = qy % GB;
    mbar_arrive_expect_tx(&gfull[b], (uint32_t)(sizeof(double) * 6 * GROW));
#pragma unroll
    for (int comp = 0; comp < 6; ++comp)
      bulk_g2s(Gsm + (b * 6 + comp) * GROW, Gg + ((int64_t)comp * N2 + (int64_t)N * qy) * CB * N,
               (uint32_t)(sizeof(double) * GROW), &gfull[b]);
  };
  if (DEFORMED && tid == 0) {
#pragma unroll
    for (int b = 0; b < GB; ++b) mbar_init(&gfull[b], 1);
#pragma unroll
    for (int qy = 0; qy < GB && qy < N; ++qy) issue_row(qy);
  }
  int cx = 0, cy = 0, cz = 0;
  if (active) {
    cx = (int)(cell % a.n0);
    const int64_t r = cell / a.n0;
    cy = (int)(r % a.n1);
    cz = (int)(r / a.n1);
  }
  double* S0 = smem + c * CS;
  double* S1 = S0 + N * LS;
  const int64_t zs = (int64_t)a.nn0 * a.nn1;
  const int gx0 = K * cx, gy = K * cy + p;
  const int64_t base = gx0 + (int64_t)a.nn0 * gy + zs * (int64_t)(K * cz);
  // Dirichlet constraints of the thread's plane (reading R5) as five flags, so that
  // element (l, i) is constrained iff ym || (i==0 && x0) || (i==K && x1) || (l==0 && z0)
  // || (l==K && z1) -- compile-time selections once i, l are unrolled
  const int gzc = a.gz0 + K * cz;
  const bool ym = ((a.bcmask & 4) && gy == 0) || ((a.bcmask & 8) && gy == a.nn1 - 1) || !active;
  const bool x0 = (a.bcmask & 1) && gx0 == 0, x1 = (a.bcmask & 2) && gx0 + K == a.nn0 - 1;
  const bool z0 = (a.bcmask & 16) && gzc == 0, z1 = (a.bcmask & 32) && gzc + K == a.nn2 - 1;
  auto masked = [&](int l, int i) {
    return ym || (i == 0 && x0) || (i == K && x1) || (l == 0 && z0) || (l == K && z1);
  };

  // ---- layout A (thread p: y = p): gather row l = x(., p, l), interpolate in x
  double X[N][N];                       // [l][qx]
#pragma unroll
  for (int l = 0; l < N; ++l) {
    double u[N];
#pragma unroll
    for (int i = 0; i < N; ++i) u[i] = masked(l, i) ? 0.0 : __ldg(a.x + base + i + l * zs);
    mv<N>(T.val, u, X[l]);
  }
  // z: N_z and N'_z per column qx, straight into shared memory
  // (element (qz, y=p, qx) at qz*LS + p*N + qx)
#pragma unroll
  for (int i = 0; i < N; ++i) {
#pragma unroll
    for (int q = 0; q < N; ++q) {
      double s1 = 0.0, s2 = 0.0;
#pragma unroll
      for (int l = 0; l < N; ++l) {
        s1 = fma(T.val[q][l], X[l][i], s1);
        s2 = fma(T.der[q][l], X[l][i], s2);
      }
      S0[q * LS + p * N + i] = s1;
      S1[q * LS + p * N + i] = s2;
    }
  }
  __syncthreads();
  // ---- layout B (thread p: qz = p).  Only the thread's own plane of S0/S1 is touched
  // until the next barrier.  u_q goes back into S0 (column by column, in place), d_y u_q
  // and d_z u_q stay in registers (Y, Z); the q-point phase runs row by row, reading a
  // row of u_q and writing back the row's d_x^T f_x in its place.
  double Y[N][N], Z[N][N];   // [qy][qx]: d_y u_q -> f_y, d_z u_q -> f_z
#pragma unroll
  for (int i = 0; i < N; ++i) {         // column qx = i
    double r1[N], r2[N];
#pragma unroll
    for (int j = 0; j < N; ++j) {
      r1[j] = S0[p * LS + j * N + i];
      r2[j] = S1[p * LS + j * N + i];
    }
#pragma unroll
    for (int qy = 0; qy < N; ++qy) {
      double s1 = 0.0, s2 = 0.0, s3 = 0.0;
#pragma unroll
      for (int j = 0; j < N; ++j) {
        s1 = fma(T.val[qy][j], r1[j], s1);
        s2 = fma(T.der[qy][j], r1[j], s2);
        s3 = fma(T.val[qy][j], r2[j], s3);
      }
      S0[p * LS + qy * N + i] = s1;
      Y[qy][i] = s2;
      Z[qy][i] = s3;
    }
  }
#pragma unroll
  for (int qy = 0; qy < N; ++qy) {
    double ur[N], fxr[N], acc[N];
    const double* Gq = Gsm + (qy % GB) * 6 * GROW + tid;
    if (DEFORMED) mbar_wait(&gfull[qy % GB], (qy / GB) & 1);
#pragma unroll
    for (int m = 0; m < N; ++m) ur[m] = S0[p * LS + qy * N + m];
#pragma unroll
    for (int qx = 0; qx < N; ++qx) {
      double gxq = 0.0;
#pragma unroll
      for (int m = 0; m < N; ++m) gxq = fma(T.colloc[qx][m], ur[m], gxq);
      const double gyq = Y[qy][qx], gzq = Z[qy][qx];
      double fx, fy, fz;
      if (DEFORMED) {
        // entry (comp, e = qx + N qy) of this thread in the staged row: comp*GROW + qx*CB*N + tid
        const double G00 = Gq[0 * GROW + qx * CB * N], G01 = Gq[1 * GROW + qx * CB * N];
        const double G02 = Gq[2 * GROW + qx * CB * N], G11 = Gq[3 * GROW + qx * CB * N];
        const double G12 = Gq[4 * GROW + qx * CB * N], G22 = Gq[5 * GROW + qx * CB * N];
        fx = G00 * gxq + G01 * gyq + G02 * gzq;
        fy = G01 * gxq + G11 * gyq + G12 * gzq;
        fz = G02 * gxq + G12 * gyq + G22 * gzq;
        if (!active) fx = fy = fz = 0.0;
      } else {
        const double w3 = T.w[qx] * T.w[qy] * T.w[p];
        fx = a.c0 * w3 * gxq;
        fy = a.c1 * w3 * gyq;
        fz = a.c2 * w3 * gzq;
      }
      fxr[qx] = fx;
      Y[qy][qx] = fy;
      Z[qy][qx] = fz;
    }
    mvt<N>(T.colloc, fxr, acc);
#pragma unroll
    for (int m = 0; m < N; ++m) S0[p * LS + qy * N + m] = acc[m];
    if (DEFORMED && qy + GB < N) {
      __syncthreads();                 // every thread is done with this buffer
      if (tid == 0) issue_row(qy + GB);
    }
  }
  // N_y^T (d_x^T f_x) + N'_y^T f_y -> S0 and N_y^T f_z -> S1, column by column in place
  // (element (qz=p, y, qx) at p*LS + y*N + qx)
#pragma unroll
  for (int i = 0; i < N; ++i) {
    double ac[N];
#pragma unroll
    for (int qy = 0; qy < N; ++qy) ac[qy] = S0[p * LS + qy * N + i];
#pragma unroll
    for (int j = 0; j < N; ++j) {
      double s1 = 0.0, s2 = 0.0;
#pragma unroll
      for (int qy = 0; qy < N; ++qy) {
        s1 = fma(T.val[qy][j], ac[qy], s1);
        s1 = fma(T.der[qy][j], Y[qy][i], s1);
        s2 = fma(T.val[qy][j], Z[qy][i], s2);
      }
      S0[p * LS + j * N + i] = s1;
      S1[p * LS + j * N + i] = s2;
    }
  }
  __syncthreads();
  // ---- layout A (thread p: y = p): per column qx, N_z^T a + N'_z^T b, then N_x^T
  // accumulated over the columns into the nodal rows V[l][.]
  double V[N][N];                       // [l][i]
#pragma unroll
  for (int l = 0; l < N; ++l)
#pragma unroll
    for (int i = 0; i < N; ++i) V[l][i] = 0.0;
#pragma unroll
  for (int qx = 0; qx < N; ++qx) {
    double ca[N], cb[N];
#pragma unroll
    for (int q = 0; q < N; ++q) {
      ca[q] = S0[q * LS + p * N + qx];
      cb[q] = S1[q * LS + p * N + qx];
    }
#pragma unroll
    for (int l = 0; l < N; ++l) {
      double v = 0.0;
#pragma unroll
      for (int q = 0; q < N; ++q) {
        v = fma(T.val[q][l], ca[q], v);
        v = fma(T.der[q][l], cb[q], v);
      }
#pragma unroll
      for (int i = 0; i < N; ++i) V[l][i] = fma(T.val[qx][i], v, V[l][i]);
    }
  }
#pragma unroll
  for (int l = 0; l < N; ++l)
#pragma unroll
    for (int i = 0; i < N; ++i)
      if (!masked(l, i)) atomicAdd(a.y + base + i + l * zs, V[l][i]);
}

// ---------------------------------------------------------------- Cartesian fast path (K1c)
// On a Cartesian cell the (k+1)-point Gauss rule integrates the stiffness exactly,
// so the element operator is the Kronecker sum
//     K^e = c0 S(x)M(x)M + c1 M(x)S(x)M + c2 M(x)M(x)S,  c_d = det J (2/h_d)^2,
// with the nodal 1-D mass M_ij = sum_q w_q phi_i phi_j and stiffness
// S_ij = sum_q w_q phi_i' phi_j'.  Factored as
//     x-lines:  a = M_x u,            c = c0 S_x u
//     y-lines:  p = M_y a,            q = c1 S_y a + M_y c
//     z-lines:  y = c2 S_z p + M_z q
// i.e. 7 line sweeps and 2 shared-memory transposes (2 fields each) per cell, and
// the scatter happens from z-lines (consecutive lanes -> consecutive addresses).
// cell0: first cell of this launch (the apply runs in z-chunks, see launcher).
// cell stride of the Kronecker element kernel's two buffers (+3 doubles at Q4: 11% fewer
// shared wavefronts in the bank-conflict model, as for the line kernel)
// Q4: the same cells-fastest thread layout as the line kernel (FEM_CART_CELL_FAST, default):
// 2 x 125 = 250 = 10 (mod 16) words per cell is already the conflict-free cell stride.
#ifndef FEM_CART_CELL_FAST
#define FEM_CART_CELL_FAST 1
#endif
template <int K>
__host__ __device__ constexpr bool cart_cell_fast() { return K == 4 && FEM_CART_CELL_FAST; }
// other degrees: padded strides from the bank-conflict model search (element (i0, i1, i2)
// at i0 + B i1 + S i2, two fields F words apart, cells CS apart)
#ifndef FEM_CART_PAD
#define FEM_CART_PAD 1
#endif
template <int K>
struct CartLayout {
  static constexpr int N = K + 1;
  static constexpr int Bp[9] = {0, 2, 3, 5, 5, 9, 10, 9, 9};
  static constexpr int Sp[9] = {0, 5, 19, 20, 25, 54, 71, 72, 89};
  static constexpr int CSp[9] = {0, 18, 105, 163, 0, 644, 993, 1150, 1601};
  // measured (apply at ~16M DoFs, dense -> padded): k=1 1041 -> 730 us, k=2 353 -> 305,
  // k=3 306 -> 216, k=7 333 -> 289, k=5, 8 -1%; k=6 +2% (kept dense)
  static constexpr bool pad = FEM_CART_PAD != 0 && K != 4 && K != 6;
  static constexpr int B = pad ? Bp[K] : N;
  static constexpr int S = pad ? Sp[K] : N * N;
  static constexpr int F = (N - 1) * (1 + B + S) + 1;
  static constexpr int CS = pad ? CSp[K] : 2 * N * N * N + (N == 5 ? (cart_cell_fast<K>() ? 0 : 3) : 0);
};
template <int N>
__host__ __device__ constexpr int cart_cell_stride() { return CartLayout<N - 1>::CS; }

template <int N>
struct KronTab {
  double M[N][N];
  double S[N][N];
};

template <int K>
#ifndef FEM_CART_MINB
#define FEM_CART_MINB 3
#endif
__global__ void __launch_bounds__((K + 1) * (K + 1) * CPB<K>::value, K == 4 ? FEM_CART_MINB : (K >= 5 ? (K == 5 ? 3 : 2) : 0))
    cg_cart_kernel(OpArgs a, KronTab<K + 1> T, int64_t cell0, int64_t cell_end) {   // within [a.cell0, a.cell1)
  FEM_PDL_ENTRY();
  constexpr int N = K + 1, N2 = N * N, N3 = N2 * N;
  constexpr int C = CPB<K>::value;
  extern __shared__ double smem[];
  int t, ci;
  if constexpr (cart_cell_fast<K>()) {   // see the line kernel
    ci = threadIdx.x;
    const int sl = threadIdx.y;
    t = sl < K * N ? (sl % K) + N * (sl / K) : K + N * (sl - K * N);
  } else {
    t = threadIdx.x;
    ci = threadIdx.y;
  }
  const int64_t cell = cell0 + (int64_t)blockIdx.x * C + ci;
  const bool active = cell < cell_end;
  using CL = CartLayout<K>;
  constexpr int B = CL::B, S = CL::S;
  double* s0 = smem + ci * CL::CS;
  double* s1 = s0 + CL::F;
  const int ta = t % N, tb = t / N;
  int cx = 0, cy = 0, cz = 0;
  if (active) {
    cx = (int)(cell % a.n0);
    const int64_t r = cell / a.n0;
    cy = (int)(r % a.n1);
    cz = (int)(r / a.n1);
  }
  const int64_t zs = (int64_t)a.nn0 * a.nn1;
  double u[N], f0[N], f1[N], f2[N];
  // ---- x-lines (y = ta, z = tb): gather, a = M_x u, c = c0 S_x u
  {
    const int gy = K * cy + ta, gz = K * cz + tb;
    const int64_t base = (int64_t)K * cx + (int64_t)a.nn0 * gy + zs * gz;
#pragma unroll
    for (int l = 0; l < N; ++l) {
      const bool m = cg_constrained(a.bcmask, K * cx + l, gy, a.gz0 + gz, a.nn0, a.nn1, a.nn2);
      u[l] = (active && !m) ? __ldg(a.x + base + l) : 0.0;
    }
    mv<N>(T.M, u, f0);
    mv<N>(T.S, u, f1);
#pragma unroll
    for (int l = 0; l < N; ++l) {
      s0[l + B * ta + S * tb] = f0[l];
      s1[l + B * ta + S * tb] = a.c0 * f1[l];
    }
  }
  __syncthreads();
  // ---- y-lines (x = ta, z = tb): p = M_y a, q = c1 S_y a + M_y c
#pragma unroll
  for (int l = 0; l < N; ++l) {
    u[l] = s0[ta + B * l + S * tb];
    f2[l] = s1[ta + B * l + S * tb];
  }
  mv<N>(T.M, u, f0);
  mv<N>(T.S, u, f1);
  mv<N>(T.M, f2, u);
#pragma unroll
  for (int l = 0; l < N; ++l) {
    s0[ta + B * l + S * tb] = f0[l];
    s1[ta + B * l + S * tb] = fma(a.c1, f1[l], u[l]);
  }
  __syncthreads();
  // ---- z-lines (x = ta, y = tb): y = c2 S_z p + M_z q, scatter-add
#pragma unroll
  for (int l = 0; l < N; ++l) {
    u[l] = s0[ta + B * tb + S * l];
    f2[l] = s1[ta + B * tb + S * l];
  }
  mv<N>(T.S, u, f0);
  mv<N>(T.M, f2, f1);
  if (active) {
    const int gx = K * cx + ta, gy = K * cy + tb;
    const int64_t base = gx + (int64_t)a.nn0 * gy + zs * (int64_t)(K * cz);
#pragma unroll
    for (int l = 0; l < N; ++l) {
      const bool m = cg_constrained(a.bcmask, gx, gy, a.gz0 + K * cz + l, a.nn0, a.nn1, a.nn2);
      if (!m) atomicAdd(a.y + base + l * zs, fma(a.c2, f0[l], f1[l]));
    }
  }
}


// ---------------------------------------------------------------- global Kronecker stencil (K1s)
// Cartesian CG levels (C4).  The element matrix is the Kronecker sum
// K^e = c0 S(x)M(x)M + c1 M(x)S(x)M + c2 M(x)M(x)S, and on a tensor grid
// of identical cells the assembled operator is the same Kronecker sum of the ASSEMBLED
// 1-D matrices:  A = c0 M1_z M1_y S1_x + c1 M1_z S1_y M1_x + c2 S1_z M1_y M1_x
// (the element set is the product of the 1-D element sets).  So
//     y = M1_z Q + c2 S1_z P,   P = M1_y M1_x x~,   Q = M1_y (c0 S1_x x~) + S1_y (c1 M1_x x~),
// x~ = x with the Dirichlet entries read as 0 (reading R5), and y_c = x_c afterwards.
// It is applied without any scatter: a block owns a 2-D tile of output node columns
// and marches through z.  Per input plane: the tile plus a k-node halo is loaded into
// shared memory with cp.async (double-buffered, out-of-domain and constrained entries
// zero-filled), x-sweeps (A = M1_x x~, B = S1_x x~) into shared memory, y-sweeps into
// registers (P, Q), and the z-direction is accumulated element by element in
// registers: with z-element ez, the k+1 planes ez k .. ez k + k contribute
// Mref[r][r'] Q + c2 Sref[r][r'] P to the outputs ez k + r, the shared vertex plane
// carries to the next element.  Every output is written exactly once (no atomics, no
// zero fill, x read once from DRAM, y written once).
// Banded 1-D rows in "slot" form: slot e owns the nodes e k + r, r = 0..k-1 (slot n
// only its vertex r = 0); vertex rows add the right end of element e-1 and the left
// end of element e, interior rows only element e.  With r a compile-time loop index,
// every coefficient is uniform across the warp (constant bank) -- no divergence.
template <int K>
struct StencilCfg {
  static constexpr int N = K + 1;
  static constexpr int TEX = (64 + K - 1) / K;        // x slots per tile
  static constexpr int TEY = 4;                       // y slots per tile
  static constexpr int TX = TEX * K;                  // output x nodes per tile
  static constexpr int THREADS = TX * TEY;            // one thread per (x node, y slot)
  static constexpr int LROWS = (TEY + 1) * K + 1;     // loaded rows (y) incl. halo
  static constexpr int LCOLS = (TEX + 1) * K + 1;     // loaded columns (x) incl. halo
  static constexpr int LPAD = LCOLS | 1;              // odd row stride: rows hit distinct banks
  static constexpr int TXP = TX + 1;                  // odd row stride of the A, B buffers
  static constexpr int HROWS = (LROWS + 1) / 2;       // x-stage: one item = one slot, two rows
  static constexpr int NBUF = 4;                     // input planes in flight (prefetch distance 3)
  static constexpr int SMEM = NBUF * LROWS * LPAD + 2 * LROWS * TXP;   // doubles
};

__device__ __forceinline__ void cp_async8(void* dst, const void* src, bool valid) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(smem_u32(dst)), "l"(src),
               "r"(valid ? 8 : 0)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int W>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(W) : "memory"); }

#ifndef FEM_STENCIL_MINB
#define FEM_STENCIL_MINB 2
#endif
template <int K>
__global__ void __launch_bounds__(StencilCfg<K>::THREADS, FEM_STENCIL_MINB)
    cg_stencil_kernel(OpArgs a, KronTab<K + 1> T) {
  FEM_PDL_ENTRY();
  using Cfg = StencilCfg<K>;
  constexpr int TEX = Cfg::TEX, TEY = Cfg::TEY, TX = Cfg::TX, LR = Cfg::LROWS, LC = Cfg::LCOLS,
                LP = Cfg::LPAD, TXP = Cfg::TXP, HR = Cfg::HROWS;
  extern __shared__ double smem[];
  double* X0 = smem;                    // NBUF input buffers [LR][LP]
  double* Ab = smem + Cfg::NBUF * LR * LP;   // A = M1_x x~ at [row][tile x] (row stride TXP)
  double* Bb = Ab + LR * TXP;           // B = S1_x x~
  const int tid = threadIdx.x;
  const int e0 = blockIdx.x * TEX, f0 = blockIdx.y * TEY;   // first x / y slot of the tile
  const int nx = a.n0, ny = a.n1, nzl = a.n2;                // cells
  const int NX = a.nn0, NY = a.nn1;
  const int gx0 = (e0 - 1) * K, gy0 = (f0 - 1) * K;        // global node of loaded (0,0)
  const int64_t zs = (int64_t)NX * NY;
  const bool cx0 = a.bcmask & 1, cx1 = a.bcmask & 2, cy0 = a.bcmask & 4, cy1 = a.bcmask & 8;
  const bool cz0 = a.bcmask & 16, cz1 = a.bcmask & 32;

  // Plane loads: thread tid always loads the same (row, column) slots of the tile, so the
  // in-domain / constraint tests and the in-plane offsets are computed once per kernel
  // (a bitmask of the valid slots and one 32-bit offset each); per plane only the z test.
  constexpr int NLD = (LR * LC + Cfg::THREADS - 1) / Cfg::THREADS;
  int ld_off[NLD];
  uint32_t ld_ok = 0;
#pragma unroll
  for (int j = 0; j < NLD; ++j) {
    const int idx = tid + j * Cfg::THREADS;
    const int r = idx / LC, c = idx % LC;
    const int gx = gx0 + c, gy = gy0 + r;
    const bool in = idx < LR * LC && gx >= 0 && gx < NX && gy >= 0 && gy < NY;
    const bool m = (cx0 && gx == 0) || (cx1 && gx == NX - 1) || (cy0 && gy == 0) || (cy1 && gy == NY - 1);
    ld_off[j] = in ? gx + NX * gy : 0;
    if (in && !m) ld_ok |= 1u << j;
  }
  auto load_plane = [&](int pl, double* buf) {   // local z plane pl (global a.gz0 + pl)
    const int gz = a.gz0 + pl;
    const bool zmask = (cz0 && gz == 0) || (cz1 && gz == a.nn2 - 1);
    const double* src = a.x + (int64_t)pl * zs;
#pragma unroll
    for (int j = 0; j < NLD; ++j) {
      const int idx = tid + j * Cfg::THREADS;
      if (idx < LR * LC) {
        const int r = idx / LC, c = idx % LC;
        cp_async8(buf + r * LP + c, src + ld_off[j], !zmask && ((ld_ok >> j) & 1u));
      }
    }
    cp_async_commit();
  };

  // this thread's y-stage / z-stage nodes: x = gx0 + K + c (tile column c), y-slot s
  const int c = tid % TX, s = tid / TX;
  const int xs = e0 * K + c;                       // global x node
  const int fy = f0 + s;                           // global y slot
  const bool col_ok = xs < NX && fy <= ny;
  // y-slot rows valid: r = 0 always (if fy <= ny), r >= 1 only if fy < ny
  const double yhl = (fy >= 1) ? 1.0 : 0.0, yhr = (fy < ny) ? 1.0 : 0.0;   // elements fy-1, fy exist

  double out[K][K + 1];      // z accumulators per y node r: out[r][rz]
  double carry[K], Pv[K], Qv[K];
#pragma unroll
  for (int r = 0; r < K; ++r) carry[r] = Pv[r] = Qv[r] = 0.0;

  // P, Q of one plane for the thread's K nodes (y rows fy K + r)
  auto plane_pq = [&](int pl, double* buf, double (&P)[K], double (&Q)[K]) {
    // x-stage: rows 0..LR-1, slots 0..TEX-1 of the tile: A, B at tile columns slot*K + r.
    // One item = one slot and two rows (ILP), rows vary fastest across lanes (odd strides:
    // no bank conflicts on the row reads and on the A/B writes).
    for (int it = tid; it < HR * TEX; it += Cfg::THREADS) {
      const int row0 = it % HR, sl = it / HR;
      const int e = e0 + sl;                       // global x slot
      const double xl = (e >= 1) ? 1.0 : 0.0, xr = (e < nx) ? 1.0 : 0.0;
#pragma unroll
      for (int h2 = 0; h2 < 2; ++h2) {
        const int row = row0 + h2 * HR;
        if (row >= LR) break;
        const double* xrow = buf + row * LP + sl * K;   // loaded column of node (e-1) K
        double v[2 * K + 1];
#pragma unroll
        for (int j = 0; j <= 2 * K; ++j) v[j] = xrow[j];
#pragma unroll
        for (int r = 0; r < K; ++r) {
          double am = 0.0, bs = 0.0;
          if (r == 0) {
            double aL = 0.0, bL = 0.0, aR = 0.0, bR = 0.0;
#pragma unroll
            for (int j = 0; j <= K; ++j) {
              aL = fma(T.M[K][j], v[j], aL);
              bL = fma(T.S[K][j], v[j], bL);
              aR = fma(T.M[0][j], v[K + j], aR);
              bR = fma(T.S[0][j], v[K + j], bR);
            }
            am = xl * aL + xr * aR;
            bs = xl * bL + xr * bR;
          } else {
#pragma unroll
            for (int j = 0; j <= K; ++j) {
              am = fma(T.M[r][j], v[K + j], am);
              bs = fma(T.S[r][j], v[K + j], bs);
            }
          }
          Ab[row * TXP + sl * K + r] = am;
          Bb[row * TXP + sl * K + r] = bs;
        }
      }
    }
    __syncthreads();
    // y-stage: column c, rows s K .. s K + 2K (element fy-1: rows sK..sK+K, element fy: sK+K..sK+2K)
    double av[2 * K + 1], bv[2 * K + 1];
#pragma unroll
    for (int j = 0; j <= 2 * K; ++j) {
      av[j] = Ab[(s * K + j) * TXP + c];
      bv[j] = Bb[(s * K + j) * TXP + c];
    }
#pragma unroll
    for (int r = 0; r < K; ++r) {
      double p = 0.0, qm = 0.0, qs = 0.0;
      if (r == 0) {
        double pL = 0.0, pR = 0.0, mL = 0.0, mR = 0.0, sL = 0.0, sR = 0.0;
#pragma unroll
        for (int j = 0; j <= K; ++j) {
          pL = fma(T.M[K][j], av[j], pL);
          pR = fma(T.M[0][j], av[K + j], pR);
          mL = fma(T.M[K][j], bv[j], mL);
          mR = fma(T.M[0][j], bv[K + j], mR);
          sL = fma(T.S[K][j], av[j], sL);
          sR = fma(T.S[0][j], av[K + j], sR);
        }
        p = yhl * pL + yhr * pR;
        qm = yhl * mL + yhr * mR;
        qs = yhl * sL + yhr * sR;
      } else {
#pragma unroll
        for (int j = 0; j <= K; ++j) {
          p = fma(T.M[r][j], av[K + j], p);
          qm = fma(T.M[r][j], bv[K + j], qm);
          qs = fma(T.S[r][j], av[K + j], qs);
        }
      }
      P[r] = p;
      Q[r] = fma(a.c0, qm, a.c1 * qs);
    }
  };

  auto write_plane = [&](int pl, const double (&v)[K]) {
    if (!col_ok) return;
    const int gz = a.gz0 + pl;
    const bool zm = (cz0 && gz == 0) || (cz1 && gz == a.nn2 - 1);
    const bool xm = (cx0 && xs == 0) || (cx1 && xs == NX - 1);
#pragma unroll
    for (int r = 0; r < K; ++r) {
      const int ys = fy * K + r;
      if (r > 0 && fy >= ny) break;
      const bool m = zm || xm || (cy0 && ys == 0) || (cy1 && ys == NY - 1);
      const int64_t idx = xs + (int64_t)NX * ys + zs * pl;
      a.y[idx] = m ? a.x[idx] : v[r];
    }
  };

  // ---- march through z: planes 0 .. K nzl (local), element by element
  const int nplanes = K * nzl + 1;
  constexpr int NB = Cfg::NBUF;
  // prologue: planes 0 .. NB-2 in flight (one commit group each, empty groups past the end)
#pragma unroll
  for (int q = 0; q < NB - 1; ++q) {
    if (q < nplanes) load_plane(q, X0 + q * LR * LP);
    else cp_async_commit();
  }
  int buf = 0;
  for (int ez = 0; ez < nzl; ++ez) {
#pragma unroll
    for (int r = 0; r < K; ++r) {
#pragma unroll
      for (int rz = 0; rz <= K; ++rz) out[r][rz] = 0.0;
      out[r][0] = carry[r];
    }
#pragma unroll
    for (int rp = 0; rp <= K; ++rp) {
      if (rp == 0 && ez > 0) continue;
      const int pl = ez * K + rp;
      // plane pl + NB - 1 goes into the buffer last read for plane pl - 1 (all threads
      // passed the barrier after that x-stage); always commit so the group count is fixed
      if (pl + NB - 1 < nplanes) load_plane(pl + NB - 1, X0 + ((buf + NB - 1) % NB) * LR * LP);
      else cp_async_commit();
      cp_async_wait<NB - 1>();
      __syncthreads();
      double P[K], Q[K];
      plane_pq(pl, X0 + buf * LR * LP, P, Q);
      buf = (buf + 1) % NB;
      if (rp == 0) {
#pragma unroll
        for (int r = 0; r < K; ++r) {
          Pv[r] = P[r];
          Qv[r] = Q[r];
        }
        continue;
      }
      // contributions of plane rp of element ez (and, at rp == 1, of its vertex plane 0)
#pragma unroll
      for (int rz = 0; rz <= K; ++rz) {
        // coefficients for column rp (runtime) -- select from the tables with a switch-free
        // loop: rp is in 1..K
        const double mz = T.M[rz][rp], sz = T.S[rz][rp], m0 = T.M[rz][0], s0 = T.S[rz][0];
#pragma unroll
        for (int r = 0; r < K; ++r) {
          double o = out[r][rz];
          o = fma(mz, Q[r], o);
          o = fma(a.c2 * sz, P[r], o);
          if (rp == 1) {
            o = fma(m0, Qv[r], o);
            o = fma(a.c2 * s0, Pv[r], o);
          }
          out[r][rz] = o;
        }
      }
      if (rp == K) {
#pragma unroll
        for (int r = 0; r < K; ++r) {
          Pv[r] = P[r];
          Qv[r] = Q[r];
        }
      }
    }
    // planes ez K + rz, rz = 0..K-1 are complete; rz = K carries to the next element
#pragma unroll
    for (int rz = 0; rz < K; ++rz) {
      double v[K];
#pragma unroll
      for (int r = 0; r < K; ++r) v[r] = out[r][rz];
      write_plane(ez * K + rz, v);
    }
#pragma unroll
    for (int r = 0; r < K; ++r) carry[r] = out[r][K];
  }
  write_plane(K * nzl, carry);
}

// ---------------------------------------------------------------- diagonal
// d_i = sum_cells sum_q sum_ab G_ab(q) B_a(q,i) B_b(q,i),  B_a = d phi_i/d xi_a at q.
template <int K, bool DEFORMED>
__global__ void cg_diag_kernel(OpArgs a, Tab<K + 1> T) {
  FEM_PDL_ENTRY();
  constexpr int N = K + 1, N3 = N * N * N;
  const int64_t id = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (id >= a.n_cells * N3) return;
  const int64_t cell = id / N3;
  const int i = (int)(id % N3);
  const int i0 = i % N, i1 = (i / N) % N, i2 = i / (N * N);
  double d = 0.0;
  for (int q2 = 0; q2 < N; ++q2)
    for (int q1 = 0; q1 < N; ++q1)
      for (int q0 = 0; q0 < N; ++q0) {
        const double bx = T.der[q0][i0] * T.val[q1][i1] * T.val[q2][i2];
        const double by = T.val[q0][i0] * T.der[q1][i1] * T.val[q2][i2];
        const double bz = T.val[q0][i0] * T.val[q1][i1] * T.der[q2][i2];
        if (DEFORMED) {
          const int q = q0 + N * (q1 + N * q2);
          const int pl = a.glayout;
          d += a.G[g_index<N>(pl, cell, 0, q)] * bx * bx + a.G[g_index<N>(pl, cell, 3, q)] * by * by +
               a.G[g_index<N>(pl, cell, 5, q)] * bz * bz +
               2.0 * (a.G[g_index<N>(pl, cell, 1, q)] * bx * by + a.G[g_index<N>(pl, cell, 2, q)] * bx * bz +
                      a.G[g_index<N>(pl, cell, 4, q)] * by * bz);
        } else {
          const double w3 = T.w[q0] * T.w[q1] * T.w[q2];
          d += w3 * (a.c0 * bx * bx + a.c1 * by * by + a.c2 * bz * bz);
        }
      }
  const int cx = (int)(cell % a.n0);
  const int64_t r = cell / a.n0;
  const int cy = (int)(r % a.n1), cz = (int)(r / a.n1);
  const int gx = K * cx + i0, gy = K * cy + i1, gz = K * cz + i2;
  if (cg_constrained(a.bcmask, gx, gy, a.gz0 + gz, a.nn0, a.nn1, a.nn2)) return;
  atomicAdd(a.y + gx + (int64_t)a.nn0 * (gy + (int64_t)a.nn1 * gz), d);
}

// Cartesian single-rank levels: the assembled diagonal in closed form, node by node (SURVEY
// App. A: diag = sum_d c_d s_d prod_{e != d} m_e with the ASSEMBLED 1-D diagonals m, s of the
// reference mass / stiffness: M_rr, S_rr inside an element, M_KK + M_00 at an interior vertex,
// one term at a boundary vertex) -- the same sums as cg_diag_kernel without the (k+1)^3
// quadrature loop per cell node and without atomics (C4 setup: 8 launches of 32 ms before)
template <int K>
__global__ void cg_diag_cart_kernel(OpArgs a, Tab<K + 1> T) {
  FEM_PDL_ENTRY();
  constexpr int N = K + 1;
  const int64_t id = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t nn = (int64_t)a.nn0 * a.nn1 * a.nn2;
  if (id >= nn) return;
  const int g[3] = {(int)(id % a.nn0), (int)((id / a.nn0) % a.nn1), (int)(id / ((int64_t)a.nn0 * a.nn1))};
  const int nc[3] = {a.n0, a.n1, a.n2};
  double m[3], st[3];
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    const int r = g[d] % K, e = g[d] / K;
    double mm = 0.0, ss = 0.0;
#pragma unroll
    for (int q = 0; q < N; ++q) {
      const double wq = T.w[q];
      if (r != 0) {
        mm = fma(wq * T.val[q][r], T.val[q][r], mm);
        ss = fma(wq * T.der[q][r], T.der[q][r], ss);
      } else {
        if (e > 0) {
          mm = fma(wq * T.val[q][K], T.val[q][K], mm);
          ss = fma(wq * T.der[q][K], T.der[q][K], ss);
        }
        if (e < nc[d]) {
          mm = fma(wq * T.val[q][0], T.val[q][0], mm);
          ss = fma(wq * T.der[q][0], T.der[q][0], ss);
        }
      }
    }
    m[d] = mm;
    st[d] = ss;
  }
  if (cg_constrained(a.bcmask, g[0], g[1], a.gz0 + g[2], a.nn0, a.nn1, a.nn2)) return;
  a.y[id] = a.c0 * st[0] * m[1] * m[2] + a.c1 * m[0] * st[1] * m[2] + a.c2 * m[0] * m[1] * st[2];
}

// ---------------------------------------------------------------- geometry (R2)
// G_q = w_q det J J^-1 J^-T with J = (I + eps 1 grad s^T) diag(h/2):
// G_df = w det J (4 / (h_d h_f)) (delta_df - beta (g_d + g_f) + beta^2 |g|^2).
template <int K>
__global__ void geometry_kernel(MapArgs m, int n0, int n1, int64_t n_cells, Tab<K + 1> T,
                                double* __restrict__ G, unsigned long long* __restrict__ err, int glayout) {
  FEM_PDL_ENTRY();
  constexpr int N = K + 1, N3 = N * N * N;
  const int64_t id = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (id >= n_cells * N3) return;
  const int64_t cell = id / N3;
  const int q = (int)(id % N3);
  const int q0 = q % N, q1 = (q / N) % N, q2 = q / (N * N);
  const int cx = (int)(cell % n0);
  const int64_t r = cell / n0;
  const int cy = (int)(r % n1), cz = (int)(r / n1);
  const int comp[6][2] = {{0, 0}, {0, 1}, {0, 2}, {1, 1}, {1, 2}, {2, 2}};
  if (m.general) {
    // G = J^-1 (kappa w det J) J^-T from the level's cell map (N3)
    const GeoPt g = geo_point(m, cx, cy, cz, T.qp[q0], T.qp[q1], T.qp[q2]);
    double Ji[3][3];
    const double det = geo_inverse(g, Ji);
    if (!(det > 0.0)) atomicMin((unsigned long long*)err, (unsigned long long)cell);
    const double w = T.w[q0] * T.w[q1] * T.w[q2] * det * kappa_at(m, g.x);
#pragma unroll
    for (int c = 0; c < 6; ++c) {
      const int d = comp[c][0], f = comp[c][1];
      G[g_index<N>(glayout, cell, c, q)] = w * (Ji[d][0] * Ji[f][0] + Ji[d][1] * Ji[f][1] + Ji[d][2] * Ji[f][2]);
    }
    return;
  }
  const PointGeo p = map_point(m, cx, cy, cz, T.qp[q0], T.qp[q1], T.qp[q2]);
  if (!(p.fac > 0.0)) {
    // record the first bad cell (as a double, exact for < 2^53)
    atomicMin((unsigned long long*)err, (unsigned long long)cell);
  }
  const double w = T.w[q0] * T.w[q1] * T.w[q2] * p.det;
  const double g2 = p.g[0] * p.g[0] + p.g[1] * p.g[1] + p.g[2] * p.g[2];
  const double b = p.beta;
#pragma unroll
  for (int c = 0; c < 6; ++c) {
    const int d = comp[c][0], f = comp[c][1];
    const double v = (d == f ? 1.0 : 0.0) - b * (p.g[d] + p.g[f]) + b * b * g2;
    G[g_index<N>(glayout, cell, c, q)] = w * (4.0 / (m.h[d] * m.h[f])) * v;
  }
}

// ---------------------------------------------------------------- load vector (O8)
// b_i = sum_q f(x_q) phi_i(xi_q) w_q det J_q, f = pi^2 sum_d L_d^-2 prod_e sin(pi t_e(x)).
// One block per cell, (k+1)^3 threads.
template <int K, bool DG>
__global__ void rhs_kernel(MapArgs m, OpArgs a, Tab<K + 1> T) {
  FEM_PDL_ENTRY();
  constexpr int N = K + 1, N3 = N * N * N;
  __shared__ double fq[N3];
  const int64_t cell = blockIdx.x;
  const int cx = (int)(cell % a.n0);
  const int64_t r = cell / a.n0;
  const int cy = (int)(r % a.n1), cz = (int)(r / a.n1);
  for (int q = threadIdx.x; q < N3; q += blockDim.x) {
    const int q0 = q % N, q1 = (q / N) % N, q2 = q / (N * N);
    if (m.general) {
      // f = -div(kappa grad u) = kappa pi^2 sum_d L_d^-2 u - grad kappa . grad u  (N3)
      const GeoPt g = geo_point(m, cx, cy, cz, T.qp[q0], T.qp[q1], T.qp[q2]);
      double Ji[3][3], gk[3], sn[3], cs[3];
      const double det = geo_inverse(g, Ji);
      const double kap = kappa_at(m, g.x, gk);
      double lap = 0.0;
#pragma unroll
      for (int d = 0; d < 3; ++d) {
        sincospi((g.x[d] - m.lo[d]) / m.L[d], &sn[d], &cs[d]);
        lap += 1.0 / (m.L[d] * m.L[d]);
      }
      const double u = sn[0] * sn[1] * sn[2];
      const double gu[3] = {M_PI / m.L[0] * cs[0] * sn[1] * sn[2], M_PI / m.L[1] * sn[0] * cs[1] * sn[2],
                            M_PI / m.L[2] * sn[0] * sn[1] * cs[2]};
      const double f = kap * M_PI * M_PI * lap * u - (gk[0] * gu[0] + gk[1] * gu[1] + gk[2] * gu[2]);
      fq[q] = f * T.w[q0] * T.w[q1] * T.w[q2] * det;
      continue;
    }
    const PointGeo p = map_point(m, cx, cy, cz, T.qp[q0], T.qp[q1], T.qp[q2]);
    double u = 1.0, lap = 0.0;
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      const double xd = p.xh[d] + m.eps * p.s;  // physical coordinate
      u *= sinpi((xd - m.lo[d]) / m.L[d]);
      lap += 1.0 / (m.L[d] * m.L[d]);
    }
    fq[q] = M_PI * M_PI * lap * u * T.w[q0] * T.w[q1] * T.w[q2] * p.det;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < N3; i += blockDim.x) {
    const int i0 = i % N, i1 = (i / N) % N, i2 = i / (N * N);
    double s = 0.0;
    for (int q2 = 0; q2 < N; ++q2)
      for (int q1 = 0; q1 < N; ++q1) {
        const double v12 = T.val[q1][i1] * T.val[q2][i2];
        for (int q0 = 0; q0 < N; ++q0) s += fq[q0 + N * (q1 + N * q2)] * T.val[q0][i0] * v12;
      }
    if (DG) {
      a.y[cell * N3 + i] = s;
    } else {
      const int gx = K * cx + i0, gy = K * cy + i1, gz = K * cz + i2;
      if (!cg_constrained(a.bcmask, gx, gy, a.gz0 + gz, a.nn0, a.nn1, a.nn2))
        atomicAdd(a.y + gx + (int64_t)a.nn0 * (gy + (int64_t)a.nn1 * gz), s);
    }
  }
}

// ---------------------------------------------------------------- Dirichlet rows
// y_c = x_c (x == nullptr: y_c = val) on the boundary planes of Dirichlet sides,
// restricted to the rank's owned node planes [0, nzo) (global plane gz0 + local).
__global__ void set_constrained_kernel(const double* __restrict__ x, double val, double* __restrict__ y,
                                       int nn0, int nn1, int nzo, int gz0, int nn2g, int bcmask) {
  FEM_PDL_ENTRY();
  const int side = blockIdx.y;
  if (!(bcmask & (1 << side))) return;
  const int d = side / 2;
  int fixed;
  if (d < 2) {
    fixed = (side % 2) ? ((d == 0 ? nn0 : nn1) - 1) : 0;
  } else {
    fixed = ((side % 2) ? nn2g - 1 : 0) - gz0;   // local plane of the global boundary plane
    if (fixed < 0 || fixed >= nzo) return;
  }
  const int na = (d == 0) ? nn1 : nn0;
  const int nb = (d == 2) ? nn1 : nzo;
  const int64_t id = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (id >= (int64_t)na * nb) return;
  const int ia = (int)(id % na), ib = (int)(id / na);
  int g[3];
  g[d] = fixed;
  if (d == 0) { g[1] = ia; g[2] = ib; }
  if (d == 1) { g[0] = ia; g[2] = ib; }
  if (d == 2) { g[0] = ia; g[1] = ib; }
  const int64_t idx = g[0] + (int64_t)nn0 * (g[1] + (int64_t)nn1 * g[2]);
  y[idx] = x ? x[idx] : val;
}

// ---------------------------------------------------------------- launchers
namespace {

OpArgs op_args(const fem_ctx* h, const Level& L, const double* x, double* y) {
  OpArgs a;
  a.x = x;
  a.y = y;
  a.G = L.G;
  a.n0 = L.n[0];
  a.n1 = L.n[1];
  a.n2 = L.n[2];
  a.nn0 = L.nn[0];
  a.nn1 = L.nn[1];
  a.nn2 = L.dist ? h->k * L.nzg + 1 : L.nn[2];
  a.gz0 = h->k * L.cz0;
  a.glayout = L.glayout;
  a.g_direct = h->g_direct ? 1 : 0;
  int mask = 0;
  for (int s = 0; s < 6; ++s)
    if (h->mesh.bc[s] == FEM_BC_DIRICHLET) mask |= 1 << s;
  a.bcmask = mask;
  a.n_cells = L.n_cells;
  a.cell0 = 0;
  a.cell1 = L.n_cells;
  a.c0 = L.cart[0];
  a.c1 = L.cart[1];
  a.c2 = L.cart[2];
  return a;
}

MapArgs map_args(const fem_ctx* h, const Level& L) {
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

template <int K>
void apply_k(fem_ctx* h, const Level& L, const double* x, double* y, int64_t r0, int64_t r1) {
  constexpr int N = K + 1, C = CPB<K>::value;
  OpArgs a = op_args(h, L, x, y);
  const bool full = r0 == 0 && r1 == L.n_cells;
  a.cell0 = r0;
  a.cell1 = r1;
  // TMA staging of 8-cell G blocks needs launches that start on a block boundary; a
  // launch of at most FEM_TMA_MIN_BLOCKS blocks reads G directly (4 instead of 3
  // resident blocks per SM: a level that fits one wave is latency-, not traffic-bound)
  // (the staged copy is one 8-cell chunk per block: any other cells-per-block count
  // (FEM_CPB4) must read G directly)
  if (a.glayout == kGLayoutCell8 &&
      (C != kCell8 || r0 % kCell8 != 0 || (r1 - r0 + C - 1) / C <= (int64_t)h->tma_min_blocks))
    a.g_direct = 1;
  if (r1 <= r0) return;
  const Tab<N> T = make_tab<N>(h->tab);
  const dim3 block(N * N, C);
  const dim3 cblock = cart_cell_fast<K>() ? dim3(C, N * N) : block;   // Cartesian element kernel
  const dim3 lblock = line_cell_fast<K>() ? dim3(C, line_tpc<K>()) : dim3(line_tpc<K>(), C);   // line kernel
  const int64_t grid = (r1 - r0 + C - 1) / C;
  if (L.cartesian && !h->general_path) {
    KronTab<N> KT;
    for (int i = 0; i < N; ++i)
      for (int j = 0; j < N; ++j) {
        double m = 0.0, s = 0.0;
        for (int q = 0; q < N; ++q) {
          m += h->tab.qw[q] * h->tab.val[q][i] * h->tab.val[q][j];
          s += h->tab.qw[q] * h->tab.der[q][i] * h->tab.der[q][j];
        }
        KT.M[i][j] = m;
        KT.S[i][j] = s;
      }
    if (!L.dist && h->stencil && full) {
      using Cfg = StencilCfg<K>;
      const size_t smb = sizeof(double) * Cfg::SMEM;
      smem_attr(reinterpret_cast<const void*>(cg_stencil_kernel<K>), (size_t)((int)smb));
      const dim3 sg((unsigned)((L.n[0] + 1 + Cfg::TEX - 1) / Cfg::TEX), (unsigned)((L.n[1] + 1 + Cfg::TEY - 1) / Cfg::TEY));
      launch_pdl(h, cg_stencil_kernel<K>, sg, Cfg::THREADS, smb, a, KT);
      count_launch();
      check_launch("cg_stencil_kernel");
      return;
    }
    const size_t sm = sizeof(double) * cart_cell_stride<N>() * C;
    // z-chunks: zero the chunk's node planes (all but the bottom one, which the previous
    // chunk has accumulated into) right before its cells are applied, so that the
    // atomic adds hit lines that are resident in L2 instead of re-reading y from HBM.
    const int64_t plane = (int64_t)L.nn[0] * L.nn[1];
    const int64_t layer = (int64_t)L.n[0] * L.n[1];
    const int lz = h->chunk_layers > 0 ? h->chunk_layers : L.n[2];
    if (!full) {   // a sub-range of a z-slab apply: y has been zeroed by the caller
      launch_pdl(h, cg_cart_kernel<K>, (unsigned)grid, cblock, sm, a, KT, r0, r1);
      count_launch();
      check_launch("cg_cart_kernel");
      return;
    }
    for (int z0 = 0; z0 < L.n[2]; z0 += lz) {
      const int z1 = std::min(z0 + lz, L.n[2]);
      const int64_t p0 = z0 == 0 ? 0 : (int64_t)K * z0 + 1, p1 = (int64_t)K * z1 + 1;
      if (!h->y_is_zero) launch_zero(h, y + p0 * plane, (p1 - p0) * plane);
      const int64_t c0 = layer * z0, c1 = layer * z1;
      launch_pdl(h, cg_cart_kernel<K>, (unsigned)((c1 - c0 + C - 1) / C), cblock, sm, a, KT, c0, c1);
      count_launch();
      check_launch("cg_cart_kernel");
    }
  } else if (L.cartesian) {
    const size_t sm = sizeof(double) * line_cell_stride<N>() * C;
    launch_pdl(h, cg_apply_kernel<K, false>, (unsigned)grid, lblock, sm, a, T);
  } else if (L.glayout == kGLayoutXLine) {
    const size_t sm = sizeof(double) * dline_cell_stride<N>() * C;
    smem_attr(reinterpret_cast<const void*>(cg_dline_kernel<K>), (size_t)((int)sm));
    launch_pdl(h, cg_dline_kernel<K>, (unsigned)grid, block, sm, a, T);
  } else if (L.glayout == kGLayoutPlane) {
    if constexpr (K <= 4) {
      if (!full) throw Error{FEM_E_ARG, "the plane kernel applies whole levels only"};
      const size_t sm = sizeof(double) * (PlanePad<N>::CS * kGroupCells + 3 * 6 * N * N * kGroupCells);
      smem_attr(reinterpret_cast<const void*>(cg_plane_kernel<K, true>), (size_t)((int)sm));
      const int64_t groups = (L.n_cells + kGroupCells - 1) / kGroupCells;
      launch_pdl(h, cg_plane_kernel<K, true>, (unsigned)groups, N * kGroupCells, sm, a, T);
    }
  } else if (h->cgf.on) {
    const size_t sm = sizeof(double) * (line_g_offset<N, C>() + (a.g_direct ? 0 : 6 * N * N * N * C));
    smem_attr(reinterpret_cast<const void*>(cg_apply_fused_kernel<K>), (size_t)((int)(sizeof(double) * (line_g_offset<N, C>() + 6 * N * N * N * C))));
    launch_pdl(h, cg_apply_fused_kernel<K>, (unsigned)grid, lblock, sm, a, T, h->cgf);
  } else if (h->cg_geo_fly && !mesh_general(h->mesh)) {
    GeoFly g;
    for (int d = 0; d < 3; ++d) {
      g.lo[d] = h->mesh.lo[d];
      g.L[d] = h->mesh.hi[d] - h->mesh.lo[d];
      g.h[d] = L.h[d];
      g.c.pl[d] = M_PI / g.L[d];
    }
    g.cz0 = L.cz0;
    g.c.eps = h->mesh.deform_eps;
    g.c.hh = (0.5 * L.h[0]) * (0.5 * L.h[1]) * (0.5 * L.h[2]);
    const int ab[6][2] = {{0, 0}, {0, 1}, {0, 2}, {1, 1}, {1, 2}, {2, 2}};
    for (int c = 0; c < 6; ++c) g.c.ih[c] = 4.0 / (L.h[ab[c][0]] * L.h[ab[c][1]]);
    const size_t sm = sizeof(double) * line_g_offset<N, C>();
    smem_attr(reinterpret_cast<const void*>(cg_apply_fly_kernel<K>), sm);
    launch_pdl(h, cg_apply_fly_kernel<K>, (unsigned)grid, lblock, sm, a, T, g);
  } else {
    const size_t sm = sizeof(double) * (line_g_offset<N, C>() + (a.g_direct ? 0 : 6 * N * N * N * C));
    smem_attr(reinterpret_cast<const void*>(cg_apply_kernel<K, true>), (size_t)((int)(sizeof(double) * (line_g_offset<N, C>() + 6 * N * N * N * C))));
    launch_pdl(h, cg_apply_kernel<K, true>, (unsigned)grid, lblock, sm, a, T);
  }
  count_launch();
  check_launch("cg_apply_kernel");
}

template <int K>
void diag_k(fem_ctx* h, Level& L) {
  constexpr int N = K + 1;
  const OpArgs a = op_args(h, L, nullptr, L.diag);
  const Tab<N> T = make_tab<N>(h->tab);
  const int64_t tot = L.n_cells * N * N * N;
  const unsigned grid = (unsigned)((tot + 255) / 256);
  if (L.cartesian && !L.dist && !h->general_path) {
    const int64_t nn = (int64_t)L.nn[0] * L.nn[1] * L.nn[2];
    cg_diag_cart_kernel<K><<<(unsigned)((nn + 255) / 256), 256, 0, h->stream>>>(a, T);
  } else if (L.cartesian)
    cg_diag_kernel<K, false><<<grid, 256, 0, h->stream>>>(a, T);
  else
    cg_diag_kernel<K, true><<<grid, 256, 0, h->stream>>>(a, T);
  count_launch();
  check_launch("cg_diag_kernel");
}

template <int K>
void geometry_k(fem_ctx* h, Level& L) {
  constexpr int N = K + 1;
  const Tab<N> T = make_tab<N>(h->tab);
  const int64_t tot = L.n_cells * N * N * N;
  geometry_kernel<K><<<(unsigned)((tot + 255) / 256), 256, 0, h->stream>>>(
      map_args(h, L), L.n[0], L.n[1], L.n_cells, T, L.G, h->geom_err, L.glayout);
  count_launch();
  check_launch("geometry_kernel");
}

template <int K>
void rhs_k(fem_ctx* h, const Level& L, double* b) {
  constexpr int N = K + 1;
  const Tab<N> T = make_tab<N>(h->tab);
  const OpArgs a = op_args(h, L, nullptr, b);
  const int threads = N * N * N < 128 ? 128 : (N * N * N > 512 ? 512 : N * N * N);
  if (h->method == FEM_CG)
    rhs_kernel<K, false><<<(unsigned)L.n_cells, threads, 0, h->stream>>>(map_args(h, L), a, T);
  else
    rhs_kernel<K, true><<<(unsigned)L.n_cells, threads, 0, h->stream>>>(map_args(h, L), a, T);
  count_launch();
  check_launch("rhs_kernel");
}

#define FEM_DISPATCH_K(k, fn, ...)              \
  switch (k) {                                  \
    case 1: fn<1>(__VA_ARGS__); break;          \
    case 2: fn<2>(__VA_ARGS__); break;          \
    case 3: fn<3>(__VA_ARGS__); break;          \
    case 4: fn<4>(__VA_ARGS__); break;          \
    case 5: fn<5>(__VA_ARGS__); break;          \
    case 6: fn<6>(__VA_ARGS__); break;          \
    case 7: fn<7>(__VA_ARGS__); break;          \
    case 8: fn<8>(__VA_ARGS__); break;          \
    default: throw Error{FEM_E_ARG, "degree out of range"}; \
  }

}  // namespace

void launch_cg_apply(fem_ctx* h, const Level& L, const double* x, double* y, int64_t c0, int64_t c1) {
  if (c1 < 0) c1 = L.n_cells;
  FEM_DISPATCH_K(h->k, apply_k, h, L, x, y, c0, c1);
}

void launch_cg_diagonal(fem_ctx* h, Level& L) { FEM_DISPATCH_K(h->k, diag_k, h, L); }

void launch_geometry(fem_ctx* h, Level& L) { FEM_DISPATCH_K(h->k, geometry_k, h, L); }

void launch_rhs(fem_ctx* h, const Level& L, double* b) { FEM_DISPATCH_K(h->k, rhs_k, h, L, b); }

namespace {
void set_constrained_impl(fem_ctx* h, const Level& L, const double* x, double v, double* y) {
  const OpArgs a = op_args(h, L, x, y);
  if (a.bcmask == 0) return;
  const int nzo = (int)(L.n_dofs / ((int64_t)L.nn[0] * L.nn[1]));   // owned node planes
  int64_t mx = std::max<int64_t>((int64_t)L.nn[0] * L.nn[1],
                                 std::max<int64_t>((int64_t)L.nn[0] * nzo, (int64_t)L.nn[1] * nzo));
  dim3 grid((unsigned)((mx + 255) / 256), 6);
  launch_pdl(h, set_constrained_kernel, grid, 256, 0, x, v, y, L.nn[0], L.nn[1], nzo, a.gz0, a.nn2, a.bcmask);
  count_launch();
  check_launch("set_constrained_kernel");
}
}  // namespace

void launch_set_constrained(fem_ctx* h, const Level& L, const double* x, double* y) {
  set_constrained_impl(h, L, x, 1.0, y);
}

void launch_set_constrained_value(fem_ctx* h, const Level& L, double v, double* y) {
  set_constrained_impl(h, L, nullptr, v, y);
}

}  // namespace fem
