// Cartesian CG levels: the operator as an atomic-free ASSEMBLED Kronecker stencil with
// warp-specialised x / (y, z) stages (K1t; the C4 kernel).
//
// On a Cartesian level every cell has the same element matrix, the Kronecker sum
//     K^e = c0 S(x)M(x)M + c1 M(x)S(x)M + c2 M(x)M(x)S,  c_d = det J (2/h_d)^2
// (exact, since the (k+1)-point Gauss rule integrates the Q_k stiffness
// and mass exactly on affine cells), so the ASSEMBLED operator is the same
// Kronecker sum of the assembled 1-D matrices M1, S1 (the element set of a tensor grid
// is the product of the 1-D element sets):
//     y = M1_z Q + S1^z_z P,   P = M1_y A,   Q = M1_y B + S1^y_y A,
//     A = M1_x x~,  B = S1^x_x x~,            S^d = c_d S,
// x~ = x with the Dirichlet entries read as 0 (reading R5).  The 1-D assembled rows
// are banded: node K e + r (r = 1..K-1) couples to element e's K+1 nodes, the vertex
// K e to the 2K+1 nodes of elements e-1 and e ("slot" form; the vertex row of an
// interior vertex uses the pre-summed coefficients M[K][j] | M[K][K]+M[0][0] | M[0][j]).
// 7 banded sweeps, ~46 DFMA per node at k = 4 (the cell-wise form needs 7 (k+1)^4 per
// cell = 68 per node, plus atomics that read y back: 1.47x the algorithmic DRAM bytes).
//
// Block = a tile of SX x SY element slots in (x, y) (output nodes [X0, X0 + K SX) x
// [Y0, Y0 + K SY), plus the far vertex column / row on the last tile) and EZ element
// layers in z, marching through z plane by plane:
//   * X warps (NXW): cp.async the x~ plane (tile + K-node halo, zero-filled outside the
//     domain and on constrained nodes) NB-1 planes ahead into shared memory, then the
//     x-stage A, B for all rows of the tile and its y-halo into a double-buffered A/B
//     plane;
//   * Y/Z warps (one thread per output column and y slot): the y-stage P, Q of the
//     thread's K rows from the A/B plane, then the z-direction element by element in
//     registers: plane r' of z-element e adds M[r][r'] Q + S^z[r][r'] P to the K+1
//     accumulators of the element's planes; the vertex plane carries to the next element.
//     Every output node is written exactly once (no atomics, no zero fill): x is read
//     once from DRAM (the halos mostly from L2), y written once -- the algorithmic
//     16 B/DoF.
// Producer/consumer hand-off through named barriers (FULL / EMPTY per A/B buffer), so
// the x-stage of plane p+1 overlaps the y/z stages of plane p on other warps.
// A z-chunk of EZ layers recomputes one halo layer below it (the bottom vertex plane's
// contribution from the element underneath); no output is written twice.
//
// Epilogues (template MODE): 0 = y = A x (constrained rows 0; y_c = x_c, when asked for, by
// the boundary-only launch_set_constrained kernel, so the epilogue never reads x);
// 1 = fused Chebyshev step (reading R8's three-term form):
//     x_new = x + c1 (x - x_old) + c2 D^-1 (b - A x)   (D^-1 = 0 on constrained rows).
#include <algorithm>

#include "device_common.cuh"

namespace fem {

// Pipeline depths per MODE (r02c A/B on C4, apply / smoother step): A/B planes in flight
// (x-stage -> y-stage hand-off) 2 for the apply (3: 766 vs 754 us apply, 2044 vs 1706 us smoother in
// r02c; re-measured at the end of round 2 on the final fused step: 3 is 1% faster there, 1443 -> 1428 us
// per smoother step, and together with the symmetric tables 1443 -> 1412-1425 us: 3 for MODE 1 / 2; MODE 0 re-measured too:
// 3 planes 664.5 -> 647.2 us per C4 apply, solve unchanged within noise: 3);
// x~ planes in flight 3 (4: 754 -> 748 us apply; smoother 1706 -> 1667 us with one element
// of L2 prefetch; 2: 1863 us).  The LR * SX - THREADS extra x-stage items of a plane
// rotate over the warps with the plane (FEM_ST_ROT; fixed on warps 0-1: 766 vs 754 us):
// every plane's EMPTY / FULL hand-off otherwise waited on the same two slow warps.
// Tried and dropped (MODE 1): parking an element's planes 1..K-1 in a 24 KB shared stash
// and writing one plane per following step (2023 us; with the operands loaded one step
// early 2517 us, spills) -- extra shared memory costs this kernel more than the burst.
#ifndef FEM_ST_NAB0
#define FEM_ST_NAB0 3
#endif
#ifndef FEM_ST_NAB1
#define FEM_ST_NAB1 3
#endif
#ifndef FEM_ST_NB0
#define FEM_ST_NB0 3
#endif
#ifndef FEM_ST_NB1
#define FEM_ST_NB1 3
#endif
#ifndef FEM_ST_ROT
#define FEM_ST_ROT 1
#endif
#ifndef FEM_ST_SYM   // exactly symmetric 1-D tables (RefTab) in the apply
#define FEM_ST_SYM 1
#endif
#ifndef FEM_ST_SYMALL   // ... and in the fused Chebyshev step (slower there in r02k, 1% faster on the final kernel)
#define FEM_ST_SYMALL 1
#endif
template <int K, int MODE = 0>
struct StCfg {
  static constexpr int N = K + 1;
  static constexpr int SX = 32 / K;               // x slots per tile (<= 32 output columns)
  static constexpr int SY = 8;                    // y slots per tile = warps per block
  static constexpr int TX = K * SX, TY = K * SY;  // output columns / rows of a tile
  static constexpr int LC = TX + K + 1;           // loaded columns [X0 - K, X0 + TX]
  static constexpr int LR = TY + K + 1;           // loaded rows (and A/B rows) [Y0 - K, Y0 + TY]
  static constexpr int LP = LC | 1;               // odd row strides: conflict-free column walks
  static constexpr int ABP = TX | 1;
  static constexpr int THREADS = 32 * SY;         // thread = (output column, y slot)
  static constexpr int NB = MODE == 0 ? FEM_ST_NB0 : FEM_ST_NB1;   // x~ planes in flight
  static constexpr int NLD = (LR * LC + THREADS - 1) / THREADS;
  static constexpr int NAB = MODE == 0 ? FEM_ST_NAB0 : FEM_ST_NAB1;
  static constexpr int NBAR = 2 * NAB + NB;
  static constexpr int SMEM = NB * LR * LP + NAB * 2 * LR * ABP + NBAR + 8;   // doubles (+ mbarriers)
  // two blocks per SM: 16 warps, 4 per SM sub-partition (16K registers each)
  static constexpr int MAXREG = 128;
};

// Compile-time reference tables (GLL Lagrange basis, (k+1)-point Gauss rule; the same
// definitions as build_tables() in tables.cu, evaluated by the compiler): folded into
// the DFMAs as constant-bank / uniform-register operands, so no vector register holds a
// coefficient (with the 127 doubles passed as kernel parameters ptxas copied them into
// vector registers and spilled).
constexpr double ct_cos(double x) {   // |x| <= pi
  double s = 0.0, t = 1.0;
  for (int k = 0; k < 40; ++k) {
    s += t;
    t *= -x * x / ((2.0 * k + 1.0) * (2.0 * k + 2.0));
  }
  return s;
}
constexpr void ct_legendre(int n, double x, double& p, double& dp) {
  double p0 = 1.0, p1 = x;
  for (int k = 2; k <= n; ++k) {
    const double p2 = ((2.0 * k - 1.0) * x * p1 - (k - 1.0) * p0) / k;
    p0 = p1;
    p1 = p2;
  }
  p = n == 0 ? 1.0 : p1;
  dp = n == 0 ? 0.0 : n * (x * p1 - p0) / (x * x - 1.0);
}
template <int K, bool SYM = false>
struct RefTab {
  static constexpr int N = K + 1;
  double gll[N] = {}, qp[N] = {}, qw[N] = {};
  double M[N][N] = {}, S[N][N] = {};      // M_ij = sum_q w_q phi_i phi_j, S_ij = sum_q w_q phi_i' phi_j'
  double Mv[2 * N - 1] = {}, Sv[2 * N - 1] = {};   // interior-vertex rows: elements e-1 and e pre-summed
  constexpr RefTab() {
    constexpr double pi = 3.14159265358979323846;
    for (int i = 0; i < N; ++i) {   // Gauss-Legendre, Newton from the Chebyshev-type guess
      double x = -ct_cos(pi * (i + 0.75) / (N + 0.5)), p = 0.0, dp = 0.0;
      for (int it = 0; it < 60; ++it) {
        ct_legendre(N, x, p, dp);
        x -= p / dp;
      }
      ct_legendre(N, x, p, dp);
      qp[i] = x;
      qw[i] = 2.0 / ((1.0 - x * x) * dp * dp);
    }
    gll[0] = -1.0;
    gll[K] = 1.0;
    for (int i = 1; i < K; ++i) {   // roots of P_K': Newton with P_K'' from the Legendre equation
      double x = -ct_cos(pi * i / K), p = 0.0, dp = 0.0;
      for (int it = 0; it < 60; ++it) {
        ct_legendre(K, x, p, dp);
        x -= dp * (1.0 - x * x) / (2.0 * x * dp - K * (K + 1.0) * p);
      }
      gll[i] = x;
    }
    double phi[N][N] = {}, dphi[N][N] = {};
    for (int q = 0; q < N; ++q)
      for (int i = 0; i < N; ++i) {
        double v = 1.0, d = 0.0;
        for (int j = 0; j < N; ++j) {
          if (j == i) continue;
          double t = 1.0;
          for (int m = 0; m < N; ++m)
            if (m != i && m != j) t *= (qp[q] - gll[m]) / (gll[i] - gll[m]);
          d += t / (gll[i] - gll[j]);
          v *= (qp[q] - gll[j]) / (gll[i] - gll[j]);
        }
        phi[q][i] = v;
        dphi[q][i] = d;
      }
    for (int i = 0; i < N; ++i)
      for (int j = 0; j < N; ++j) {
        double m = 0.0, s = 0.0;
        for (int q = 0; q < N; ++q) {
          m += qw[q] * phi[q][i] * phi[q][j];
          s += qw[q] * dphi[q][i] * dphi[q][j];
        }
        M[i][j] = m;
        S[i][j] = s;
      }
    // SYM: exact symmetry M_ij = M_ji = M_{K-i,K-j} (S likewise) -- mathematically so (GLL
    // nodes and Gauss points symmetric about 0), in floating point up to an ulp.  With one
    // value per orbit the k = 4 matrices hold 9 distinct coefficients instead of 25, and the
    // compiler reuses registers across the sweeps instead of re-materialising near-equal
    // literals (2 IMAD.MOV / UMOV per use)
    if (SYM) {
      for (int i = 0; i < N; ++i)
        for (int j = 0; j < N; ++j) {
          int bi = i, bj = j;
          const int ci[3] = {j, K - i, K - j}, cj[3] = {i, K - j, K - i};
          for (int t = 0; t < 3; ++t)
            if (ci[t] < bi || (ci[t] == bi && cj[t] < bj)) bi = ci[t], bj = cj[t];
          M[i][j] = M[bi][bj];
          S[i][j] = S[bi][bj];
        }
    }
    for (int j = 0; j <= 2 * K; ++j) {
      Mv[j] = (j <= K ? M[K][j] : 0.0) + (j >= K ? M[0][j - K] : 0.0);
      Sv[j] = (j <= K ? S[K][j] : 0.0) + (j >= K ? S[0][j - K] : 0.0);
    }
  }
};
template <int K, bool SYM = false>
__device__ constexpr RefTab<K, SYM> kRef{};
// the same tables in the constant bank: DFMAs take them as uniform-register operands
// loaded two doubles per LDCU.128 (compile-time literals cost two UMOVs per use)
template <int K>
__constant__ RefTab<K> cRef = RefTab<K>();
// MODE 1 epilogue operands: prefetch.global.L2 per 128-byte line at the element's start
// (C4 solve, 5 its, NB 4: bulk cp.async.bulk.prefetch.L2 one element ahead 141.2 ms, none
// 132.5, per line one ahead 131.8, two ahead 125.1, three 133.1, four 135.3; with NB 3:
// one ahead 122.2 ms, two ahead 124.4, at the element's start 118.4 ms: smoother step 1600 us,
// DRAM 4.7 GB read vs 3.24 GB algorithmic.  Reading the epilogue's x from copies parked out of
// the x~ tile brought DRAM reads to 3.39 GB but the step to 1712 us: not bandwidth-bound)
#ifndef FEM_ST_PF_AHEAD
#define FEM_ST_PF_AHEAD 0
#endif
#ifndef FEM_ST_PF_X   // also prefetch x
#define FEM_ST_PF_X 1
#endif
#ifndef FEM_ST_PF_LINES
#define FEM_ST_PF_LINES 1
#endif
#ifndef FEM_ST_SUSPEND_NS
#define FEM_ST_SUSPEND_NS 100000
#endif
// MODE 1 / 2 epilogue (write_element): 64-bit node offsets.  Plane base + 32-bit offsets, the
// form that helps the x~ copies and the MODE 0 stores, measured 1596-1842 us per C4 smoother
// step vs 1480 us (with __ldg / ld.global / generic / .cg loads alike).
#ifndef FEM_ST_EPI_DV   // the rows' D^-1 loads issued with the x, x_old, b loads (1451 vs 1481 us)
#define FEM_ST_EPI_DV 1
#endif
// (prefetch.global.L1 of the operands 1 / 2 / all planes ahead inside the epilogue: 1459 / 1473
// / 1469 vs 1447 us)
// (plane q+1's operand loads issued before plane q's stores, in registers: 92 B of spills,
// 1558 vs 1445 us; the __restrict__ function form below: neutral, the compiler still keeps the
// plane order)
#ifndef FEM_ST_EPI_FN   // __restrict__-parameter function form
#define FEM_ST_EPI_FN 0
#endif
#ifndef FEM_ST_WP   // MODE 0 store: 1 st.global.wb, 0 generic store
#define FEM_ST_WP 1
#endif
#ifndef FEM_ST_CBANK
#define FEM_ST_CBANK 0
#endif
#if FEM_ST_CBANK
#define ST_TAB(K) cRef<K>  // (SYMT unused)
#else
#define ST_TAB(K) kRef<K, SYMT>
#endif

struct StArgs {
  const double* __restrict__ x;
  double* __restrict__ y;          // MODE 0: A x;  MODE 1: x_new
  const double* __restrict__ xo;   // MODE 1: x_old (nullptr: none)
  const double* __restrict__ b;    // MODE 1
  const double* __restrict__ dinv; // MODE 1 (unused when dcls is set)
  const double* __restrict__ dcls; // MODE 1: D^-1 per node class, (K+2)^3 (api.cu), or nullptr
  double c1, c2;                   // MODE 1
  double c0, cy, cz;               // Cartesian metric det J (2/h_d)^2 of x, y, z
  int nx, ny, nz;                  // cells
  int NX, NY, NZ;                  // nodes
  int bcmask;
  int ez_per_block;
};

__device__ __forceinline__ void bar_sync_n(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ void bar_arrive_n(int id, int n) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ void st_cp_async8(void* dst, const void* src, bool valid) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(smem_u32(dst)), "l"(src),
               "r"(valid ? 8 : 0)
               : "memory");
}
__device__ __forceinline__ void st_cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int W>
__device__ __forceinline__ void st_cp_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(W) : "memory"); }

enum { kBarX = 1, kBarFull = 2, kBarEmpty = 4 };

// a plane's base pointer made opaque to the compiler, so that an address is formed as
// plane base + 32-bit in-plane offset (one IMAD.WIDE / LEA pair) instead of the 64-bit
// re-associated (plane offset + node offset) * 8 + array base (5 instructions per access;
// NX * NY < 2^31 is checked by use_stencil2)
template <typename T>
__device__ __forceinline__ T* st_plane(T* p) {
  asm("mov.b64 %0, %0;" : "+l"(p));
  return p;
}

// banded 1-D row of slot node r from 2K+1 consecutive values v (v[0] = node K(e-1)):
// r = 0 the vertex (elements e-1: left, e: right), r >= 1 element e only.  STIFF selects
// the reference stiffness S instead of the mass M.
template <int K, bool STIFF, bool SYMT>
__device__ __forceinline__ double band_row(const double* v, int r, bool both, bool left) {
  double s = 0.0;
  if (r == 0) {
    if (both) {   // two half-length chains (DFMA latency), one extra add
      double s2 = 0.0;
#pragma unroll
      for (int j = 0; j < K; ++j) s = fma(STIFF ? ST_TAB(K).Sv[j] : ST_TAB(K).Mv[j], v[j], s);
#pragma unroll
      for (int j = K; j <= 2 * K; ++j) s2 = fma(STIFF ? ST_TAB(K).Sv[j] : ST_TAB(K).Mv[j], v[j], s2);
      s += s2;
    } else if (left) {
#pragma unroll
      for (int j = 0; j <= K; ++j) s = fma(STIFF ? ST_TAB(K).S[K][j] : ST_TAB(K).M[K][j], v[j], s);
    } else {
#pragma unroll
      for (int j = 0; j <= K; ++j) s = fma(STIFF ? ST_TAB(K).S[0][j] : ST_TAB(K).M[0][j], v[K + j], s);
    }
  } else {
#pragma unroll
    for (int j = 0; j <= K; ++j) s = fma(STIFF ? ST_TAB(K).S[r][j] : ST_TAB(K).M[r][j], v[K + j], s);
  }
  return s;
}

// wait for the phase with the given parity; the suspend-time hint lets the warp sleep in
// the barrier unit until the phase completes instead of spinning on try_wait (the spin
// loop cost ~10% of the issue slots of this issue-bound kernel)
__device__ __forceinline__ void mbar_wait_sleep(uint64_t* bar, uint32_t phase) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(phase), "r"(FEM_ST_SUSPEND_NS)
      : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
// arrive on bar when all of this thread's prior cp.async copies have landed
__device__ __forceinline__ void mbar_arrive_cp_async(uint64_t* bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// MODE 1 / 2 epilogue of one z-element as a function with __restrict__ parameters: the
// compiler may then issue a plane's operand loads ahead of the previous plane's stores
template <int K, int MODE>
__device__ __forceinline__ void st_write_element(const double* __restrict__ x, const double* __restrict__ xo,
                                                 const double* __restrict__ b, const double* __restrict__ dcls,
                                                 double* __restrict__ y, const double (&out)[K][K + 1], int rowo0,
                                                 int64_t NXY, int NX, int NZ, uint32_t rvalid, const int (&clxy)[K],
                                                 int ez, int nq, double c1, double c2, double cy) {
#pragma unroll
  for (int q = 0; q <= K; ++q) {
    if (q >= nq) break;
    const int pz = K * ez + q;
    const int cz = pz == 0 ? 0 : pz == NZ - 1 ? K + 1 : (pz % K == 0 ? K : pz % K);
    const int clz = (K + 2) * (K + 2) * cz;
    const int64_t po = rowo0 + NXY * pz;
    double xv[K], xov[K], bv[K], dv[K];
#pragma unroll
    for (int r = 0; r < K; ++r) {
      const bool ok = (rvalid >> r) & 1u;
      const int64_t o = po + (int64_t)NX * r;
      xv[r] = ok ? x[o] : 0.0;
      xov[r] = MODE == 1 && ok ? xo[o] : 0.0;
      bv[r] = ok ? b[o] : 0.0;
      dv[r] = dcls[clxy[r] + clz];
    }
#pragma unroll
    for (int r = 0; r < K; ++r) {
      if (!((rvalid >> r) & 1u)) continue;
      const double v = cy * out[r][q];
      y[po + (int64_t)NX * r] = fma(c2 * dv[r], bv[r] - v, fma(c1, xv[r] - xov[r], xv[r]));
    }
  }
}

template <int K, int MODE, bool ISO>
__global__ void __launch_bounds__(StCfg<K>::THREADS) __maxnreg__(StCfg<K>::MAXREG)
    cg_stencil2_kernel(StArgs a) {
  FEM_PDL_ENTRY();
  using C = StCfg<K, MODE>;
  // exactly symmetric tables for the apply (C4 665 vs 683 us); the fused step measured slower
  // with them (1530 vs 1482 us: register allocation), so it keeps the computed ones
  constexpr bool SYMT = FEM_ST_SYM && (MODE == 0 || FEM_ST_SYMALL);
  constexpr int N = K + 1, SX = C::SX, LR = C::LR, LC = C::LC, LP = C::LP, ABP = C::ABP, NB = C::NB;
  constexpr int NAB = C::NAB;
  extern __shared__ double smem[];
  double* Xt = smem;                           // [NB][LR][LP]
  double* AB = smem + NB * LR * LP;            // [2 buffers][A, B][LR][ABP]
  uint64_t* bars = reinterpret_cast<uint64_t*>(AB + NAB * 2 * LR * ABP);
  uint64_t* full = bars;                       // [NAB] A/B buffer written by every thread
  uint64_t* empty = bars + NAB;                // [NAB] A/B buffer read by every thread
  uint64_t* landed = bars + 2 * NAB;           // [NB]  x~ plane copies of every thread landed
  const int tid = threadIdx.x;
  const int e0 = blockIdx.x * SX, f0 = blockIdx.y * C::SY;
  const int X0 = K * e0, Y0 = K * f0;
  const int ez0 = blockIdx.z * a.ez_per_block;
  const int ez1 = min(ez0 + a.ez_per_block, a.nz);
  const int ezs = max(ez0 - 1, 0);             // first element layer processed (halo layer)
  const int NP = (ez1 - ezs) * K + 1;          // planes K ezs .. K ez1
  const int pz0 = K * ezs;
  const int64_t NXY = (int64_t)a.NX * a.NY;
  const int bm = a.bcmask;
  // this thread's output column and y slot (rows K s + r)
  const int c = tid & 31, s = tid >> 5;
  const int gx = X0 + c;
  const int f = f0 + s;
  const bool colin = c < C::TX && gx < a.NX;
  const int rowo0 = gx + a.NX * (Y0 + K * s);   // in-plane offset of the thread's row 0 (row r: + NX r)
  uint32_t rvalid = 0, rcons = 0;              // per row r: inside the domain / constrained (x, y)
  {
    const bool xm = ((bm & 1) && gx == 0) || ((bm & 2) && gx == a.NX - 1);
#pragma unroll
    for (int r = 0; r < K; ++r) {
      const int gy = Y0 + K * s + r;
      if (colin && gy < a.NY) rvalid |= 1u << r;
      if (xm || ((bm & 4) && gy == 0) || ((bm & 8) && gy == a.NY - 1)) rcons |= 1u << r;
    }
  }
  auto epilogue = [&](int pz, int r, double v, bool m) {   // output (row r, plane pz)
    const int64_t pb = NXY * pz;
    const int o = rowo0 + a.NX * r;
    if constexpr (MODE == 0) {   // constrained rows: 0 here, x_c by launch_set_constrained
      __stwb(st_plane(a.y + pb) + o, m ? 0.0 : v);
    } else {   // D^-1 = 0 on constrained rows
      const double xv = __ldg(st_plane(a.x + pb) + o);
      const double xov = MODE == 1 ? __ldg(st_plane(a.xo + pb) + o) : 0.0;
      __stwb(st_plane(a.y + pb) + o,
             fma(a.c2 * __ldg(st_plane(a.dinv + pb) + o), __ldg(st_plane(a.b + pb) + o) - v, fma(a.c1, xv - xov, xv)));
    }
  };
  // tiles holding only the far boundary column / row of a Dirichlet side: every output
  // is a constrained row
  if ((X0 == a.NX - 1 && (bm & 2)) || (Y0 == a.NY - 1 && (bm & 8))) {
    const int q1 = K * ez1 + (ez1 == a.nz ? 1 : 0);
    for (int pz = K * ez0; pz < q1; ++pz)
#pragma unroll
      for (int r = 0; r < K; ++r)
        if ((rvalid >> r) & 1u) epilogue(pz, r, 0.0, true);
    return;
  }
  if (tid == 0) {
    for (int b = 0; b < C::NBAR; ++b) mbar_init(bars + b, C::THREADS);
  }
  __syncthreads();

  // ---- loads: the same (row, column) slots of the tile in every plane
  int ld_off[C::NLD];
  uint32_t ld_ok = 0;
#pragma unroll
  for (int j = 0; j < C::NLD; ++j) {
    const int idx = tid + j * C::THREADS;
    const int r = idx / LC, cc = idx % LC;
    const int lx = X0 - K + cc, ly = Y0 - K + r;
    const bool in = idx < LR * LC && lx >= 0 && lx < a.NX && ly >= 0 && ly < a.NY;
    const bool m = ((bm & 1) && lx == 0) || ((bm & 2) && lx == a.NX - 1) || ((bm & 4) && ly == 0) ||
                   ((bm & 8) && ly == a.NY - 1);
    ld_off[j] = in ? lx + a.NX * ly : 0;
    if (in && !m) ld_ok |= 1u << j;
  }
  auto load_plane = [&](int i) {   // plane index i (global plane pz0 + i) into buffer i % NB
    if (i >= NP) return;
    const int gz = pz0 + i;
    const bool zm = ((bm & 16) && gz == 0) || ((bm & 32) && gz == a.NZ - 1);
    const double* src = st_plane(a.x + (int64_t)gz * NXY);
    double* dst = Xt + (i % NB) * LR * LP;
    const uint32_t ok = zm ? 0u : ld_ok;   // source sizes of this plane's copies: 8 or 0 bytes
#pragma unroll
    for (int j = 0; j < C::NLD; ++j) {
      const int idx = tid + j * C::THREADS;
      if (idx < LR * LC) {
        const int so = LP == LC ? idx : (idx / LC) * LP + idx % LC;
        if constexpr (MODE == 0) {   // source size 8 or 0 straight from the mask bit
          asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(smem_u32(dst + so)),
                       "l"(src + ld_off[j]), "r"(((ok >> j) & 1u) << 3)
                       : "memory");
        } else {   // (MODE 1: this form measured better, the register allocation differs)
          st_cp_async8(dst + so, src + ld_off[j], !zm && ((ld_ok >> j) & 1u));
        }
      }
    }
    mbar_arrive_cp_async(landed + i % NB);
  };

  // ---- x-stage of plane i: A = M_x x~, B = rx S_x x~ at every tile column, all LR rows.
  // Item = (row, slot): 2K+1 loaded values -> K outputs per field.  Slot e's vertex row
  // uses the pre-summed coefficients; on a domain boundary (e = 0 or e = nx) the missing
  // element's inputs are zero-filled and the vertex value is halved (M[K][K] = M[0][0],
  // S[K][K] = S[0][0]), so the same row gives the one-element sum without a branch.
  const int nsl = min(SX, a.nx - e0 + 1);
  const int nitems = LR * nsl;
  const double rx = a.c0 / a.cy, rz = a.cz / a.cy;   // metric folded: y = c_y (M_z Q + r_z S_z P)
  static_assert(C::LR * C::SX <= 2 * C::THREADS, "x-stage items per thread");
  // the thread's (at most two) items, loop-invariant: shared-memory read and write
  // offsets packed into one word each (both < 2^16), the boundary halving in bit 31
  // (MODE 0 only: in MODE 1 the two extra registers made the epilogue spill)
  uint32_t xit[2];
#pragma unroll
  for (int u = 0; u < 2; ++u) {
    const int it = tid + u * C::THREADS;
    const int row = it % LR, sl = it / LR;
    const bool edge = e0 + sl == 0 || e0 + sl == a.nx;
    xit[u] = (uint32_t)(row * LP + sl * K) | ((uint32_t)(row * ABP + sl * K) << 16) | (edge ? 0x80000000u : 0u);
  }
  auto x_stage = [&](int i) {
    const double* xb = Xt + (i % NB) * LR * LP;
    double* Ab = AB + (i % NAB) * 2 * LR * ABP;
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      // the LR * SX - THREADS extra items of a plane go to two warps that rotate with the
      // plane (FEM_ST_ROT), so that no warp is the slow one on every plane
      const int it = u == 0 ? tid : C::THREADS + (FEM_ST_ROT ? ((tid - 64 * (i & 3)) & (C::THREADS - 1)) : tid);
      if (it >= nitems) break;
      const double* v;
      double* ao;
      bool edge;
      if (MODE == 0 && u == 0) {
        v = xb + (xit[u] & 0xffffu);
        ao = Ab + ((xit[u] >> 16) & 0x7fffu);
        edge = xit[u] >> 31;
      } else {
        const int row = it % LR, sl = it / LR;
        v = xb + row * LP + sl * K;
        ao = Ab + row * ABP + sl * K;
        edge = e0 + sl == 0 || e0 + sl == a.nx;
      }
      // v: loaded column of node K (e-1)
      double w[2 * K + 1];
#pragma unroll
      for (int j = 0; j <= 2 * K; ++j) w[j] = v[j];
      const double wk = w[K];
      w[K] = edge ? 0.5 * wk : wk;
      double* bo = ao + LR * ABP;
      ao[0] = band_row<K, false, SYMT>(w, 0, true, false);
      bo[0] = ISO ? band_row<K, true, SYMT>(w, 0, true, false) : rx * band_row<K, true, SYMT>(w, 0, true, false);
      w[K] = wk;
#pragma unroll
      for (int r = 1; r < K; ++r) {
        ao[r] = band_row<K, false, SYMT>(w, r, true, false);
        bo[r] = ISO ? band_row<K, true, SYMT>(w, r, true, false) : rx * band_row<K, true, SYMT>(w, r, true, false);
      }
    }
  };

  // ---- y/z stages (thread = column c, y slot s)
  const double hy = (f == 0 || f == a.ny) ? 0.5 : 1.0;
  double out[K][N];
#pragma unroll
  for (int r = 0; r < K; ++r)
#pragma unroll
    for (int q = 0; q < N; ++q) out[r][q] = 0.0;
  // P = r_z M_y A, Q = M_y B + S_y A  (vertex row: halved centre on the boundary)
  auto y_stage = [&](const double (&av)[2 * K + 1], const double (&bv)[2 * K + 1], double (&P)[K], double (&Q)[K]) {
    {
      double p1 = 0.0, p2 = 0.0, q1 = 0.0, q2 = 0.0;
#pragma unroll
      for (int j = 0; j <= 2 * K; ++j) {
        const double aj = j == K ? hy * av[j] : av[j], bj = j == K ? hy * bv[j] : bv[j];
        if (j < K) {
          p1 = fma(ST_TAB(K).Mv[j], aj, p1);
          q1 = fma(ST_TAB(K).Sv[j], aj, fma(ST_TAB(K).Mv[j], bj, q1));
        } else {
          p2 = fma(ST_TAB(K).Mv[j], aj, p2);
          q2 = fma(ST_TAB(K).Sv[j], aj, fma(ST_TAB(K).Mv[j], bj, q2));
        }
      }
      P[0] = ISO ? p1 + p2 : rz * (p1 + p2);
      Q[0] = q1 + q2;
    }
#pragma unroll
    for (int r = 1; r < K; ++r) {
      double p = 0.0, q = 0.0;
#pragma unroll
      for (int j = 0; j <= K; ++j) {
        p = fma(ST_TAB(K).M[r][j], av[K + j], p);
        q = fma(ST_TAB(K).S[r][j], av[K + j], fma(ST_TAB(K).M[r][j], bv[K + j], q));
      }
      P[r] = ISO ? p : rz * p;
      Q[r] = q;
    }
  };
  auto accumulate = [&](int rp, const double (&P)[K], const double (&Q)[K]) {
#pragma unroll
    for (int q = 0; q < N; ++q)
#pragma unroll
      for (int r = 0; r < K; ++r)
        out[r][q] = fma(ST_TAB(K).S[q][rp], P[r], fma(ST_TAB(K).M[q][rp], Q[r], out[r][q]));
  };
  auto write_plane = [&](int pz, int q) {   // MODE 0: c_y out[.][q] -> global plane pz
    const bool zm = ((bm & 16) && pz == 0) || ((bm & 32) && pz == a.NZ - 1);
    double* yp = st_plane(a.y + NXY * pz);
#pragma unroll
    for (int r = 0; r < K; ++r)
      if ((rvalid >> r) & 1u) {
        const double v = zm || ((rcons >> r) & 1u) ? 0.0 : a.cy * out[r][q];
        if (FEM_ST_WP) __stwb(yp + rowo0 + a.NX * r, v);
        else yp[rowo0 + a.NX * r] = v;
      }
  };
  // MODE 1: node classes of D^-1 (see api.cu): 0 first node, r inside an element, K interior
  // vertex, K+1 last node
  auto ncls = [&](int g, int nn) { return g == 0 ? 0 : g == nn - 1 ? K + 1 : (g % K == 0 ? K : g % K); };
  int clxy[K];   // x and y class part of the D^-1 class index
#pragma unroll
  for (int r = 0; r < K; ++r)
    clxy[r] = ncls(min(gx, a.NX - 1), a.NX) + (K + 2) * ncls(min(Y0 + K * s + r, a.NY - 1), a.NY);
  // MODE 1: the element's K output planes (plus the top plane at the domain end): all
  // operand loads of a pair of planes are issued before any store (a store may alias them,
  // so the compiler would otherwise serialise one DRAM round trip per output)
  auto write_element = [&](int ez, int nq) {
#if FEM_ST_EPI_FN
    st_write_element<K, MODE>(a.x, a.xo, a.b, a.dcls, a.y, out, rowo0, NXY, a.NX, a.NZ, rvalid, clxy, ez, nq,
                              a.c1, a.c2, a.cy);
#else
#pragma unroll
    for (int q = 0; q < N; ++q) {
      if (q >= nq) break;
      const int pz = K * ez + q;
      const int clz = (K + 2) * (K + 2) * ncls(pz, a.NZ);
      const int64_t po = rowo0 + NXY * pz;
      const double* xp = a.x + po;
      const double* bp = a.b + po;
      const double* op = MODE == 1 ? a.xo + po : nullptr;
      double* yp = a.y + po;
      double xv[K], xov[K], bv2[K], dv[K];
#pragma unroll
      for (int r = 0; r < K; ++r) {
        const bool ok = (rvalid >> r) & 1u;
        xv[r] = ok ? xp[a.NX * r] : 0.0;
        xov[r] = MODE == 1 && ok ? op[a.NX * r] : 0.0;
        bv2[r] = ok ? bp[a.NX * r] : 0.0;
        if (FEM_ST_EPI_DV) dv[r] = __ldg(a.dcls + clxy[r] + clz);
      }
#pragma unroll
      for (int r = 0; r < K; ++r) {
        if (!((rvalid >> r) & 1u)) continue;
        if (!FEM_ST_EPI_DV) dv[r] = __ldg(a.dcls + clxy[r] + clz);
        const double v = a.cy * out[r][q];
        yp[a.NX * r] = fma(a.c2 * dv[r], bv2[r] - v, fma(a.c1, xv[r] - xov[r], xv[r]));
      }
    }
#endif
  };

  // MODE 1: the epilogue reads x, x_old, b (D^-1 from the class table) of the element's
  // output planes; a burst of dependent loads at the element end stalls the warps for a
  // DRAM round trip, so the warp prefetches its 4 rows x (K planes) x the arrays into L2
  // FEM_ST_PF_AHEAD elements ahead (lanes split the 256-byte row ranges).
  auto prefetch_epilogue = [&](int ez) {
    if constexpr (MODE != 0) {
      if (ez < ez0) return;
      const int nq = K + (ez + 1 == a.nz ? 1 : 0);
      const int ncol = min(C::TX, a.NX - X0);
      for (int t = c; t < 4 * K * nq; t += 32) {
        const int arr = t & 3, rq = t >> 2, r = rq % K, q = rq / K;
        const int gy = Y0 + K * s + r;
        if (gy >= a.NY) continue;
        const double* base = arr == 0 ? (FEM_ST_PF_X ? a.x : nullptr) : arr == 1 ? (MODE == 1 ? a.xo : nullptr)
                                                                        : arr == 2 ? a.b : nullptr;
        if (!base) continue;
#if FEM_ST_PF_LINES
        {   // per 128-byte line
          const double* p0 = base + X0 + (int64_t)a.NX * gy + NXY * (K * ez + q);
          for (int o = 0; o < ncol; o += 16) asm volatile("prefetch.global.L2 [%0];" ::"l"(p0 + o));
        }
#else
        prefetch_l2_range(base + X0 + (int64_t)a.NX * gy + NXY * (K * ez + q), sizeof(double) * ncol);
#endif
      }
    }
  };

  // ---- pipeline (mbarriers: a warp may run up to one plane ahead of the slowest one).
  // Iteration i: x-stage of plane i+1 into A/B buffer (i+1)&1, then the y/z stages of
  // plane i from buffer i&1; plane i+NB is copied into the x~ buffer plane i used.
#pragma unroll
  for (int i = 0; i < NB; ++i) load_plane(i);
  mbar_wait_sleep(landed, 0);
  x_stage(0);
  mbar_arrive(full);
  double P[K], Q[K];
  int i = 0;
  auto step = [&]() {
    if (i + 1 < NP) {
      if (i + 1 >= NAB)   // y/z stages of plane i + 1 - NAB done
        mbar_wait_sleep(empty + (i + 1) % NAB, ((i + 1) / NAB - 1) & 1);
      mbar_wait_sleep(landed + (i + 1) % NB, ((i + 1) / NB) & 1);
      x_stage(i + 1);
      mbar_arrive(full + (i + 1) % NAB);
    }
    mbar_wait_sleep(full + i % NAB, (i / NAB) & 1);       // x-stage of plane i done (x~ buffer i % NB free)
    load_plane(i + NB);
    double av[2 * K + 1], bv[2 * K + 1];
    {
      const double* Ab = AB + (i % NAB) * 2 * LR * ABP + (K * s) * ABP + c;
      const double* Bb = Ab + LR * ABP;
#pragma unroll
      for (int j = 0; j <= 2 * K; ++j) {
        av[j] = Ab[j * ABP];
        bv[j] = Bb[j * ABP];
      }
    }
    mbar_arrive(empty + i % NAB);
    y_stage(av, bv, P, Q);
    ++i;
  };
  step();
  accumulate(0, P, Q);
  for (int d = 0; d < FEM_ST_PF_AHEAD; ++d) prefetch_epilogue(ez0 + d);
  for (int ez = ezs; ez < ez1; ++ez) {
    if (ez + FEM_ST_PF_AHEAD < ez1) prefetch_epilogue(ez + FEM_ST_PF_AHEAD);   // elements ahead
#pragma unroll
    for (int rp = 1; rp <= K; ++rp) {
      step();
      accumulate(rp, P, Q);
    }
    // planes K ez .. K ez + K - 1 are complete; the vertex plane carries
    if (ez >= ez0) {
      if constexpr (MODE == 0) {
#pragma unroll
        for (int q = 0; q < K; ++q) write_plane(K * ez + q, q);
      } else {
        write_element(ez, ez + 1 == a.nz ? K + 1 : K);   // the top plane (q = K) too at the end
      }
    }
#pragma unroll
    for (int r = 0; r < K; ++r) {
      out[r][0] = out[r][K];
#pragma unroll
      for (int q = 1; q < N; ++q) out[r][q] = 0.0;
    }
    if (ez + 1 < ez1) accumulate(0, P, Q);   // the same plane is r' = 0 of the next element
  }
  if constexpr (MODE == 0) {
    if (ez1 == a.nz) write_plane(K * a.nz, 0);
  }
}

// ---------------------------------------------------------------- launcher
template <int K, int MODE>
void stencil_k(fem_ctx* h, const Level& L, const StArgs& a0) {
  using C = StCfg<K, MODE>;
  StArgs a = a0;
  a.nx = L.n[0];
  a.ny = L.n[1];
  a.nz = L.n[2];
  a.NX = L.nn[0];
  a.NY = L.nn[1];
  a.NZ = L.nn[2];
  int mask = 0;
  for (int s = 0; s < 6; ++s)
    if (h->mesh.bc[s] == FEM_BC_DIRICHLET) mask |= 1 << s;
  a.bcmask = mask;
  const int gx = (a.NX + C::TX - 1) / C::TX, gy = (a.NY + C::TY - 1) / C::TY;
  // z-element layers per block: about 8 waves of 2 blocks per SM (wave quantisation,
  // small levels) without making the recomputed halo layer (1/ez of the work) large
  int ez = h->stencil_ez;
  if (ez <= 0) {
    const long tiles = (long)gx * gy;
    // MODE 0 (no epilogue burst) prefers longer z-chunks -- fewer recomputed halo layers --
    // over wave balance: C4 apply ez 16 -> 32: 747 -> 724 us (solve 118.6 -> 116.4 ms at 5 its); the
    // fused step does not (ez 32 for it: 1591 -> 1646 us)
    ez = (int)std::lround((double)a.nz * tiles / ((MODE == 0 ? 4.0 : 8.0) * 2 * 148));
    ez = std::max(4, std::min(ez, 32));
  }
  ez = std::max(1, std::min(ez, a.nz));
  a.ez_per_block = ez;
  const int gz = (a.nz + ez - 1) / ez;
  a.c0 = L.cart[0];
  a.cy = L.cart[1];
  a.cz = L.cart[2];
  const size_t sm = sizeof(double) * C::SMEM;
  const bool iso = L.cart[0] == L.cart[1] && L.cart[1] == L.cart[2];
  auto kern = iso ? cg_stencil2_kernel<K, MODE, true> : cg_stencil2_kernel<K, MODE, false>;
  smem_attr(reinterpret_cast<const void*>(kern), sm);
  launch_pdl(h, kern, dim3(gx, gy, gz), dim3(C::THREADS), sm, a);
  count_launch();
  check_launch("cg_stencil2_kernel");
}

// y = A x (setc: y_c = x_c on constrained rows, else 0).  Single-rank Cartesian CG levels, k <= 4.
void launch_cg_stencil_apply(fem_ctx* h, const Level& L, const double* x, double* y, bool setc) {
  StArgs a{};
  a.x = x;
  a.y = y;
  switch (h->k) {
    case 1: stencil_k<1, 0>(h, L, a); break;
    case 2: stencil_k<2, 0>(h, L, a); break;
    case 3: stencil_k<3, 0>(h, L, a); break;
    case 4: stencil_k<4, 0>(h, L, a); break;
    default: throw Error{FEM_E_ARG, "stencil kernel: k in 1..4"};
  }
  if (setc) launch_set_constrained(h, L, x, y);   // boundary rows only
}

// x_new = x + c1 (x - x_old) + c2 D^-1 (b - A x)  (fused Chebyshev step, R7)
void launch_cg_stencil_cheb(fem_ctx* h, const Level& L, const double* x, const double* xo, const double* b,
                            double* xnew, double c1, double c2) {
  StArgs a{};
  a.x = x;
  a.y = xnew;
  a.xo = xo;
  a.b = b;
  a.dinv = L.dinv;
  a.dcls = L.dinv_cls;
  a.c1 = c1;
  a.c2 = c2;
  if (!a.dcls) throw Error{FEM_E_ARG, "stencil Chebyshev step: no D^-1 class table"};
  // MODE 1: x_old read; MODE 2: first step of the recurrence, x_old = 0 (no stream)
  switch (h->k * 4 + (xo ? 1 : 2)) {
    case 5: stencil_k<1, 1>(h, L, a); break;
    case 6: stencil_k<1, 2>(h, L, a); break;
    case 9: stencil_k<2, 1>(h, L, a); break;
    case 10: stencil_k<2, 2>(h, L, a); break;
    case 13: stencil_k<3, 1>(h, L, a); break;
    case 14: stencil_k<3, 2>(h, L, a); break;
    case 17: stencil_k<4, 1>(h, L, a); break;
    case 18: stencil_k<4, 2>(h, L, a); break;
    default: throw Error{FEM_E_ARG, "stencil kernel: k in 1..4"};
  }
}

}  // namespace fem
