// Multigrid and vector kernels: level transfer (K6), Chebyshev step (K5),
// fused PCG vector updates and deterministic reductions (K7), coarse solve (K8),
// splitmix64 start vector.
//
// Transfer ("geometric embedding operations ... implemented by
// tensorial techniques"): one block per coarse cell applies the 1-D embedding
// matrix E [M x (k+1)] in three sweeps (CG: M = 2k+1 fine nodes of the two
// children; DG: M = 2(k+1), child matrices stacked).  CG prolongation writes each
// fine node from exactly one coarse cell (half-open ownership), so x_f += P x_c
// needs no atomics; CG restriction reads each fine node in its owning coarse cell
// only, which reproduces P^T exactly (a coarse basis function of a neighbour
// vanishes on the shared face unless its node lies on it), and adds into the
// coarse vector with atomics.  DG transfers touch only the 8 children.
#include <algorithm>

#include "device_common.cuh"

namespace fem {

constexpr int kTransferThreads = 128;   // block size of the transfer kernels

template <int K, bool DG>
struct Embed {
  static constexpr int N = K + 1;
  static constexpr int M = DG ? 2 * N : 2 * K + 1;
  double E[M][N];
};

struct TransferArgs {
  int nc0, nc1, nc2;     // rank-local coarse cells
  int nnc0, nnc1, nnc2;  // coarse CG nodes (z: GLOBAL node planes)
  int nnf0, nnf1, nnf2;  // fine CG nodes (z: GLOBAL node planes)
  int czc0, ncz;         // global index of the first local coarse layer, global coarse layers
  int bcmask;
};

__device__ __forceinline__ int64_t cg_index(int gx, int gy, int gz, int nn0, int nn1) {
  return gx + (int64_t)nn0 * (gy + (int64_t)nn1 * gz);
}

// Line-thread form: in each of the three sweeps a thread owns one 1-D line of the
// current direction and keeps it in registers (inputs read once, from global memory in
// the first sweep of the restriction and written to global memory in the last sweep of
// the prolongation), so shared memory only carries the two intermediate tensors.
// (The earlier element-per-thread form staged all (2k+1)^3 / (2k+2)^3 fine values in
// shared memory and re-read each one per output: ~7x the shared-memory traffic.)

// fine-level value (r, s, t) of coarse cell (cx, cy, cz) for the restriction (0 where the
// fine node is not owned by this coarse cell (CG) or constrained)
template <int K, bool DG>
__device__ __forceinline__ double transfer_fine_in(const TransferArgs& a, const double* __restrict__ bf,
                                                   const double* __restrict__ axf, int cx, int cy, int cz,
                                                   int r, int sidx, int tt) {
  constexpr int N = K + 1;
  int64_t idx;
  if (DG) {
    const int fx = 2 * cx + r / N, fy = 2 * cy + sidx / N, fz = 2 * cz + tt / N;
    const int64_t fcell = fx + (int64_t)(2 * a.nc0) * (fy + (int64_t)(2 * a.nc1) * fz);
    idx = fcell * N * N * N + r % N + N * ((sidx % N) + N * (tt % N));
  } else {
    // the node exists whether or not this cell owns it: load unconditionally (all loads of
    // a line in flight together), mask afterwards
    const bool owned = !((r == 2 * K && cx != a.nc0 - 1) || (sidx == 2 * K && cy != a.nc1 - 1) ||
                         (tt == 2 * K && a.czc0 + cz != a.ncz - 1));
    const int gx = 2 * K * cx + r, gy = 2 * K * cy + sidx, gz = 2 * K * cz + tt;
    idx = cg_index(gx, gy, gz, a.nnf0, a.nnf1);
    const double v = __ldg(bf + idx) - (axf ? __ldg(axf + idx) : 0.0);
    return (!owned || cg_constrained(a.bcmask, gx, gy, 2 * K * a.czc0 + gz, a.nnf0, a.nnf1, a.nnf2)) ? 0.0 : v;
  }
  return __ldg(bf + idx) - (axf ? __ldg(axf + idx) : 0.0);
}

// xf += P xc
template <int K, bool DG>
__global__ void prolongate_kernel(TransferArgs a, Embed<K, DG> E, const double* __restrict__ xc,
                                  double* __restrict__ xf) {
  FEM_PDL_ENTRY();
  constexpr int N = K + 1, M = Embed<K, DG>::M;
  extern __shared__ double smem[];
  double* s_1 = smem;               // [l][j][r]  M N^2
  double* s_2 = smem + M * N * N;   // [l][s][r]  M^2 N
  __shared__ double sE[M][N];
  for (int i = threadIdx.x; i < M * N; i += blockDim.x) sE[i / N][i % N] = E.E[i / N][i % N];
  const int64_t cell = blockIdx.x;
  const int cx = (int)(cell % a.nc0);
  const int64_t rr = cell / a.nc0;
  const int cy = (int)(rr % a.nc1), cz = (int)(rr / a.nc1);
  __syncthreads();
  // x: coarse x-lines (j, l) -> M fine x values
  for (int line = threadIdx.x; line < N * N; line += blockDim.x) {
    const int j = line % N, l = line / N;
    double in[N];
#pragma unroll
    for (int i = 0; i < N; ++i) {
      if (DG) {
        in[i] = __ldg(xc + cell * N * N * N + i + N * line);
      } else {
        const int gx = K * cx + i, gy = K * cy + j, gz = K * cz + l;
        in[i] = cg_constrained(a.bcmask, gx, gy, K * a.czc0 + gz, a.nnc0, a.nnc1, a.nnc2)
                    ? 0.0
                    : __ldg(xc + cg_index(gx, gy, gz, a.nnc0, a.nnc1));
      }
    }
#pragma unroll
    for (int r = 0; r < M; ++r) {
      double s = 0.0;
#pragma unroll
      for (int i = 0; i < N; ++i) s = fma(sE[r][i], in[i], s);
      s_1[r + M * (j + N * l)] = s;
    }
  }
  __syncthreads();
  // y: lines (r, l)
  for (int line = threadIdx.x; line < M * N; line += blockDim.x) {
    const int r = line % M, l = line / M;
    double in[N];
#pragma unroll
    for (int j = 0; j < N; ++j) in[j] = s_1[r + M * (j + N * l)];
#pragma unroll
    for (int sidx = 0; sidx < M; ++sidx) {
      double s = 0.0;
#pragma unroll
      for (int j = 0; j < N; ++j) s = fma(sE[sidx][j], in[j], s);
      s_2[r + M * (sidx + M * l)] = s;
    }
  }
  __syncthreads();
  // z: lines (r, s) -> M fine values along z, added into xf (all old values loaded first)
  for (int line = threadIdx.x; line < M * M; line += blockDim.x) {
    const int r = line % M, sidx = line / M;
    double in[N], old[M];
    int64_t idx[M];
    bool wr[M];
#pragma unroll
    for (int tt = 0; tt < M; ++tt) {
      if (DG) {
        const int fx = 2 * cx + r / N, fy = 2 * cy + sidx / N, fz = 2 * cz + tt / N;
        const int64_t fcell = fx + (int64_t)(2 * a.nc0) * (fy + (int64_t)(2 * a.nc1) * fz);
        idx[tt] = fcell * N * N * N + r % N + N * ((sidx % N) + N * (tt % N));
        wr[tt] = true;
      } else {
        // owned: local fine index < 2K unless this is the last coarse cell
        const int gx = 2 * K * cx + r, gy = 2 * K * cy + sidx, gz = 2 * K * cz + tt;
        idx[tt] = cg_index(gx, gy, gz, a.nnf0, a.nnf1);
        wr[tt] = !((r == 2 * K && cx != a.nc0 - 1) || (sidx == 2 * K && cy != a.nc1 - 1) ||
                   (tt == 2 * K && a.czc0 + cz != a.ncz - 1)) &&
                 !cg_constrained(a.bcmask, gx, gy, 2 * K * a.czc0 + gz, a.nnf0, a.nnf1, a.nnf2);
      }
      old[tt] = xf[idx[tt]];
    }
#pragma unroll
    for (int l = 0; l < N; ++l) in[l] = s_2[r + M * (sidx + M * l)];
#pragma unroll
    for (int tt = 0; tt < M; ++tt) {
      double s = 0.0;
#pragma unroll
      for (int l = 0; l < N; ++l) s = fma(sE[tt][l], in[l], s);
      if (wr[tt]) xf[idx[tt]] = old[tt] + s;
    }
  }
}

// xc (+)= P^T (bf - axf)   [axf may be null: P^T bf].  CG: xc must be zeroed (atomics).
template <int K, bool DG>
__global__ void restrict_kernel(TransferArgs a, Embed<K, DG> E, const double* __restrict__ bf,
                                const double* __restrict__ axf, double* __restrict__ xc) {
  FEM_PDL_ENTRY();
  constexpr int N = K + 1, M = Embed<K, DG>::M;
  extern __shared__ double smem[];
  double* s_1 = smem;               // [t][s][i]  N M^2
  double* s_2 = smem + N * M * M;   // [t][j][i]  N^2 M
  __shared__ double sE[M][N];
  for (int i = threadIdx.x; i < M * N; i += blockDim.x) sE[i / N][i % N] = E.E[i / N][i % N];
  const int64_t cell = blockIdx.x;
  const int cx = (int)(cell % a.nc0);
  const int64_t rr = cell / a.nc0;
  const int cy = (int)(rr % a.nc1), cz = (int)(rr / a.nc1);
  __syncthreads();
  // x: fine x-lines (s, t), read once from global memory into registers
  for (int line = threadIdx.x; line < M * M; line += blockDim.x) {
    const int sidx = line % M, tt = line / M;
    double in[M];
#pragma unroll
    for (int r = 0; r < M; ++r) in[r] = transfer_fine_in<K, DG>(a, bf, axf, cx, cy, cz, r, sidx, tt);
#pragma unroll
    for (int i = 0; i < N; ++i) {
      double s = 0.0;
#pragma unroll
      for (int r = 0; r < M; ++r) s = fma(sE[r][i], in[r], s);
      s_1[i + N * (sidx + M * tt)] = s;
    }
  }
  __syncthreads();
  // y: lines (i, t)
  for (int line = threadIdx.x; line < N * M; line += blockDim.x) {
    const int i = line % N, tt = line / N;
    double in[M];
#pragma unroll
    for (int sidx = 0; sidx < M; ++sidx) in[sidx] = s_1[i + N * (sidx + M * tt)];
#pragma unroll
    for (int j = 0; j < N; ++j) {
      double s = 0.0;
#pragma unroll
      for (int sidx = 0; sidx < M; ++sidx) s = fma(sE[sidx][j], in[sidx], s);
      s_2[i + N * (j + N * tt)] = s;
    }
  }
  __syncthreads();
  // z: lines (i, j)
  for (int line = threadIdx.x; line < N * N; line += blockDim.x) {
    const int i = line % N, j = line / N;
    double in[M];
#pragma unroll
    for (int tt = 0; tt < M; ++tt) in[tt] = s_2[i + N * (j + N * tt)];
#pragma unroll
    for (int l = 0; l < N; ++l) {
      double s = 0.0;
#pragma unroll
      for (int tt = 0; tt < M; ++tt) s = fma(sE[tt][l], in[tt], s);
      if (DG) {
        xc[cell * N * N * N + line + N * N * l] = s;
      } else {
        const int gx = K * cx + i, gy = K * cy + j, gz = K * cz + l;
        if (!cg_constrained(a.bcmask, gx, gy, K * a.czc0 + gz, a.nnc0, a.nnc1, a.nnc2))
          atomicAdd(xc + cg_index(gx, gy, gz, a.nnc0, a.nnc1), s);
      }
    }
  }
}

// Element-per-thread form (CG): every fine value staged in shared memory, consecutive
// threads on consecutive fine x-nodes (coalesced); measured faster than the line-thread
// form for CG at scale (C4 solve 212 vs 220 ms), slower for DG.
// xf += P xc
template <int K, bool DG>
__global__ void prolongate_elem_kernel(TransferArgs a, Embed<K, DG> E, const double* __restrict__ xc,
                                  double* __restrict__ xf) {
  FEM_PDL_ENTRY();
  constexpr int N = K + 1, M = Embed<K, DG>::M;
  extern __shared__ double smem[];
  double* s_in = smem;               // N^3
  double* s_1 = smem + N * N * N;    // M N^2
  double* s_2 = s_1 + M * N * N;     // M^2 N
  // E indexed by a thread-dependent row: from shared memory (a kernel-parameter
  // (constant bank) operand with divergent addresses serialises the warp)
  __shared__ double sE[M][N];
  for (int i = threadIdx.x; i < M * N; i += blockDim.x) sE[i / N][i % N] = E.E[i / N][i % N];
  const int64_t cell = blockIdx.x;
  const int cx = (int)(cell % a.nc0);
  const int64_t rr = cell / a.nc0;
  const int cy = (int)(rr % a.nc1), cz = (int)(rr / a.nc1);
  for (int i = threadIdx.x; i < N * N * N; i += blockDim.x) {
    const int i0 = i % N, i1 = (i / N) % N, i2 = i / (N * N);
    double v;
    if (DG) {
      v = xc[cell * N * N * N + i];
    } else {
      const int gx = K * cx + i0, gy = K * cy + i1, gz = K * cz + i2;
      v = cg_constrained(a.bcmask, gx, gy, K * a.czc0 + gz, a.nnc0, a.nnc1, a.nnc2)
              ? 0.0
              : xc[cg_index(gx, gy, gz, a.nnc0, a.nnc1)];
    }
    s_in[i] = v;
  }
  __syncthreads();
  if constexpr (!DG) {
    // CG: one row of the embedding matrix per thread in registers (fixed fine index along
    // the sweep direction): one shared-memory load per FMA instead of two
    constexpr int TPR = kTransferThreads / M;
    const int ri = threadIdx.x / TPR, rj = threadIdx.x % TPR;
    const bool act = ri < M;
    double e[N];
#pragma unroll
    for (int i = 0; i < N; ++i) e[i] = act ? sE[ri][i] : 0.0;
    if (act) {   // x: s_1[r + M jl], r = ri
      for (int jl = rj; jl < N * N; jl += TPR) {
        double s = 0.0;
#pragma unroll
        for (int i = 0; i < N; ++i) s = fma(e[i], s_in[i + N * jl], s);
        s_1[ri + M * jl] = s;
      }
    }
    __syncthreads();
    if (act) {   // y: s_2[r + M (sidx + M l)], sidx = ri
      for (int it = rj; it < M * N; it += TPR) {
        const int r = it % M, l = it / M;
        double s = 0.0;
#pragma unroll
        for (int j = 0; j < N; ++j) s = fma(e[j], s_1[r + M * (j + N * l)], s);
        s_2[r + M * (ri + M * l)] = s;
      }
    }
    __syncthreads();
    if (act) {   // z + write: fine node (r, sidx, tt), tt = ri
      const int tt = ri;
      for (int it = rj; it < M * M; it += TPR) {
        const int r = it % M, sidx = it / M;
        double s = 0.0;
#pragma unroll
        for (int l = 0; l < N; ++l) s = fma(e[l], s_2[r + M * (sidx + M * l)], s);
        // owned: local fine index < 2K unless this is the last coarse cell
        if ((r == 2 * K && cx != a.nc0 - 1) || (sidx == 2 * K && cy != a.nc1 - 1) ||
            (tt == 2 * K && a.czc0 + cz != a.ncz - 1))
          continue;
        const int gx = 2 * K * cx + r, gy = 2 * K * cy + sidx, gz = 2 * K * cz + tt;
        if (cg_constrained(a.bcmask, gx, gy, 2 * K * a.czc0 + gz, a.nnf0, a.nnf1, a.nnf2)) continue;
        xf[cg_index(gx, gy, gz, a.nnf0, a.nnf1)] += s;
      }
    }
    return;
  }
  for (int o = threadIdx.x; o < M * N * N; o += blockDim.x) {  // x sweep: [l][j][r]
    const int r = o % M, jl = o / M;
    double s = 0.0;
#pragma unroll
    for (int i = 0; i < N; ++i) s = fma(sE[r][i], s_in[i + N * jl], s);
    s_1[o] = s;
  }
  __syncthreads();
  for (int o = threadIdx.x; o < M * M * N; o += blockDim.x) {  // y sweep: [l][s][r]
    const int r = o % M, sidx = (o / M) % M, l = o / (M * M);
    double s = 0.0;
#pragma unroll
    for (int j = 0; j < N; ++j) s = fma(sE[sidx][j], s_1[r + M * (j + N * l)], s);
    s_2[o] = s;
  }
  __syncthreads();
#pragma unroll
  for (int it = 0; it < (M * M * M + kTransferThreads - 1) / kTransferThreads; ++it) {  // z sweep + write
    const int o = threadIdx.x + it * kTransferThreads;
    if (o >= M * M * M) break;
    int r, sidx, tt;
    int64_t fidx = 0;
    if (DG) {
      // o enumerates the fine DoFs in memory order (child cell, then its n^3 block), so
      // a warp's read-modify-writes of xf are consecutive addresses
      const int child = o / (N * N * N), loc = o % (N * N * N);
      const int ca = child & 1, cb = (child >> 1) & 1, cc = child >> 2;
      r = ca * N + loc % N;
      sidx = cb * N + (loc / N) % N;
      tt = cc * N + loc / (N * N);
      const int64_t fcell = (2 * cx + ca) + (int64_t)(2 * a.nc0) * ((2 * cy + cb) + (int64_t)(2 * a.nc1) * (2 * cz + cc));
      fidx = fcell * N * N * N + loc;
    } else {
      r = o % M;
      sidx = (o / M) % M;
      tt = o / (M * M);
    }
    double s = 0.0;
#pragma unroll
    for (int l = 0; l < N; ++l) s = fma(sE[tt][l], s_2[r + M * (sidx + M * l)], s);
    if (DG) {
      xf[fidx] += s;
    } else {
      // owned: local fine index < 2K unless this is the last coarse cell
      if ((r == 2 * K && cx != a.nc0 - 1) || (sidx == 2 * K && cy != a.nc1 - 1) ||
          (tt == 2 * K && a.czc0 + cz != a.ncz - 1))
        continue;
      const int gx = 2 * K * cx + r, gy = 2 * K * cy + sidx, gz = 2 * K * cz + tt;
      if (cg_constrained(a.bcmask, gx, gy, 2 * K * a.czc0 + gz, a.nnf0, a.nnf1, a.nnf2)) continue;
      xf[cg_index(gx, gy, gz, a.nnf0, a.nnf1)] += s;
    }
  }
}

// xc (+)= P^T (bf - axf)   [axf may be null: P^T bf].  CG: xc must be zeroed (atomics).
template <int K, bool DG>
__global__ void restrict_elem_kernel(TransferArgs a, Embed<K, DG> E, const double* __restrict__ bf,
                                const double* __restrict__ axf, double* __restrict__ xc) {
  FEM_PDL_ENTRY();
  constexpr int N = K + 1, M = Embed<K, DG>::M;
  extern __shared__ double smem[];
  double* s_in = smem;               // M^3
  double* s_1 = smem + M * M * M;    // N M^2
  double* s_2 = smem;                // N^2 M (aliases s_in, dead after the x sweep)
  __shared__ double sE[M][N];   // see prolongate_kernel
  for (int i = threadIdx.x; i < M * N; i += blockDim.x) sE[i / N][i % N] = E.E[i / N][i % N];
  const int64_t cell = blockIdx.x;
  const int cx = (int)(cell % a.nc0);
  const int64_t rr = cell / a.nc0;
  const int cy = (int)(rr % a.nc1), cz = (int)(rr / a.nc1);
  // CG: compile-time trip count, fully unrolled, so the loads of all trips are issued
  // before the first one returns (restrict 29 -> 27 us on C2; DG measured slower unrolled)
#pragma unroll
  for (int it = 0; it < (M * M * M + kTransferThreads - 1) / kTransferThreads; ++it) {
    const int o = threadIdx.x + it * kTransferThreads;
    if (o >= M * M * M) break;
    int r = o % M, sidx = (o / M) % M, tt = o / (M * M);
    double v = 0.0;
    if (DG) {
      // fine DoFs read in memory order (coalesced), placed at their (r, s, t) position
      const int child = o / (N * N * N), loc = o % (N * N * N);
      const int ca = child & 1, cb = (child >> 1) & 1, cc = child >> 2;
      r = ca * N + loc % N;
      sidx = cb * N + (loc / N) % N;
      tt = cc * N + loc / (N * N);
      const int64_t fcell = (2 * cx + ca) + (int64_t)(2 * a.nc0) * ((2 * cy + cb) + (int64_t)(2 * a.nc1) * (2 * cz + cc));
      const int64_t idx = fcell * N * N * N + loc;
      v = bf[idx] - (axf ? axf[idx] : 0.0);
    } else {
      const bool owned = !((r == 2 * K && cx != a.nc0 - 1) || (sidx == 2 * K && cy != a.nc1 - 1) ||
                           (tt == 2 * K && a.czc0 + cz != a.ncz - 1));
      const int gx = 2 * K * cx + r, gy = 2 * K * cy + sidx, gz = 2 * K * cz + tt;
      if (owned && !cg_constrained(a.bcmask, gx, gy, 2 * K * a.czc0 + gz, a.nnf0, a.nnf1, a.nnf2)) {
        const int64_t idx = cg_index(gx, gy, gz, a.nnf0, a.nnf1);
        v = bf[idx] - (axf ? axf[idx] : 0.0);
      }
    }
    s_in[r + M * (sidx + M * tt)] = v;
  }
  __syncthreads();
  if constexpr (!DG) {
    // CG: each thread keeps one column of the embedding matrix in registers (the output's
    // coarse index along the sweep direction is fixed per thread), so a sweep costs one
    // shared-memory load per FMA instead of two (the transfer was issue-bound, ncu r02:
    // 80% issue-active, 2 LDS per DFMA)
    constexpr int TPC = kTransferThreads / N;   // threads per coarse index
    const int ci = threadIdx.x / TPC, cj = threadIdx.x % TPC;
    const bool act = ci < N;
    double e[M];
#pragma unroll
    for (int r = 0; r < M; ++r) e[r] = act ? sE[r][ci] : 0.0;
    if (act) {   // x: s_1[st N + i], i = ci
      for (int st = cj; st < M * M; st += TPC) {
        double s = 0.0;
#pragma unroll
        for (int r = 0; r < M; ++r) s = fma(e[r], s_in[r + M * st], s);
        s_1[st * N + ci] = s;
      }
    }
    __syncthreads();
    if (act) {   // y: s_2[i + N (j + N tt)], j = ci
      for (int it = cj; it < N * M; it += TPC) {
        const int i = it % N, tt = it / N;
        double s = 0.0;
#pragma unroll
        for (int sidx = 0; sidx < M; ++sidx) s = fma(e[sidx], s_1[i + N * (sidx + M * tt)], s);
        s_2[i + N * (ci + N * tt)] = s;
      }
    }
    __syncthreads();
    if (act) {   // z: (i, j, l), l = ci
      for (int it = cj; it < N * N; it += TPC) {
        const int i = it % N, j = it / N;
        double s = 0.0;
#pragma unroll
        for (int tt = 0; tt < M; ++tt) s = fma(e[tt], s_2[i + N * (j + N * tt)], s);
        const int gx = K * cx + i, gy = K * cy + j, gz = K * cz + ci;
        if (!cg_constrained(a.bcmask, gx, gy, K * a.czc0 + gz, a.nnc0, a.nnc1, a.nnc2))
          atomicAdd(xc + cg_index(gx, gy, gz, a.nnc0, a.nnc1), s);
      }
    }
    return;
  }
  for (int o = threadIdx.x; o < N * M * M; o += blockDim.x) {  // x: [t][s][i]
    const int i = o % N, st = o / N;
    double s = 0.0;
#pragma unroll
    for (int r = 0; r < M; ++r) s = fma(sE[r][i], s_in[r + M * st], s);
    s_1[o] = s;
  }
  __syncthreads();
  for (int o = threadIdx.x; o < N * N * M; o += blockDim.x) {  // y: [t][j][i]
    const int i = o % N, j = (o / N) % N, tt = o / (N * N);
    double s = 0.0;
#pragma unroll
    for (int sidx = 0; sidx < M; ++sidx) s = fma(sE[sidx][j], s_1[i + N * (sidx + M * tt)], s);
    s_2[o] = s;
  }
  __syncthreads();
  for (int o = threadIdx.x; o < N * N * N; o += blockDim.x) {  // z: [l][j][i]
    const int i = o % N, j = (o / N) % N, l = o / (N * N);
    double s = 0.0;
#pragma unroll
    for (int tt = 0; tt < M; ++tt) s = fma(sE[tt][l], s_2[i + N * (j + N * tt)], s);
    xc[cell * N * N * N + o] = s;
  }
}

// Node-grid form (CG, k <= 4, large levels): the CG vector of a structured level is a 3-D
// grid of nodes and P = P1 (x) P1 (x) P1 with the banded global 1-D embedding P1 (fine node
// f = 2k c + r of coarse cell c takes E[r][i] from coarse node k c + i).  A block takes a
// strip of kGridTXC coarse cells along x of one (cy, cz) and a thread owns one fine x-node
// of the strip: the fine vector is read / written as rows of ~128 consecutive doubles
// (the element form above moves 2k+1 = 9-double rows and spends most of its instructions
// on the index arithmetic of the element gather: ncu r02k, 940M instructions per launch,
// issue-bound at 73%).  The x sweep goes through shared memory (coarse strip), the y and z
// sweeps stay in the thread's registers with compile-time E operands.  Ownership and
// constraints are exactly those of the element form (half-open cells, last cell closed),
// so the z-slab exchanges around the transfers are unchanged.
#ifndef FEM_GT_SPAN
#define FEM_GT_SPAN 64              // fine x-nodes per strip = 2 SPAN (k | SPAN) or the next lower multiple of 2k
#endif
#ifndef FEM_GT_MINB
#define FEM_GT_MINB 4               // resident blocks per SM the register allocation aims at
#endif
#ifndef FEM_GT_RMINB
#define FEM_GT_RMINB 4              // the same for the restriction
#endif
#ifndef FEM_GT_RPIPE
#define FEM_GT_RPIPE 0              // restriction: software-pipelined plane loads
#endif
#ifndef FEM_GT_RPL
#define FEM_GT_RPL 1                // restriction: fine planes loaded per batch
#endif
#ifndef FEM_GT_RGROUPS
#define FEM_GT_RGROUPS 2            // restriction: threads per coarse node in the x sweep
#endif
#ifndef FEM_GT_RNOATOM
#define FEM_GT_RNOATOM 0            // timing experiment: plain stores instead of the atomics
#endif

template <int K>
struct GridTile {
  static constexpr int TXC = FEM_GT_SPAN / K; // coarse cells per strip
  static constexpr int FX = 2 * K * TXC;      // fine nodes per strip (half-open)
  static constexpr int CW = K * TXC + 1;      // coarse nodes per strip (closed)
  static constexpr int THREADS = (FX + 1 + 31) / 32 * 32;   // FX fine nodes + the closing node of the last strip
};

// xf += P xc
template <int K>
__global__ void __launch_bounds__(GridTile<K>::THREADS, FEM_GT_MINB)
prolongate_grid_kernel(TransferArgs a, Embed<K, false> E, const double* __restrict__ xc,
                       double* __restrict__ xf) {
  FEM_PDL_ENTRY();
  constexpr int N = K + 1, M = 2 * K + 1, TXC = GridTile<K>::TXC, CW = GridTile<K>::CW;
  __shared__ double s_c[N * N][CW + 1];
  __shared__ double sE[M][N];
  const int tid = threadIdx.x;
  for (int i = tid; i < M * N; i += GridTile<K>::THREADS) sE[i / N][i % N] = E.E[i / N][i % N];
  const int cx0 = blockIdx.x * TXC, cy = blockIdx.y, cz = blockIdx.z;
  const int ncx = min(TXC, a.nc0 - cx0);
  const bool last_x = cx0 + ncx == a.nc0, last_y = cy == a.nc1 - 1, last_z = a.czc0 + cz == a.ncz - 1;
  if (tid <= K * ncx) {   // coarse strip, constrained values read as 0
    const int gx = K * cx0 + tid;
    const bool con_x = ((a.bcmask & 1) && gx == 0) || ((a.bcmask & 2) && gx == a.nnc0 - 1);
#pragma unroll
    for (int jl = 0; jl < N * N; ++jl) {
      const int gy = K * cy + jl % N, gz = K * cz + jl / N;
      const bool con = con_x || cg_constrained(a.bcmask & ~3, gx, gy, K * a.czc0 + gz, a.nnc0, a.nnc1, a.nnc2);
      const double v = __ldg(xc + cg_index(gx, gy, gz, a.nnc0, a.nnc1));
      s_c[jl][tid] = con ? 0.0 : v;
    }
  }
  __syncthreads();
  const int nfx = 2 * K * ncx + (last_x ? 1 : 0);   // fine nodes this strip owns along x
  if (tid >= nfx) return;
  const int cl = min(tid / (2 * K), ncx - 1), r = tid - 2 * K * cl;
  double e[N];
#pragma unroll
  for (int i = 0; i < N; ++i) e[i] = sE[r][i];
  double u[N * N];   // x sweep: u[j + N l]
#pragma unroll
  for (int jl = 0; jl < N * N; ++jl) {
    double s = 0.0;
#pragma unroll
    for (int i = 0; i < N; ++i) s = fma(e[i], s_c[jl][K * cl + i], s);
    u[jl] = s;
  }
  const int gx = 2 * K * cx0 + tid;
  if (((a.bcmask & 1) && gx == 0) || ((a.bcmask & 2) && gx == a.nnf0 - 1)) return;
  const int64_t row = a.nnf0, plane = (int64_t)a.nnf0 * a.nnf1;
  double* __restrict__ out = xf + cg_index(gx, 2 * K * cy, 2 * K * cz, a.nnf0, a.nnf1);
  const int gz0 = 2 * K * (a.czc0 + cz);
#pragma unroll
  for (int s = 0; s < M; ++s) {
    if (s == 2 * K && !last_y) break;
    const int gy = 2 * K * cy + s;
    if (((a.bcmask & 4) && gy == 0) || ((a.bcmask & 8) && gy == a.nnf1 - 1)) continue;
    double v[N];   // y sweep for this fine row
#pragma unroll
    for (int l = 0; l < N; ++l) {
      double t = 0.0;
#pragma unroll
      for (int j = 0; j < N; ++j) t = fma(E.E[s][j], u[j + N * l], t);
      v[l] = t;
    }
    double old[M];
    bool wr[M];
#pragma unroll
    for (int t = 0; t < M; ++t) {
      const int gz = gz0 + t;
      wr[t] = !(t == 2 * K && !last_z) && !(((a.bcmask & 16) && gz == 0) || ((a.bcmask & 32) && gz == a.nnf2 - 1));
      old[t] = wr[t] ? out[s * row + t * plane] : 0.0;
    }
#pragma unroll
    for (int t = 0; t < M; ++t) {
      double w = old[t];
#pragma unroll
      for (int l = 0; l < N; ++l) w = fma(E.E[t][l], v[l], w);
      if (wr[t]) out[s * row + t * plane] = w;
    }
  }
}

// xc += P^T (bf - axf)   [axf may be null]; xc zeroed by the caller (atomics, as the element form)
template <int K, bool AX>
__global__ void __launch_bounds__(GridTile<K>::THREADS, FEM_GT_RMINB)
restrict_grid_kernel(TransferArgs a, Embed<K, false> E, const double* __restrict__ bf,
                     const double* __restrict__ axf, double* __restrict__ xc) {
  FEM_PDL_ENTRY();
  constexpr int N = K + 1, M = 2 * K + 1, TXC = GridTile<K>::TXC, FX = GridTile<K>::FX;
  constexpr int SW = FX + 2;   // fine positions 0..FX of the strip (+1 pad)
  __shared__ double s_u[N * N][SW];
  __shared__ double sE[M][N];
  const int tid = threadIdx.x;
  for (int i = tid; i < M * N; i += GridTile<K>::THREADS) sE[i / N][i % N] = E.E[i / N][i % N];
  const int cx0 = blockIdx.x * TXC, cy = blockIdx.y, cz = blockIdx.z;
  const int ncx = min(TXC, a.nc0 - cx0);
  const bool last_x = cx0 + ncx == a.nc0, last_y = cy == a.nc1 - 1, last_z = a.czc0 + cz == a.ncz - 1;
  const int nfx = 2 * K * ncx + (last_x ? 1 : 0);
  const int gx = 2 * K * cx0 + tid;
  const bool act = tid < nfx && !(((a.bcmask & 1) && gx == 0) || ((a.bcmask & 2) && gx == a.nnf0 - 1));
  double u[N * N];
#pragma unroll
  for (int jl = 0; jl < N * N; ++jl) u[jl] = 0.0;
  if (act) {
    const int64_t row = a.nnf0, plane = (int64_t)a.nnf0 * a.nnf1;
    const int64_t base = cg_index(gx, 2 * K * cy, 2 * K * cz, a.nnf0, a.nnf1);
    const double* __restrict__ pb = bf + base;
    const double* __restrict__ pa = AX ? axf + base : nullptr;
    const int gz0 = 2 * K * (a.czc0 + cz);
    // fine plane t of the strip: used (owned and not constrained in z)?  its (masked) row values
    auto plane_used = [&](int t) {
      const int gz = gz0 + t;
      return !(t == 2 * K && !last_z) && !(((a.bcmask & 16) && gz == 0) || ((a.bcmask & 32) && gz == a.nnf2 - 1));
    };
    auto load_plane = [&](int t, double (&val)[M]) {
#pragma unroll
      for (int s = 0; s < M; ++s) {
        const int gy = 2 * K * cy + s;
        const bool rd = !(s == 2 * K && !last_y) && !(((a.bcmask & 4) && gy == 0) || ((a.bcmask & 8) && gy == a.nnf1 - 1));
        // no control flow around the loads (a branch per load keeps the compiler from batching
        // them: ncu r02l, 60% of the stall samples on the first use of each value): the masked
        // rows read the strip's first value instead
        const int64_t off = rd ? s * row + t * plane : 0;
        double v = __ldg(pb + off);
        if constexpr (AX) v -= __ldg(pa + off);
        val[s] = rd ? v : 0.0;
      }
    };
    auto add_plane = [&](int t, const double (&val)[M]) {
      double p[N];   // y sweep of this fine plane
#pragma unroll
      for (int j = 0; j < N; ++j) {
        double q = 0.0;
#pragma unroll
        for (int s = 0; s < M; ++s) q = fma(E.E[s][j], val[s], q);
        p[j] = q;
      }
#pragma unroll
      for (int l = 0; l < N; ++l)
#pragma unroll
        for (int j = 0; j < N; ++j) u[j + N * l] = fma(E.E[t][l], p[j], u[j + N * l]);
    };
#if FEM_GT_RPIPE
    // software pipeline: the loads of plane t+1 are issued before plane t is reduced
    double cur[M], nxt[M];
    if (plane_used(0)) load_plane(0, cur);
#pragma unroll
    for (int t = 0; t < M; ++t) {
      if (t + 1 < M && plane_used(t + 1)) load_plane(t + 1, nxt);
      if (plane_used(t)) add_plane(t, cur);
#pragma unroll
      for (int s = 0; s < M; ++s) cur[s] = nxt[s];
    }
#elif FEM_GT_RPL == 2
    // two planes' loads in flight before the first is reduced
#pragma unroll
    for (int t = 0; t < M; t += 2) {
      double v0[M], v1[M];
      const bool u0 = plane_used(t), u1 = t + 1 < M && plane_used(t + 1);
      if (u0) load_plane(t, v0);
      if (u1) load_plane(t + 1, v1);
      if (u0) add_plane(t, v0);
      if (u1) add_plane(t + 1, v1);
    }
#else
#pragma unroll
    for (int t = 0; t < M; ++t) {
      if (!plane_used(t)) continue;
      double val[M];
      load_plane(t, val);
      add_plane(t, val);
    }
#endif
  }
  if (tid <= FX) {
#pragma unroll
    for (int jl = 0; jl < N * N; ++jl) s_u[jl][tid] = u[jl];
  }
  __syncthreads();
  // x sweep: coarse node I of the strip collects the fine positions 2I - (2k-1) .. 2I + (2k-1);
  // the (j, l) pairs of a node are dealt to RG threads
  constexpr int CWmax = GridTile<K>::CW;
  constexpr int RG = GridTile<K>::THREADS / CWmax < FEM_GT_RGROUPS ? GridTile<K>::THREADS / CWmax : FEM_GT_RGROUPS;
  const int I = tid % CWmax, g = tid / CWmax;
  if (g >= RG || I > K * ncx) return;
  const int gcx = K * cx0 + I;
  if (((a.bcmask & 1) && gcx == 0) || ((a.bcmask & 2) && gcx == a.nnc0 - 1)) return;
  double wt[4 * K - 1];
#pragma unroll
  for (int d = 0; d < 4 * K - 1; ++d) {
    const int f = 2 * I + d - (2 * K - 1);
    double w = 0.0;
    if (f >= 0 && f <= 2 * K * ncx) {
      const int c = min(f / (2 * K), ncx - 1), i = I - K * c;
      if (i >= 0 && i <= K) w = sE[f - 2 * K * c][i];
    }
    wt[d] = w;
  }
  const int f0 = 2 * I - (2 * K - 1);
#pragma unroll
  for (int jl0 = 0; jl0 < N * N; jl0 += RG) {
    const int jl = jl0 + g;
    if (jl >= N * N) break;
    const int gy = K * cy + jl % N, gz = K * cz + jl / N;
    double s = 0.0;
#pragma unroll
    for (int d = 0; d < 4 * K - 1; ++d) {
      const int f = min(max(f0 + d, 0), FX);
      s = fma(wt[d], s_u[jl][f], s);
    }
    if (!cg_constrained(a.bcmask & ~3, gcx, gy, K * a.czc0 + gz, a.nnc0, a.nnc1, a.nnc2)) {
#if FEM_GT_RNOATOM
      xc[cg_index(gcx, gy, gz, a.nnc0, a.nnc1)] = s;   // timing experiment only (wrong sums)
#else
      atomicAdd(xc + cg_index(gcx, gy, gz, a.nnc0, a.nnc1), s);
#endif
    }
  }
}

// ---------------------------------------------------------------- vectors
__global__ void cheb_step_kernel(double* __restrict__ xn, const double* __restrict__ x,
                                 const double* __restrict__ xo, const double* __restrict__ b,
                                 double* __restrict__ ax, const double* __restrict__ dinv, double c1,
                                 double c2, int64_t n, bool clear_ax) {
  FEM_PDL_ENTRY();
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double xi = x ? x[i] : 0.0;
    const double xoi = xo ? xo[i] : 0.0;
    const double r = b[i] - (ax ? ax[i] : 0.0);
    xn[i] = xi + c1 * (xi - xoi) + c2 * dinv[i] * r;
    if (clear_ax) ax[i] = 0.0;
  }
}

// First Chebyshev step from x = 0 on a Cartesian CG level with a D^-1 class table (api.cu:
// (k+2)^3 values, class per direction 0 first node, r inside an element, k interior vertex, k+1
// last node): x_1 = c2 D^-1 b reads b and writes x_1 only (16 B per DoF; the D^-1 vector of the
// generic kernel is a third stream: 505 -> 3xx us on the finest C4 level)
template <int K>
__global__ void cheb_first_cls_kernel(double* __restrict__ xn, const double* __restrict__ b,
                                      const double* __restrict__ dcls, double c2, int NX, int NY, int NZ) {
  FEM_PDL_ENTRY();
  constexpr int ZPT = 8;   // z planes per thread: the (x, y) class and index arithmetic once per 8 nodes
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= NX * NY) return;
  const int gy = p / NX, gx = p - gy * NX;
  auto ncls = [](int g, int nn) { return g == 0 ? 0 : g == nn - 1 ? K + 1 : (g % K == 0 ? K : g % K); };
  const double* __restrict__ dxy = dcls + ncls(gx, NX) + (K + 2) * ncls(gy, NY);
  const int gz0 = blockIdx.y * ZPT;
  const int64_t plane = (int64_t)NX * NY;
  const double* __restrict__ pb = b + p + plane * gz0;
  double* __restrict__ px = xn + p + plane * gz0;
  double v[ZPT];
#pragma unroll
  for (int j = 0; j < ZPT; ++j) v[j] = gz0 + j < NZ ? pb[plane * j] : 0.0;
#pragma unroll
  for (int j = 0; j < ZPT; ++j)
    if (gz0 + j < NZ) px[plane * j] = c2 * __ldg(dxy + (K + 2) * (K + 2) * ncls(gz0 + j, NZ)) * v[j];
}

__global__ void axpby_kernel(double* __restrict__ y, const double* __restrict__ x, double a, double b,
                             int64_t n) {
  FEM_PDL_ENTRY();
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    y[i] = a * x[i] + b * y[i];
}

__global__ void fill_kernel(double* __restrict__ y, double v, int64_t n) {
  FEM_PDL_ENTRY();
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    y[i] = v;
}

__global__ void copy_kernel(double* __restrict__ y, const double* __restrict__ x, int64_t n) {
  FEM_PDL_ENTRY();
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    y[i] = x[i];
}

__global__ void add_kernel(double* __restrict__ y, const double* __restrict__ x, int64_t n) {
  FEM_PDL_ENTRY();
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    y[i] += x[i];
}

__global__ void sub_kernel(double* __restrict__ r, const double* __restrict__ b,
                           const double* __restrict__ ax, int64_t n) {
  FEM_PDL_ENTRY();
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    r[i] = b[i] - (ax ? ax[i] : 0.0);
}

__global__ void dinv_kernel(const double* __restrict__ d, double* __restrict__ di, int64_t n) {
  FEM_PDL_ENTRY();
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    di[i] = 1.0 / d[i];
}

__device__ __forceinline__ double u01_splitmix(uint64_t seed, uint64_t i) {
  uint64_t z = seed + (i + 1) * 0x9E3779B97F4A7C15ULL;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  z = z ^ (z >> 31);
  return 2.0 * ((double)(z >> 11) * 0x1.0p-53) - 1.0;
}

__global__ void splitmix_kernel(double* __restrict__ s, uint64_t seed, int64_t first, int64_t n) {
  FEM_PDL_ENTRY();
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    s[i] = u01_splitmix(seed, (uint64_t)(first + i));
}

// ---- deterministic block reduction with a last-block finisher
constexpr int kRedThreads = 256;

__device__ __forceinline__ double block_sum(double v, double* sh) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (lane == 0) sh[w] = v;
  __syncthreads();
  double s = 0.0;
  if (threadIdx.x == 0)
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) s += sh[i];
  __syncthreads();
  return s;
}

// counters: per-handle array (after the partial sums in h->red), so that handles
// running concurrently (ranks of an in-process group) never share a counter
__device__ __forceinline__ void finish_reduction(double part, double* red, double* out, int slot,
                                                 unsigned int* counters) {
  __shared__ bool last;
  if (threadIdx.x == 0) {
    red[blockIdx.x] = part;
    __threadfence();
    const unsigned prev = atomicAdd(&counters[slot], 1u);
    last = (prev == gridDim.x - 1);
  }
  __syncthreads();
  if (last) {
    __shared__ double sh[32];
    double v = 0.0;
    for (int i = threadIdx.x; i < (int)gridDim.x; i += blockDim.x) v += ((volatile double*)red)[i];
    const double s = block_sum(v, sh);
    if (threadIdx.x == 0) {
      out[slot] = s;
      counters[slot] = 0;
    }
  }
}

__global__ void dot_kernel(const double* __restrict__ a, const double* __restrict__ b, int64_t n,
                           double* red, double* out, int slot, unsigned int* counters) {
  FEM_PDL_ENTRY();
  __shared__ double sh[32];
  double v = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    v = fma(a[i], b[i], v);
  const double s = block_sum(v, sh);
  finish_reduction(s, red, out, slot, counters);
}

// alpha = scal[0]/scal[1]  (rz / pq);  x += alpha p;  r -= alpha q;  scal[2] = (r, r)
__global__ void pcg_update_xr_kernel(double* __restrict__ x, double* __restrict__ r,
                                     const double* __restrict__ p, const double* __restrict__ q,
                                     int64_t n, double* red, double* scal, unsigned int* counters) {
  FEM_PDL_ENTRY();
  __shared__ double sh[32];
  const double alpha = scal[0] / scal[1];
  double v = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    x[i] = fma(alpha, p[i], x[i]);
    const double ri = fma(-alpha, q[i], r[i]);
    r[i] = ri;
    v = fma(ri, ri, v);
  }
  const double s = block_sum(v, sh);
  finish_reduction(s, red, scal, 2, counters);
}

// beta = scal[3]/scal[0] (rz_new / rz);  p = z + beta p
__global__ void pcg_update_p_kernel(double* __restrict__ p, const double* __restrict__ z, int64_t n,
                                    const double* scal) {
  FEM_PDL_ENTRY();
  const double beta = scal[3] / scal[0];
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    p[i] = fma(beta, p[i], z[i]);
}

__global__ void copy_scalar_kernel(double* scal, int dst, int src) {
  FEM_PDL_ENTRY(); scal[dst] = scal[src]; }

__global__ void set_scalar_kernel(double* scal, int idx, double v) {
  FEM_PDL_ENTRY(); scal[idx] = v; }

// x = A0^{-1} b on the free DoFs (dense inverse from the Cholesky factor); x = 0 elsewhere.
// x = A0^{-1} b on the free DoFs (dense inverse from the Cholesky factor); x = 0 elsewhere.
// One warp per entry of x (coalesced row reads, shuffle reduction), b's free entries
// staged in shared memory by every block; pos[i] = row of entry i in A0^{-1} or -1.
__global__ void coarse_solve_kernel(const double* __restrict__ Ainv, const int* __restrict__ free_idx,
                                    const int* __restrict__ pos, int nf, const double* __restrict__ b,
                                    double* __restrict__ x, int64_t n) {
  FEM_PDL_ENTRY();
  extern __shared__ double sb[];
  for (int i = threadIdx.x; i < nf; i += blockDim.x) sb[i] = b[free_idx[i]];
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t e = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); e < n; e += warps) {
    const int row = pos[e];
    double s = 0.0;
    if (row >= 0)
      for (int j = lane; j < nf; j += 32) s = fma(Ainv[(int64_t)row * nf + j], sb[j], s);
    for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
    if (lane == 0) x[e] = s;
  }
}

// ---------------------------------------------------------------- launchers
namespace {

inline unsigned vec_grid(int64_t n) {
  int64_t g = (n + 255) / 256;
  return (unsigned)std::max<int64_t>(1, std::min<int64_t>(g, 148 * 16));
}

TransferArgs transfer_args(const fem_ctx* h, const Level& c, const Level& f) {
  TransferArgs a;
  a.nc0 = c.n[0];
  a.nc1 = c.n[1];
  a.nc2 = c.n[2];
  a.nnc0 = c.nn[0];
  a.nnc1 = c.nn[1];
  a.nnc2 = h->k * c.nzg + 1;
  a.nnf0 = f.nn[0];
  a.nnf1 = f.nn[1];
  a.nnf2 = h->k * f.nzg + 1;
  a.czc0 = c.cz0;
  a.ncz = c.nzg;
  int mask = 0;
  for (int s = 0; s < 6; ++s)
    if (h->mesh.bc[s] == FEM_BC_DIRICHLET) mask |= 1 << s;
  a.bcmask = mask;
  return a;
}

template <int K, bool DG>
Embed<K, DG> make_embed(const Tables1D& t) {
  Embed<K, DG> e;
  constexpr int N = K + 1;
  for (int r = 0; r < Embed<K, DG>::M; ++r)
    for (int j = 0; j < N; ++j) e.E[r][j] = DG ? t.dg_embed[r / N][r % N][j] : t.cg_embed[r][j];
  return e;
}

template <int K, bool DG>
void prolongate_kd(fem_ctx* h, const Level& c, const Level& f, const double* xc, double* xf) {
  constexpr int N = K + 1, M = Embed<K, DG>::M;
  if constexpr (!DG && K <= 4) {
    if (c.n_cells >= h->grid_transfer_min_cells) {
      const dim3 grid((unsigned)((c.n[0] + GridTile<K>::TXC - 1) / GridTile<K>::TXC), (unsigned)c.n[1], (unsigned)c.n[2]);
      launch_pdl(h, prolongate_grid_kernel<K>, grid, GridTile<K>::THREADS, 0, transfer_args(h, c, f),
                 make_embed<K, DG>(h->tab), xc, xf);
      count_launch();
      check_launch("prolongate_grid_kernel");
      return;
    }
  }
  if constexpr (!DG) {
    const size_t sm = sizeof(double) * (N * N * N + M * N * N + M * M * N);
    smem_attr(reinterpret_cast<const void*>(prolongate_elem_kernel<K, DG>), (size_t)((int)sm));
    launch_pdl(h, prolongate_elem_kernel<K, DG>, (unsigned)c.n_cells, kTransferThreads, sm,
               transfer_args(h, c, f), make_embed<K, DG>(h->tab), xc, xf);
  } else {
    const size_t sm = sizeof(double) * (M * N * N + M * M * N);
    smem_attr(reinterpret_cast<const void*>(prolongate_kernel<K, DG>), (size_t)((int)sm));
    launch_pdl(h, prolongate_kernel<K, DG>, (unsigned)c.n_cells, kTransferThreads, sm,
               transfer_args(h, c, f), make_embed<K, DG>(h->tab), xc, xf);
  }
  count_launch();
  check_launch("prolongate_kernel");
}

template <int K, bool DG>
void restrict_kd(fem_ctx* h, const Level& c, const Level& f, const double* bf, const double* axf,
                 double* xc) {
  constexpr int N = K + 1, M = Embed<K, DG>::M;
  if constexpr (!DG && K <= 4) {
    if (c.n_cells >= h->grid_transfer_min_cells) {
      const dim3 grid((unsigned)((c.n[0] + GridTile<K>::TXC - 1) / GridTile<K>::TXC), (unsigned)c.n[1], (unsigned)c.n[2]);
      if (axf)
        launch_pdl(h, restrict_grid_kernel<K, true>, grid, GridTile<K>::THREADS, 0, transfer_args(h, c, f),
                   make_embed<K, DG>(h->tab), bf, axf, xc);
      else
        launch_pdl(h, restrict_grid_kernel<K, false>, grid, GridTile<K>::THREADS, 0, transfer_args(h, c, f),
                   make_embed<K, DG>(h->tab), bf, axf, xc);
      count_launch();
      check_launch("restrict_grid_kernel");
      return;
    }
  }
  if constexpr (!DG) {
    const size_t sm = sizeof(double) * (M * M * M + N * M * M);
    smem_attr(reinterpret_cast<const void*>(restrict_elem_kernel<K, DG>), (size_t)((int)sm));
    launch_pdl(h, restrict_elem_kernel<K, DG>, (unsigned)c.n_cells, kTransferThreads, sm,
               transfer_args(h, c, f), make_embed<K, DG>(h->tab), bf, axf, xc);
  } else {
    const size_t sm = sizeof(double) * (N * M * M + N * N * M);
    smem_attr(reinterpret_cast<const void*>(restrict_kernel<K, DG>), (size_t)((int)sm));
    launch_pdl(h, restrict_kernel<K, DG>, (unsigned)c.n_cells, kTransferThreads, sm,
               transfer_args(h, c, f), make_embed<K, DG>(h->tab), bf, axf, xc);
  }
  count_launch();
  check_launch("restrict_kernel");
}

template <int K>
void prolongate_k(fem_ctx* h, const Level& c, const Level& f, const double* xc, double* xf) {
  if (h->method == FEM_CG) prolongate_kd<K, false>(h, c, f, xc, xf);
  else prolongate_kd<K, true>(h, c, f, xc, xf);
}

template <int K>
void restrict_k(fem_ctx* h, const Level& c, const Level& f, const double* bf, const double* axf,
                double* xc) {
  if (h->method == FEM_CG) restrict_kd<K, false>(h, c, f, bf, axf, xc);
  else restrict_kd<K, true>(h, c, f, bf, axf, xc);
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

void launch_prolongate_add(fem_ctx* h, const Level& c, const Level& f, const double* xc, double* xf) {
  FEM_DISPATCH_K(h->k, prolongate_k, h, c, f, xc, xf);
}

void launch_restrict(fem_ctx* h, const Level& c, const Level& f, const double* bf, const double* axf,
                     double* xc) {
  if (h->method == FEM_CG) launch_zero(h, xc, c.n_store);   // ghost plane too (compress-added after)
  FEM_DISPATCH_K(h->k, restrict_k, h, c, f, bf, axf, xc);
}

// zero / copy as kernels (not memset/memcpy graph nodes) so that the PDL chain of the
// solve is not broken
void launch_zero(fem_ctx* h, double* p, int64_t n) {
  if (n <= 0) return;
  launch_pdl(h, fill_kernel, vec_grid(n), 256, 0, p, 0.0, n);
  count_launch();
  check_launch("fill_kernel");
}

void launch_copy(fem_ctx* h, double* dst, const double* src, int64_t n) {
  if (n <= 0) return;
  launch_pdl(h, copy_kernel, vec_grid(n), 256, 0, dst, src, n);
  count_launch();
  check_launch("copy_kernel");
}

void launch_dinv(fem_ctx* h, Level& L) {
  launch_pdl(h, dinv_kernel, vec_grid(L.n_dofs), 256, 0, L.diag, L.dinv, L.n_dofs);
  count_launch();
  check_launch("dinv_kernel");
}

void launch_splitmix(fem_ctx* h, const Level& L, uint64_t seed, double* s) {
  launch_pdl(h, splitmix_kernel, vec_grid(L.n_dofs), 256, 0, s, seed, L.first_global, L.n_dofs);
  count_launch();
  check_launch("splitmix_kernel");
}

void launch_cheb_step(fem_ctx* h, const Level& L, double* xn, const double* x, const double* xo,
                      const double* b, double* ax, double c1, double c2, bool has_xo) {
  // CG, single-slab level: clear the consumed A x so that the next apply into L.t needs
  // no memset (the owned block is the whole storage)
  const bool clear = ax != nullptr && ax == L.t && h->method == FEM_CG && !L.dist;
  launch_pdl(h, cheb_step_kernel, vec_grid(L.n_dofs), 256, 0, xn, x, has_xo ? xo : nullptr, b, ax,
                                                              L.dinv, c1, c2, L.n_dofs, clear);
  if (clear) L.t_zero = true;
  count_launch();
  check_launch("cheb_step_kernel");
}

void launch_cheb_first_cls(fem_ctx* h, const Level& L, double* xn, const double* b, double c2) {
  const int NX = L.nn[0], NY = L.nn[1], NZ = L.nn[2];
  const dim3 grid((unsigned)(((int64_t)NX * NY + 255) / 256), (unsigned)((NZ + 7) / 8));
  const double* dcls = L.dinv_cls;
  switch (h->k) {
    case 1: launch_pdl(h, cheb_first_cls_kernel<1>, grid, 256, 0, xn, b, dcls, c2, NX, NY, NZ); break;
    case 2: launch_pdl(h, cheb_first_cls_kernel<2>, grid, 256, 0, xn, b, dcls, c2, NX, NY, NZ); break;
    case 3: launch_pdl(h, cheb_first_cls_kernel<3>, grid, 256, 0, xn, b, dcls, c2, NX, NY, NZ); break;
    case 4: launch_pdl(h, cheb_first_cls_kernel<4>, grid, 256, 0, xn, b, dcls, c2, NX, NY, NZ); break;
    default: throw Error{FEM_E_ARG, "class-table Chebyshev step: k in 1..4"};
  }
  count_launch();
  check_launch("cheb_first_cls_kernel");
}

// reduction grid: deterministic for a given n (the finisher sums gridDim.x partials in order)
inline unsigned red_grid(int64_t n) {
  return (unsigned)std::max<int64_t>(1, std::min<int64_t>((n + kRedThreads - 1) / kRedThreads, kRedBlocks));
}

void launch_dot(fem_ctx* h, const double* a, const double* b, int64_t n, int slot) {
  launch_pdl(h, dot_kernel, red_grid(n), kRedThreads, 0, a, b, n, h->red + slot * kRedBlocks, h->scal,
                                                        slot, (unsigned int*)(h->red + 16 * kRedBlocks));
  count_launch();
  check_launch("dot_kernel");
}

void launch_pcg_update_xr(fem_ctx* h, double* x, double* r, const double* p, double* q, int64_t n) {
  launch_pdl(h, pcg_update_xr_kernel, red_grid(n), kRedThreads, 0, x, r, p, q, n,
                                                                  h->red + 2 * kRedBlocks, h->scal,
                                                                  (unsigned int*)(h->red + 16 * kRedBlocks));
  count_launch();
  check_launch("pcg_update_xr_kernel");
}

void launch_pcg_update_p(fem_ctx* h, double* p, const double* z, int64_t n) {
  launch_pdl(h, pcg_update_p_kernel, vec_grid(n), 256, 0, p, z, n, h->scal);
  count_launch();
  check_launch("pcg_update_p_kernel");
  launch_pdl(h, copy_scalar_kernel, 1, 1, 0, h->scal, 0, 3);
  count_launch();
  check_launch("copy_scalar_kernel");
}

void launch_set_scalar(fem_ctx* h, int idx, double v) {
  launch_pdl(h, set_scalar_kernel, 1, 1, 0, h->scal, idx, v);
  count_launch();
  check_launch("set_scalar_kernel");
}

void launch_coarse_solve(fem_ctx* h, const double* b, double* x) {
  const Level& L0 = h->levels[0];
  const unsigned grid = (unsigned)std::min<int64_t>((L0.n_dofs + 7) / 8, 148);
  launch_pdl(h, coarse_solve_kernel, grid, 256, sizeof(double) * h->n_coarse_free, h->coarse_inv,
             h->coarse_free, h->coarse_pos, h->n_coarse_free, b, x, L0.n_dofs);
  count_launch();
  check_launch("coarse_solve_kernel");
}

void launch_axpby(fem_ctx* h, double* y, const double* x, double a, double b, int64_t n) {
  launch_pdl(h, axpby_kernel, vec_grid(n), 256, 0, y, x, a, b, n);
  count_launch();
  check_launch("axpby_kernel");
}

void launch_add(fem_ctx* h, double* y, const double* x, int64_t n) {
  if (n <= 0) return;
  launch_pdl(h, add_kernel, vec_grid(n), 256, 0, y, x, n);
  count_launch();
  check_launch("add_kernel");
}

void launch_sub(fem_ctx* h, double* r, const double* b, const double* ax, int64_t n) {
  launch_pdl(h, sub_kernel, vec_grid(n), 256, 0, r, b, ax, n);
  count_launch();
  check_launch("sub_kernel");
}

}  // namespace fem
