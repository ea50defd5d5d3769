// libfem internals: 1-D tables, level hierarchy, handle.  B200 / sm_100a, FP64.
// Nothing here is shared with oracle/ (the CPU reference re-derives everything).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <memory>
#include <utility>
#include <string>
#include <vector>

#include "../../include/fem.h"

// Q4 CG line kernel thread layout (kernels_cg.cu): 1 = cells fastest (default)
#ifndef FEM_LINE_CELL_FAST
#define FEM_LINE_CELL_FAST 1
#endif

namespace fem {

constexpr int kMaxDeg = 8;
constexpr int kMaxN = kMaxDeg + 1;

// ---------------------------------------------------------------- errors
void set_error(const std::string& msg);
struct Error {
  int code;
  std::string msg;
};
#define FEM_CUDA_TRY(expr)                                                              \
  do {                                                                                  \
    cudaError_t e_ = (expr);                                                            \
    if (e_ != cudaSuccess)                                                              \
      throw ::fem::Error{e_ == cudaErrorMemoryAllocation ? FEM_E_OOM : FEM_E_CUDA,       \
                         std::string(#expr) + ": " + cudaGetErrorString(e_)};           \
  } while (0)

void count_launch(int n = 1);
void check_launch(const char* what);

// ---------------------------------------------------------------- 1-D tables
// GLL Lagrange basis at the (k+1)-point Gauss rule.
struct Tables1D {
  int k = 0, n = 0;
  double gll[kMaxN];              // GLL nodes on [-1,1]
  double qp[kMaxN], qw[kMaxN];    // Gauss points / weights
  double val[kMaxN][kMaxN];       // [q][i] phi_i(qp_q)
  double der[kMaxN][kMaxN];       // [q][i] phi_i'(qp_q)
  double colloc[kMaxN][kMaxN];    // [q][p] l_p'(qp_q), l = Lagrange basis on Gauss points
  double dface[2][kMaxN];         // [side][i] phi_i'(-1), phi_i'(+1)
  double cg_embed[2 * kMaxDeg + 1][kMaxN];  // [fine node r of the 2 children][coarse j]
  double dg_embed[2][kMaxN][kMaxN];         // [child][fine i][coarse j]
};
void build_tables(int k, Tables1D& t);
void gll_points(int l, double* x);   // GLL(l) nodes (mapping support points)
// the level's cell map uses the general (table-driven) path: shell, polynomial mapping or kappa (N3)
inline bool mesh_general(const fem_mesh& m) {
  return m.geometry != FEM_GEOM_BOX || m.mapping_degree != 0 || m.kappa_amplitude != 0.0;
}

// ---------------------------------------------------------------- communication
// Transport of the z-slab exchanges: NCCL between processes, or an
// in-process group of threads sharing one device (comm.cu).  All calls are
// enqueued on the caller's stream; every rank issues the same sequence.
class Comm {
 public:
  struct Msg {
    int peer;      // other rank
    int tag;       // matches a send of the peer with a recv here (in-process transport)
    double* ptr;   // device buffer
    int64_t n;     // doubles
  };
  int rank = 0, nranks = 1;
  virtual ~Comm() {}
  virtual void exchange(const std::vector<Msg>& sends, const std::vector<Msg>& recvs, cudaStream_t s) = 0;
  virtual void allreduce_sum(double* p, int64_t n, cudaStream_t s) = 0;
  virtual bool graph_capturable() const = 0;
  // asynchronous transport errors (NCCL: ncclCommGetAsyncError); throws FEM_E_NCCL
  virtual void check() {}
};
std::unique_ptr<Comm> make_nccl_comm(const void* id, int rank, int nranks);
std::unique_ptr<Comm> make_local_comm(void* group, int rank, int nranks);

// ---------------------------------------------------------------- level data
// Vector convention: every level vector pointer points at the rank's OWNED block;
// ghost data lives in the same allocation (CG: the ghost node plane right after
// the owned planes; SIPG: one ghost cell layer before and one after the owned
// cells).  Vector kernels touch [0, n_dofs); operator kernels read the ghosts.
struct Level {
  int idx = 0;
  int n[3] = {0, 0, 0};          // rank-local cells per direction (z: slab layers)
  int nn[3] = {0, 0, 0};         // CG nodes per direction held locally (z: k n[2] + 1)
  int nzg = 0;                   // cells in z of the whole level
  int cz0 = 0;                   // global index of the first local cell layer
  bool dist = false;             // z-slab of this rank (else replicated / single rank)
  int ghost_lo = -1, ghost_hi = -1;  // neighbour ranks (dist only)
  double h[3] = {0, 0, 0};
  int64_t n_cells = 0;           // local cells
  int64_t n_dofs = 0;            // owned DoFs (vector length)
  int64_t n_store = 0;           // owned + ghost DoFs
  int64_t own_off = 0;           // owned block offset inside the allocation
  int64_t first_global = 0, n_global = 0;
  bool cartesian = true;
  double cart[3] = {0, 0, 0};    // Cartesian metric: det(J) (2/h_d)^2
  double* G = nullptr;           // deformed: geometry table, layout g_index (device_common.cuh)
  int glayout = 0;               // kGLayout* of G (device_common.cuh)
  double* face = nullptr;        // SIPG deformed: face data, see kernels_dg.cu
  double* diag = nullptr;        // diag(A)
  double* dinv = nullptr;        // 1/diag on free DoFs, 0 on constrained
  double lam = 0.0;
  // work vectors for the V-cycle (level >= 1 need all, level 0 needs b, x)
  double *b = nullptr, *x = nullptr, *x2 = nullptr, *x3 = nullptr, *t = nullptr, *b2 = nullptr;
  // host-side knowledge that t is all zeros (the Chebyshev step clears the A x it
  // consumes), so that the next CG apply into t needs no memset; reset at graph capture
  mutable bool t_zero = false;
  // CG single-rank deformed levels: three A x buffers rotated by the fused Chebyshev
  // sequences (each fused kernel clears the buffer the next one accumulates into)
  double* tf[3] = {nullptr, nullptr, nullptr};
  // Cartesian SIPG single-rank levels: D^-1 depends on the cell only through which of its
  // faces lie on the boundary (3 classes per direction): 27 x n^3 values copied from dinv
  double* dinv_cls = nullptr;
  // PCG vectors (finest level, allocated on first cg_solve)
  double *pcg_r = nullptr, *pcg_p = nullptr, *pcg_q = nullptr, *pcg_z = nullptr;
  double* halo = nullptr;        // CG dist: receive buffer of one node plane (compress-add)
  // last distributed level above a replicated one: the whole-level twin used for
  // the transfers (gathered residual gb, prolongated correction gx; no geometry)
  std::unique_ptr<Level> full;
  double *gb = nullptr, *gx = nullptr;
};

// Chebyshev step fused into an element-centric (SIPG) operator apply: the kernel writes
// x_new = x + c1 (x - x_old) + c2 D^-1 (b - A x) instead of A x.
struct ChebFuse {
  const double* xo = nullptr;    // x_old (nullptr: first step)
  const double* b = nullptr;
  const double* dinv = nullptr;
  const double* dinv_cls = nullptr;   // Cartesian SIPG: D^-1 per cell class (27 x n^3), or nullptr
  double c1 = 0.0, c2 = 0.0;
  int on = 0;
};

// Chebyshev step fused into the CG line-kernel gather (kernels_cg.cu, FUSED)
struct CgFuse {
  const double* xo = nullptr;    // x_old (nullptr: none)
  const double* b = nullptr;
  const double* dinv = nullptr;
  const double* t = nullptr;     // A x of the kernel's input x
  double* xnew = nullptr;        // the new iterate (written by the owning cells)
  int materialize = 1;           // 0: apply x itself (only zbuf is cleared)
  double* zbuf = nullptr;        // cleared by the owning cells (the next target), or nullptr
  double c1 = 0.0, c2 = 0.0;
  int on = 0;
};

struct Profile {
  bool on = false;
  int mode = 0;                  // fem_options.profile: 1 PCG applies, 2 finest-level smoother steps
  std::vector<cudaEvent_t> ev;   // pairs (start, stop) recorded eagerly
  std::vector<double> evb;       // algorithmic bytes of each eager pair
  size_t used = 0;
  double ms = 0.0;
  double bytes = 0.0;            // algorithmic bytes of the timed launches (mode 2)
  int64_t launches = 0;
  // while a graph is being captured, event pairs go here (owned by the graph)
  bool capturing = false;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>>* cap = nullptr;
  std::vector<double>* capb = nullptr;   // bytes of each captured pair
};

// One PCG iteration as two CUDA graphs (P:L1144-1148 loop body):
//   g_pre = V-cycle z = V(r), (r,z), p = z + beta p
//   g_upd = q = A p, (p,q), x += alpha p, r -= alpha q, (r,r), scalars -> pinned host
struct SolveGraphs {
  cudaGraphExec_t g_pre = nullptr, g_upd = nullptr;
  int64_t k_pre = 0, k_upd = 0;   // kernels per replay
  const double* b = nullptr;
  double* x = nullptr;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> ev_pre, ev_upd;
  std::vector<double> evb_pre, evb_upd;   // algorithmic bytes per timed launch (profile mode 2)
  // the whole PCG loop as one graph: a conditional WHILE node around both parts and an
  // on-device stopping test (single rank, no profiling); cond_failed: not supported, host loop
  cudaGraphExec_t g_loop = nullptr;
  bool cond_failed = false;
  int64_t k_iter = 0;
  double* hist_dev = nullptr;   // [kCondHist] relative residuals of the device loop
};
constexpr int kCondHist = 4096;

}  // namespace fem

struct fem_ctx {
  int k = 0, method = 0;
  fem_mesh mesh{};
  fem_options opt{};
  int device = 0;
  cudaStream_t stream = nullptr;
  fem::Tables1D tab;
  std::vector<fem::Level> levels;
  // coarse solve: free DoFs of level 0 and the dense inverse (via Cholesky)
  int n_coarse_free = 0;
  int* coarse_free = nullptr;
  int* coarse_pos = nullptr;       // [n] row of each level-0 entry in the inverse, -1 if constrained
  double* coarse_inv = nullptr;
  // reductions
  double* red = nullptr;          // partial sums [kRedBlocks * 4]
  double* scal = nullptr;         // device scalars [16]
  double* hscal = nullptr;        // pinned host mirror [16]
  // host staging
  double* stage[3] = {nullptr, nullptr, nullptr};
  int64_t stage_len = 0;
  unsigned long long* geom_err = nullptr;  // device: first cell with det J <= 0
  fem::Profile prof;
  cudaStream_t cap_stream = nullptr;   // non-blocking stream used only for graph capture
  fem::SolveGraphs sg;
  std::vector<double> hist;             // ||r_i|| / ||b|| of the last cg_solve, i = 0 .. iterations
  std::unique_ptr<fem::Comm> comm;      // nranks > 1
  int rank = 0, nranks = 1;
  bool use_graphs = true;               // PCG iteration as CUDA graphs (not with the in-process transport)
  bool overlap = true;                  // FEM_OVERLAP=0: halo exchanges serialised with the applies
  cudaStream_t comm_stream = nullptr;   // halo exchanges of distributed levels
  cudaEvent_t ev_fork = nullptr, ev_import = nullptr, ev_export = nullptr;
  int chunk_layers = 0;                 // Cartesian CG apply: cell layers per z-chunk (FEM_CHUNK_LAYERS; 0 = one launch)
  bool general_path = false;           // FEM_GENERAL_PATH=1: quadrature kernel on Cartesian levels too
  bool plane_kernel = false;           // FEM_PLANE=1: plane kernel on deformed CG levels (K <= 4)
  int64_t tma_min_blocks = 0;          // FEM_TMA_MIN_BLOCKS: launches this small read G directly
  bool g_direct = true;                // line kernel reads G from global (else TMA-staged; default at Q4); FEM_G_DIRECT
  bool y_is_zero = false;              // set around launch_cg_apply: the output is known to be zero
  fem::ChebFuse fuse;                   // set around a fused Chebyshev apply (SIPG levels)
  fem::CgFuse cgf;                      // set around a fused Chebyshev step + apply (CG levels)
  bool pdl = true;                     // FEM_PDL=0: plain launches (no programmatic dependent launch)
  int64_t fuse_max_cells = 512;        // FEM_FUSE_CELLS: CG levels up to this many cells use the fused step
  bool dinv_classes = true;            // FEM_DINV_CLASSES=0: fused SIPG epilogue reads the full D^-1
  bool fuse_cheb = true;               // FEM_FUSE_CHEB=0: separate Chebyshev-step kernels
  bool line_cell_fast = FEM_LINE_CELL_FAST != 0;   // Q4 line kernel: cells-fastest layout, G in kGLayoutCell8
  bool dg_kron = true;                 // FEM_DG_KRON=0: quadrature cell+face kernel on Cartesian SIPG levels
  bool cg_geo_fly = false;              // FEM_CG_GEO_FLY=1: deformed CG recomputes G from the analytic box map (measured slower: C2 apply 62.6 vs 57.1 us)
  bool dg_cgeo_fly = false;            // FEM_DG_CGEO_FLY=1: deformed SIPG cell metric from the analytic map
  bool dg_fgeo_fly = false;            // FEM_DG_FGEO_FLY=1: deformed SIPG recomputes the face geometry (measured slower: C5 7.28 vs 5.35 ms)
  bool stencil = false;                // FEM_STENCIL=1: atomic-free global Kronecker stencil on Cartesian CG levels (K1s, study)
  bool stencil2 = true;                // FEM_STENCIL2=0: warp-specialised assembled stencil (K1t) off
  bool cheb_first_cls = true;   // FEM_CHEB_FIRST_CLS: first Chebyshev step from x = 0 reads D^-1 from the class table (K1t levels)
  int64_t grid_transfer_min_cells = 4096;  // FEM_GT_MIN_CELLS: node-grid CG transfers (k <= 4) onto coarse levels with >= this many local cells
  int64_t stencil2_min_cells = 32768;  // FEM_ST_MIN_CELLS: K1t on single-rank Cartesian CG levels with >= this many cells
                                       // (C4 solve, 5 its: 4096 118.6 ms, 32768 116.9, 262144 116.4-119.2, 2097152 124.4: below
                                       // 32^3 cells the few z-marching blocks of K1t are latency-bound, 47 us at 16^3)
  int stencil_ez = 0;                  // FEM_ST_EZ: K1t z-element layers per block (0: 32)
  bool dbasis = false;                 // FEM_DBASIS=1: derivative-basis line kernel (measured slower, kept for study)
};

namespace fem {

constexpr int kRedBlocks = 1184;  // 8 x 148 SMs (256 threads each: full occupancy for the HBM-bound passes)

// kernels (kernels_*.cu)
void launch_geometry(fem_ctx* h, Level& L);
void launch_apply(fem_ctx* h, const Level& L, const double* x, double* y, bool accumulate_into_zeroed);
void launch_diagonal(fem_ctx* h, Level& L);
void launch_rhs(fem_ctx* h, const Level& L, double* b);
void launch_prolongate_add(fem_ctx* h, const Level& coarse, const Level& fine, const double* xc,
                           double* xf);
void launch_restrict(fem_ctx* h, const Level& coarse, const Level& fine, const double* bf,
                     const double* axf, double* xc);
void launch_set_constrained(fem_ctx* h, const Level& L, const double* x, double* y);  // y_c = x_c (x null: 1)
void launch_set_constrained_value(fem_ctx* h, const Level& L, double v, double* y);    // y_c = v
void launch_zero(fem_ctx* h, double* p, int64_t n);
void launch_copy(fem_ctx* h, double* dst, const double* src, int64_t n);
void launch_dinv(fem_ctx* h, Level& L);
void launch_splitmix(fem_ctx* h, const Level& L, uint64_t seed, double* s);
// Chebyshev three-term step:  xn = x + c1 (x - xo) + c2 Dinv (b - Ax); Ax <- 0.
void launch_cheb_step(fem_ctx* h, const Level& L, double* xn, const double* x, const double* xo,
                      const double* b, double* ax, double c1, double c2, bool has_xo);
// x_1 = c2 D^-1 b from the D^-1 class table (Cartesian CG levels with L.dinv_cls)
void launch_cheb_first_cls(fem_ctx* h, const Level& L, double* xn, const double* b, double c2);
// reductions into h->scal[slot] (device)
void launch_dot(fem_ctx* h, const double* a, const double* b, int64_t n, int slot);
// PCG pieces
void launch_pcg_update_xr(fem_ctx* h, double* x, double* r, const double* p, double* q, int64_t n);
void launch_pcg_update_p(fem_ctx* h, double* p, const double* z, int64_t n);
void launch_coarse_solve(fem_ctx* h, const double* b, double* x);
void launch_set_scalar(fem_ctx* h, int idx, double v);
void launch_axpby(fem_ctx* h, double* y, const double* x, double a, double b, int64_t n);
void launch_sub(fem_ctx* h, double* r, const double* b, const double* ax, int64_t n);

// level helpers
inline bool is_cg(const fem_ctx* h) { return h->method == FEM_CG; }

// Launch with programmatic dependent launch (PDL, sm_90+): the kernel may be scheduled
// while its predecessor on the stream drains; it must begin with pdl_entry()
// (device_common.cuh), which waits for the predecessor's completion and memory flush
// before anything that reads its results.  Captured into the PCG graphs as
// programmatic edges; it removes most of the launch gap between the many small
// kernels of the coarse multigrid levels.
template <typename... KArgs, typename... Args>
inline void launch_pdl(fem_ctx* h, void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = h->stream;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = h->pdl ? 1 : 0;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  const cudaError_t e = cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
  if (e != cudaSuccess) throw Error{FEM_E_CUDA, std::string("cudaLaunchKernelEx: ") + cudaGetErrorString(e)};
}

// Raise a kernel's dynamic shared-memory limit to at least `bytes` on the current
// device (once per kernel, device and size; thread-safe).
void smem_attr(const void* func, size_t bytes);

// z-slab exchanges (api.cu); no-ops on replicated levels / single rank
void halo_import(fem_ctx* h, const Level& L, double* v);      // ghosts <- neighbours' owned data
void halo_export_add(fem_ctx* h, const Level& L, double* v);  // CG: ghost plane added into the owner
void allreduce(fem_ctx* h, double* p, int64_t n);             // sum over ranks (device buffer)
void launch_add(fem_ctx* h, double* y, const double* x, int64_t n);  // y += x

// Cartesian CG single-rank levels, k = 2..4: atomic-free assembled stencil (kernels_stencil.cu)
inline bool use_stencil2(const fem_ctx* h, const Level& L) {
  return h->method == FEM_CG && h->stencil2 && L.cartesian && !L.dist && !h->general_path &&
         h->k >= 1 && h->k <= 4 && L.n_cells >= h->stencil2_min_cells &&
         (int64_t)L.nn[0] * L.nn[1] < (int64_t(1) << 31);   // 32-bit in-plane offsets
}
void launch_cg_stencil_apply(fem_ctx* h, const Level& L, const double* x, double* y, bool setc);
void launch_cg_stencil_cheb(fem_ctx* h, const Level& L, const double* x, const double* xo, const double* b,
                            double* xnew, double c1, double c2);

}  // namespace fem
