/*
 * libfem — B200 (sm_100a) FP64 matrix-free high-order Laplace operator (CG and
 * SIPG on hexahedral Q_k elements) and its geometric-multigrid preconditioned
 * conjugate gradient solver.  C ABI: plain pointers and sizes only.
 *
 * Method: arXiv 1611.03029 (Kronbichler & Wall), cited as P:L<line> of
 * /root/reference/PAPER.md, section/equation labels in brackets:
 *   operator           eq:poisson_fem, eq:poisson_dgsip,
 *                      eq:bc_dgsip, matrix-free evaluation eq:mf_eval
 *                       with sum factorization;
 *   solver             P:L1144-1148 (PCG + V-cycle, relative residual stop),
 *                      P:L1159-1185 (Chebyshev-Jacobi smoother on
 *                      [0.06, 1.2] lambda_max, 15 CG iterations for lambda_max,
 *                      tensorial level transfer, small coarse solve).
 * Readings where the paper is silent are listed in DESIGN.md ("Readings").
 *
 * VECTORS.  Every vector argument is a contiguous array of doubles of the
 * length the call states.  It may live in DEVICE memory (cudaMalloc, torch CUDA
 * tensor on the handle's device) or in HOST memory (pageable or pinned); the
 * library detects which with cudaPointerGetAttributes.  Device vectors are
 * used in place; host vectors are staged through library-owned device buffers
 * (copy in, compute, copy out) inside the call.  The caller owns every vector
 * and the library keeps no pointer after a call returns.
 *   CG layout:   global lexicographic node index g_x + (k n_x + 1)(g_y + (k n_y + 1) g_z),
 *                node (g_x, g_y, g_z) = (k c_x + i, k c_y + j, k c_z + l); the vector
 *                includes Dirichlet-constrained entries.
 *   SIPG layout: cell-major, cell c = c_x + n_x (c_y + n_y c_z), local index
 *                i + (k+1) j + (k+1)^2 l.
 *   Multi-rank (nranks > 1): vectors are the rank's owned z-slab slice in
 *   global order (see fem_info).
 *
 * ASYNCHRONY.  Calls on device vectors are enqueued on the handle's stream and
 * return before completion unless stated otherwise; host-vector calls and
 * cg_solve are synchronous.  A handle is not thread-safe; separate handles are
 * independent.
 *
 * ERRORS.  Every int-returning call returns FEM_OK (0) or a negative FEM_E_*
 * code (cg_solve may also return FEM_NOT_CONVERGED = 1); fem_last_error()
 * returns a thread-local message describing the last failure.
 */
#ifndef LIBFEM_FEM_H
#define LIBFEM_FEM_H

#include <stdint.h>

#if defined(__GNUC__)
#define FEM_API __attribute__((visibility("default")))
#else
#define FEM_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

#define FEM_OK 0
#define FEM_NOT_CONVERGED 1       /* cg_solve: maxit reached; x holds the last iterate   */
#define FEM_E_ARG (-1)            /* bad degree/method/mesh, null pointer, bad level       */
#define FEM_E_SIZE (-2)           /* vector length differs from the length the call needs  */
#define FEM_E_GEOMETRY (-3)       /* det J <= 0 at some quadrature point; message names cell */
#define FEM_E_BREAKDOWN (-4)      /* p^T A p <= 0, NaN/Inf residual or Lanczos breakdown   */
#define FEM_E_CUDA (-5)           /* CUDA runtime error                                    */
#define FEM_E_NCCL (-6)           /* NCCL error (multi-rank)                               */
#define FEM_E_OOM (-7)            /* device allocation failed                              */

typedef struct fem_ctx* fem_handle;     /* opaque; created by fem_setup, owned by libfem */

typedef enum { FEM_CG = 0, FEM_SIPG = 1 } fem_method;
typedef enum { FEM_BC_DIRICHLET = 0, FEM_BC_NEUMANN = 1 } fem_bc;
typedef enum { FEM_GEOM_BOX = 0, FEM_GEOM_SHELL = 1 } fem_geometry;

/* Structured hexahedral mesh of the box [lo, hi] (cells are images of
 * [-1,1]^3).  Optional smooth deformation x_d += eps * prod_e sin(pi t_e),
 * t = (xhat - lo)/(hi - lo) (BASELINE.json configs[1], [4]); eps = 0 => Cartesian.
 *
 * SURVEY §8f N3 (zero-initialised fields keep the box / exact map / kappa = 1):
 * geometry FEM_GEOM_SHELL: the n[0] x n[1] x n[2] cells tile one of the six
 *   cube-sphere patches of the paper's spherical shell 0.5 < r < 1:
 *   t = (c + (xi+1)/2)/n, a = tan(pi/2 (t0 - 1/2)), b = tan(pi/2 (t1 - 1/2)),
 *   r = 0.5 + 0.5 t2, x = r (1, a, b)/|(1, a, b)|  (lo, hi and deform_eps unused);
 * mapping_degree l in [1, 8]: every cell is mapped by the degree-l polynomial through
 *   the exact map at its tensor GLL(l) support points (the paper's shell
 *   uses l = 5); 0 = the exact map's analytic Jacobian;
 * kappa_amplitude A != 0: diffusivity kappa(x) = 1 + A prod_{e=1}^{3} cos(2 pi x_e + 0.1 e)
 *   (eq:diffusivity_shell; the paper's A = 1e6 makes kappa negative on
 *   parts of the domain -- DESIGN.md reading N3-c -- which the apply accepts and the
 *   PCG solver does not, it needs kappa > 0).  kappa is folded into the geometry
 *   tables (G_q = kappa w det J J^-1 J^-T, face JxW), so it costs no apply bandwidth.
 * Any of the three selects the general (table-driven) operator path on every level. */
typedef struct {
  int32_t n[3];          /* cells per direction on the finest level (>= 1)            */
  double lo[3], hi[3];   /* box corners                                               */
  double deform_eps;     /* deformation amplitude; 0 => Cartesian fast path           */
  int32_t bc[6];         /* fem_bc of the sides -x,+x,-y,+y,-z,+z                      */
  int32_t rank, nranks;  /* z-slab partition (nranks = 1: single GPU); n[2] % nranks == 0 */
  const void* nccl_id;   /* host pointer to a 128-byte ncclUniqueId (fem_nccl_unique_id on
                            one rank, broadcast by the caller), or NULL                     */
  void* local_group;     /* fem_local_group_create() handle: the nranks ranks are threads of
                            ONE process sharing one device (test transport), or NULL.
                            nranks > 1 needs exactly one of nccl_id / local_group.        */
  int32_t geometry;      /* fem_geometry (FEM_GEOM_BOX)                                   */
  int32_t mapping_degree;/* 0 = exact map; l in [1, 8] = degree-l polynomial mapping        */
  double kappa_amplitude;/* A of eq:diffusivity_shell; 0 => kappa = 1                      */
} fem_mesh;

/* Solver knobs; pass NULL to fem_setup for the defaults in brackets. */
typedef struct {
  double penalty_factor;          /* SIPG sigma_F = c (k+1)^2 / h_F        [2.0]  */
  int32_t cheb_degree;            /* Chebyshev error-polynomial degree     [5]    */
  double cheb_lo, cheb_hi;        /* interval factors on lambda_max        [0.06, 1.2] */
  int32_t eig_iters;              /* CG iterations for lambda_max          [15] */
  int32_t coarse_cells;           /* stop coarsening at max cells/dir <=   [1]    */
  uint64_t eig_seed;              /* splitmix64 seed of the start vector   [0x5eed] */
  const double* lambda_override;  /* host array [n_levels] or NULL (tests)        */
  void* stream;                   /* cudaStream_t; NULL => legacy default stream  */
  int32_t device;                 /* CUDA device ordinal; -1 => current device    */
  int32_t profile;                /* 1 => time the finest PCG applies with events,
                                     2 => time the finest-level smoother steps  */
  int32_t slab_min_layers;        /* multi-rank: a level is split into z-slabs while
                                     every rank keeps >= this many cell layers     [1] */
  int64_t slab_min_dofs;          /* ... and >= this many DoFs per rank; coarser
                                     levels are replicated on every rank (they are
                                     latency-bound: a halo exchange per apply would
                                     cost more than the redundant work)        [32768] */
} fem_options;

/* Fills *opt with the defaults above.  Returns FEM_OK or FEM_E_ARG (opt NULL). */
FEM_API int fem_default_options(fem_options* opt);

/* Builds the level hierarchy (halving while every n_d is even and max n_d >
 * coarse_cells), the geometry tables (R2), diagonals (R6), lambda_max estimates
 * and the coarse Cholesky factor (R9).  degree k in [1, 8].
 * Synchronous.  Errors: FEM_E_ARG (bad degree/method/mesh/options),
 * FEM_E_GEOMETRY (det J <= 0, message names the level and cell), FEM_E_CUDA,
 * FEM_E_OOM, FEM_E_BREAKDOWN (Lanczos breakdown), FEM_E_NCCL.  *out is set only
 * on success. */
FEM_API int fem_setup(const fem_mesh* mesh, int32_t degree, int32_t method, const fem_options* opt,
              fem_handle* out);

/* ---- multi-rank z-slab partition ----
 * Rank r of P owns the cell layers c_z in [r n_z/P, (r+1) n_z/P) of every
 * distributed level.  CG: it owns the node planes [k z0, k z1) (the last rank also
 * the top plane k n_z) and keeps the plane k z1 of rank r+1 as a ghost (imported
 * before every operator apply, its contributions compress-added back after it).
 * SIPG: it owns its cells' blocks and keeps one ghost cell layer from each
 * neighbour rank.  PCG dot products are all-reduced.  Levels coarser than the
 * last one that still gives every rank slab_min_layers layers and slab_min_dofs DoFs
 * are replicated: the
 * residual of the last distributed level is gathered (all-reduce of zero-padded
 * owned slices) and the coarse levels run redundantly on every rank.
 * fem_partition is pure host arithmetic (no device needed): it describes, level by
 * level (0 = coarsest), what fem_setup will build for `mesh->rank`. */
typedef struct {
  int32_t cells[3];          /* rank-local cells per direction                          */
  int32_t global_cells[3];   /* cells per direction of the whole level                  */
  int32_t cell_z0;           /* global index of the first local cell layer              */
  int32_t distributed;       /* 1: z-slab of this rank; 0: replicated on every rank     */
  int64_t n_owned;           /* owned DoFs = length of the rank-local vectors           */
  int64_t first_global;      /* global index of the first owned DoF                     */
  int64_t n_global;          /* DoFs of the whole level                                 */
  int64_t n_stored;          /* owned + ghost DoFs the rank keeps                       */
  int32_t ghost_lo, ghost_hi;/* neighbour ranks whose data is imported (-1: none)       */
} fem_level_part;

/* Fills out[0 .. *n_levels) (coarsest first) for mesh->rank; max_levels bounds out.
 * opt may be NULL (defaults).  The finest level is always distributed and the
 * coarsest always replicated when nranks > 1.  Errors: FEM_E_ARG (bad
 * degree/method/mesh, n[2] not divisible by nranks, a multi-rank mesh that does
 * not coarsen at least once, max_levels too small). */
FEM_API int fem_partition(const fem_mesh* mesh, int32_t degree, int32_t method, const fem_options* opt,
                  fem_level_part* out, int32_t max_levels, int32_t* n_levels);

/* Writes a fresh 128-byte ncclUniqueId into id (host memory, len >= 128); call on
 * one rank and broadcast.  NCCL is loaded at run time (libnccl.so.2; the copy the
 * process already has, e.g. torch's, is reused).  Errors: FEM_E_NCCL. */
FEM_API int fem_nccl_unique_id(void* id, int64_t len);

/* In-process transport for nranks threads sharing one device (tests, and to run
 * the multi-rank path on a single GPU).  Each thread calls the collective entry
 * points of its own handle; exchanges are device-to-device copies ordered by
 * events between the ranks' streams (no kernel waits on another).  Destroy after
 * every handle using it.  Errors: FEM_E_ARG. */
FEM_API int fem_local_group_create(int32_t nranks, void** group);
FEM_API void fem_local_group_destroy(void* group);

/* Sizes: rank-local and global DoF counts of the finest level, first global
 * index owned, number of levels.  Any output pointer may be NULL. */
FEM_API int fem_info(fem_handle h, int64_t* n_local, int64_t* n_global, int64_t* first_global,
             int32_t* n_levels);

/* y = A x on the finest level (eq:mf_eval).  CG: constrained entries of x are
 * read as 0 and y_c = x_c (Dirichlet row/column elimination).
 * nx, ny must equal n_local.  x and y must not alias. */
FEM_API int fem_apply(fem_handle h, const double* x, int64_t nx, double* y, int64_t ny);

/* d = diag(A) on the finest level (1 on constrained CG rows): "the matrix diagonal that
 * is pre-computed and stored" for the Jacobi part of the smoother, the
 * diagonal of the operator of eq:poisson_fem / eq:poisson_dgsip (cell and face terms). */
FEM_API int fem_diagonal(fem_handle h, double* d, int64_t nd);

/* z = V(r): one multigrid V-cycle, z overwritten: Chebyshev-Jacobi pre-smoothing from
 * zero, residual, restriction, the coarser V-cycle, prolongation, post-smoothing
 * (P:L1159-1170 smoother, P:L1181-1185 transfer and coarse solve; the V-cycle of
 * P:L1144-1146's preconditioner).  Linear in r and symmetric. */
FEM_API int mg_vcycle(fem_handle h, const double* r, int64_t nr, double* z, int64_t nz);

/* Preconditioned CG from the caller's x (pass zeros) until
 * ||r|| <= rtol ||b|| or maxit iterations.  Synchronous.  iters/relres may be
 * NULL.  Returns FEM_OK, FEM_NOT_CONVERGED, or FEM_E_BREAKDOWN (message names
 * the iteration). */
FEM_API int cg_solve(fem_handle h, const double* b, int64_t nb, double* x, int64_t nx, double rtol,
             int32_t maxit, int32_t* iters, double* relres);

/* The same solve from the zero start vector (the usual preconditioned-CG call):
 * x is OUTPUT only -- its contents on entry are ignored, a host x is not copied to the device
 * (8 bytes per DoF less host-to-device traffic than cg_solve) and the ||x_0|| test is skipped.
 * Same arithmetic, return codes and history as cg_solve called with x = 0. */
FEM_API int cg_solve_zero(fem_handle h, const double* b, int64_t nb, double* x, int64_t nx, double rtol,
                  int32_t maxit, int32_t* iters, double* relres);

/* Residual history of the last cg_solve on this handle: rel[i] = ||r_i|| / ||b|| for
 * i = 0 .. iterations (r_0 = b - A x_0; r_i the recursively updated residual after the
 * i-th x update, the quantity of the stopping test).  Copies at most cap
 * entries; *n (may be NULL) receives the full length (0 before any solve).  Host
 * memory.  Errors: FEM_E_ARG (rel NULL with cap > 0). */
FEM_API int cg_history(fem_handle h, double* rel, int32_t cap, int32_t* n);

/* Load vector of the manufactured solution u = prod sin(pi t_d), f = -Laplace u
 * ((k+1)^3 Gauss points, CG Dirichlet rows 0); SURVEY §8c O8. */
FEM_API int fem_rhs(fem_handle h, double* b, int64_t nb);

/* ---- level-wise entry points (one per §8a row, used by the parity tests) ----
 * level in [0, n_levels): 0 = coarsest, n_levels-1 = finest.  Lengths are the
 * level's rank-local (owned) DoF count (fem_level_info); on multi-rank handles
 * every call is collective. */
FEM_API int fem_level_info(fem_handle h, int32_t level, int64_t* n_dofs, int32_t cells[3]);
FEM_API int fem_level_apply(fem_handle h, int32_t level, const double* x, int64_t nx, double* y,
                    int64_t ny);
FEM_API int fem_level_diagonal(fem_handle h, int32_t level, double* d, int64_t nd);
/* lambda_max estimate used by the smoother on `level` (level >= 1); host double. */
FEM_API int fem_level_lambda(fem_handle h, int32_t level, double* lam);
/* Geometry table of `level` (R2): per cell, per quadrature point q (x fastest),
 * the 6 entries (00,01,02,11,12,22) of G_q = w_q det J_q J_q^-1 J_q^-T, layout
 * [cell][6][q]; nG = n_cells (k+1)^3 * 6.  Cartesian levels store no table: the
 * call still fills the array (from the per-level constants). */
FEM_API int fem_level_geometry(fem_handle h, int32_t level, double* G, int64_t nG);
/* x <- S(x, b): one Chebyshev smoothing pass of degree cheb_degree on `level`
 * (>= 1); x_is_zero != 0 means x = 0 on entry (p-1 operator applies, else p). */
FEM_API int mg_smooth(fem_handle h, int32_t level, const double* b, int64_t nb, double* x, int64_t nx,
              int32_t x_is_zero);
/* xf += P xc, P: level-1 -> level (nodal interpolation). */
FEM_API int mg_prolongate_add(fem_handle h, int32_t level, const double* xc, int64_t nc, double* xf,
                      int64_t nf);
/* xc = P^T xf, P: level-1 -> level. */
FEM_API int mg_restrict(fem_handle h, int32_t level, const double* xf, int64_t nf, double* xc,
                int64_t nc);
/* x = A_0^{-1} b on the coarsest level (dense Cholesky on free DoFs, R9). */
FEM_API int mg_coarse_solve(fem_handle h, const double* b, int64_t nb, double* x, int64_t nx);

/* ---- instrumentation ---- */
/* Blocks until all work enqueued by the handle is done. */
FEM_API int fem_sync(fem_handle h);
/* Number of CUDA kernels this library launched (all handles) since load. */
FEM_API int64_t fem_kernel_launches(void);
/* profile = 1 only: total device milliseconds and launch count of the timed
 * finest-level operator-apply kernels since the last reset: the PCG apply q = A p
 * of every cg_solve iteration (the smoother's applies launch the same kernel and
 * are not bracketed, so that the events do not perturb the solve) and every
 * fem_apply / fem_level_apply on the finest level. */
FEM_API int fem_profile_read(fem_handle h, double* ms, int64_t* launches, int32_t reset);
/* profile = 2: every Chebyshev step of the finest level (the fused smoother launches of
 * R7, reading R8) of mg_smooth / mg_vcycle / cg_solve is bracketed; *bytes = their
 * algorithmic bytes (read x, x_old if present, b; write x_new: 24 or 32 B per DoF). */
FEM_API int fem_profile_read_bytes(fem_handle h, double* ms, int64_t* launches, double* bytes, int32_t reset);
/* Switch the profile mode (0, 1, 2) of an existing handle; the cached PCG graphs are dropped
 * (re-captured with the new event nodes on the next cg_solve). */
FEM_API int fem_profile_mode(fem_handle h, int32_t mode);

FEM_API const char* fem_last_error(void);
FEM_API void fem_destroy(fem_handle h);

#ifdef __cplusplus
}
#endif
#endif /* LIBFEM_FEM_H */
