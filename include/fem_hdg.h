/* libfem -- HDG matrix-free operators, C ABI.
 *
 * Hybridizable DG for the Poisson problem, sec:discret_hdg of arXiv 1611.03029
 * (/root/reference/PAPER.md, cited P:L<line>): q = -grad u, u_h and q_h in Q_k DG
 * (GLL nodal), trace lambda_h in Q_k(F) on every face (eq:trace_space),
 * numerical flux q^.n = q.n + tau (u - lambda), tau = 5 (kappa = 1),
 * matrices of eq:hdg_matrix.  Box meshes (n[0] x n[1] x n[2] cells of [lo, hi]):
 * Cartesian, or deformed by the map of reading R2 (deform_eps != 0, degree 1..4: the local inverse
 * is then stored per cell, the paper's design; mixed form and post-processing: Cartesian only).
 *
 * Vectors are DEVICE pointers (CUDA float64, e.g. torch.cuda tensors), asynchronous on
 * the handle's stream unless stated otherwise; host pointers give FEM_E_ARG.
 * Layouts:
 *   trace vector  faces normal to x first ((n0+1) n1 n2 faces, index
 *                 i_x + (n0+1)(c_y + n1 c_z)), then y (n0 (n1+1) n2, c_x + n0 (i_y + (n1+1) c_z)),
 *                 then z (n0 n1 (n2+1), c_x + n0 (c_y + n1 i_z)); each face (k+1)^2 GLL nodes,
 *                 the lower of its two tangential directions fastest.  Length hdg_info n_trace.
 *   cell vector   u (and each q component): cell-major, lexicographic cells (x fastest), per
 *                 cell (k+1)^3 nodes, x fastest (the SIPG layout).  Length n_cells (k+1)^3.
 * Dirichlet sides: their faces' trace entries are constrained (homogeneous g_D, "imposed
 * strongly on the trace space"): inputs read as 0, outputs y_c = x_c.
 * Return codes as in fem.h (FEM_OK, FEM_E_ARG, FEM_E_SIZE, FEM_E_CUDA, FEM_E_BREAKDOWN,
 * FEM_NOT_CONVERGED); fem_last_error() gives the text.
 */
#ifndef FEM_HDG_H
#define FEM_HDG_H

#include <stdint.h>

#include "fem.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct hdg_ctx* hdg_handle;   /* opaque; created by hdg_setup, owned by libfem */

/* Setup: the 1-D tables (GLL basis, Gauss rule, mass M, derivative Dm, inverse mass, and the
 * generalized eigenpairs of the inner Schur complement's 1-D factors, see hdg_apply), on deformed
 * meshes the per-cell inverses of the inner Schur complement, the diagonal and the stream.  mesh:
 * n, lo, hi, bc, deform_eps used (geometry BOX, no mapping degree / kappa, nranks 1); degree 1..8
 * (1..4 deformed); tau > 0 (the paper's 5).  stream: cudaStream_t or NULL. */
FEM_API int hdg_setup(const fem_mesh* mesh, int32_t degree, double tau, void* stream, hdg_handle* out);
FEM_API int hdg_info(hdg_handle h, int64_t* n_trace, int64_t* n_cells);

/* y = K lambda, the statically condensed trace operator (eq:hdg_matrix_condensed),
 * evaluated matrix-free in the three steps of "HDG trace matrix-free":
 * (1) [C^T; G^T] lambda, (2) the local inverse by the inner Schur complement
 * U = (D + E A^-1 E^T)^-1 (R_u - E A^-1 R_q), Q = A^-1 (R_q + E^T U), (3) [C G] and H.
 * On Cartesian cells the Schur complement's inverse is applied by tensor-product fast
 * diagonalization (exact) instead of the paper's stored dense matrix; on
 * deformed cells (or with FEM_HDG_DENSE=1) the stored dense inverse is used. */
FEM_API int hdg_apply(hdg_handle h, const double* lambda, int64_t n, double* y, int64_t ny);
/* d = diag(K) (1 on constrained entries). */
FEM_API int hdg_diagonal(hdg_handle h, double* d, int64_t nd);
/* r = sum_K [C G] L^-1 [0; F] with F = (f, v), f = -lap u for the manufactured
 * u = prod sin(pi (x - lo)/(hi - lo)); constrained entries 0. */
FEM_API int hdg_rhs(hdg_handle h, double* r, int64_t nr);
/* Local recovery: u (cell vector) from the trace and, if with_f, the manufactured load F;
 * q (3 cell vectors, component-major: q_x, q_y, q_z) if q != NULL. */
FEM_API int hdg_local_solve(hdg_handle h, const double* lambda, int64_t n, int32_t with_f, double* u,
                            int64_t nu, double* q, int64_t nq);
/* "HDG mixed matrix-free": [y_q; y_u] = [A -E^T; E D] [q; u] + [C^T; -G^T] lambda^(q, u)
 * with lambda^ = H_F^-1 sum_K (C q + G u) on every free face (point-wise on Cartesian faces), 0 on
 * constrained faces.  qu and y: 4 cell vectors (q_x, q_y, q_z, u), length 4 n_cells (k+1)^3. */
FEM_API int hdg_mixed_apply(hdg_handle h, const double* qu, int64_t n, double* y, int64_t ny);
/* Element-by-element post-processing: u* in Q_{k+1}(K) with (grad u*, grad w)_K =
 * -(q, grad w)_K for all w in Q_{k+1}(K) and (u*, 1)_K = (u, 1)_K, from q (3 cell vectors) and u of
 * hdg_local_solve; converges at order k+2.  ustar: cell-major, (k+2)^3 GLL(k+1) nodes per cell,
 * x fastest.  Cartesian meshes, degree 1..7. */
FEM_API int hdg_postprocess(hdg_handle h, const double* q, int64_t nq, const double* u, int64_t nu, double* ustar,
                            int64_t nus);
/* PCG with the diagonal of K on K lambda = b from the caller's lambda (pass zeros), stopping
 * test ||r|| <= rtol ||b|| on the updated residual (reading R13).  Synchronous. */
FEM_API int hdg_cg_solve(hdg_handle h, const double* b, int64_t nb, double* lambda, int64_t n, double rtol,
                         int32_t maxit, int32_t* iters, double* relres);
FEM_API void hdg_destroy(hdg_handle h);

#ifdef __cplusplus
}
#endif

#endif /* FEM_HDG_H */
