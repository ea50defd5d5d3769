"""CPU oracle for the matrix-free CG / SIPG Laplace operator and its GMG-CG solver.

TEST INFRASTRUCTURE ONLY.  Only `tests/`, `__graft_entry__.smoke()` and the
`cpu_baseline` / `--impl reference` legs of `bench.py` may import this package.
The product path (`paper_1611_03029_b200/`, `libfem.so`) never imports, links or
executes anything here, and this package never imports the product.

What it is: a plain, slow, FP64 numpy/scipy implementation of what the paper
(arXiv 1611.03029, `/root/reference/PAPER.md`, cited `P:L<line>`) computes,
with no sum factorization:

* `basis`      1-D Gauss and Gauss-Lobatto rules, Lagrange basis
* `mesh`       structured hex mesh, deformation map, Jacobians, numbering
* `cg`         CG element matrices by full 3-D tensor quadrature, CSR assembly,
               dense-B element-wise apply, diagonal (eq:poisson_fem, eq:mf_eval)
* `sipg`       SIPG cell + face matrices / apply / diagonal (eq:poisson_dgsip, eq:bc_dgsip)
* `transfer`   nodal-interpolation prolongation P and restriction P^T
* `multigrid`  Chebyshev-Jacobi smoother, lambda_max estimate, V-cycle, PCG
* `problem`    manufactured right-hand side and L2 error
* `hdg`        HDG: quadrature-built local matrices, the statically
               condensed trace operator K and its right-hand side (eq:hdg_matrix_condensed),
               local recovery, the mixed (flux-substituted) operator, Jacobi-PCG

Parity status of every function is listed in DESIGN.md ("Oracle pins").
"""
