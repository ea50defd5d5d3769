"""B200-native matrix-free CG / SIPG Laplace operator with GMG-preconditioned CG
(arXiv 1611.03029 hot path).  The product is libfem.so (include/fem.h); this
package holds its CUDA sources (csrc/), the in-tree build (build.py) and the thin
ctypes binding (fem.py).  Import `paper_1611_03029_b200.fem` to load the library."""
