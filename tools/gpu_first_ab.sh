#!/bin/bash
# A/B of the class-table first Chebyshev step (FEM_CHEB_FIRST_CLS) on the C4 solve
python -m pytest tests/test_gpu_stencil.py -m gpu -x -q 2>&1 | tail -2
for v in 1 0 1 0; do echo "FEM_CHEB_FIRST_CLS=$v"; FEM_CHEB_FIRST_CLS=$v PROBE_SOLVE=1 python tools/probe.py C4 2>&1 | tail -2; done
