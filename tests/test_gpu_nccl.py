"""Two-process NCCL z-slab path (one process per GPU; skipped when fewer than two GPUs
are visible).  tests/mp/nccl_worker.py runs under torchrun and compares the distributed
operator, V-cycle and PCG with a single-rank handle (and the operator with the CPU
oracle), with the PCG iteration captured into CUDA graphs (NCCL calls and the
comm-stream halo overlap inside the graphs) and eagerly (FEM_NO_GRAPHS=1, FEM_OVERLAP=0).
Bars as tests/test_gpu_slabs.py: 1e-12 operator, 1e-11 V-cycle (lambda pinned),
PCG iterations +-1.
"""
import json
import os
import random
import subprocess
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.skipif(not torch.cuda.is_available() or torch.cuda.device_count() < 2,
                    reason="needs two GPUs (one NCCL rank each)")
@pytest.mark.parametrize("env", [{}, {"FEM_NO_GRAPHS": "1"}, {"FEM_OVERLAP": "0"}])
def test_nccl_two_ranks_match_single_rank(env, tmp_path):
    out = tmp_path / "nccl.json"
    e = dict(os.environ, FEM_NCCL_OUT=str(out), **env)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", str(random.randint(20000, 40000)),
           os.path.join(ROOT, "tests", "mp", "nccl_worker.py")]
    p = subprocess.run(cmd, env=e, cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, p.stderr[-4000:]
    res = json.loads(out.read_text())
    for name, r in res.items():
        assert r["apply_vs_single"] <= 1e-12, (name, r)
        assert r["apply_vs_oracle"] <= 1e-12, (name, r)
        assert r["vcycle_vs_single"] <= 1e-11, (name, r)
        assert r["converged"] and abs(r["its"] - r["its_single"]) <= 1, (name, r)
        assert r["x_vs_single"] <= 1e-8, (name, r)
