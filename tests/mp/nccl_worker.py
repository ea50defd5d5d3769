"""Multi-process NCCL z-slab worker (launched by tests/test_gpu_nccl.py under torchrun).

Each rank owns a z-slab of the mesh (one process per GPU, libfem's NCCL transport:
grouped send/recv halo exchange, all-reduced dot products, optionally captured into
the PCG CUDA graphs with the comm-stream overlap).  Rank 0 gathers the distributed
results and compares them with a single-rank handle and the CPU oracle; the verdict is
written as JSON to $FEM_NCCL_OUT.
"""
import json
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import fem_inputs  # noqa: E402
from paper_1611_03029_b200 import fem  # noqa: E402

D, N = fem.FEM_BC_DIRICHLET, fem.FEM_BC_NEUMANN
CASES = [
    dict(name="cg_q3_deformed", cells=(4, 4, 8), degree=3, method=fem.FEM_CG, deform_eps=0.05, bc=(D,) * 6),
    dict(name="cg_q4_cartesian", cells=(4, 4, 8), degree=4, method=fem.FEM_CG, deform_eps=0.0,
         bc=(D, N, D, D, N, D)),
    dict(name="sipg_q2_deformed", cells=(2, 2, 8), degree=2, method=fem.FEM_SIPG, deform_eps=0.05,
         bc=(D, N, D, D, N, D)),
]


def gather(v, n_global, first, world):
    """Owned slices of all ranks -> the global vector on every rank."""
    full = torch.zeros(n_global, dtype=torch.float64, device="cuda")
    full[first:first + v.numel()] = v
    dist.all_reduce(full)
    return full


def relmax(a, b):
    return float((a - b).abs().max() / b.abs().max().clamp_min(1e-300))


def run_case(c, rank, world):
    from oracle import cg as ocg, sipg as osipg
    from oracle.mesh import Mesh
    kw = {k: v for k, v in c.items() if k != "name"}
    cells, k, method = kw.pop("cells"), kw.pop("degree"), kw.pop("method")
    single = fem.Fem(cells, k, method, **kw)
    lam = [single.fem_level_lambda(l) if l else 0.0 for l in range(single.n_levels)]
    uid = [fem.nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(uid, src=0)
    F = fem.Fem(cells, k, method, rank=rank, nranks=world, nccl_id=uid[0], lambda_override=lam, **kw)
    single_l = fem.Fem(cells, k, method, lambda_override=lam, **kw)
    n, ng, first = F.n_local, F.n_global, F.first_global
    xg = torch.from_numpy(fem_inputs.uniform_pm1(3, ng)).cuda()
    # operator
    y = torch.zeros(n, dtype=torch.float64, device="cuda")
    F.fem_apply(xg[first:first + n].contiguous(), y)
    yg = gather(y, ng, first, world)
    y1 = torch.zeros(ng, dtype=torch.float64, device="cuda")
    single.fem_apply(xg, y1)
    m = Mesh(cells, k, eps=c["deform_eps"], bc=c["bc"])
    yo = ocg.apply(m, xg.cpu().numpy()) if method == fem.FEM_CG else osipg.apply(m, xg.cpu().numpy())
    res = {"apply_vs_single": relmax(yg, y1), "apply_vs_oracle": relmax(yg.cpu(), torch.from_numpy(yo))}
    # V-cycle (lambda pinned to the single-rank estimates)
    b = torch.zeros(n, dtype=torch.float64, device="cuda")
    F.fem_rhs(b)
    bg = gather(b, ng, first, world)
    z = torch.zeros_like(b)
    F.mg_vcycle(b, z)
    zg = gather(z, ng, first, world)
    z1 = torch.zeros_like(bg)
    single_l.mg_vcycle(bg, z1)
    res["vcycle_vs_single"] = relmax(zg, z1)
    # PCG
    x = torch.zeros_like(b)
    its, rr, ok = F.cg_solve(b, x, rtol=1e-10)
    xg2 = gather(x, ng, first, world)
    x1 = torch.zeros_like(bg)
    its1, rr1, ok1 = single_l.cg_solve(bg, x1, rtol=1e-10)
    res.update(its=its, its_single=its1, converged=bool(ok and ok1), relres=rr,
               x_vs_single=relmax(xg2, x1), history=F.cg_history())
    for h in (F, single, single_l):
        h.close()
    return res


def main():
    rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    out = {c["name"]: run_case(c, rank, world) for c in CASES}
    if rank == 0:
        with open(os.environ["FEM_NCCL_OUT"], "w") as f:
            json.dump(out, f, indent=1)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
