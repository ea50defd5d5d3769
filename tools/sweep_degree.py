"""Degree sweep k = 1..8 of the operator apply: the B200 version of the
paper's fig:matvec / fig:mv_roofline.

    python tools/sweep_degree.py [out.json] [target_dofs]

For CG and SIPG, Cartesian and deformed (eps = 0.05), every k: a mesh of n^3 cells
with about `target_dofs` (default 1.6e7, the paper measured at ~1e7 so that vectors
come from DRAM), x ~ U[-1,1) (seed 0), 20 back-to-back applies timed with
CUDA events after a warm-up.  Reported: actual and equivalent DoFs/s (n_cells k^3 / t,
P:L399-404), the algorithmic bytes per apply (x read + y written, 16 B/DoF; the
geometry table on deformed meshes, 48 B per cell quadrature point; SIPG deformed
face records, 7 doubles per face quadrature point) and the fraction of the measured
HBM bandwidth they imply.  Single-level handles (coarse_cells = n): no multigrid
setup is needed for an apply.
"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import fem_inputs  # noqa: E402
from paper_1611_03029_b200 import fem  # noqa: E402


def hbm_peak():
    p = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            return float(json.load(f)["hbm_gbs"])
    except OSError:
        return 6650.0


def time_apply(F, x, y, reps=20):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(3):
        F.fem_apply(x, y)
    torch.cuda.synchronize()
    s.record()
    for _ in range(reps):
        F.fem_apply(x, y)
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) * 1e-3 / reps


def main():
    out = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/degree_sweep.json"
    target = float(sys.argv[2]) if len(sys.argv) > 2 else 1.6e7
    peak = hbm_peak()
    rows = []
    only_m = os.environ.get("SWEEP_METHODS", "CG,SIPG").split(",")
    only_g = os.environ.get("SWEEP_GEOM", "Cartesian,deformed").split(",")
    ks = [int(v) for v in os.environ.get("SWEEP_K", "1,2,3,4,5,6,7,8").split(",")]
    for method, mname in ((fem.FEM_CG, "CG"), (fem.FEM_SIPG, "SIPG")):
        if mname not in only_m:
            continue
        for eps in (0.0, 0.05):
            if ("deformed" if eps else "Cartesian") not in only_g:
                continue
            for k in ks:
                per = k if method == fem.FEM_CG else k + 1
                n = max(2, int(round(target ** (1 / 3) / per)))
                F = fem.Fem((n, n, n), k, method, deform_eps=eps, coarse_cells=n)
                nd, nc, N = F.n_local, n ** 3, k + 1
                x = torch.from_numpy(fem_inputs.uniform_pm1(0, nd)).cuda()
                y = torch.zeros_like(x)
                t = time_apply(F, x, y)
                bytes_ = 16 * nd
                if eps:
                    bytes_ += 48 * N ** 3 * nc
                    if method == fem.FEM_SIPG:
                        nfaces = 3 * n * n * (n + 1)
                        bytes_ += 8 * 7 * N * N * nfaces
                r = {"method": mname, "geometry": "deformed" if eps else "Cartesian", "k": k, "cells": n,
                     "dofs": nd, "t_apply_s": t, "dofs_per_s": nd / t, "equiv_dofs_per_s": nc * k ** 3 / t,
                     "alg_bytes": bytes_, "alg_bytes_per_dof": bytes_ / nd, "hbm_gbs": bytes_ / t / 1e9,
                     "hbm_frac": bytes_ / t / 1e9 / peak}
                rows.append(r)
                print(f"{mname:4s} {r['geometry']:9s} k={k} n={n:3d} dofs={nd:9d} t={t*1e6:9.1f}us "
                      f"{nd/t/1e9:7.2f} GDoF/s equiv {r['equiv_dofs_per_s']/1e9:7.2f} "
                      f"B/DoF {r['alg_bytes_per_dof']:6.1f} HBM {100*r['hbm_frac']:5.1f}%", flush=True)
                F.close()
                del x, y
                torch.cuda.empty_cache()
    os.makedirs(os.path.dirname(out) or ".", exist_ok=True)
    with open(out, "w") as f:
        json.dump({"hbm_peak_gbs": peak, "target_dofs": target, "rows": rows}, f, indent=1)


if __name__ == "__main__":
    main()
