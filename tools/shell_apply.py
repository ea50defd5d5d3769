"""Apply throughput on the paper's "curved mesh, variable coefficient" case:
the cube-sphere shell patch with the degree-5 polynomial mapping and eq:diffusivity_shell
(amplitude 1e6), CG and SIPG, k = 1..8, ~`target` DoFs (default 2.5e7, the
paper's fig:matvec "curved" points were measured at 25.4M DoFs for Q4).

    python tools/shell_apply.py [out.json] [target_dofs]

kappa is folded into the geometry tables, so the bytes per apply equal the deformed
box's (16 B/DoF + 48 B per cell quadrature point, + 56 B per SIPG face point); the
table is reported next to the time.  Single-level handles (coarse_cells = n).
"""
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import fem_inputs  # noqa: E402
from paper_1611_03029_b200 import fem  # noqa: E402
from sweep_degree import hbm_peak, time_apply  # noqa: E402


def main():
    out = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/shell_apply.json"
    target = float(sys.argv[2]) if len(sys.argv) > 2 else 2.5e7
    ks = [int(v) for v in os.environ.get("KS", "1,2,3,4,5,6,7,8").split(",")]
    peak = hbm_peak()
    rows = []
    for method, mname in ((fem.FEM_CG, "CG"), (fem.FEM_SIPG, "SIPG")):
        for k in ks:
            per = k if method == fem.FEM_CG else k + 1
            n = max(2, int(round(target ** (1 / 3) / per)))
            t0 = time.time()
            F = fem.Fem((n, n, n), k, method, geometry=fem.FEM_GEOM_SHELL, mapping_degree=5,
                        kappa_amplitude=1e6, coarse_cells=n)
            torch.cuda.synchronize()
            setup = time.time() - t0
            nd, nc, N = F.n_local, n ** 3, k + 1
            x = torch.from_numpy(fem_inputs.uniform_pm1(0, nd)).cuda()
            y = torch.zeros_like(x)
            t = time_apply(F, x, y)
            bytes_ = 16 * nd + 48 * N ** 3 * nc
            if method == fem.FEM_SIPG:
                bytes_ += 8 * 7 * N * N * 3 * n * n * (n + 1)
            r = {"method": mname, "k": k, "cells": n, "dofs": nd, "setup_s": setup, "t_apply_s": t,
                 "dofs_per_s": nd / t, "equiv_dofs_per_s": nc * k ** 3 / t, "alg_bytes": bytes_,
                 "hbm_frac": bytes_ / t / 1e9 / peak}
            rows.append(r)
            print(f"{mname:4s} k={k} n={n:3d} dofs={nd:9d} setup={setup:6.2f}s t={t*1e3:8.3f}ms "
                  f"{nd/t/1e9:7.2f} GDoF/s equiv {r['equiv_dofs_per_s']/1e9:7.2f} HBM {100*r['hbm_frac']:5.1f}%",
                  flush=True)
            F.close()
            del x, y
            torch.cuda.empty_cache()
    os.makedirs(os.path.dirname(out) or ".", exist_ok=True)
    with open(out, "w") as f:
        json.dump({"hbm_peak_gbs": peak, "target_dofs": target, "kappa_amplitude": 1e6, "mapping_degree": 5,
                   "rows": rows}, f, indent=1)


if __name__ == "__main__":
    main()
