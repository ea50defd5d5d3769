"""N4: the paper's design (inner Schur complement inverse stored per cell) against the
fast-diagonalization kernel on Cartesian Q_k meshes, and the stored-inverse kernel on the
deformed mesh (development aid; writes gpurun_out/hdg_designs.json)."""
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import fem_inputs  # noqa: E402
from paper_1611_03029_b200 import fem  # noqa: E402

HBM = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json"))).get("hbm_gbs", 6534.5) if os.path.exists("MEASURED_PEAKS.json") else 6534.5


def run(cells, k, eps, dense, reps=10):
    os.environ["FEM_HDG_DENSE"] = "1" if dense else "0"
    t0 = time.perf_counter()
    H = fem.Hdg(cells, k, deform_eps=eps)
    torch.cuda.synchronize()
    setup = time.perf_counter() - t0
    x = torch.from_numpy(fem_inputs.uniform_pm1(0, H.n_trace)).cuda()
    y = torch.empty_like(x)
    H.hdg_apply(x, y)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        H.hdg_apply(x, y)
    e.record()
    torch.cuda.synchronize()
    t = s.elapsed_time(e) * 1e-3 / reps
    m = (k + 1) ** 3
    stored = H.n_cells * m * m * 8 if dense else 0
    bytes_ = 16 * H.n_trace + stored
    b = torch.zeros_like(x)
    H.hdg_rhs(b)
    lam = torch.zeros_like(b)
    its, rr, ok = H.hdg_cg_solve(b, lam, rtol=1e-10)
    r = {"cells": list(cells), "k": k, "eps": eps, "design": "stored S^-1 per cell (paper)" if dense else "fast diagonalization",
         "n_trace": H.n_trace, "setup_s": round(setup, 3), "apply_us": t * 1e6,
         "trace_dofs_per_s": H.n_trace / t, "equivalent_dofs_per_s": H.n_cells * k ** 3 / t,
         "algorithmic_bytes": bytes_, "hbm_frac": bytes_ / t / 1e9 / HBM, "jacobi_pcg_its": its, "relres": rr}
    H.close()
    del x, y, b, lam
    torch.cuda.empty_cache()
    print(json.dumps(r), flush=True)
    return r


rows = []
for k in (2, 3, 4):
    n = {2: 48, 3: 40, 4: 32}[k]
    rows.append(run((n, n, n), k, 0.0, False))
    rows.append(run((n, n, n), k, 0.0, True))
    rows.append(run((n, n, n), k, 0.05, True))
os.makedirs("gpurun_out", exist_ok=True)
json.dump(rows, open("gpurun_out/hdg_designs.json", "w"), indent=1)
