"""Operator-apply driver for ncu captures (development aid, not the bench contract).

    python tools/ncu_apply.py C2 [reps]

Sets up the config, then brackets `reps` finest-level applies with
cudaProfilerStart/Stop so that `ncu --profile-from-start off` sees only them.
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import fem_inputs  # noqa: E402
from paper_1611_03029_b200 import fem  # noqa: E402

w = fem_inputs.CONFIGS[sys.argv[1]]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
F = fem.Fem(w.cells, w.degree, w.method, deform_eps=w.deform_eps, bc=w.bc, penalty_factor=w.penalty_factor)
x = torch.from_numpy(fem_inputs.uniform_pm1(w.seed, F.n_local)).cuda()
y = torch.zeros_like(x)
F.fem_apply(x, y)
torch.cuda.synchronize()
smooth = os.environ.get("NCU_SMOOTH") == "1"   # finest-level smoother instead (fused Chebyshev)
xs = torch.zeros_like(x)
torch.cuda.cudart().cudaProfilerStart()
for _ in range(reps):
    if smooth:
        F.mg_smooth(F.n_levels - 1, y, xs, False)
    else:
        F.fem_apply(x, y)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
print(f"{w.name}: {reps} applies ok, |y|_max = {y.abs().max().item():.6e}")
F.close()
