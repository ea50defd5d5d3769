"""One V-cycle on a config under cudaProfilerStart/Stop (development aid for ncu captures of the
transfer and smoother kernels)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import fem_inputs  # noqa: E402
from paper_1611_03029_b200 import fem  # noqa: E402

w = fem_inputs.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C4"]
F = fem.Fem(w.cells, w.degree, w.method, deform_eps=w.deform_eps, bc=w.bc, penalty_factor=w.penalty_factor)
r = torch.from_numpy(fem_inputs.uniform_pm1(w.seed, F.n_local)).cuda()
z = torch.zeros_like(r)
F.mg_vcycle(r, z)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
F.mg_vcycle(r, z)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
print("ok", float(z.abs().max()))
