"""HDG apply driver for ncu (development aid): trace and mixed applies at Q<k> on n^3 cells."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import fem_inputs  # noqa: E402
from paper_1611_03029_b200 import fem  # noqa: E402

n, k = int(sys.argv[1]), int(sys.argv[2])
H = fem.Hdg((n, n, n), k)
x = torch.from_numpy(fem_inputs.uniform_pm1(0, H.n_trace)).cuda()
y = torch.empty_like(x)
qu = torch.from_numpy(fem_inputs.uniform_pm1(1, 4 * H.n_cell_dofs)).cuda()
yq = torch.empty_like(qu)
H.hdg_apply(x, y)
H.hdg_mixed_apply(qu, yq)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
H.hdg_apply(x, y)
H.hdg_mixed_apply(qu, yq)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
print("ok", float(y.abs().max()), float(yq.abs().max()))
