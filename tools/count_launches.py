import sys, torch
sys.path.insert(0,'.')
import fem_inputs
from paper_1611_03029_b200 import fem
w=fem_inputs.C2
F=fem.Fem(w.cells,w.degree,w.method,deform_eps=w.deform_eps)
b=torch.zeros(F.n_local,dtype=torch.float64,device='cuda'); F.fem_rhs(b); x=torch.zeros_like(b)
F.cg_solve(b,x)
for i in range(3):
    x.zero_(); l0=fem.kernel_launches(); its,rr,ok=F.cg_solve(b,x); torch.cuda.synchronize(); print('launches per solve', fem.kernel_launches()-l0, 'its', its)
