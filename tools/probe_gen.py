import sys, os, torch
sys.path.insert(0, '/root/repo' if os.path.exists('/root/repo') else '.')
import fem_inputs
from paper_1611_03029_b200 import fem
def t(F, reps=50):
    n=F.n_local; x=torch.from_numpy(fem_inputs.uniform_pm1(0,n)).cuda(); y=torch.zeros_like(x)
    F.fem_apply(x,y); torch.cuda.synchronize()
    s,e=torch.cuda.Event(enable_timing=True),torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps): F.fem_apply(x,y)
    e.record(); torch.cuda.synchronize(); return s.elapsed_time(e)/reps*1e3
for eps in (0.05, 0.0):
    F=fem.Fem((32,32,32),4,fem.FEM_CG,deform_eps=eps)
    print("eps",eps,"general_path",os.environ.get("FEM_GENERAL_PATH"),"apply us %.1f"%t(F))
    F.close()
