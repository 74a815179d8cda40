"""Profiling driver for ncu: one synthesis + analysis at nrhs=1 and nrhs=32 on
a workload's plan (built with the GPU builder if not cached).  No oracle."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import mht_inputs as mi
from paper_2605_21828_b200 import workloads as W, mht

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
w = mi.WORKLOADS[name]
path = W.plan_cache_path(w)
if not os.path.exists(path):
    W.build_workload_plan(w, path + ".build", builder="gpu", log=None)
    os.replace(path + ".build", path)
torch.cuda.empty_cache()
P = mht.Plan(path)
for r in sorted(set((1,) + tuple(w.nrhs))):
    c = torch.from_numpy(mi.workload_coefficients(w, r)).cuda()
    y = torch.from_numpy(mi.workload_adjoint_input(w, r)).cuda()
    P.apply(c); P.adjoint(y)
torch.cuda.synchronize()
print("prof_run ok", name)
