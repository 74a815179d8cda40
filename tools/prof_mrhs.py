"""Profiling driver for ncu: one eager multi-RHS synthesis and analysis of a
workload's plan, per-stage launches (python tools/prof_mrhs.py c4 64)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import mht_inputs as mi
from paper_2605_21828_b200 import workloads as W, mht

name, nrhs = sys.argv[1], int(sys.argv[2])
w = mi.WORKLOADS[name]
P = mht.Plan(W.ensure_plan(w, builder="gpu", log=None))
P.set_graphs(False)
c = torch.from_numpy(mi.workload_coefficients(w, nrhs)).cuda()
y = torch.from_numpy(mi.workload_adjoint_input(w, nrhs)).cuda()
P.apply(c)
P.adjoint(y)
torch.cuda.synchronize()
print("prof_mrhs ok", name, nrhs)
