"""Profiling driver for ncu: one eager (no graph) nrhs = 1 synthesis and
analysis of a workload's plan, per-stage launches.  E.g. the forward kernel of
stage 4 of c1 (stages 2..7 launch in order):
    ncu --set full -k regex:fwd_kernel -s 2 -c 1 -o gpurun_out/c1_s4 python tools/prof_nrhs1.py c1
"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import mht_inputs as mi
from paper_2605_21828_b200 import workloads as W, mht

name = sys.argv[1] if len(sys.argv) > 1 else "c1"
w = mi.WORKLOADS[name]
path = W.ensure_plan(w, builder="gpu", log=None)
P = mht.Plan(path)
P.set_graphs(False)
c = torch.from_numpy(mi.workload_coefficients(w, 1)).cuda()
y = torch.from_numpy(mi.workload_adjoint_input(w, 1)).cuda()
P.apply(c)
P.adjoint(y)
torch.cuda.synchronize()
print("prof_nrhs1 ok", name)
