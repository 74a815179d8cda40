"""Profiling driver for ncu: nrhs = 1 synthesis and analysis of a workload's
plan in the one-launch dataflow mode (mht_set_persistent), two warm-up applies
per direction first.  Capture the third launch of the flow kernel, e.g.
    ncu --set full -k regex:flow_kernel -s 4 -c 1 -o gpurun_out/flow python tools/prof_flow.py c2
"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import mht_inputs as mi
from paper_2605_21828_b200 import workloads as W, mht

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
w = mi.WORKLOADS[name]
path = W.ensure_plan(w, builder="gpu", log=None)
torch.cuda.empty_cache()
P = mht.Plan(path)
P.set_graphs(False)
P.set_persistent(True)
c = torch.from_numpy(mi.workload_coefficients(w, 1)).cuda()
y = torch.from_numpy(mi.workload_adjoint_input(w, 1)).cuda()
for _ in range(3):
    P.apply(c)
    P.adjoint(y)
torch.cuda.synchronize()
print("prof_flow ok", name)
