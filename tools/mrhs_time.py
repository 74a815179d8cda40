"""Per-apply device time of a workload's multi-RHS synthesis and analysis
(cold L2, CPU enqueued ahead, CUDA events per apply, median):
    python tools/mrhs_time.py c4 64"""
import os, sys, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import mht_inputs as mi
from paper_2605_21828_b200 import mht, workloads as W
tag = os.environ.get("TAG", "")
name, nrhs = sys.argv[1], int(sys.argv[2])
w = mi.WORKLOADS[name]
P = mht.Plan(W.ensure_plan(w, builder="gpu", log=None))
c = torch.from_numpy(mi.workload_coefficients(w, nrhs)).cuda()
y = torch.from_numpy(mi.workload_adjoint_input(w, nrhs)).cuda()
flush = torch.empty(64 * 2**20, dtype=torch.float32, device="cuda")
for kind, fn in (("fwd", lambda: P.apply(c)), ("adj", lambda: P.adjoint(y))):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    ev = []
    for _ in range(25):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); ev.append((e0, e1))
    torch.cuda.synchronize()
    ts = [a.elapsed_time(b) * 1e3 for a, b in ev[3:]]
    print(f"{tag} {name} nrhs={nrhs} {kind} median {statistics.median(ts):.1f} us", flush=True)
