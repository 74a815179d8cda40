"""Time the multi-RHS kernels of one workload's plan (variant chosen by MHT_MMA)
and check them against the nrhs=1 GEMV path column by column (self-consistency,
not the oracle)."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import mht_inputs as mi
from paper_2605_21828_b200 import workloads as W, mht
name = sys.argv[1] if len(sys.argv) > 1 else "c2"
w = mi.WORKLOADS[name]
path = W.plan_cache_path(w)
if not os.path.exists(path):
    W.build_workload_plan(w, path + ".build", builder="gpu", log=None); os.replace(path + ".build", path)
torch.cuda.empty_cache()
P = mht.Plan(path)
r = max(w.nrhs)
c = torch.from_numpy(mi.workload_coefficients(w, r)).cuda()
y = torch.from_numpy(mi.workload_adjoint_input(w, r)).cuda()
f = P.apply(c); a = P.adjoint(y)
f1 = torch.stack([P.apply(c[i:i+1])[0] for i in range(3)]); a1 = torch.stack([P.adjoint(y[i:i+1])[0] for i in range(3)])
err = max(((f[:3]-f1).norm()/f1.norm()).item(), ((a[:3]-a1).norm()/a1.norm()).item())
res = {"variant": os.environ.get("MHT_MMA", "default"), "nrhs": r, "consistency": err}
for nm, fn in (("fwd", lambda: P.apply(c, out=f)), ("adj", lambda: P.adjoint(y, out=a))):
    for _ in range(2): fn()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); e0.record()
    for _ in range(5): fn()
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    res[nm + "_ms"] = round(ms, 3)
    res[nm + "_TF"] = round((8 if P.is_complex else 2) * P.info.factor_entries * r / ms / 1e9, 2)
print(json.dumps(res), flush=True)
