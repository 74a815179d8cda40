"""Compare the multi-RHS result of one workload under the current kernel
selection against the nrhs = 1 path, per direction (prints where they differ)."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import mht_inputs as mi
from paper_2605_21828_b200 import workloads as W, mht
name = sys.argv[1]; r = int(sys.argv[2]) if len(sys.argv) > 2 else 32
w = mi.WORKLOADS[name]
path = W.plan_cache_path(w)
if not os.path.exists(path):
    W.build_workload_plan(w, path + ".build", builder="gpu", log=None); os.replace(path + ".build", path)
P = mht.Plan(path)
c = torch.from_numpy(mi.workload_coefficients(w, r)).cuda()
y = torch.from_numpy(mi.workload_adjoint_input(w, r)).cuda()
f = P.apply(c).cpu().numpy(); a = P.adjoint(y).cpu().numpy()
out = {"ws": os.environ.get("MHT_MMA_WS"), "nrhs": r}
for nm, full, one in (("fwd", f, lambda i: P.apply(c[i:i+1])[0]), ("adj", a, lambda i: P.adjoint(y[i:i+1])[0])):
    errs = []
    for i in (0, 1, r - 1):
        ref = one(i).cpu().numpy()
        d = np.abs(full[i] - ref)
        errs.append([float(np.linalg.norm(d) / np.linalg.norm(ref)), int(np.count_nonzero(d > 1e-9 * np.abs(ref).max())),
                     [int(x) for x in np.argsort(-d)[:5]]])
    out[nm] = errs
print(json.dumps(out))
