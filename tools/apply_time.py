"""Per-apply device time (python tools/apply_time.py c1 c4) with the CPU running ahead (all launches enqueued,
one sync): cold L2 (64 MB flush before each apply), CUDA events per apply."""
import os, sys, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import mht_inputs as mi
from paper_2605_21828_b200 import mht, workloads as W
tag = os.environ.get("TAG", "")
for name in sys.argv[1:]:
    w = mi.WORKLOADS[name]
    P = mht.Plan(W.ensure_plan(w, builder="gpu", log=None))
    if os.environ.get("RING"): P.set_ring(True)
    c = torch.from_numpy(mi.workload_coefficients(w, 1)).cuda()
    y = torch.from_numpy(mi.workload_adjoint_input(w, 1)).cuda()
    flush = torch.empty(64 * 2**20, dtype=torch.float32, device="cuda")
    for kind, fn in (("fwd", lambda: P.apply(c)), ("adj", lambda: P.adjoint(y))):
        for _ in range(5): fn()
        torch.cuda.synchronize()
        ev = []
        for _ in range(40):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(); fn(); e1.record(); ev.append((e0, e1))
        torch.cuda.synchronize()
        ts = [a.elapsed_time(b) * 1e3 for a, b in ev[5:]]
        print(f"{tag} {name} {kind} median {statistics.median(ts):.1f} us min {min(ts):.1f}", flush=True)
    P.close()
