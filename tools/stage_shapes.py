"""Per-stage block-shape statistics of a workload's plan (host only, from the
plan file): block kinds, r_out / n_red distributions and the number of 64-row
tiles, to explain per-stage kernel rates (bench.py stage_ms).

    python tools/stage_shapes.py c3 [> profiles/r01_stage_shapes_c3.txt]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import mht_inputs as mi
from paper_2605_21828_b200 import workloads as W
from paper_2605_21828_b200.precompute.planfile import PlanView

name = sys.argv[1] if len(sys.argv) > 1 else "c3"
w = mi.WORKLOADS[name]
path = W.plan_cache_path(w)
if not os.path.exists(path):
    W.build_workload_plan(w, path + ".build", builder="gpu" if os.environ.get("CUDA_VISIBLE_DEVICES", "x") != "" else "cpu", log=None)
    os.replace(path + ".build", path)
pv = PlanView(path)
print(f"# {name}: n={pv.n} m={pv.m} L={pv.L} complex={pv.complex} entries={pv.entries}")
print("stage nblk identity id dense | r_out p10/p50/p90/max | n_red p10/p50/p90/max | tiles64 | mean K per tile")
for s, st in enumerate(pv.stages):
    b = st.blocks
    kind = np.asarray(b["kind"])
    ro, ri = np.asarray(b["r_out"], np.int64), np.asarray(b["r_in"], np.int64)
    nred = np.where(kind == 1, ri - ro, np.where(kind == 2, ri, 0))
    ex = kind != 0
    tiles = int(((ro[ex] + 63) // 64).sum())
    q = lambda a: "/".join(str(int(x)) for x in (np.percentile(a, [10, 50, 90]).tolist() + [a.max()])) if a.size else "-"
    meank = float((nred[ex] * ((ro[ex] + 63) // 64)).sum() / max(tiles, 1))
    print(f"{s:5d} {st.nblk:5d} {int((kind == 0).sum()):8d} {int((kind == 1).sum()):3d} {int((kind == 2).sum()):5d} | "
          f"{q(ro[ex])} | {q(nred[ex])} | {tiles} | {meank:.1f}")
