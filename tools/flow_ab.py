"""A/B of the nrhs = 1 execution modes on one or more workloads' plans:
per-stage launches (graph replay) vs the one-launch dataflow kernel
(mht_set_persistent).  Cold L2 (a 256 MiB buffer rewritten before every
apply), CUDA events on the launching stream, median of --reps applies per
direction.  Prints one JSON line per (workload, mode).

    python tools/flow_ab.py c1 c4 [--reps 50]
"""
import argparse
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch

import mht_inputs as mi
from paper_2605_21828_b200 import _build, mht
from paper_2605_21828_b200 import workloads as W


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("workloads", nargs="+")
    ap.add_argument("--reps", type=int, default=50)
    ap.add_argument("--builder", default="gpu")
    a = ap.parse_args()
    _build.build()
    flush = torch.empty(64 * 2**20, dtype=torch.float32, device="cuda")
    for name in a.workloads:
        w = mi.WORKLOADS[name]
        path = W.ensure_plan(w, builder=a.builder, log=None)
        P = mht.Plan(path)
        coef = sum(s["coef_bytes"] for s in P.stage_stats())
        sb = P.scalar_bytes
        c = torch.from_numpy(mi.workload_coefficients(w, 1)).cuda()
        y = torch.from_numpy(mi.workload_adjoint_input(w, 1)).cuda()
        res = {}
        for mode in (False, True):
            P.set_persistent(mode)
            out = {}
            for kind in ("fwd", "adj"):
                fn = (lambda: P.apply(c)) if kind == "fwd" else (lambda: P.adjoint(y))
                for _ in range(3):
                    r = fn()
                torch.cuda.synchronize()
                ts = []
                for _ in range(a.reps):
                    flush.zero_()
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record()
                    r = fn()
                    e1.record()
                    torch.cuda.synchronize()
                    ts.append(e0.elapsed_time(e1))
                med = statistics.median(ts)
                byts = coef + (w.m + w.n) * sb
                out[kind] = {"ms_median": med, "ms_min": min(ts), "GBps": byts / (med / 1e3) / 1e9,
                             "frac_of_6454": byts / (med / 1e3) / 1e9 / 6454.6}
                res[(mode, kind)] = r.clone()
            print(json.dumps({"workload": name, "mode": "flow" if mode else "per-stage", "coef_bytes": coef,
                              **out}), flush=True)
            if mode:  # phase completion stamps of one profiled (eager) apply per direction
                P.set_profiling(True)
                for d, fn in ((0, lambda: P.apply(c)), (1, lambda: P.adjoint(y))):
                    flush.zero_()
                    fn()
                    ph = P.phase_times(d)
                    print(json.dumps({"workload": name, "dir": d, "phase_completion_deltas_ms":
                                      [(s_, k_, round(ms_, 4)) for s_, k_, ms_ in ph]}), flush=True)
                P.set_profiling(False)
                P.profile_reset()
        for kind in ("fwd", "adj"):
            a0, a1 = res[(False, kind)], res[(True, kind)]
            err = (torch.linalg.vector_norm(a0 - a1) / torch.linalg.vector_norm(a0)).item()
            mx = ((a0 - a1).abs().max() / a0.abs().max()).item()
            print(json.dumps({"workload": name, "check": kind, "rel_l2_flow_vs_stage": err, "maxabs_rel": mx}),
                  flush=True)
        P.close()


if __name__ == "__main__":
    main()
