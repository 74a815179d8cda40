#!/usr/bin/env python
"""bench.py — butterfly MHT apply/adjoint on B200 (driver contract).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl mht|reference] [--workload c2]

A *step* is one pass of the whole hot path over
one batch of synthetic input: synthesis f = Phi c and analysis c = Phi^* f at
nrhs = 1 and at the workload's multi-RHS width (32 for configs[1]), i.e.
2 * (1 + 32) = 66 column transforms per step.  ``value`` is column transforms
per second summed over all ranks (weak scaling: every rank is an independent
replica over its own right-hand sides — "replicas only").

Workload: configs[1] (flat periodic square, n = m = 65,536, tol 1e-8) — the
configuration BASELINE.json's metric is quoted on.  The plan (tens of GB) is
far larger than L2, so no L2 flush is needed; for small workloads (< 4 x L2)
a 256 MiB buffer is rewritten between timed steps.

``--impl reference`` times the oracle (independent CPU butterfly apply O2,
``oracle/``) on this box's host cores on a bounded sample of the same workload
(rank 0 only; other ranks exit 0).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import mht_inputs as mi  # noqa: E402

METRIC = "MHT applies/sec (fp64) and achieved HBM GB/s / FP64 % of peak at nrhs=1 and 32"
UNIT = "column transforms/s"
L2_BYTES = 126 * 2**20


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="mht", choices=["mht", "reference"])
    ap.add_argument("--workload", default="c2", choices=sorted(mi.WORKLOADS))
    ap.add_argument("--builder", default="gpu", choices=["gpu", "cpu"])
    ap.add_argument("--e2e-steps", type=int, default=10)
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--mode", default="replicas", choices=["replicas", "shard"],
                    help="replicas (default): every rank holds the whole plan and transforms its own columns "
                         "(weak scaling, no data-path collective); shard: the plan is split across the ranks "
                         "and every transform is done jointly with one NCCL all-to-all (strong scaling)")
    ap.add_argument("--exchange", default="nccl", choices=["nccl", "fused"],
                    help="--mode shard only: nccl = one all_to_all_single of z_ls per direction between the "
                         "kernel sequences; fused = the switch stage's kernels store z_ls straight into the peers' "
                         "receive buffers over NVLink peer memory (CUDA IPC) with arrival flags (DESIGN.md §7)")
    ap.add_argument("--cpu-table", action="store_true",
                    help="cpu_baseline leg only: time the oracle (O2 at 1 and all threads, O1 dense sum full or on "
                         "a labelled row subset) on this host for --workload, print one JSON line, exit")
    return ap.parse_args()


def log(*a):
    print(*a, file=sys.stderr, flush=True)


# ---------------------------------------------------------------- clocks
class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        self.p = None

    def start(self, settle: float = 0.3):
        """Start sampling; then wait `settle` s so nvidia-smi's start-up (NVML
        initialisation, which can stall the driver for milliseconds) is over
        before the caller's timed region begins."""
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                                       "-lms", "200", "-i", str(self.idx)], stdout=self.f, stderr=subprocess.DEVNULL)
            time.sleep(settle)
        except Exception:
            self.p = None

    def stop(self):
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.p.terminate()
        self.p.wait()
        self.f.flush()
        rows = [r.split(",") for r in open(self.f.name).read().strip().splitlines() if r.strip()]
        os.unlink(self.f.name)
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            r = [x.strip() for x in r]
            if len(r) < 9:
                continue
            try:
                sm.append(float(r[1]))
                smax.append(float(r[2]))
            except ValueError:
                continue
            for nm, v in zip(names, r[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------- setup
def dist_setup(args):
    import torch

    from paper_2605_21828_b200 import replicas

    ws, rank, lrank = replicas.env_world()
    gpu = torch.cuda.is_available()
    if gpu:
        torch.cuda.set_device(lrank)
    if ws > 1:
        import torch.distributed as dist

        if gpu:
            dist.init_process_group("nccl", device_id=torch.device("cuda", lrank))
        else:
            dist.init_process_group("gloo")
    return ws, rank, lrank


def barrier(ws):
    from paper_2605_21828_b200 import replicas

    replicas.barrier(ws)


def allreduce_max(x, ws):
    import torch

    from paper_2605_21828_b200 import replicas

    return replicas.allreduce_max(x, ws, device="cuda" if torch.cuda.is_available() else None)


def get_plan(w, args, ws, rank, lrank):
    from paper_2605_21828_b200 import workloads as W

    import torch

    path = W.plan_cache_path(w)
    if rank == 0 and not os.path.exists(path):
        t0 = time.time()
        builder = args.builder if torch.cuda.is_available() else "cpu"
        st = W.build_workload_plan(w, path + ".build", builder=builder, device=f"cuda:{lrank}",
                                   log=lambda s: log(s))
        os.replace(path + ".build", path)
        log(f"[bench] plan built ({builder}) in {time.time() - t0:.1f}s: {st['entries']} entries "
            f"({st['entries'] / st['dense_entries']:.3f} of dense), {st['plan_bytes'] / 1e9:.2f} GB")
        if torch.cuda.is_available():
            torch.cuda.empty_cache()
    barrier(ws)
    return path


def phases_for(w):
    ph = [("fwd", 1), ("adj", 1)]
    for r in w.nrhs:
        if r > 1:
            ph += [("fwd", r), ("adj", r)]
    return ph


def dtype_tag(w):
    return "c128" if w.dtype == "complex128" else "f64"


def workload_desc(w):
    if w.family == "flat":
        return f"{w.name}: flat periodic square, n=m={w.n}, k in [-{w.extra['side'] // 2},{w.extra['side'] // 2 - 1}]^2, tol {w.tol:g}"
    if w.family == "sphere":
        return f"{w.name}: unit sphere, n={w.n}, real SH l<={w.extra['lmax']}, tol {w.tol:g}"
    return f"{w.name}: torus mesh n={w.n}, m={w.m}, tol {w.tol:g}"


# ---------------------------------------------------------------- oracle (CPU) legs
def time_oracle(path, w, seconds, steps=None, warmup=0):
    """O2 forward + adjoint at nrhs = 1, repeated; returns (transforms/s, reps, s, threads)."""
    import oracle

    O = oracle.Plan(path, verify_checksum=False)
    c = mi.workload_coefficients(w, 1)
    y = mi.workload_adjoint_input(w, 1)
    for _ in range(warmup):
        O.apply(c)
        O.adjoint(y)
    reps, t0 = 0, time.perf_counter()
    while True:
        O.apply(c)
        O.adjoint(y)
        reps += 1
        el = time.perf_counter() - t0
        if (steps is not None and reps >= steps) or (steps is None and el >= seconds):
            break
    O.close()
    return 2 * reps / el, reps, el, oracle.num_threads()


def run_reference(args, w, path):
    v, reps, el, cores = time_oracle(path, w, None, steps=args.steps, warmup=args.warmup)
    sample = (f"oracle O2 (independent CPU butterfly apply, C + OpenMP) on the full {w.name} plan: "
              f"synthesis + analysis at nrhs=1 per step, {reps} steps in {el:.1f}s")
    out = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * el / reps,
           "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": dtype_tag(w),
           "data": "synthetic (seeded, mht_inputs)",
           "config": {"workload": workload_desc(w), "nrhs": [1], "plan": os.path.basename(path)},
           "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": sample},
           "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


def run_cpu_table(args, w, path):
    """SURVEY.md §8(d) CPU protocol: O2 (butterfly) with all threads and with
    one; O1 (dense sum) in full for c1 and c4, on a 4,096-row subset for the
    others (extrapolated x n/4096, labelled).  Bounded: each figure is the
    mean over reps within ~args.cpu_seconds."""
    import oracle

    out = {"impl": "cpu_table", "workload": workload_desc(w), "unit": "ms per column transform",
           "host_cores": len(os.sched_getaffinity(0))}
    try:
        out["cpu_model"] = [l.split(":", 1)[1].strip() for l in open("/proc/cpuinfo") if l.startswith("model name")][0]
    except Exception:
        pass
    c = mi.workload_coefficients(w, 1)
    y = mi.workload_adjoint_input(w, 1)
    for threads in (oracle.num_threads(), 1):
        oracle.set_threads(threads)
        O = oracle.Plan(path, verify_checksum=False)
        for kind, fn, arg in (("apply", O.apply, c), ("adjoint", O.adjoint, y)):
            reps, t0 = 0, time.perf_counter()
            while True:
                fn(arg)
                reps += 1
                if time.perf_counter() - t0 >= args.cpu_seconds / 4 or reps >= 200:
                    break
            out[f"O2_{kind}_threads{threads}"] = 1e3 * (time.perf_counter() - t0) / reps
        O.close()
    oracle.set_threads(out["host_cores"])
    rows = np.arange(w.n) if w.n * w.m <= 2**27 else np.sort(np.random.default_rng(7).choice(w.n, 4096, replace=False))
    t0 = time.perf_counter()
    if w.family == "flat":
        oracle.flat_synth(mi.flat_points(w.n)[rows], mi.flat_workload_modes(w), c)
    elif w.family == "sphere":
        th, ph, _ = mi.sphere_points(w.n)
        oracle.sphere_synth(th[rows], ph[rows], w.extra["lmax"], c)
    else:
        from mht_inputs import mesh as mm

        Phi = mm.torus_workload_inputs(w.extra["nu"], w.extra["nv"], w.m)[3]
        t0 = time.perf_counter()
        oracle.dense_synth(Phi[rows], c)
    el = time.perf_counter() - t0
    out["O1_synth_ms"] = 1e3 * el * w.n / len(rows)
    out["O1_rows_timed"] = int(len(rows))
    out["O1_note"] = ("full" if len(rows) == w.n else f"extrapolated from a {len(rows)}-row subset (x n/{len(rows)})")
    out["threads_all"] = out["host_cores"]
    print(json.dumps(out), flush=True)


# ---------------------------------------------------------------- main
def main():
    args = parse()
    import torch

    w = mi.WORKLOADS[args.workload]
    ws, rank, lrank = dist_setup(args)
    if args.cpu_table:
        if rank == 0:
            run_cpu_table(args, w, get_plan(w, args, 1, rank, lrank))
        return
    if args.impl == "reference":
        # the reference arm (the oracle on host cores) runs on rank 0 only;
        # other ranks exit 0 without work
        if rank == 0:
            run_reference(args, w, get_plan(w, args, 1, rank, lrank))
        return
    path = get_plan(w, args, ws, rank, lrank)
    if args.mode == "shard" and ws > 1:
        return run_shard(args, w, path, ws, rank, lrank)

    from paper_2605_21828_b200 import mht, replicas

    P = mht.Plan(path, lrank)
    dev = torch.device("cuda", lrank)
    phases = phases_for(w)
    widths = sorted({r for _, r in phases})
    P.reserve(max(widths))
    sb = P.scalar_bytes
    # inputs (each rank its own right-hand sides: replicas over RHS columns)
    ins, outs = {}, {}
    for r in widths:
        c = replicas.rank_coefficients(w, r, rank)
        y = replicas.rank_adjoint_inputs(w, r, rank)
        ins[("fwd", r)] = torch.from_numpy(c).to(dev)
        ins[("adj", r)] = torch.from_numpy(y).to(dev)
        outs[("fwd", r)] = torch.empty((r, w.n), dtype=P.torch_dtype, device=dev)
        outs[("adj", r)] = torch.empty((r, w.m), dtype=P.torch_dtype, device=dev)

    def step():
        for kind, r in phases:
            if kind == "fwd":
                P.apply(ins[(kind, r)], out=outs[(kind, r)])
            else:
                P.adjoint(ins[(kind, r)], out=outs[(kind, r)])

    flush = None
    if P.info.plan_bytes < 4 * L2_BYTES:
        flush = torch.empty(2 * L2_BYTES // 4, dtype=torch.float32, device=dev)
    for _ in range(max(args.warmup, 0)):
        step()
    torch.cuda.synchronize()

    def timed_steps():
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
        barrier(ws)
        torch.cuda.synchronize()
        for k in range(args.steps):
            if flush is not None:
                flush.zero_()
            ev[k][0].record()
            step()
            ev[k][1].record()
        torch.cuda.synchronize()
        barrier(ws)
        return allreduce_max(sum(a.elapsed_time(b) for a, b in ev), ws)

    # ---- the timed region: the library's default mode (each apply replays its
    # captured CUDA graph), CUDA events on the launching stream, max over ranks
    clocks = ClockSampler(lrank)
    clocks.start()
    total_ms = timed_steps()
    clk = clocks.stop()
    transforms = sum(r for _, r in phases)
    value = replicas.job_throughput(transforms * args.steps, ws, total_ms / 1e3)

    # ---- kernel pass: the same K steps again with every launch bracketed by the
    # library's own events on its stream (eager launches), for the per-kernel
    # breakdown and the roofline
    P.set_profiling(True)
    P.profile_reset()
    prof_ms = timed_steps()

    # ---- per-kernel live timing (events bracket every launch on its stream)
    stats = P.stage_stats()
    coef_bytes = sum(s["coef_bytes"] for s in stats)
    entries = P.info.factor_entries
    per = {}
    for kind_i, kind in ((0, "fwd"), (1, "adj"), (2, "sum")):
        for r in widths:
            ms, nl = P.profile_get(kind_i, -1, r)
            if nl:
                per[(kind, r)] = (ms, nl)
    # per-stage device time (ms per apply) of every phase, with the stage's factor bytes
    stage_ms = {}
    for kind_i, kind in ((0, "fwd"), (1, "adj"), (2, "sum")):
        for r in widths:
            row = {}
            for s_ in range(0, P.L + 2):
                ms, nl = P.profile_get(kind_i, s_, r)
                if nl:
                    row[str(s_)] = round(ms / args.steps, 4)
            if kind == "sum":  # stage -1 (the final sums into c) = all - the per-stage ones
                ms, nl = P.profile_get(kind_i, -1, r)
                if nl:
                    row["c"] = round(ms / args.steps - sum(row.values()), 4)
            if row:
                stage_ms[f"{kind}_nrhs{r}"] = row
    P.set_profiling(False)
    breakdown = {}
    for (kind, r), (ms, nl) in per.items():
        applies = args.steps
        byts = (coef_bytes + (w.m + w.n) * r * sb) * applies if kind != "sum" else None
        flops = (8 if P.is_complex else 2) * entries * r * applies
        breakdown[f"{kind}_nrhs{r}"] = {
            "ms_per_apply": ms / applies, "launches_per_apply": nl / applies,
            "GBps": (byts / (ms / 1e3) / 1e9) if byts else None,
            "TFLOPs": (flops / (ms / 1e3) / 1e12) if kind != "sum" else None}
    peaks = _peaks()
    dom = max(((k, v) for k, v in per.items() if k[0] in ("fwd", "adj")), key=lambda kv: kv[1][0])
    (dkind, dr), (dms, dn) = dom
    per_launch_ms = dms / dn
    traffic = _traffic(w.name, f"{dkind}@{dr}")
    if dr == 1:
        alg = (coef_bytes + (w.m + w.n) * sb) / (dn / args.steps)        # bytes per launch (average)
        achieved = alg / (per_launch_ms / 1e3) / 1e9
        kname = f"{dkind}_kernel nrhs=1"
        roof = {"bound": "hbm", "achieved": achieved, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                "frac": achieved / peaks["hbm_gbs"], "frac_of_nominal_8TBs": achieved / 8000.0,
                "traffic": traffic, "algorithmic_bytes_per_launch": alg,
                "kernel": kname, "peak_source": peaks["hbm_src"]}
    else:
        # the multi-RHS stages run on the FP64 tensor pipe (DMMA): its own measured peak
        alg = (8 if P.is_complex else 2) * entries * dr / (dn / args.steps)
        achieved = alg / (per_launch_ms / 1e3) / 1e12
        roof = {"bound": "tensor", "achieved": achieved, "peak": peaks["dmma_tflops"], "unit": "TFLOP/s",
                "frac": achieved / peaks["dmma_tflops"], "frac_of_burst_peak": achieved / peaks["dmma_tflops_burst"],
                "frac_of_nominal": achieved / (148 * 64 * 2 * 1.965e9 / 1e12),  # 37.2 TF: 148 SMs x 64 FMA/clk x 2 x 1.965 GHz
                "traffic": traffic, "algorithmic_flops_per_launch": alg,
                "kernel": _mma_kernel_name(P.is_complex, dkind, dr),
                "peak_source": peaks["dmma_src"]}
        if P.is_complex:
            roof["note"] = ("achieved counts 8 real flops per complex multiply-add (algorithmic); the kernel "
                            "issues 3 real DMMA products per complex product (Gauss), so pipe work is 3/4 of that")
            roof["pipe_frac"] = 0.75 * achieved / peaks["dmma_tflops"]  # issued DMMA work / the pipe's peak
        else:
            roof["pipe_frac"] = achieved / peaks["dmma_tflops"]
    if traffic is not None:
        roof["traffic_source"] = _traffic_src(w.name)
    roof["per_launch_ms"] = per_launch_ms
    roof["launches_per_apply"] = dn / args.steps

    out = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
           "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
           "scaling": "weak", "vs_baseline": None, "dtype": dtype_tag(w),
           "data": "synthetic (seeded generators in mht_inputs; no paper dataset)",
           "config": {"workload": workload_desc(w), "phases": [f"{k}@nrhs{r}" for k, r in phases],
                      "transforms_per_step_per_gpu": transforms, "parallelism": f"replicas{ws}",
                      "plan_bytes": P.info.plan_bytes, "factor_entries": entries,
                      "factor_fraction_of_dense": entries / (w.n * w.m),
                      "l2": ("plan larger than L2 (no flush)" if flush is None else "L2 flushed between steps")},
           "roofline": roof, "breakdown": breakdown, "clocks": clk,
           "kernel_pass": {"ms_per_step": prof_ms / args.steps,
                           "value": replicas.job_throughput(transforms * args.steps, ws, prof_ms / 1e3),
                           "note": "the same steps launched eagerly with every kernel bracketed by CUDA events "
                                   "(breakdown, stage_ms and roofline come from this pass); value above is the "
                                   "graph-replay timed region"},
           "stage_ms": stage_ms, "stage_coef_bytes": {str(x["stage"]): x["coef_bytes"] for x in stats},
           # counted: every launch of the timed region is bracketed by the library's events
           "gpu_launches": int(sum(nl for _, nl in per.values()))}

    # ---- end to end through the C ABI with pinned host buffers
    if not args.no_e2e:
        out["e2e"] = _e2e(P, phases, w, ws, args, device_ms_per_step=total_ms / args.steps)
    # ---- CPU oracle baseline (rank 0, N = 1)
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        v, reps, el, cores = time_oracle(path, w, args.cpu_seconds)
        out["cpu_baseline"] = {"value": v, "unit": UNIT, "cores": cores, "kind": "oracle",
                               "sample": f"O2 synthesis+analysis at nrhs=1 on the full {w.name} plan, "
                                         f"{reps} reps in {el:.1f}s (bounded sample of the step's phases)"}
    if rank == 0:
        print(json.dumps(out), flush=True)
    P.close()
    if ws > 1:
        import torch.distributed as dist

        dist.destroy_process_group()


def run_shard(args, w, path, ws, rank, lrank):
    """--mode shard under torchrun: rank g holds shard g of the plan (frequency
    subtrees up to the switch level, space subtrees after it);
    every transform of the step is done jointly by all ranks, the exchange is
    one torch.distributed (NCCL) all_to_all_single of z_ls per direction."""
    import torch

    from paper_2605_21828_b200 import replicas
    from paper_2605_21828_b200 import shard as SH

    dev = torch.device("cuda", lrank)
    S = SH.ShardPlan(path, ws, rank, lrank)
    phases = phases_for(w)
    if args.exchange == "fused":
        S.fuse(max(r for _, r in phases))
    ins, outs = {}, {}
    for kind, r in phases:
        if kind == "fwd":
            ins[(kind, r)] = torch.from_numpy(mi.workload_coefficients(w, r)).to(dev)
            outs[(kind, r)] = torch.zeros((r, w.n), dtype=S.torch_dtype, device=dev)
        else:
            ins[(kind, r)] = torch.from_numpy(mi.workload_adjoint_input(w, r)).to(dev)
            outs[(kind, r)] = torch.zeros((r, w.m), dtype=S.torch_dtype, device=dev)

    def step():
        for kind, r in phases:
            if kind == "fwd":
                S.apply(ins[(kind, r)], outs[(kind, r)])
            else:
                S.adjoint(ins[(kind, r)], outs[(kind, r)])

    for _ in range(max(args.warmup, 0)):
        step()
    torch.cuda.synchronize()
    clocks = ClockSampler(lrank)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    barrier(ws)
    torch.cuda.synchronize()
    clocks.start()
    for k in range(args.steps):
        ev[k][0].record()
        step()
        ev[k][1].record()
    torch.cuda.synchronize()
    clk = clocks.stop()
    barrier(ws)
    total_ms = allreduce_max(sum(a.elapsed_time(b) for a, b in ev), ws)
    transforms = sum(r for _, r in phases)
    exch = int(sum(S.send_len) - S.send_len[rank])  # entries this rank sends per RHS column and direction
    out = {"metric": METRIC, "value": transforms * args.steps / (total_ms / 1e3), "unit": UNIT, "n_gpus": ws,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": total_ms / args.steps,
           "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": dtype_tag(w),
           "data": "synthetic (seeded generators in mht_inputs; no paper dataset)",
           "config": {"workload": workload_desc(w), "phases": [f"{k}@nrhs{r}" for k, r in phases],
                      "transforms_per_step": transforms, "parallelism": f"shard{ws} (switch level {S.ls})",
                      "exchange": ("fused: switch-stage stores into the peers' receive buffers (CUDA IPC, NVLink)"
                                   if args.exchange == "fused" else "NCCL all_to_all_single"),
                      "factor_entries_this_rank": S.info.factor_entries,
                      "exchange_bytes_per_rhs_per_direction_this_rank": exch * S.scalar_bytes},
           "clocks": clk, "gpu_launches": None}
    if rank == 0:
        print(json.dumps(out), flush=True)
    S.close()
    import torch.distributed as dist

    dist.destroy_process_group()


def _e2e(P, phases, w, ws, args, device_ms_per_step=None):
    """The same step through the C ABI's host-buffer call mht_apply_host_batch:
    every phase copies its input from pinned host memory, replays the apply
    and copies the result back, inside the timed region, the copies of one
    phase overlapping the transforms of its neighbours (one call per step,
    which returns when all of the step's outputs are in host memory).  Also measures the host<->device link on this box (pinned torch
    copies of the widest phase's vectors, CUDA events, each direction alone)
    so the e2e time can be checked against device time + bytes / link rate."""
    import torch

    host_in, host_out = {}, {}
    h2d = d2h = 0
    for kind, r in phases:
        nout = w.n if kind == "fwd" else w.m
        src = (mi.workload_coefficients(w, r) if kind == "fwd" else mi.workload_adjoint_input(w, r))
        ti = torch.from_numpy(src).pin_memory()
        to = torch.empty((r, nout), dtype=P.torch_dtype).pin_memory()
        host_in[(kind, r)], host_out[(kind, r)] = ti, to
        h2d += ti.numel() * P.scalar_bytes
        d2h += to.numel() * P.scalar_bytes

    # one pipelined host batch per step (mht_apply_host_batch): each phase's
    # input copy and the previous phase's output copy overlap the transforms;
    # the call returns when the step's outputs are all in host memory
    jobs = [(0 if kind == "fwd" else 1, r, host_in[(kind, r)].data_ptr(), host_out[(kind, r)].data_ptr())
            for kind, r in phases]

    def step():
        P.host_batch_ptr(jobs)

    # two warm-up steps: the first grows the host staging to the widest phase
    # (which drops the graphs captured for the narrower ones), the second
    # captures every phase's graph outside the timed region
    step()
    step()
    # at least args.e2e_steps steps and ~0.2 s of them (small plans: 1 ms steps),
    # the same count on every rank
    nsteps = args.e2e_steps
    if device_ms_per_step:
        nsteps = max(nsteps, int(math.ceil(200.0 / max(device_ms_per_step, 1e-3))))
    nsteps = int(allreduce_max(nsteps, ws))
    barrier(ws)
    clocks = ClockSampler(torch.cuda.current_device())
    clocks.start()
    t0 = time.perf_counter()
    for _ in range(nsteps):
        step()
    el = allreduce_max(time.perf_counter() - t0, ws)
    clk = clocks.stop()
    transforms = sum(r for _, r in phases)
    # link rates on this box: the widest phase's input (H2D) and output (D2H)
    big_in = max(host_in.values(), key=lambda t: t.numel())
    big_out = max(host_out.values(), key=lambda t: t.numel())
    dev_in = torch.empty_like(big_in, device="cuda")
    dev_out = torch.empty_like(big_out, device="cuda")
    rates = {}
    for name, dst, src_ in (("h2d", dev_in, big_in), ("d2h", big_out, dev_out)):
        best = None
        for _ in range(5):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            dst.copy_(src_, non_blocking=True)
            b.record()
            torch.cuda.synchronize()
            t = a.elapsed_time(b)
            best = t if best is None else min(best, t)
        rates[name] = src_.numel() * P.scalar_bytes / (best / 1e3) / 1e9
    out = {"value": ws * transforms * nsteps / el, "unit": UNIT, "h2d_bytes_per_step": h2d,
           "d2h_bytes_per_step": d2h, "steps": nsteps, "ms_per_step": 1e3 * el / nsteps,
           "link_GBps": {"h2d": rates["h2d"], "d2h": rates["d2h"],
                         "how": "pinned torch copy of the widest phase's vector, best of 5, CUDA events"},
           "clocks": clk,
           "api": "mht_apply_host_batch: the step's phases as one pipelined host batch (pinned host buffers, every "
                  "copy in the timed region, host-to-device / device-to-host overlapping the transforms)"}
    if device_ms_per_step is not None:
        out["copy_floor_ms_per_step"] = 1e3 * (h2d / (rates["h2d"] * 1e9) + d2h / (rates["d2h"] * 1e9))
        out["device_ms_per_step"] = device_ms_per_step
    return out


def _mma_kernel_name(cplx, kind, nrhs):
    """The multi-RHS kernel libmht dispatches for this width (csrc/mht_kernels.cu mma_dispatch)."""
    if cplx and nrhs >= 16:
        return (f"mma_ws_kernel {kind} nrhs={nrhs} (DMMA m16n8k4 f64, TMA + warp-specialised, "
                f"{32 if nrhs >= 32 else 16} RHS per CTA)")
    if not cplx and nrhs >= 32:
        return f"mma_real_kernel {kind} nrhs={nrhs} (DMMA m16n8k4 f64, cp.async ring, 6 CTAs/SM)"
    return f"mma_kernel {kind} nrhs={nrhs} (DMMA m16n8k4 f64, {16 if nrhs >= 16 else 8} RHS per CTA)"


def _peaks():
    """Roofline denominators: MEASURED_PEAKS.json (driver-written) for HBM; FP64
    from the measured DFMA microbenchmark in profiles/ if present, else derived
    from unit counts and clocks."""
    out = {}
    mp = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        d = json.load(open(mp))
        out["hbm_gbs"] = float(d["hbm_gbs"])
        out["hbm_src"] = "measured (MEASURED_PEAKS.json hbm_gbs)"
        smax = float(d.get("sm_max_mhz", 1965.0))
    except Exception:
        out["hbm_gbs"] = 6650.0
        out["hbm_src"] = "fallback (B200_PROFILING.md 6.65 TB/s)"
        smax = 1965.0
    cands = sorted(f for f in os.listdir(os.path.join(ROOT, "profiles")) if f.endswith("fp64_peak.json"))
    fp = os.path.join(ROOT, "profiles", cands[-1]) if cands else ""
    try:
        d = json.load(open(fp))
        # the kernels are timed inside long steps: the sustained figure (the
        # burst one is reported beside it)
        sus = "dmma_m16n8k4_tflops_sustained" in d
        out["fp64_tflops"] = float(d["dfma_tflops_sustained" if sus else "dfma_tflops"])
        out["dmma_tflops"] = float(d["dmma_m16n8k4_tflops_sustained" if sus else "dmma_m16n8k4_tflops"])
        out["dmma_tflops_burst"] = float(d["dmma_m16n8k4_tflops"])
        clk = d.get("clocks", {})
        out["fp64_src"] = f"measured DFMA microbenchmark ({os.path.relpath(fp, ROOT)})"
        out["dmma_src"] = (f"measured DMMA m16n8k4 microbenchmark, {'sustained 3 s' if sus else 'burst'} "
                           f"({os.path.relpath(fp, ROOT)}; SM clock median {clk.get('sm_mhz')} MHz, "
                           f"reasons {clk.get('reasons')})")
    except Exception:
        out["fp64_tflops"] = out["dmma_tflops"] = out["dmma_tflops_burst"] = 148 * 64 * 2 * smax * 1e6 / 1e12
        out["fp64_src"] = out["dmma_src"] = "derived: 148 SMs x 64 FP64 FMA/clk x 2 x sm_max_mhz"
    return out


def _traffic_file(workload):
    cands = sorted(f for f in os.listdir(os.path.join(ROOT, "profiles"))
                   if f.endswith(f"_traffic_{workload}.json"))
    return os.path.join(ROOT, "profiles", cands[-1]) if cands else None


def _traffic(workload, phase):
    """DRAM bytes per launch of the dominant phase from the committed ncu capture
    (profiles/rNN_traffic_<workload>.json, tools/ncu_traffic.py), else None."""
    f = _traffic_file(workload)
    if f is None:
        return None
    try:
        return json.load(open(f))["phases"][phase]["dram_bytes_per_launch"]
    except Exception:
        return None


def _traffic_src(workload):
    f = _traffic_file(workload)
    return os.path.relpath(f, ROOT) if f else None


if __name__ == "__main__":
    main()
