"""Driver for compute-sanitizer (racecheck / synccheck / memcheck): every
libmht kernel family on two small plans, one apply of each kind.

    compute-sanitizer --tool racecheck --racecheck-report all python tools/sanitize_run.py
    compute-sanitizer --tool synccheck python tools/sanitize_run.py

Plans: a complex flat plan (n = m = 4096, L = 6, tol 1e-8: c1's shape) and a
real sphere plan (n = 4096, l <= 63, L = 6, tol 1e-10), built by the CPU
builder.  Widths: nrhs = 1 (fwd_kernel, adj_kernel, reduce_kernel), 17 (mma_kernel), 32 and 40 (mma_ws_kernel for complex,
mma_real_kernel for real; 40 = a partial second RHS chunk).  Graphs off so
every launch is a plain launch the tool instruments.  Prints one line per case
with the max relative difference against the nrhs = 1 path (a self-check
only; parity against the oracle is tests/test_gpu_parity.py).
"""
import os
import sys
import tempfile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np
import torch

import mht_inputs as mi
from paper_2605_21828_b200 import _build, mht
from paper_2605_21828_b200 import workloads as W


def main():
    _build.build()
    mht.load_library()
    root = tempfile.mkdtemp(prefix="mht_san_")
    cases = [(W.flat_workload(4096, 64, 6, 1e-8, name="san_flat"), mi.complex_gaussian),
             (W.sphere_workload(4096, 63, 6, 1e-10, name="san_sph"), mi.real_gaussian)]
    widths = [int(x) for x in os.environ.get("SAN_WIDTHS", "1,17,32,40").split(",")]
    for w, gen in cases:
        path = os.path.join(root, f"{w.name}.plan")
        W.build_workload_plan(w, path, workers=8, log=None)
        P = mht.Plan(path)
        P.set_graphs(False)
        for nrhs in widths:
            c = torch.from_numpy(gen(nrhs, w.m, 10 + nrhs)).cuda()
            y = torch.from_numpy(gen(nrhs, w.n, 20 + nrhs)).cuda()
            f = P.apply(c)
            a = P.adjoint(y)
            torch.cuda.synchronize()
            f1 = torch.stack([P.apply(c[r:r + 1])[0] for r in range(min(nrhs, 2))])
            a1 = torch.stack([P.adjoint(y[r:r + 1])[0] for r in range(min(nrhs, 2))])
            ef = (torch.linalg.vector_norm(f[:2] - f1) / torch.linalg.vector_norm(f1)).item()
            ea = (torch.linalg.vector_norm(a[:2] - a1) / torch.linalg.vector_norm(a1)).item()
            print(f"{w.name} nrhs={nrhs}: fwd vs nrhs=1 {ef:.2e}, adj {ea:.2e}", flush=True)
        P.close()
    print("sanitize_run done", flush=True)


if __name__ == "__main__":
    main()
