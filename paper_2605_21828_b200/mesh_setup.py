"""configs[3] setup: torus mesh, stored eigenvectors (inputs from mht_inputs.mesh)
and the Fiedler-tree spatial ordering (§3)."""
from __future__ import annotations

import sys
import time

import mht_inputs as mi
from mht_inputs import mesh as mm

from .precompute.basis import DenseBasis
from .precompute.fiedler import fiedler_tree


def mesh_workload(nu: int, nv: int, m: int, L: int, tol: float, name: str = "mesh"):
    return mi.Workload(name, "mesh", nu * nv, m, "float64", tol, L, (1,), {"nu": nu, "nv": nv})


def setup_mesh(w: mi.Workload):
    t0 = time.time()
    V, F, lam, Phi, mass = mm.torus_workload_inputs(w.extra["nu"], w.extra["nv"], w.m)
    t1 = time.time()
    perm, sp_off = fiedler_tree(V, F, w.L)
    print(f"[mesh_setup] eigenbasis {t1 - t0:.1f}s, Fiedler tree {time.time() - t1:.1f}s", file=sys.stderr)
    return DenseBasis(Phi), perm, sp_off
