"""Convergence / timing of the GPU eigensolver on the configs[3] torus."""
import os, sys, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from mht_inputs import mesh as mm
V, F = mm.torus_mesh()
K, mass = mm.cotan_fem(V, F)
for deg in (24, 48):
    info = {}
    t = time.time()
    try:
        lam, Q = mm.chebyshev_subspace_eigs(K, mass, 2048, device="cuda", degree=deg, info=info)
        ok = True
    except RuntimeError as e:
        ok = str(e)
    el = time.time() - t
    print(json.dumps({"degree": deg, "seconds": round(el, 1), "ok": ok, **info}), flush=True)
