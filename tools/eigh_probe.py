"""Why does the c4 eigen-solve take ~650 s on the box?  Time torch.linalg.eigh
on the GPU for the 32,768 x 32,768 float64 matrix and report any exception."""
import os, sys, time, traceback
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from mht_inputs import mesh as mm
V, F = mm.torus_mesh()
K, mass = mm.cotan_fem(V, F)
s = 1.0 / np.sqrt(mass)
A = (K.multiply(s[:, None]).multiply(s[None, :])).toarray()
A = 0.5 * (A + A.T)
print("matrix", A.shape, A.dtype, flush=True)
for drv in ("default",):
    try:
        t = time.time()
        At = torch.as_tensor(A, device="cuda")
        lam, Q = torch.linalg.eigh(At)
        torch.cuda.synchronize()
        print("torch eigh ok", round(time.time() - t, 1), "s", float(lam[0]), float(lam[2047]), flush=True)
    except Exception:
        traceback.print_exc()
