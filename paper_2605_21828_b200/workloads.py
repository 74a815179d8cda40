"""Workload -> (basis, trees) -> plan file.  Host precompute, outside the timed path.

Geometry, modes and coefficient vectors come from ``mht_inputs`` (the seeded
generators shared with the oracle); the butterfly factorization is built here.
"""
from __future__ import annotations

import dataclasses
import os

import numpy as np

import mht_inputs as mi

from .precompute.basis import DenseBasis, FlatBasis, SphereBasis
from .precompute.builder import build_plan
from .precompute.trees import freq_tree, kd_tree


def flat_workload(n: int, side: int, L: int, tol: float, name: str = "flat", seed: int = mi.SEED_GEOMETRY):
    """A flat-square workload with n random points and side^2 modes."""
    return mi.Workload(name, "flat", n, side * side, "complex128", tol, L, (1,), {"side": side, "seed": seed})


def sphere_workload(n: int, lmax: int, L: int, tol: float, name: str = "sphere"):
    return mi.Workload(name, "sphere", n, (lmax + 1) ** 2, "float64", tol, L, (1,), {"lmax": lmax})


def freq_plan_order(w: mi.Workload):
    """(plan mode list, perm_k) of a flat workload.  The user's c is in
    eigenvalue order (mht_inputs.flat_workload_modes).  The quadtree-frequency
    variant (extra["ftree"] == "kd", reading A18) factorizes the columns in the
    2-D kd order of the frequency box and stores perm_k (plan position -> user
    index) in the plan, so the library reads and writes c in the user's order;
    otherwise the plan order is the user's order and there is no perm_k."""
    k_user = mi.flat_workload_modes(w)
    if w.extra.get("ftree") != "kd":
        return k_user, None
    k_plan = mi.flat_modes_kd(w.extra["side"], w.L)[: w.m]
    idx = {tuple(v): i for i, v in enumerate(k_user.tolist())}
    perm_k = np.array([idx[tuple(v)] for v in k_plan.tolist()], dtype=np.int32)
    return k_plan, perm_k


def setup(w: mi.Workload):
    """Return (basis, perm, sp_off, fr_off, perm_k); perm_k is None unless the
    plan's frequency order differs from the user's (freq_plan_order)."""
    perm_k = None
    if w.family == "flat":
        x = mi.flat_points(w.n, seed=w.extra.get("seed", mi.SEED_GEOMETRY))
        k, perm_k = freq_plan_order(w)
        basis = FlatBasis(x, k)
        perm, sp_off = kd_tree(x, w.L, alternate=True)
    elif w.family == "sphere":
        th, ph, p = mi.sphere_points(w.n)
        basis = SphereBasis(th, ph, w.extra["lmax"])
        perm, sp_off = kd_tree(p, w.L, alternate=False)
    elif w.family == "mesh":
        from . import mesh_setup

        basis, perm, sp_off = mesh_setup.setup_mesh(w)
    else:
        raise ValueError(w.family)
    fr_off = freq_tree(w.m, w.L)
    return basis, perm, sp_off, fr_off, perm_k


def build_workload_plan(w: mi.Workload, path: str, workers=None, log=print, precompute_sphere=None,
                        builder: str = "cpu", device="cuda"):
    """builder = "cpu" (numpy/scipy CPQR, multiprocess) or "gpu" (libmht's
    construction kernels on the device, include/mht_build.h; same
    factorization, same file format)."""
    basis, perm, sp_off, fr_off, perm_k = setup(w)
    if builder == "gpu":
        from .precompute import gpu_builder as G

        if w.family == "flat":
            tb = G.DeviceFlatBasis(basis.x, basis.k, device)
        elif w.family == "sphere":
            tb = G.DeviceTableBasis(G.sphere_table(basis.theta, basis.phi, basis.lmax, device), np.float64)
        else:
            import torch

            tb = G.DeviceTableBasis(torch.as_tensor(np.asarray(basis.Phi), device=device), basis.dtype)
        try:
            return G.build_plan_gpu(tb, perm, sp_off, fr_off, w.L, w.tol, path, device=device, log=log,
                                    perm_k=perm_k)
        finally:
            del tb
    if isinstance(basis, SphereBasis) and (precompute_sphere or (precompute_sphere is None and w.n * w.m <= 6e9)):
        basis.precompute_all()
    return build_plan(basis, perm, sp_off, fr_off, w.L, w.tol, path, workers=workers, log=log, perm_k=perm_k)


# bump when the builders' numerics change so cached plans are never reused across versions
BUILDER_VERSION = 6  # 5: quadtree-frequency plans carry perm_k (plan v2); 6: device CPQR kernel (per-block stop)


def plan_cache_path(w: mi.Workload, root: str | None = None) -> str:
    root = root or os.environ.get("MHT_PLAN_DIR") or ("/dev/shm/mht_plans" if os.path.isdir("/dev/shm") else "/tmp/mht_plans")
    os.makedirs(root, exist_ok=True)
    tag = f"{w.name}_{w.family}_n{w.n}_m{w.m}_L{w.L}_tol{w.tol:g}"
    ex = "_".join(f"{k}{v}" for k, v in sorted(w.extra.items()))
    return os.path.join(root, f"{tag}_{ex}_b{BUILDER_VERSION}.plan")


def ensure_plan(w: mi.Workload, workers=None, log=print, root=None, builder="cpu", device="cuda") -> str:
    """Build the plan unless a complete file for this workload already exists
    (a cache only; a fresh box always rebuilds)."""
    p = plan_cache_path(w, root)
    if not os.path.exists(p):
        build_workload_plan(w, p, workers=workers, log=log, builder=builder, device=device)
    return p


__all__ = ["flat_workload", "sphere_workload", "setup", "build_workload_plan", "ensure_plan",
           "plan_cache_path", "DenseBasis", "dataclasses", "np"]
