"""Pins for the oracle's O2 (independent CPU butterfly apply/adjoint).

O2 is checked against O1 (itself pinned by FFTs, closed forms and brute force):
an (numerically) exact full-rank plan must reproduce the dense sum to ~1e-13,
an eps-plan must agree with it to <= 10 eps, and
the factored form must satisfy the adjoint identity, linearity and the exact
zero/rank-1/rank-0 special cases.
"""
import numpy as np
import pytest

import mht_inputs as mi
from paper_2605_21828_b200 import workloads as W
from paper_2605_21828_b200.precompute import build_plan, freq_tree, kd_tree
from paper_2605_21828_b200.precompute.basis import DenseBasis
from paper_2605_21828_b200.precompute.planfile import PlanView


def rel(a, b):
    return np.linalg.norm(a - b) / np.linalg.norm(b)


def flat_plan(tmp, n, side, L, tol, m=None, name="f"):
    w = W.flat_workload(n, side, L, tol, name=name)
    if m is not None:
        w = mi.Workload(name, "flat", n, m, "complex128", tol, L, (1,), {"side": side})
    path = str(tmp / f"{name}_{n}_{side}_{L}_{tol:g}_{w.m}.plan")
    W.build_workload_plan(w, path, workers=2, log=None)
    x = mi.flat_points(n)
    k = mi.flat_modes(side)[: w.m]
    return path, x, k, w


@pytest.mark.parametrize("n,side,L", [(64, 8, 1), (256, 16, 2), (1024, 32, 4)])
def test_full_rank_plan_equals_dense(oracle_lib, tmp_plans, n, side, L):
    """tol ~ 0: every ID is exact, so BF c == Phi c to rounding."""
    path, x, k, w = flat_plan(tmp_plans, n, side, L, 1e-15)
    P = oracle_lib.Plan(path)
    assert P.validate() == 0
    c = mi.complex_gaussian(2, w.m, 1)
    assert rel(P.apply(c), oracle_lib.flat_synth(x, k, c)) < 1e-12
    y = mi.complex_gaussian(2, n, 2)
    assert rel(P.adjoint(y), oracle_lib.flat_analysis(x, k, y)) < 1e-12


@pytest.mark.parametrize("tol", [1e-4, 1e-6, 1e-8])
def test_eps_plan_within_10_eps_of_dense(oracle_lib, tmp_plans, tol):
    path, x, k, w = flat_plan(tmp_plans, 2048, 32, 4, tol)
    P = oracle_lib.Plan(path)
    c = mi.complex_gaussian(3, w.m, 1)
    f, fd = P.apply(c), oracle_lib.flat_synth(x, k, c)
    for r in range(3):
        assert rel(f[r], fd[r]) <= 10 * tol
    y = mi.complex_gaussian(3, w.n, 2)
    ca, cd = P.adjoint(y), oracle_lib.flat_analysis(x, k, y)
    for r in range(3):
        assert rel(ca[r], cd[r]) <= 10 * tol
    # compression happened at the looser tolerances
    if tol >= 1e-6:
        assert P.entries() < w.n * w.m


def test_adjoint_identity_linearity_zero(oracle_lib, tmp_plans):
    path, x, k, w = flat_plan(tmp_plans, 2048, 32, 4, 1e-6)
    P = oracle_lib.Plan(path)
    c = mi.complex_gaussian(2, w.m, 5)
    y = mi.complex_gaussian(2, w.n, 6)
    f = P.apply(c)
    ca = P.adjoint(y)
    for r in range(2):
        lhs, rhs = np.vdot(y[r], f[r]), np.vdot(ca[r], c[r])
        assert abs(lhs - rhs) <= 1e-12 * np.linalg.norm(y[r]) * np.linalg.norm(c[r]) * w.n
    a, b = 0.3 - 1.1j, 2.0 + 0.5j
    lin = P.apply(a * c[0] + b * c[1])[0]
    assert rel(lin, a * f[0] + b * f[1]) < 1e-12
    assert np.all(P.apply(np.zeros(w.m, complex)) == 0)
    assert np.all(P.adjoint(np.zeros(w.n, complex)) == 0)


def test_uneven_leaves_and_partial_mode_list(oracle_lib, tmp_plans):
    """n and m not multiples of 2^L: ragged leaves on both trees."""
    path, x, k, w = flat_plan(tmp_plans, 1000, 32, 4, 1e-9, m=1000, name="ragged")
    P = oracle_lib.Plan(path)
    V = PlanView(path)
    assert len(set(np.diff(V.sp_off))) > 1 and len(set(np.diff(V.fr_off))) > 1
    c = mi.complex_gaussian(1, 1000, 1)
    assert rel(P.apply(c), oracle_lib.flat_synth(x, k, c)) < 1e-7


def test_L0_plan_is_dense_product(oracle_lib, tmp_plans):
    path, x, k, w = flat_plan(tmp_plans, 64, 8, 0, 1e-12)
    P = oracle_lib.Plan(path)
    c = mi.complex_gaussian(1, 64, 1)
    assert rel(P.apply(c), oracle_lib.flat_synth(x, k, c)) < 1e-12


def test_sphere_plan(oracle_lib, tmp_plans):
    lmax = 23
    w = W.sphere_workload(1024, lmax, 3, 1e-10)
    path = str(tmp_plans / "sph.plan")
    W.build_workload_plan(w, path, workers=2, log=None)
    th, ph, _ = mi.sphere_points(1024)
    P = oracle_lib.Plan(path)
    assert P.dtype == np.float64
    c = mi.sphere_coefficients(2, lmax)
    f, fd = P.apply(c), oracle_lib.sphere_synth(th, ph, lmax, c)
    assert rel(f, fd) <= 1e-9
    y = mi.real_gaussian(2, 1024, 2)
    assert rel(P.adjoint(y), oracle_lib.sphere_analysis(th, ph, lmax, y)) <= 1e-9


def _dense_plan(tmp, Phi, L, tol, name):
    n, m = Phi.shape
    rng = np.random.default_rng(0)
    pts = rng.uniform(size=(n, 2))
    perm, sp_off = kd_tree(pts, L)
    path = str(tmp / f"{name}.plan")
    build_plan(DenseBasis(Phi), perm, sp_off, freq_tree(m, L), L, tol, path, workers=1, log=None)
    return path


def test_rank_one_and_zero_matrices(oracle_lib, tmp_plans):
    """Rank-1 Phi gives every non-identity block rank 1; Phi = 0 gives rank 0
    and BF c == 0 exactly."""
    rng = np.random.default_rng(3)
    u, v = rng.standard_normal(256), rng.standard_normal(256)
    path = _dense_plan(tmp_plans, np.outer(u, v), 2, 1e-12, "rank1")
    V = PlanView(path)
    for s in range(1, V.L + 1):
        assert np.all(V.stages[s].blocks["r_out"] == 1)
    P = oracle_lib.Plan(path)
    c = rng.standard_normal((1, 256))
    assert rel(P.apply(c)[0], u * (v @ c[0])) < 1e-12
    path0 = _dense_plan(tmp_plans, np.zeros((256, 256)), 2, 1e-12, "rank0")
    V0 = PlanView(path0)
    assert np.all(V0.stages[1].blocks["r_out"] == 0)
    P0 = oracle_lib.Plan(path0)
    assert np.all(P0.apply(c) == 0)
    assert np.all(P0.adjoint(rng.standard_normal((1, 256))) == 0)


def test_plan_invariants_and_checksum(oracle_lib, tmp_plans):
    path, x, k, w = flat_plan(tmp_plans, 2048, 32, 4, 1e-6)
    V = PlanView(path)
    assert V.verify_checksum()
    assert V.entries == oracle_lib.Plan(path).entries()
    assert V.entries <= w.n * w.m
    # chain invariant r_in = r_out(p, c1) + r_out(p, c2)
    nl = 1 << V.L
    for s in range(1, V.L + 1):
        nf, nfp = nl >> s, nl >> (s - 1)
        prev = V.stages[s - 1].blocks["r_out"]
        for b in range(nl):
            t, v = divmod(b, nf)
            p = t >> 1
            assert V.stages[s].blocks["r_in"][b] == prev[p * nfp + 2 * v] + prev[p * nfp + 2 * v + 1]
    # a corrupted byte is caught by the oracle's reader
    bad = str(tmp_plans / "bad.plan")
    raw = bytearray(open(path, "rb").read())
    raw[-100] ^= 0xFF
    open(bad, "wb").write(raw)
    with pytest.raises(ValueError):
        oracle_lib.Plan(bad)
