"""Pins for the oracle's LSQR (oracle/lsqr.py), the reference for the inverse
MHT of PAPER.md §7.1 (Eq. inverse-MHT).

* iterate by iterate against scipy.sparse.linalg.lsqr (the library routine of
  the same algorithm, atol = btol = 0 so both run exactly k steps);
* at convergence against numpy.linalg.lstsq (the least-squares solution by
  its plain definition), real and complex;
* with the operator given by the oracle's O2 butterfly on a full-rank plan,
  the converged LSQR solution solves the dense least-squares problem.
"""
import numpy as np
import pytest
import scipy.sparse.linalg as spla

import mht_inputs as mi
from paper_2605_21828_b200 import workloads as W

pytestmark = pytest.mark.filterwarnings("ignore")


def _ops(A):
    return (lambda v: A @ v), (lambda u: A.conj().T @ u)


@pytest.mark.parametrize("cplx", [False, True])
@pytest.mark.parametrize("k", [1, 2, 5, 17])
def test_lsqr_matches_scipy_iterates(cplx, k):
    from oracle.lsqr import lsqr

    rng = np.random.default_rng(3 + k)
    A = rng.standard_normal((80, 30))
    b = rng.standard_normal(80)
    if cplx:
        A = A + 1j * rng.standard_normal((80, 30))
        b = b + 1j * rng.standard_normal(80)
    x, rnorm, arnorm, _ = lsqr(*_ops(A), b, k)
    ref = spla.lsqr(A, b, atol=0.0, btol=0.0, conlim=0.0, iter_lim=k)
    assert np.linalg.norm(x - ref[0]) <= 1e-12 * np.linalg.norm(ref[0])
    assert abs(rnorm - ref[3]) <= 1e-10 * ref[3]
    # the residual estimate is the true residual (exact arithmetic identity)
    assert abs(rnorm - np.linalg.norm(b - A @ x)) <= 1e-10 * np.linalg.norm(b)


@pytest.mark.parametrize("cplx", [False, True])
def test_lsqr_converges_to_lstsq(cplx):
    from oracle.lsqr import lsqr_block

    rng = np.random.default_rng(11)
    A = rng.standard_normal((120, 40))
    B = rng.standard_normal((3, 120))
    if cplx:
        A = A + 1j * rng.standard_normal((120, 40))
        B = B + 1j * rng.standard_normal((3, 120))
    X, rn, an = lsqr_block(*_ops(A), B, 120)
    Xs = np.linalg.lstsq(A, B.T, rcond=None)[0].T
    assert np.linalg.norm(X - Xs) <= 1e-10 * np.linalg.norm(Xs)
    # normal equations A^*(b - A x) = 0 at the solution
    assert np.linalg.norm(A.conj().T @ (B.T - A @ X.T)) <= 1e-9 * np.linalg.norm(A) * np.linalg.norm(B)
    assert np.all(an <= 1e-8 * np.linalg.norm(A) * rn + 1e-12)


def test_lsqr_with_o2_operator_solves_dense_problem(oracle_lib, tmp_plans):
    """Tall flat problem (n = 1024 points, m = 256 modes) on a full-rank plan:
    LSQR driven by O2 recovers the dense least-squares solution."""
    from oracle.lsqr import lsqr_block

    w = W.flat_workload(1024, 16, 2, 1e-15, name="lsqr_tall")
    path = str(tmp_plans / "lsqr_tall.plan")
    W.build_workload_plan(w, path, workers=2, log=None)
    O = oracle_lib.Plan(path)
    x = mi.flat_points(w.n)
    k = mi.flat_modes(16)
    Phi = np.exp(1j * (x @ k.T.astype(float)))
    B = mi.complex_gaussian(2, w.n, 5)
    X, _, _ = lsqr_block(lambda v: O.apply(v[None, :])[0], lambda u: O.adjoint(u[None, :])[0], B, 60)
    Xs = np.linalg.lstsq(Phi, B.T, rcond=None)[0].T
    assert np.linalg.norm(X - Xs) <= 1e-9 * np.linalg.norm(Xs)
