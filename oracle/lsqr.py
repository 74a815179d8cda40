"""ORACLE — TEST INFRASTRUCTURE ONLY (see oracle/__init__.py for the rules).

LSQR for the inverse MHT  c = argmin ||Phi c - b||_2  (§7.1,
Eq. (inverse-MHT): "we use the BF-MHT within the LSQR iterative
least squares algorithm [Paige & Saunders 1982]").  The paper
gives no algorithm of its own; this is Paige & Saunders' LSQR (Golub-Kahan
bidiagonalisation + Givens QR of the bidiagonal, no damping) written out step
by step in plain numpy, one right-hand side at a time, with the operator
passed in as two callables (the oracle's O2 apply / adjoint, or a dense
matrix).  Pinned in tests/test_oracle_lsqr.py against scipy.sparse.linalg.lsqr
iterate by iterate and against numpy.linalg.lstsq at convergence.
"""
from __future__ import annotations

import math

import numpy as np


def lsqr(matvec, rmatvec, b, iters: int):
    """``iters`` LSQR iterations from x0 = 0 for one right-hand side b.

    Returns (x, rnorm, arnorm, anorm): the iterate and Paige & Saunders'
    running estimates of ||b - A x||, ||A^*(b - A x)|| and ||A||_F."""
    b = np.asarray(b)
    beta = float(np.linalg.norm(b))
    u = b / beta if beta > 0 else b.copy()
    v = rmatvec(u)
    x = np.zeros_like(v)
    alpha = float(np.linalg.norm(v))
    if alpha > 0:
        v = v / alpha
    w = v.copy()
    phibar, rhobar = beta, alpha
    anorm2 = 0.0
    c = 1.0
    for _ in range(iters):
        # bidiagonalisation:  beta u = A v - alpha u,   alpha v = A^* u - beta v
        u = matvec(v) - alpha * u
        beta = float(np.linalg.norm(u))
        if beta > 0:
            u = u / beta
        anorm2 += alpha * alpha + beta * beta
        v = rmatvec(u) - beta * v
        alpha = float(np.linalg.norm(v))
        if alpha > 0:
            v = v / alpha
        # plane rotation eliminating the subdiagonal beta
        rho = math.hypot(rhobar, beta)
        c = rhobar / rho if rho > 0 else 1.0
        s = beta / rho if rho > 0 else 0.0
        theta = s * alpha
        rhobar = -c * alpha
        phi = c * phibar
        phibar = s * phibar
        # solution and search direction updates
        if rho > 0:
            x = x + (phi / rho) * w
            w = v - (theta / rho) * w
    return x, phibar, phibar * alpha * abs(c), math.sqrt(anorm2)


def lsqr_block(matvec, rmatvec, B, iters: int):
    """Column-by-column LSQR for B of shape (nrhs, n) (ABI layout); the
    operators act on single vectors.  Returns X (nrhs, m) and per-column
    (rnorm, arnorm)."""
    B = np.atleast_2d(B)
    xs, rn, an = [], [], []
    for r in range(B.shape[0]):
        x, rnorm, arnorm, _ = lsqr(matvec, rmatvec, B[r], iters)
        xs.append(x)
        rn.append(rnorm)
        an.append(arnorm)
    return np.stack(xs), np.array(rn), np.array(an)
