"""Column interpolative decomposition (host precompute).

PAPER.md P:236-239 (§2) leaves the low-rank primitive open ("SVD, QR,
interpolative decomposition"); P:333-336 mentions randomized subsampling.
Reading A5: column ID by (optionally sketched) column-pivoted
QR; rank k = first i with |R_ii| <= eps |R_00|; T = R11^{-1} R12.

    A(:, red) ~= A(:, skel) T,   i.e.  A ~= A(:, skel) [I T] Pi.

For tall blocks (rows >> cols) the pivoting runs on a Gaussian sketch
Y = G A with cols + 16 rows (Halko–Martinsson–Tropp style), otherwise on A.
"""
from __future__ import annotations

import numpy as np
import scipy.linalg as sl

OVERSAMPLE = 16


def column_id(A: np.ndarray, tol: float, seed: int = 0):
    """Return (k, skel, red, T) with A(:, red) ~= A(:, skel) @ T (T is k x (c-k)).

    k == c means full column rank (the caller emits an IDENTITY block)."""
    r, c = A.shape
    if c == 0:
        return 0, np.zeros(0, np.int64), np.zeros(0, np.int64), np.zeros((0, 0), A.dtype)
    Y = A
    if r > 2 * (c + OVERSAMPLE):
        rng = np.random.default_rng(seed)
        if np.iscomplexobj(A):
            G = (rng.standard_normal((c + OVERSAMPLE, r)) + 1j * rng.standard_normal((c + OVERSAMPLE, r)))
        else:
            G = rng.standard_normal((c + OVERSAMPLE, r))
        Y = G @ A
    R, P = sl.qr(Y, mode="r", pivoting=True, check_finite=False)
    d = np.abs(np.diag(R))
    if d.size == 0 or d[0] == 0.0:
        return 0, np.zeros(0, np.int64), np.arange(c), np.zeros((0, c), A.dtype)
    small = np.nonzero(d <= tol * d[0])[0]
    k = int(small[0]) if small.size else int(d.size)
    if k == c:
        return c, np.arange(c), np.zeros(0, np.int64), np.zeros((c, 0), A.dtype)
    T = sl.solve_triangular(R[:k, :k], R[:k, k:], check_finite=False)
    return k, P[:k].astype(np.int64), P[k:].astype(np.int64), T
