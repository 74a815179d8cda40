"""Builder-side evaluators of blocks Phi(tau, nu) (host precompute, not timed).

Independent of ``oracle/`` (which has its own C evaluators); both take their
geometry and mode lists from ``mht_inputs``.

* FlatBasis:   Phi_jk = exp(i k.x_j)  (§1 Eq. 2D-DFT)
* SphereBasis: real orthonormal spherical harmonics (reading A11), evaluated
  per point set by the normalised associated-Legendre recurrence, vectorised
  over (points x m) with a Python loop over l.
* DenseBasis:  stored Phi (meshes).
"""
from __future__ import annotations

import numpy as np


class FlatBasis:
    dtype = np.complex128

    def __init__(self, x, k):
        self.x = np.ascontiguousarray(x, dtype=np.float64)
        self.k = np.ascontiguousarray(k, dtype=np.float64)
        self.n, self.m = self.x.shape[0], self.k.shape[0]

    def block(self, rows, cols):
        ph = self.x[rows] @ self.k[cols].T
        return np.exp(1j * ph)


def _legendre_table(lmax, theta):
    """P[l][m] arrays: fully normalised assoc. Legendre (no Condon-Shortley),
    returned as array (lmax+1, lmax+1, npts) with zeros for m > l."""
    x = np.cos(theta)
    s = np.sin(theta)
    npts = theta.shape[0]
    P = np.zeros((lmax + 1, lmax + 1, npts))
    P[0, 0] = 1.0 / np.sqrt(4.0 * np.pi)
    for m in range(1, lmax + 1):
        P[m, m] = np.sqrt((2.0 * m + 1.0) / (2.0 * m)) * s * P[m - 1, m - 1]
    mm = np.arange(lmax + 1, dtype=np.float64)
    for l in range(1, lmax + 1):
        # m = l - 1 diagonal-adjacent term
        P[l, l - 1] = np.sqrt(2.0 * (l - 1) + 3.0) * x * P[l - 1, l - 1]
        if l >= 2:
            m = mm[: l - 1]
            a = np.sqrt((4.0 * l * l - 1.0) / (l * l - m * m))
            b = np.sqrt(((l - 1.0) ** 2 - m * m) / (4.0 * (l - 1.0) ** 2 - 1.0))
            P[l, : l - 1] = a[:, None] * (x[None, :] * P[l - 1, : l - 1] - b[:, None] * P[l - 2, : l - 1])
    return P


class SphereBasis:
    dtype = np.float64

    def __init__(self, theta, phi, lmax, cache_rows: int = 0):
        self.theta = np.asarray(theta, dtype=np.float64)
        self.phi = np.asarray(phi, dtype=np.float64)
        self.lmax = int(lmax)
        self.n = self.theta.shape[0]
        self.m = (lmax + 1) ** 2
        ls = np.repeat(np.arange(lmax + 1), 2 * np.arange(lmax + 1) + 1)
        self.mode_l = ls
        self.mode_m = np.arange(self.m) - ls * ls - ls
        self._cache = None

    def rows_all(self, rows):
        """Y(rows, :) for all modes, (len(rows), m)."""
        th = self.theta[rows]
        ph = self.phi[rows]
        P = _legendre_table(self.lmax, th)          # (l, m>=0, pts)
        am = np.abs(self.mode_m)
        val = P[self.mode_l, am, :].T                 # (pts, modes)
        scale = np.where(self.mode_m == 0, 1.0, np.sqrt(2.0))
        mph = np.outer(ph, am.astype(np.float64))
        trig = np.where(self.mode_m[None, :] >= 0, np.cos(mph), np.sin(mph))
        return val * scale[None, :] * trig

    def block(self, rows, cols):
        if self._cache is not None:
            return self._cache[np.asarray(rows)][:, cols]
        return self.rows_all(rows)[:, cols]

    def precompute_all(self, chunk=2048):
        Y = np.empty((self.n, self.m))
        for s in range(0, self.n, chunk):
            Y[s:s + chunk] = self.rows_all(np.arange(s, min(self.n, s + chunk)))
        self._cache = Y
        return Y


class DenseBasis:
    def __init__(self, Phi):
        self.Phi = np.asarray(Phi)
        self.dtype = self.Phi.dtype
        self.n, self.m = self.Phi.shape

    def block(self, rows, cols):
        return self.Phi[np.ix_(np.asarray(rows), np.asarray(cols))]
