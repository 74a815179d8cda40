"""Seeded synthetic input generators shared by the oracle and the GPU path.

This module is the ONLY code the oracle (``oracle/``) and the product package
(``paper_2605_21828_b200``) have in common.  It holds none of the method's
arithmetic: no basis evaluation, no tree, no factorization, no transform.  It
only draws points, coefficient vectors and adjoint inputs from fixed seeds and
lists the modes (the column order of Phi) that define each workload.

Recipes follow SURVEY.md §8(d) (reading A13):

* RNG: ``numpy.random.default_rng(seed)`` (PCG64).  Seeds: 0 for geometry
  (points, jitter, mesh noise), 1 for coefficients c (an (nrhs, m) array drawn
  in one call), 2 for adjoint inputs f (an (nrhs, n) array).
* complex Gaussian = (a + i b)/sqrt(2), a, b ~ N(0, 1).
* Flat periodic square [-pi, pi]^2 (Eq. (1) "2D-DFT"):
  modes k in [-s/2, s/2-1]^2 sorted by (k1^2 + k2^2, k1, k2) (reading A8 —
  eigenvalue order with lexicographic ties).
* Unit sphere (configs[2]): Fibonacci lattice z_j = 1 - (2j+1)/n,
  phi_j = j*pi*(3 - sqrt 5), each point rotated by an angle U[0, 0.1 d] in a
  uniformly random tangent direction, d = sqrt(4 pi / n).  Modes (l, m),
  l <= lmax, m = -l..l, index l^2 + l + m (reading A8).  c_lm ~ N(0, 1/(1+l))
  (variance, reading A13).

Arrays use the layouts of the C ABI (include/mht.h): coefficient blocks are
(nrhs, m) C-contiguous, i.e. column-major m x nrhs.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

SEED_GEOMETRY = 0
SEED_COEF = 1
SEED_ADJ = 2


# ----------------------------------------------------------------------------
# flat periodic square  (§1 Eq. "2D-DFT")
# ----------------------------------------------------------------------------
def flat_points(n: int, seed: int = SEED_GEOMETRY) -> np.ndarray:
    """n points i.i.d. uniform in [-pi, pi)^2, shape (n, 2) float64."""
    rng = np.random.default_rng(seed)
    return rng.uniform(-np.pi, np.pi, size=(n, 2))


def grid_points(N: int) -> np.ndarray:
    """Uniform N x N grid x = -pi + 2 pi j / N, row-major (j1 slow), (N*N, 2)."""
    g = -np.pi + 2.0 * np.pi * np.arange(N) / N
    x1, x2 = np.meshgrid(g, g, indexing="ij")
    return np.stack([x1.ravel(), x2.ravel()], axis=1)


def flat_modes(side: int) -> np.ndarray:
    """All integer modes k in [-side/2, side/2 - 1]^2, shape (side^2, 2) int64,
    sorted by (|k|^2, k1, k2) — eigenvalue order lambda = k1^2 + k2^2
    with lexicographic ties (reading A8)."""
    h = side // 2
    r = np.arange(-h, side - h, dtype=np.int64)
    k1, k2 = np.meshgrid(r, r, indexing="ij")
    k1 = k1.ravel()
    k2 = k2.ravel()
    order = np.lexsort((k2, k1, k1 * k1 + k2 * k2))
    return np.stack([k1[order], k2[order]], axis=1)


def flat_modes_kd(side: int, L: int) -> np.ndarray:
    """The modes of [-side/2, side/2 - 1]^2 (side a power of two) in the order of
    a 2-D kd tree over the FREQUENCY box (the quadtree-in-frequency variant,
    PAPER.md §5): depth d halves the current box along k1 (d even) or
    k2 (d odd) at its midpoint, so the nodes at even depths are exactly the
    quadtree's squares; 2^L leaves of side^2 / 2^L modes, each leaf in
    eigenvalue order (|k|^2, k1, k2) inside.  Returns (side^2, 2) int64."""
    s = int(round(math.log2(side)))
    assert 1 << s == side and 0 <= L <= 2 * s
    h = side // 2
    k = flat_modes(side)
    i1, i2 = k[:, 0] + h, k[:, 1] + h           # 0 .. side - 1
    leaf = np.zeros(k.shape[0], dtype=np.int64)
    for d in range(L):                          # bit d of the path: axis d % 2, split number d // 2
        bit = ((i1 if d % 2 == 0 else i2) >> (s - 1 - d // 2)) & 1
        leaf = (leaf << 1) | bit
    order = np.argsort(leaf, kind="stable")     # stable: eigenvalue order inside a leaf
    return k[order].copy()


def flat_workload_modes(w) -> np.ndarray:
    """The mode list of a flat workload in the user's c order: eigenvalue order
    (reading A7/A8).  (A quadtree-frequency plan factorizes in the kd order of
    flat_modes_kd and maps it back with its perm_k; the user's order is this one.)"""
    return flat_modes(w.extra["side"])[: w.m]


def flat_modes_first(m: int) -> np.ndarray:
    """The first m modes of Z^2 in eigenvalue order (for m not a square)."""
    side = 2 * int(math.ceil(math.sqrt(m) / 2.0 + 2))
    return flat_modes(side)[:m].copy()


# ----------------------------------------------------------------------------
# sphere
# ----------------------------------------------------------------------------
def sphere_points(n: int, seed: int = SEED_GEOMETRY, jitter: float = 0.1):
    """Jittered Fibonacci lattice on S^2.

    Returns (theta, phi, xyz): colatitude in [0, pi], longitude in (-pi, pi],
    and unit vectors (n, 3)."""
    j = np.arange(n, dtype=np.float64)
    z = 1.0 - (2.0 * j + 1.0) / n
    lon = j * np.pi * (3.0 - np.sqrt(5.0))
    rho = np.sqrt(np.maximum(0.0, 1.0 - z * z))
    p = np.stack([rho * np.cos(lon), rho * np.sin(lon), z], axis=1)
    if jitter > 0:
        rng = np.random.default_rng(seed)
        d = np.sqrt(4.0 * np.pi / n)
        ang = rng.uniform(0.0, jitter * d, size=n)
        psi = rng.uniform(0.0, 2.0 * np.pi, size=n)
        # orthonormal tangent frame (e_theta, e_phi) at each point
        th0 = np.arccos(np.clip(z, -1.0, 1.0))
        e_t = np.stack([np.cos(th0) * np.cos(lon), np.cos(th0) * np.sin(lon), -np.sin(th0)], axis=1)
        e_p = np.stack([-np.sin(lon), np.cos(lon), np.zeros(n)], axis=1)
        t = np.cos(psi)[:, None] * e_t + np.sin(psi)[:, None] * e_p
        p = np.cos(ang)[:, None] * p + np.sin(ang)[:, None] * t
        p /= np.linalg.norm(p, axis=1, keepdims=True)
    theta = np.arccos(np.clip(p[:, 2], -1.0, 1.0))
    phi = np.arctan2(p[:, 1], p[:, 0])
    return theta, phi, p


def sphere_modes(lmax: int) -> np.ndarray:
    """(l, m) pairs, l = 0..lmax, m = -l..l, in index order l^2 + l + m; int64 (M, 2)."""
    out = [(l, mm) for l in range(lmax + 1) for mm in range(-l, l + 1)]
    return np.asarray(out, dtype=np.int64)


def gauss_legendre_grid(nlat: int, nlon: int):
    """Quadrature grid on S^2: Gauss-Legendre in cos(theta) x uniform longitude.

    Returns (theta, phi, w) flattened, w summing to 4 pi.  Exact for products of
    spherical harmonics of total degree < min(2 nlat, nlon)."""
    xg, wg = np.polynomial.legendre.leggauss(nlat)
    th = np.arccos(xg)
    ph = -np.pi + 2.0 * np.pi * np.arange(nlon) / nlon
    T, P = np.meshgrid(th, ph, indexing="ij")
    W = np.repeat(wg[:, None], nlon, axis=1) * (2.0 * np.pi / nlon)
    return T.ravel(), P.ravel(), W.ravel()


# ----------------------------------------------------------------------------
# coefficient / data vectors
# ----------------------------------------------------------------------------
def complex_gaussian(nrhs: int, length: int, seed: int) -> np.ndarray:
    """(nrhs, length) complex128, entries (a + i b)/sqrt(2), drawn in one call."""
    rng = np.random.default_rng(seed)
    ab = rng.standard_normal((nrhs, length, 2))
    return ((ab[..., 0] + 1j * ab[..., 1]) / np.sqrt(2.0)).astype(np.complex128)


def real_gaussian(nrhs: int, length: int, seed: int, scale=None) -> np.ndarray:
    """(nrhs, length) float64 N(0, 1) (times ``scale`` per column if given)."""
    rng = np.random.default_rng(seed)
    v = rng.standard_normal((nrhs, length))
    if scale is not None:
        v = v * np.asarray(scale, dtype=np.float64)[None, :]
    return v


def sphere_coefficients(nrhs: int, lmax: int, seed: int = SEED_COEF) -> np.ndarray:
    """c_lm ~ N(0, 1/(1+l)) (variance; reading A13), (nrhs, (lmax+1)^2)."""
    l = sphere_modes(lmax)[:, 0].astype(np.float64)
    return real_gaussian(nrhs, len(l), seed, scale=1.0 / np.sqrt(1.0 + l))


# ----------------------------------------------------------------------------
# workload registry (BASELINE.json configs)
# ----------------------------------------------------------------------------
@dataclass(frozen=True)
class Workload:
    name: str
    family: str          # "flat" | "sphere" | "mesh"
    n: int
    m: int
    dtype: str           # "complex128" | "float64"
    tol: float
    L: int
    nrhs: tuple = (1,)
    extra: dict = field(default_factory=dict)


WORKLOADS = {
    # configs[0]: flat, n = m = 4096, k in [-32,31]^2, tol 1e-8, leaf 64
    "c1": Workload("c1", "flat", 4096, 4096, "complex128", 1e-8, 6, (1,), {"side": 64}),
    # configs[1]: flat, n = m = 65536, k in [-128,127]^2, tol 1e-8, nrhs 1 and 32
    "c2": Workload("c2", "flat", 65536, 65536, "complex128", 1e-8, 10, (1, 32), {"side": 256}),
    # configs[2]: sphere, n = m = 65536, l <= 255, tol 1e-10, nrhs 1 and 32
    "c3": Workload("c3", "sphere", 65536, 65536, "float64", 1e-10, 10, (1, 32), {"lmax": 255}),
    # configs[3]: torus mesh 256 x 128, m = 2048, tol 1e-8, nrhs 1 and 64
    "c4": Workload("c4", "mesh", 32768, 2048, "float64", 1e-8, 5, (1, 64), {"nu": 256, "nv": 128}),
    # configs[4]: flat, n = m = 2^20, k in [-512,511]^2, tol 1e-6, nrhs 1 and 16
    "c5": Workload("c5", "flat", 1 << 20, 1 << 20, "complex128", 1e-6, 14, (1, 16), {"side": 1024}),
    # configs[4] protocol: n = m = 2^18 on the box [-256,255]^2 at tol
    # 1e-6 probes to 285 GB (profiles/r02_probe_c5p18.json): it does not fit one B200.  The labelled
    # stand-in is the largest flat square that does: n = m = 2^17 points / modes, the 2^17 lowest
    # eigenvalues (|k| <= ~204, taken from the [-256,255]^2 box in eigenvalue order), tol 1e-6,
    # nrhs 1 and 16
    "c5p18": Workload("c5p18", "flat", 1 << 18, 1 << 18, "complex128", 1e-6, 12, (1, 16), {"side": 512}),
    "c5s": Workload("c5s", "flat", 1 << 17, 1 << 17, "complex128", 1e-6, 11, (1, 16), {"side": 512}),
    # the quadtree-in-frequency plan variant (§5; NEXT-3): configs[0] / [1]
    # with the frequency tree a 2-D kd tree over the frequency box instead of eigenvalue ranges
    "c1kd": Workload("c1kd", "flat", 4096, 4096, "complex128", 1e-8, 6, (1,), {"side": 64, "ftree": "kd"}),
    "c2kd": Workload("c2kd", "flat", 65536, 65536, "complex128", 1e-8, 10, (1, 32), {"side": 256, "ftree": "kd"}),
}


def workload_points(w: Workload):
    """Geometry of a workload: flat -> (n,2) array; sphere -> (theta, phi)."""
    if w.family == "flat":
        return flat_points(w.n)
    if w.family == "sphere":
        th, ph, _ = sphere_points(w.n)
        return th, ph
    raise ValueError("mesh geometry: use mht_inputs.mesh")


def workload_modes(w: Workload):
    if w.family == "flat":
        return flat_workload_modes(w)
    if w.family == "sphere":
        return sphere_modes(w.extra["lmax"])
    raise ValueError("mesh modes are eigen-indices 0..m-1")


def workload_coefficients(w: Workload, nrhs: int) -> np.ndarray:
    if w.family == "flat":
        return complex_gaussian(nrhs, w.m, SEED_COEF)
    if w.family == "sphere":
        return sphere_coefficients(nrhs, w.extra["lmax"], SEED_COEF)
    return real_gaussian(nrhs, w.m, SEED_COEF)


def workload_adjoint_input(w: Workload, nrhs: int) -> np.ndarray:
    if w.dtype == "complex128":
        return complex_gaussian(nrhs, w.n, SEED_ADJ)
    return real_gaussian(nrhs, w.n, SEED_ADJ)
