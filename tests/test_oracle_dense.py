"""Pins for the oracle's O1 dense sums (CPU, -m "not gpu").

Each test checks the oracle against something other than itself: a library FFT
on a uniform grid, closed forms (addition theorem, Y_00), exact Gauss-Legendre
quadrature orthonormality, scipy's spherical harmonics, and brute-force
Python loops at n = m = 64 (SURVEY.md §8(c) "Pins").
"""
import cmath
import math

import numpy as np
import pytest
import scipy.special as sps

import mht_inputs as mi


def rel(a, b):
    return np.linalg.norm(a - b) / np.linalg.norm(b)


# ---------------------------------------------------------------- flat -----
@pytest.mark.parametrize("N", [16, 64])
def test_flat_synth_equals_fft_on_uniform_grid(oracle_lib, N):
    """PAPER.md P:53-64 (Eq. 2D-DFT): on x = -pi + 2 pi j / N with all N^2 modes,
    f = N^2 ifft2(C), C[k mod N] = c_k (-1)^(k1+k2)."""
    x = mi.grid_points(N)
    k = mi.flat_modes(N)
    c = mi.complex_gaussian(2, N * N, 1)
    f = oracle_lib.flat_synth(x, k, c)
    C = np.zeros((2, N, N), complex)
    C[:, k[:, 0] % N, k[:, 1] % N] = c * ((-1.0) ** (k[:, 0] + k[:, 1]))
    F = (N * N * np.fft.ifft2(C)).reshape(2, -1)
    assert rel(f, F) < 1e-12


@pytest.mark.parametrize("N", [16, 64])
def test_flat_analysis_equals_fft_on_uniform_grid(oracle_lib, N):
    x = mi.grid_points(N)
    k = mi.flat_modes(N)
    f = mi.complex_gaussian(3, N * N, 2)
    c = oracle_lib.flat_analysis(x, k, f)
    Fh = np.fft.fft2(f.reshape(3, N, N))
    ref = Fh[:, k[:, 0] % N, k[:, 1] % N] * ((-1.0) ** (k[:, 0] + k[:, 1]))
    assert rel(c, ref) < 1e-12


def test_flat_synth_equals_fft_at_c2_mode_box(oracle_lib):
    """SURVEY §8(c) pin at N = 256: the whole [-128, 127]^2 mode box of
    configs[1] (65,536 modes) on the 256 x 256 uniform grid, against numpy's
    FFT on 512 seeded grid points (the dense sum over every mode for each;
    the row subset keeps the CPU suite fast), synthesis and analysis."""
    N = 256
    x = mi.grid_points(N)
    k = mi.flat_modes(N)
    rows = np.sort(np.random.default_rng(11).choice(N * N, 512, replace=False))
    c = mi.complex_gaussian(1, N * N, 3)
    f = oracle_lib.flat_synth(x[rows], k, c)
    C = np.zeros((1, N, N), complex)
    C[:, k[:, 0] % N, k[:, 1] % N] = c * ((-1.0) ** (k[:, 0] + k[:, 1]))
    F = (N * N * np.fft.ifft2(C)).reshape(1, -1)[:, rows]
    assert rel(f, F) < 1e-12
    # analysis of f supported on the sampled points: sum over those rows only
    y = np.zeros((1, N * N), complex)
    y[:, rows] = mi.complex_gaussian(1, 512, 4)
    a = oracle_lib.flat_analysis(x[rows], k, y[:, rows])
    Fh = np.fft.fft2(y.reshape(1, N, N))
    ref = Fh[:, k[:, 0] % N, k[:, 1] % N] * ((-1.0) ** (k[:, 0] + k[:, 1]))
    assert rel(a, ref) < 1e-12


def test_flat_gram_is_N2_identity_on_alias_free_grid(oracle_lib):
    """Phi^* Phi = N^2 I on the alias-free grid."""
    N = 32
    x = mi.grid_points(N)
    k = mi.flat_modes(N)
    c = mi.complex_gaussian(1, N * N, 7)
    back = oracle_lib.flat_analysis(x, k, oracle_lib.flat_synth(x, k, c))
    assert rel(back, N * N * c) < 1e-12


def test_flat_unit_vector_gives_plane_wave(oracle_lib):
    """c = e_k -> f_j = exp(i k.x_j), |f_j| = 1."""
    x = mi.flat_points(200)
    k = mi.flat_modes(16)
    q = 77
    c = np.zeros((1, k.shape[0]), complex)
    c[0, q] = 1.0
    f = oracle_lib.flat_synth(x, k, c)[0]
    assert np.allclose(np.abs(f), 1.0, atol=1e-14)
    j = 5
    ref = cmath.exp(1j * (k[q, 0] * x[j, 0] + k[q, 1] * x[j, 1]))
    assert abs(f[j] - ref) < 1e-13


def test_flat_brute_force_64(oracle_lib):
    """n = m = 64, modes [-4,3]^2, Phi built entrywise with cmath."""
    x = mi.flat_points(64, seed=11)
    k = mi.flat_modes(8)
    Phi = np.array([[cmath.exp(1j * (int(kk[0]) * xx[0] + int(kk[1]) * xx[1])) for kk in k] for xx in x])
    c = mi.complex_gaussian(2, 64, 12)
    f = oracle_lib.flat_synth(x, k, c)
    fb = np.array([[sum(Phi[j, q] * c[r, q] for q in range(64)) for j in range(64)] for r in range(2)])
    assert rel(f, fb) < 1e-13
    y = mi.complex_gaussian(2, 64, 13)
    cb = np.array([[sum(Phi[j, q].conjugate() * y[r, j] for j in range(64)) for q in range(64)] for r in range(2)])
    assert rel(oracle_lib.flat_analysis(x, k, y), cb) < 1e-13


def test_flat_modes_order():
    """Ordering example m = 5 -> (0,0), (-1,0), (0,-1), (0,1), (1,0)."""
    k = mi.flat_modes(8)[:5]
    assert [tuple(v) for v in k] == [(0, 0), (-1, 0), (0, -1), (0, 1), (1, 0)]


# ---------------------------------------------------------------- sphere ---
def scipy_real_ylm(lmax, theta, phi):
    """Real orthonormal harmonics from scipy's complex Y_l^m (which carries the
    Condon-Shortley phase): ours = sqrt2 (-1)^m Re/Im Y_l^m (reading A11)."""
    cols = []
    for l in range(lmax + 1):
        for mm in range(-l, l + 1):
            a = abs(mm)
            Y = sps.sph_harm_y(l, a, theta, phi)
            if mm == 0:
                cols.append(Y.real)
            elif mm > 0:
                cols.append(math.sqrt(2.0) * (-1) ** a * Y.real)
            else:
                cols.append(math.sqrt(2.0) * (-1) ** a * Y.imag)
    return np.stack(cols, axis=1)


def test_sphere_matches_scipy(oracle_lib):
    th, ph, _ = mi.sphere_points(300, seed=3)
    Y = oracle_lib.sphere_matrix(th, ph, 20)
    Ys = scipy_real_ylm(20, th, ph)
    assert np.abs(Y - Ys).max() < 1e-12


def test_sphere_high_degree_matches_scipy(oracle_lib):
    """Stability of the recurrence up to l = 255 (all configs[2] modes)."""
    th, ph, _ = mi.sphere_points(64, seed=4)
    Y = oracle_lib.sphere_matrix(th, ph, 255)
    for (l, mm) in [(255, 0), (255, 7), (255, -200), (255, 255), (200, -3), (128, 64)]:
        a = abs(mm)
        Ys = sps.sph_harm_y(l, a, th, ph)
        ref = Ys.real if mm == 0 else math.sqrt(2) * (-1) ** a * (Ys.real if mm > 0 else Ys.imag)
        assert np.abs(Y[:, l * l + l + mm] - ref).max() < 1e-11, (l, mm)


def test_sphere_Y00(oracle_lib):
    th, ph, _ = mi.sphere_points(10)
    Y = oracle_lib.sphere_matrix(th, ph, 3)
    assert np.allclose(Y[:, 0], 1.0 / math.sqrt(4 * math.pi), atol=1e-15)


@pytest.mark.parametrize("l", [1, 5, 60, 255])
def test_sphere_addition_theorem(oracle_lib, l):
    """sum_m Y_lm(x) Y_lm(y) = (2l+1)/(4 pi) P_l(x.y)."""
    th, ph, p = mi.sphere_points(6, seed=9)
    Y = oracle_lib.sphere_matrix(th, ph, l)
    blk = Y[:, l * l: (l + 1) ** 2]
    G = blk @ blk.T
    Pl = sps.eval_legendre(l, np.clip(p @ p.T, -1, 1))
    assert np.abs(G - (2 * l + 1) / (4 * math.pi) * Pl).max() < 1e-10 * (2 * l + 1)


def test_sphere_quadrature_orthonormality(oracle_lib):
    """Gauss-Legendre(nlat) x uniform(nlon) quadrature: sum_j w_j Y_k Y_k' = delta."""
    lmax = 40
    th, ph, w = mi.gauss_legendre_grid(lmax + 1, 2 * lmax + 2)
    Y = oracle_lib.sphere_matrix(th, ph, lmax)
    G = Y.T @ (w[:, None] * Y)
    assert np.abs(G - np.eye(G.shape[0])).max() < 1e-12


def test_sphere_synth_analysis_quadrature_roundtrip(oracle_lib):
    """Phi^T W Phi c = c at lmax = 95 through the synth/analysis sums."""
    lmax = 95
    th, ph, w = mi.gauss_legendre_grid(lmax + 1, 2 * lmax + 2)
    c = mi.sphere_coefficients(1, lmax, seed=5)
    f = oracle_lib.sphere_synth(th, ph, lmax, c)
    back = oracle_lib.sphere_analysis(th, ph, lmax, f * w[None, :])
    assert rel(back, c) < 1e-12


def test_sphere_brute_force_64(oracle_lib):
    """n = m = 64, l <= 7: Phi from scipy, products by Python loops."""
    th, ph, _ = mi.sphere_points(64, seed=21)
    Phi = scipy_real_ylm(7, th, ph)
    c = mi.sphere_coefficients(2, 7, seed=22)
    fb = np.array([[sum(Phi[j, q] * c[r, q] for q in range(64)) for j in range(64)] for r in range(2)])
    assert rel(oracle_lib.sphere_synth(th, ph, 7, c), fb) < 1e-13
    y = mi.real_gaussian(2, 64, 23)
    cb = np.array([[sum(Phi[j, q] * y[r, j] for j in range(64)) for q in range(64)] for r in range(2)])
    assert rel(oracle_lib.sphere_analysis(th, ph, 7, y), cb) < 1e-13


# ---------------------------------------------------------------- dense ----
@pytest.mark.parametrize("cplx", [False, True])
def test_dense_brute_force(oracle_lib, cplx):
    rng = np.random.default_rng(0)
    n, m = 40, 24
    Phi = rng.standard_normal((n, m)) + (1j * rng.standard_normal((n, m)) if cplx else 0)
    c = rng.standard_normal((3, m)) + (1j * rng.standard_normal((3, m)) if cplx else 0)
    fb = np.array([[sum(Phi[j, q] * c[r, q] for q in range(m)) for j in range(n)] for r in range(3)])
    assert rel(oracle_lib.dense_synth(Phi, c), fb) < 1e-14
    y = rng.standard_normal((3, n)) + (1j * rng.standard_normal((3, n)) if cplx else 0)
    cb = np.array([[sum(np.conj(Phi[j, q]) * y[r, j] for j in range(n)) for q in range(m)] for r in range(3)])
    assert rel(oracle_lib.dense_analysis(Phi, y), cb) < 1e-14


def test_flat_adjoint_identity_random_points(oracle_lib):
    """<Phi c, y> = <c, Phi^* y> for the O1 sums at random points."""
    x = mi.flat_points(300)
    k = mi.flat_modes(16)
    c = mi.complex_gaussian(1, 256, 1)[0]
    y = mi.complex_gaussian(1, 300, 2)[0]
    lhs = np.vdot(y, oracle_lib.flat_synth(x, k, c)[0])
    rhs = np.vdot(oracle_lib.flat_analysis(x, k, y)[0], c)
    assert abs(lhs - rhs) < 1e-12 * abs(lhs) * 100
