"""Pins for the configs[3] inputs (torus mesh, cotangent FEM, eigenbasis) and the
Fiedler tree.  Closed forms: the cotangent stiffness of a regular right-
triangle grid is the 5-point Laplacian stencil with lumped mass h^2; the
torus area is 4 pi^2 R r; eigen-residual, M-orthonormality, the constant
null vector and Weyl's law N(lambda) ~ A lambda / (4 pi) (reading A4)."""
import numpy as np
import pytest

from mht_inputs import mesh as mm
from paper_2605_21828_b200.precompute.fiedler import fiedler_tree


def test_cotan_is_five_point_stencil_on_regular_grid():
    N, h = 8, 0.25
    g = np.arange(N) * h
    X, Y = np.meshgrid(g, g, indexing="ij")
    V = np.stack([X.ravel(), Y.ravel(), np.zeros(N * N)], 1)
    idx = lambda i, j: i * N + j
    F = []
    for i in range(N - 1):
        for j in range(N - 1):
            a, b, c, d = idx(i, j), idx(i + 1, j), idx(i + 1, j + 1), idx(i, j + 1)
            F += [(a, b, c), (a, c, d)]
    K, mass = mm.cotan_fem(V, np.array(F))
    Kd = K.toarray()
    i = idx(3, 4)
    assert Kd[i, i] == pytest.approx(4.0, abs=1e-12)
    for nb in (idx(2, 4), idx(4, 4), idx(3, 3), idx(3, 5)):
        assert Kd[i, nb] == pytest.approx(-1.0, abs=1e-12)
    assert abs(Kd[i, idx(4, 5)]) < 1e-12 and abs(Kd[i, idx(2, 3)]) < 1e-12  # diagonal edges: cot 90 = 0
    assert mass[i] == pytest.approx(h * h, rel=1e-12)
    assert np.abs(Kd.sum(1)).max() < 1e-12


def test_torus_mesh_area_and_topology():
    V, F = mm.torus_mesh(64, 32, sigma=0.0)
    assert V.shape == (2048, 3) and F.shape == (4096, 3)
    E = {tuple(sorted(e)) for f in F for e in ((f[0], f[1]), (f[1], f[2]), (f[2], f[0]))}
    assert V.shape[0] - len(E) + F.shape[0] == 0        # genus 1
    # polyhedral area -> 4 pi^2 R r at second order in the mesh size
    errs = []
    for nu, nv in ((64, 32), (128, 64)):
        Vr, Fr = mm.torus_mesh(nu, nv, sigma=0.0)
        errs.append(abs(mm.cotan_fem(Vr, Fr)[1].sum() / (8 * np.pi ** 2) - 1))
    assert errs[1] < 1e-3 and 3.5 < errs[0] / errs[1] < 4.5


def test_eigenbasis_properties():
    V, F = mm.torus_mesh(32, 16, sigma=0.01)
    lam, Phi, mass, K = mm.mesh_eigenbasis(V, F, 200)
    assert np.abs(Phi.T @ (mass[:, None] * Phi) - np.eye(200)).max() < 1e-10
    res = K @ Phi - mass[:, None] * Phi * lam[None, :]
    assert np.linalg.norm(res) <= 1e-10 * np.linalg.norm(K.toarray()) * np.linalg.norm(Phi)
    assert abs(lam[0]) < 1e-10 and np.ptp(Phi[:, 0]) < 1e-10
    assert np.all(np.diff(lam) >= -1e-12)
    j = np.argmax(np.abs(Phi), 0)
    assert np.all(Phi[j, np.arange(200)] > 0)  # sign convention
    # Weyl: N(lambda) ~ A lambda / (4 pi) within O(sqrt(lambda)) at low frequencies
    A = mass.sum()
    lam_k = lam[100]
    assert abs(101 - A * lam_k / (4 * np.pi)) < 4 * np.sqrt(A * lam_k / (4 * np.pi)) + 10


def test_fiedler_tree_partitions_and_balances():
    V, F = mm.torus_mesh(32, 16, sigma=0.01)
    perm, sp_off = fiedler_tree(V, F, 3)
    assert np.array_equal(np.sort(perm), np.arange(V.shape[0]))
    sizes = np.diff(sp_off)
    assert sizes.size == 8 and sizes.min() > 0.5 * sizes.mean()
    # every leaf is a connected patch of the mesh
    import scipy.sparse as sp
    import scipy.sparse.csgraph as csg

    for t in range(8):
        idx = perm[sp_off[t]:sp_off[t + 1]]
        loc = -np.ones(V.shape[0], int)
        loc[idx] = np.arange(idx.size)
        Fs = loc[F[np.all(loc[F] >= 0, 1)]]
        G = sp.coo_matrix((np.ones(3 * len(Fs)), (Fs.ravel(), np.roll(Fs, 1, 1).ravel())), shape=(idx.size,) * 2)
        assert csg.connected_components(G, directed=False)[0] == 1


def test_chebyshev_subspace_eigs_match_dense():
    """The sparse Chebyshev-filtered subspace solver (used for configs[3] on a
    GPU) reproduces the dense eigh: same eigenvalues, residual and
    M-orthonormality at the same bars, on a 48 x 24 noisy torus (CPU)."""
    V, F = mm.torus_mesh(48, 24, sigma=0.01)
    lam_d, Phi_d, mass, K = mm.mesh_eigenbasis(V, F, 160, method="dense")
    lam_c, Phi_c, _, _ = mm.mesh_eigenbasis(V, F, 160, method="chebyshev")
    assert np.abs(lam_c - lam_d).max() <= 1e-9 * max(1.0, lam_d.max())
    assert np.abs(Phi_c.T @ (mass[:, None] * Phi_c) - np.eye(160)).max() < 1e-10
    res = K @ Phi_c - mass[:, None] * Phi_c * lam_c[None, :]
    assert np.linalg.norm(res) <= 1e-10 * np.linalg.norm(K.toarray()) * np.linalg.norm(Phi_c)
    # same invariant subspaces: for non-degenerate eigenvalues the vectors agree (signs fixed)
    gaps = np.minimum(np.diff(lam_d, prepend=-1e9), np.diff(lam_d, append=1e9))
    iso = np.where(gaps > 1e-6 * max(1.0, lam_d.max()))[0]
    assert iso.size > 20
    assert np.abs(Phi_c[:, iso] - Phi_d[:, iso]).max() < 1e-7
