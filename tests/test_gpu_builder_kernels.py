"""NEXT-1: libmht's plan-construction kernels (include/mht_build.h)
on the B200, each against an independent reference — numpy's exp for the flat
blocks, scipy's spherical harmonics (and the pinned oracle evaluator) for the
sphere table, LAPACK's column-pivoted QR (geqp3) for the batched CPQR — and the
plans the device builder writes with them against the dense sum (O1) and,
through libmht, against the oracle butterfly (O2)."""
import numpy as np
import pytest
import scipy.linalg as sl
import torch

import mht_inputs as mi
from paper_2605_21828_b200.precompute import freq_tree, kd_tree
from paper_2605_21828_b200.precompute.basis import FlatBasis

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def dk():
    if not torch.cuda.is_available():
        pytest.fail("GPU test run without a GPU")
    from paper_2605_21828_b200 import _build
    from paper_2605_21828_b200.precompute import devkern

    _build.build()
    return devkern


def test_flat_blocks_kernel_matches_numpy(dk):
    """exp(i k.x) in-kernel vs numpy on the host, with zero padding."""
    x, k = mi.flat_points(300), mi.flat_modes(16)
    nb = FlatBasis(x, k)
    xd, kd = torch.as_tensor(x).cuda(), torch.as_tensor(k.astype(np.float64)).cuda()
    rows = torch.tensor([[3, 5, 7, -1], [0, 1, 2, 3], [299, 0, -1, -1]]).cuda()
    cols = torch.tensor([[1, 2, -1], [10, 11, 12], [255, -1, 0]]).cuda()
    At = dk.flat_blocks(xd, kd, rows, cols).cpu().numpy()
    assert At.shape == (3, 3, 4) and At.dtype == np.complex128
    assert np.abs(At[0, :2, :3] - nb.block([3, 5, 7], [1, 2]).T).max() < 1e-14
    assert np.all(At[0, 2] == 0) and np.all(At[0, :, 3] == 0)
    assert np.abs(At[1] - nb.block([0, 1, 2, 3], [10, 11, 12]).T).max() < 1e-14
    assert np.all(At[2, 1] == 0) and np.all(At[2, :, 2:] == 0)
    assert np.abs(At[2, 0, :2] - nb.block([299, 0], [255])[:, 0]).max() < 1e-14
    # a larger batch: |Phi| = 1 exactly up to rounding, against numpy entry by entry
    rng = np.random.default_rng(3)
    r = rng.integers(0, 300, (5, 200))
    c = rng.integers(0, 256, (5, 77))
    At = dk.flat_blocks(xd, kd, torch.as_tensor(r).cuda(), torch.as_tensor(c).cuda()).cpu().numpy()
    ref = np.exp(1j * np.einsum("bcd,brd->bcr", k[c].astype(np.float64), x[r]))
    assert np.abs(At - ref).max() < 1e-12
    assert np.abs(np.abs(At) - 1).max() < 1e-14


def test_sphere_table_kernel_matches_scipy_and_oracle(dk, oracle_lib):
    """Y_lm (reading A11) in-kernel vs scipy.special.sph_harm_y and the pinned
    oracle evaluator, up to l = 255."""
    from scipy.special import sph_harm_y

    th, ph, _ = mi.sphere_points(257, seed=5)
    for lmax in (0, 7, 63, 255):
        Y = dk.sphere_table(torch.as_tensor(th).cuda(), torch.as_tensor(ph).cuda(), lmax).cpu().numpy()
        assert np.abs(Y - oracle_lib.sphere_matrix(th, ph, lmax)).max() < 1e-12
    # scipy (complex, Condon-Shortley phase) -> real, no CS phase
    lmax = 255
    Y = dk.sphere_table(torch.as_tensor(th).cuda(), torch.as_tensor(ph).cuda(), lmax).cpu().numpy()
    for l in (0, 1, 17, 128, 255):
        for m in sorted({0, 1, l // 2, l}):
            if m > l:
                continue
            z = sph_harm_y(l, m, th, ph)
            cs = (-1.0) ** m
            if m == 0:
                ref_p, ref_n = z.real, None
            else:
                ref_p = np.sqrt(2.0) * cs * z.real
                ref_n = np.sqrt(2.0) * cs * z.imag
            assert np.abs(Y[:, l * l + l + m] - ref_p).max() < 1e-11, (l, m)
            if ref_n is not None:
                assert np.abs(Y[:, l * l + l - m] - ref_n).max() < 1e-11, (l, -m)


def _lowrank(rng, R, C, rank, cplx, noise=1e-13):
    U = rng.standard_normal((R, rank)) + (1j * rng.standard_normal((R, rank)) if cplx else 0)
    V = rng.standard_normal((rank, C)) + (1j * rng.standard_normal((rank, C)) if cplx else 0)
    return U @ V + noise * rng.standard_normal((R, C))


@pytest.mark.parametrize("cplx", [False, True])
def test_cpqr_kernel_matches_lapack(dk, cplx):
    """Full-rank blocks: the kernel's pivots equal LAPACK geqp3's and its R
    equals LAPACK's R up to a unit phase per row (|R| entrywise, 1e-12 of
    |R_00|); rank-deficient blocks: the rank rule of reading A5 and the ID
    property |A[:, red] - A[:, skel] T| <= 10 tol |A| with T = R11^-1 R12."""
    rng = np.random.default_rng(1)
    dt = np.complex128 if cplx else np.float64
    for (B, R, C) in ((3, 40, 60), (2, 200, 90), (4, 17, 17)):
        mats = [rng.standard_normal((R, C)) + (1j * rng.standard_normal((R, C)) if cplx else 0) for _ in range(B)]
        At = torch.as_tensor(np.stack([m.T for m in mats]).astype(dt)).cuda().contiguous()
        ranks, perm = dk.cpqr(At, 0.0)
        At, ranks, perm = At.cpu().numpy(), ranks.cpu().numpy(), perm.cpu().numpy()
        k = min(R, C)
        for b in range(B):
            assert ranks[b] == k
            Rl, Pl = sl.qr(mats[b], mode="r", pivoting=True)
            assert np.array_equal(perm[b][:k], Pl[:k]), b
            Rk = At[b].T[:k, :]  # R rows 0..k-1 over column positions
            assert np.abs(np.abs(np.triu(Rk)) - np.abs(Rl[:k, :])).max() <= 1e-12 * abs(Rl[0, 0])
            assert sorted(perm[b].tolist()) == list(range(C))
    # rank-deficient blocks (low rank + 1e-13 noise), tol 1e-10
    B, R, C, rank, tol = 3, 60, 80, 17, 1e-10
    mats = [_lowrank(rng, R, C, rank, cplx) for _ in range(B)]
    At = torch.as_tensor(np.stack([m.T for m in mats]).astype(dt)).cuda().contiguous()
    ranks, perm = dk.cpqr(At, tol)
    At, ranks, perm = At.cpu().numpy(), ranks.cpu().numpy(), perm.cpu().numpy()
    for b in range(B):
        assert ranks[b] == rank
        Rm = At[b].T
        R11, R12 = Rm[:rank, :rank], Rm[:rank, rank:]
        T = sl.solve_triangular(R11, R12)
        skel, red = perm[b][:rank], perm[b][rank:]
        A = mats[b]
        assert np.linalg.norm(A[:, red] - A[:, skel] @ T) <= 10 * tol * np.linalg.norm(A)


def test_cpqr_kernel_edge_cases(dk):
    """Zero block -> rank 0; zero padding columns are never pivoted ahead of
    non-zero ones; a block too tall for the Householder vector in shared memory
    (R = 16,000 complex: the global-scratch path) still matches LAPACK."""
    z = torch.zeros((2, 5, 7), dtype=torch.complex128, device="cuda")
    ranks, perm = dk.cpqr(z, 1e-8)
    assert ranks.cpu().tolist() == [0, 0]
    rng = np.random.default_rng(7)
    A = rng.standard_normal((30, 6))
    At = np.zeros((1, 10, 30))
    At[0, [0, 2, 4, 6, 8, 9]] = A.T                         # columns 1, 3, 5, 7 are zero padding
    t = torch.as_tensor(At).cuda()
    ranks, perm = dk.cpqr(t, 1e-12)
    assert int(ranks[0]) == 6
    assert set(perm[0, :6].cpu().tolist()) == {0, 2, 4, 6, 8, 9}
    R, C = 16000, 6
    M = rng.standard_normal((R, C)) + 1j * rng.standard_normal((R, C))
    t = torch.as_tensor(np.ascontiguousarray(M.T)[None]).cuda()
    ranks, perm = dk.cpqr(t, 0.0)
    Rl, Pl = sl.qr(M, mode="r", pivoting=True)
    assert int(ranks[0]) == C and np.array_equal(perm[0].cpu().numpy(), Pl)
    Rk = t[0].cpu().numpy().T[:C, :]
    assert np.abs(np.abs(np.triu(Rk)) - np.abs(Rl[:C, :])).max() <= 1e-12 * abs(Rl[0, 0])


@pytest.mark.parametrize("family", ["flat", "sphere", "mesh"])
def test_device_builder_plans(dk, oracle_lib, tmp_path, family):
    """Plans written by the device builder (kernels above): within 10 tol of
    the dense sum (O1) in the oracle's butterfly, and libmht on the same file
    equal to the oracle butterfly (O2) element by element (1e-12)."""
    from paper_2605_21828_b200 import mht
    from paper_2605_21828_b200.precompute.gpu_builder import (DeviceFlatBasis, DeviceTableBasis, build_plan_gpu,
                                                              sphere_table)

    L = 4
    if family == "flat":
        n, side, tol = 1024, 32, 1e-8
        x, k = mi.flat_points(n), mi.flat_modes(side)
        perm, sp = kd_tree(x, L)
        basis = DeviceFlatBasis(x, k, "cuda")
        m = side * side
        c = mi.complex_gaussian(2, m, 1)
        ref = oracle_lib.flat_synth(x, k, c)
    elif family == "sphere":
        n, lmax, tol = 1024, 31, 1e-10
        th, ph, p = mi.sphere_points(n)
        perm, sp = kd_tree(p, L, alternate=False)
        basis = DeviceTableBasis(sphere_table(th, ph, lmax, "cuda"), np.float64)
        m = (lmax + 1) ** 2
        c = mi.sphere_coefficients(2, lmax)
        ref = oracle_lib.sphere_synth(th, ph, lmax, c)
    else:
        from mht_inputs import mesh as mm
        from paper_2605_21828_b200.precompute.fiedler import fiedler_tree

        V, F = mm.torus_mesh(32, 16, sigma=0.01)
        lam, Phi, mass, _ = mm.mesh_eigenbasis(V, F, 256)
        L, tol, m = 2, 1e-8, 256
        perm, sp = fiedler_tree(V, F, L)
        basis = DeviceTableBasis(torch.as_tensor(Phi).cuda(), np.float64)
        c = mi.real_gaussian(2, m, 1)
        ref = oracle_lib.dense_synth(Phi, c)
    path = str(tmp_path / f"{family}.plan")
    stats = build_plan_gpu(basis, perm, sp, freq_tree(m, L), L, tol, path, device="cuda", log=None)
    assert stats["entries"] > 0
    O = oracle_lib.Plan(path)
    assert O.validate() == 0
    f = O.apply(c)
    for r in range(2):
        assert np.linalg.norm(f[r] - ref[r]) / np.linalg.norm(ref[r]) <= 10 * tol
    P = mht.Plan(path, 0)
    fg = P.apply(torch.from_numpy(c).cuda()).cpu().numpy()
    for r in range(2):
        assert np.abs(fg[r] - f[r]).max() <= 1e-12 * np.abs(f[r]).max()
    P.close()
