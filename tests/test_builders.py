"""Host-precompute checks (CPU): the device builder's evaluators and batched
CPQR (run here through torch on the CPU) against independent references, and
its plans against the dense sum."""
import numpy as np
import pytest
import scipy.linalg as sl
import torch

import mht_inputs as mi
from paper_2605_21828_b200.precompute import freq_tree, kd_tree
from paper_2605_21828_b200.precompute.basis import FlatBasis, SphereBasis
from paper_2605_21828_b200.precompute.gpu_builder import (TorchFlatBasis, TorchTableBasis, build_plan_gpu,
                                                          cpqr_batched, sphere_table_torch)


def test_sphere_table_torch_matches_oracle(oracle_lib):
    th, ph, _ = mi.sphere_points(257, seed=5)
    for lmax in (7, 63):
        Y = oracle_lib.sphere_matrix(th, ph, lmax)
        Yt = sphere_table_torch(th, ph, lmax, "cpu").numpy()
        assert np.abs(Y - Yt).max() < 1e-12
    # host (numpy) evaluator too
    Yn = SphereBasis(th, ph, 63).rows_all(np.arange(257))
    assert np.abs(oracle_lib.sphere_matrix(th, ph, 63) - Yn).max() < 1e-12


def test_flat_block_torch_matches_numpy():
    x, k = mi.flat_points(300), mi.flat_modes(16)
    tb, nb = TorchFlatBasis(x, k, "cpu"), FlatBasis(x, k)
    rows = torch.tensor([[3, 5, 7, -1], [0, 1, 2, 3]])
    cols = torch.tensor([[1, 2, -1], [10, 11, 12]])
    At = tb.block_t(rows, cols).numpy()
    ref = nb.block([3, 5, 7], [1, 2])
    assert np.allclose(At[0, :2, :3], ref.T, atol=1e-14)
    assert np.all(At[0, 2] == 0) and np.all(At[0, :, 3] == 0)      # zero padding
    assert np.allclose(At[1], nb.block([0, 1, 2, 3], [10, 11, 12]).T, atol=1e-14)


@pytest.mark.parametrize("cplx", [False, True])
def test_cpqr_batched_matches_lapack(cplx):
    rng = np.random.default_rng(1)
    B, R, C, rank = 3, 40, 60, 17
    mats = []
    for _ in range(B):
        U = rng.standard_normal((R, rank)) + (1j * rng.standard_normal((R, rank)) if cplx else 0)
        V = rng.standard_normal((rank, C)) + (1j * rng.standard_normal((rank, C)) if cplx else 0)
        mats.append(U @ V + 1e-13 * rng.standard_normal((R, C)))
    At = torch.tensor(np.stack([m.T for m in mats]))
    ranks, perm = cpqr_batched(At.clone(), 1e-10)
    for b in range(B):
        assert ranks[b].item() == rank
        Rl, Pl = sl.qr(mats[b], mode="r", pivoting=True)
        k = int(np.sum(np.abs(np.diag(Rl)) > 1e-10 * abs(Rl[0, 0])))
        assert k == rank
        # the first pivot is the largest column (same rule as LAPACK)
        assert perm[b, 0].item() == Pl[0]


@pytest.mark.parametrize("family", ["flat", "sphere"])
def test_device_builder_plan_accuracy(oracle_lib, tmp_path, family):
    L = 4
    if family == "flat":
        n, side, tol = 1024, 32, 1e-8
        x, k = mi.flat_points(n), mi.flat_modes(side)
        perm, sp = kd_tree(x, L)
        basis = TorchFlatBasis(x, k, "cpu")
        m = side * side
        c = mi.complex_gaussian(2, m, 1)
        ref = oracle_lib.flat_synth(x, k, c)
    else:
        n, lmax, tol = 1024, 31, 1e-10
        th, ph, p = mi.sphere_points(n)
        perm, sp = kd_tree(p, L, alternate=False)
        basis = TorchTableBasis(sphere_table_torch(th, ph, lmax, "cpu"), np.float64)
        m = (lmax + 1) ** 2
        c = mi.sphere_coefficients(2, lmax)
        ref = oracle_lib.sphere_synth(th, ph, lmax, c)
    path = str(tmp_path / f"{family}.plan")
    build_plan_gpu(basis, perm, sp, freq_tree(m, L), L, tol, path, device="cpu", log=None)
    P = oracle_lib.Plan(path)
    assert P.validate() == 0
    f = P.apply(c)
    for r in range(2):
        assert np.linalg.norm(f[r] - ref[r]) / np.linalg.norm(ref[r]) <= 10 * tol


@pytest.mark.parametrize("builder", ["cpu", "device"])
def test_mesh_plan_fiedler(oracle_lib, tmp_path, builder):
    """configs[3] pipeline at small size: torus mesh, stored eigenvectors,
    Fiedler-tree rows (uneven leaves), plan within 10 tol of the dense sum."""
    from mht_inputs import mesh as mm
    from paper_2605_21828_b200.precompute import build_plan
    from paper_2605_21828_b200.precompute.basis import DenseBasis
    from paper_2605_21828_b200.precompute.fiedler import fiedler_tree

    V, F = mm.torus_mesh(32, 16, sigma=0.01)
    lam, Phi, mass, _ = mm.mesh_eigenbasis(V, F, 256)
    L, tol = 2, 1e-8
    perm, sp = fiedler_tree(V, F, L)
    path = str(tmp_path / f"mesh_{builder}.plan")
    if builder == "cpu":
        build_plan(DenseBasis(Phi), perm, sp, freq_tree(256, L), L, tol, path, workers=2, log=None)
    else:
        build_plan_gpu(TorchTableBasis(torch.as_tensor(Phi), np.float64), perm, sp, freq_tree(256, L), L, tol,
                       path, device="cpu", log=None)
    P = oracle_lib.Plan(path)
    c = mi.real_gaussian(2, 256, 1)
    f, fd = P.apply(c), oracle_lib.dense_synth(Phi, c)
    y = mi.real_gaussian(2, V.shape[0], 2)
    a, ad = P.adjoint(y), oracle_lib.dense_analysis(Phi, y)
    for r in range(2):
        assert np.linalg.norm(f[r] - fd[r]) / np.linalg.norm(fd[r]) <= 10 * tol
        assert np.linalg.norm(a[r] - ad[r]) / np.linalg.norm(ad[r]) <= 10 * tol
