"""Streaming post-order factorization (§4, Alg. 3;
paper_2605_21828_b200/precompute/streaming.py), CPU only.

Pins: on the same basis values, trees, tolerance and ID seeds, the post-order
builder writes the SAME plan file, byte for byte, as the stage-order builder
(§2 recursion, already pinned against the dense sums and O2 in
tests/test_oracle_butterfly.py / test_builders.py); the plan matches the
oracle's dense sum within 10 x tol; the kept skeleton columns stay below the
basis size; the band file streams exact columns.
"""
import numpy as np
import pytest

import mht_inputs as mi
from paper_2605_21828_b200.precompute import build_plan, freq_tree, kd_tree
from paper_2605_21828_b200.precompute.basis import DenseBasis, FlatBasis
from paper_2605_21828_b200.precompute.streaming import BandFile, ClosedFormBands, build_plan_streaming


class _Mem:
    def __init__(self, Phi):
        self.Phi = Phi
        self.n, self.m = Phi.shape
        self.dtype = Phi.dtype

    def __call__(self, c0, c1):
        return self.Phi[:, c0:c1]


def _both(tmp_path, Phi, L, tol, name, pts=None):
    n, m = Phi.shape
    pts = np.random.default_rng(0).uniform(size=(n, 2)) if pts is None else pts
    perm, sp_off = kd_tree(pts, L)
    fr_off = freq_tree(m, L)
    a, b = str(tmp_path / f"{name}_stage.plan"), str(tmp_path / f"{name}_stream.plan")
    build_plan(DenseBasis(Phi), perm, sp_off, fr_off, L, tol, a, workers=1, log=None)
    st = build_plan_streaming(_Mem(Phi), perm, sp_off, fr_off, L, tol, b, workers=4, log=None)
    return a, b, st, perm


def _smooth_kernel(n, m, seed):
    # a numerically low-rank (butterfly-compressible) real matrix: exp(-|x - y|) between point sets
    rng = np.random.default_rng(seed)
    x = np.sort(rng.uniform(0, 1, n))
    y = np.sort(rng.uniform(0, 1, m))
    return np.exp(-4.0 * np.abs(x[:, None] - y[None, :])) + 0.5 * np.cos(3.0 * x[:, None] * y[None, :])


@pytest.mark.parametrize("case", ["real_lowrank", "real_random", "complex_flat"])
def test_streaming_plan_identical_to_stage_order(tmp_path, case):
    if case == "real_lowrank":
        Phi, L, tol = _smooth_kernel(777, 512, 3), 3, 1e-8
    elif case == "real_random":
        Phi, L, tol = np.random.default_rng(5).standard_normal((300, 256)), 2, 1e-10
    else:
        x = mi.flat_points(1024)
        k = mi.flat_modes(32)
        Phi, L, tol = FlatBasis(x, k).block(np.arange(1024), np.arange(1024)), 4, 1e-8
    a, b, st, _ = _both(tmp_path, Phi, L, tol, case)
    assert open(a, "rb").read() == open(b, "rb").read()
    if case == "real_lowrank":
        assert st["entries"] < 0.6 * Phi.size          # it compressed
        assert st["kept_bytes_peak"] < Phi.nbytes      # never held Phi


def test_streaming_plan_matches_dense_sum(tmp_path, oracle_lib):
    """Flat n = m = 2048 at tol 1e-8 built from closed-form bands: O2 on the
    streaming plan vs O1 (dense sum) within 10 x tol, synthesis and analysis."""
    n, side, L, tol = 2048, 32, 4, 1e-8
    x = mi.flat_points(n)
    k = mi.flat_modes(side)[: side * side]
    perm, sp_off = kd_tree(x, L, alternate=True)
    fr_off = freq_tree(k.shape[0], L)
    path = str(tmp_path / "flat_stream.plan")
    st = build_plan_streaming(ClosedFormBands(FlatBasis(x, k)), perm, sp_off, fr_off, L, tol, path, log=None)
    O = oracle_lib.Plan(path)
    c = mi.complex_gaussian(2, k.shape[0], 1)
    y = mi.complex_gaussian(2, n, 2)
    fd, cd = oracle_lib.flat_synth(x, k, c), oracle_lib.flat_analysis(x, k, y)
    f, ca = O.apply(c), O.adjoint(y)
    for r in range(2):
        assert np.linalg.norm(f[r] - fd[r]) / np.linalg.norm(fd[r]) <= 10 * tol
        assert np.linalg.norm(ca[r] - cd[r]) / np.linalg.norm(cd[r]) <= 10 * tol
    assert st["kept_bytes_peak"] < n * k.shape[0] * 16


def test_band_file_roundtrip(tmp_path):
    Phi = np.random.default_rng(1).standard_normal((123, 70))
    bf = BandFile.write(str(tmp_path / "phi.bands"), Phi, chunk=16)
    for c0, c1 in ((0, 7), (7, 64), (64, 70), (3, 3)):
        assert np.array_equal(bf(c0, c1), Phi[:, c0:c1])
