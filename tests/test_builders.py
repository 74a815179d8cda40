"""Host-precompute checks (CPU): the host evaluators and the CPU builder's
plans against independent references and the dense sum.  The device builder's
kernels (include/mht_build.h) are checked on the GPU in
tests/test_gpu_builder_kernels.py."""
import numpy as np
import pytest

import mht_inputs as mi
from paper_2605_21828_b200.precompute import freq_tree
from paper_2605_21828_b200.precompute.basis import SphereBasis


def test_sphere_host_evaluator_matches_oracle(oracle_lib):
    th, ph, _ = mi.sphere_points(257, seed=5)
    Yn = SphereBasis(th, ph, 63).rows_all(np.arange(257))
    assert np.abs(oracle_lib.sphere_matrix(th, ph, 63) - Yn).max() < 1e-12


def test_mesh_plan_fiedler(oracle_lib, tmp_path):
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
    path = str(tmp_path / "mesh_cpu.plan")
    build_plan(DenseBasis(Phi), perm, sp, freq_tree(256, L), L, tol, path, workers=2, log=None)
    P = oracle_lib.Plan(path)
    c = mi.real_gaussian(2, 256, 1)
    f, fd = P.apply(c), oracle_lib.dense_synth(Phi, c)
    y = mi.real_gaussian(2, V.shape[0], 2)
    a, ad = P.adjoint(y), oracle_lib.dense_analysis(Phi, y)
    for r in range(2):
        assert np.linalg.norm(f[r] - fd[r]) / np.linalg.norm(fd[r]) <= 10 * tol
        assert np.linalg.norm(a[r] - ad[r]) / np.linalg.norm(ad[r]) <= 10 * tol
