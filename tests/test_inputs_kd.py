"""The quadtree-in-frequency mode order (mht_inputs.flat_modes_kd; §5
P:543-553, NEXT-3): a permutation of the mode box whose tree nodes are
axis-aligned boxes — at even depths exactly the quadtree's squares — with the
frequency tree's equal-count leaves (reading A7) landing on those boxes."""
import numpy as np
import pytest

import mht_inputs as mi
from paper_2605_21828_b200.precompute.trees import freq_tree


@pytest.mark.parametrize("side,L", [(8, 4), (16, 5), (64, 6), (256, 10)])
def test_kd_modes_are_boxes(side, L):
    k = mi.flat_modes_kd(side, L)
    ref = mi.flat_modes(side)
    assert sorted(map(tuple, k)) == sorted(map(tuple, ref))          # a permutation of the box
    fr = freq_tree(side * side, L)
    for d in range(L + 1):                                          # every tree node is a box
        nodes = 1 << d
        w = (side * side) >> d
        e1, e2 = side >> ((d + 1) // 2), side >> (d // 2)           # k1 split ceil(d/2) times, k2 floor(d/2)
        for t in range(0, nodes, max(1, nodes // 8)):
            blk = k[t * w:(t + 1) * w]
            assert np.ptp(blk[:, 0]) == e1 - 1 and np.ptp(blk[:, 1]) == e2 - 1
            if d % 2 == 0:
                assert e1 == e2                                     # quadtree squares at even depths
    leaf = k[fr[0]:fr[1]]
    lam = (leaf ** 2).sum(1)
    assert np.all(np.diff(lam) >= 0)                                # eigenvalue order inside a leaf


def test_kd_workloads_registered():
    from paper_2605_21828_b200 import workloads as W

    for name, base in (("c1kd", "c1"), ("c2kd", "c2")):
        w, b = mi.WORKLOADS[name], mi.WORKLOADS[base]
        assert (w.n, w.m, w.L, w.tol, w.dtype) == (b.n, b.m, b.L, b.tol, b.dtype)
        # the user's c order is the same eigenvalue order; the plan's is the kd order
        assert np.array_equal(mi.flat_workload_modes(w), mi.flat_workload_modes(b))
        k_plan, perm_k = W.freq_plan_order(w)
        assert np.array_equal(k_plan, mi.flat_workload_modes(w)[perm_k])
        assert W.freq_plan_order(b)[1] is None


def test_plan_frequency_permutation_oracle(tmp_path, oracle_lib):
    """Plan v2 (perm_k, reading A18): the oracle's O2 on a quadtree-frequency
    plan with c in the user's eigenvalue order equals, bitwise, O2 on the same
    factorization written without perm_k (v1) applied to c[perm_k] — synthesis
    and analysis — and matches the dense sum with the eigenvalue-order modes."""
    from paper_2605_21828_b200 import workloads as W
    from paper_2605_21828_b200.precompute import build_plan
    from paper_2605_21828_b200.precompute.basis import FlatBasis
    from paper_2605_21828_b200.precompute.trees import freq_tree, kd_tree

    w = mi.Workload("kdsmall", "flat", 1024, 1024, "complex128", 1e-8, 4, (1,), {"side": 32, "ftree": "kd"})
    p2 = str(tmp_path / "kd_v2.plan")
    W.build_workload_plan(w, p2, workers=2, log=None)
    x = mi.flat_points(w.n)
    k_plan, perm_k = W.freq_plan_order(w)
    perm, sp_off = kd_tree(x, w.L, alternate=True)
    p1 = str(tmp_path / "kd_v1.plan")
    build_plan(FlatBasis(x, k_plan), perm, sp_off, freq_tree(w.m, w.L), w.L, w.tol, p1, workers=2, log=None)
    O2, O1 = oracle_lib.Plan(p2), oracle_lib.Plan(p1)
    c = mi.complex_gaussian(3, w.m, 1)
    y = mi.complex_gaussian(3, w.n, 2)
    assert np.array_equal(O2.apply(c), O1.apply(c[:, perm_k]))
    a1 = O1.adjoint(y)
    a2 = np.empty_like(a1)
    a2[:, perm_k] = a1
    assert np.array_equal(O2.adjoint(y), a2)
    k_user = mi.flat_workload_modes(w)
    fd, cd = oracle_lib.flat_synth(x, k_user, c), oracle_lib.flat_analysis(x, k_user, y)
    f, ca = O2.apply(c), O2.adjoint(y)
    for r in range(3):
        assert np.linalg.norm(f[r] - fd[r]) / np.linalg.norm(fd[r]) <= 10 * w.tol
        assert np.linalg.norm(ca[r] - cd[r]) / np.linalg.norm(cd[r]) <= 10 * w.tol
