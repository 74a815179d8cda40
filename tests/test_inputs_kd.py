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
    for name, base in (("c1kd", "c1"), ("c2kd", "c2")):
        w, b = mi.WORKLOADS[name], mi.WORKLOADS[base]
        assert (w.n, w.m, w.L, w.tol, w.dtype) == (b.n, b.m, b.L, b.tol, b.dtype)
        k = mi.flat_workload_modes(w)
        assert k.shape == (w.m, 2) and not np.array_equal(k, mi.flat_workload_modes(b))
