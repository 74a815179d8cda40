"""Index trees T_x (space) and T_lambda (frequency) — host precompute.

PAPER.md §2 P:224-229 assumes binary trees on the rows and columns of Phi;
§3 P:355-362 builds T_lambda on [0, lambda_m] and T_x from a 2-D
parameterisation / quadtree (or a Fiedler tree, Alg. 2).

Representation: both trees have exactly 2^L leaves.  A node at depth d,
index t covers leaves [t 2^(L-d), (t+1) 2^(L-d)), i.e. a contiguous range of
tree positions; ``perm[pos]`` maps tree positions back to user point indices
and ``off[leaf]`` gives the leaf boundaries.

* ``freq_tree``  — equal-count contiguous ranges of the eigenvalue-sorted modes
  (reading A7).
* ``kd_tree``    — median splits (reading A9): alternate axes for d = 2,
  the axis of largest spread for d = 3; ties broken by original index.
* ``fiedler_tree`` lives in ``fiedler.py`` (meshes).
"""
from __future__ import annotations

import numpy as np


def freq_tree(m: int, L: int) -> np.ndarray:
    nl = 1 << L
    return np.array([(i * m) // nl for i in range(nl + 1)], dtype=np.int64)


def kd_tree(points: np.ndarray, L: int, alternate: bool = True):
    """Return (perm int32[n], sp_off int64[2^L+1])."""
    pts = np.asarray(points, dtype=np.float64)
    n, dim = pts.shape
    order = [np.arange(n)]
    for depth in range(L):
        nxt = []
        for idx in order:
            if alternate and dim == 2:
                ax = depth % dim
            else:
                sub = pts[idx]
                ax = int(np.argmax(sub.max(axis=0) - sub.min(axis=0))) if len(idx) else 0
            key = pts[idx, ax]
            o = np.lexsort((idx, key))          # stable: ties by original index
            idx = idx[o]
            h = len(idx) // 2
            nxt.append(idx[:h])
            nxt.append(idx[h:])
        order = nxt
    perm = np.concatenate(order).astype(np.int32)
    sizes = np.array([len(o) for o in order], dtype=np.int64)
    sp_off = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
    return perm, sp_off


def node_rows(perm, sp_off, L, depth, t):
    """User point indices of space node (depth, t)."""
    w = 1 << (L - depth)
    return perm[sp_off[t * w]: sp_off[(t + 1) * w]]


def node_cols(fr_off, L, height, v):
    """Mode indices (c order) of frequency node (height, v)."""
    w = 1 << height
    return np.arange(fr_off[v * w], fr_off[(v + 1) * w])
