"""Fiedler tree on a triangle mesh (host precompute, not timed).

PAPER.md §3 (Alg. 2 — body missing, reading A16): recursively
split the manifold by the sign of the second eigenfunction phi_2 of the
Neumann Laplace–Beltrami problem on each sub-manifold.  Reading
A10:

* per node, the cotangent stiffness and lumped mass are re-assembled from the
  triangles entirely inside the node (natural = homogeneous Neumann BC);
* the split is by the pointwise vertex sign of phi_2 (mesh-free
  variant), zero going to the non-negative side; phi_2's sign is fixed so its
  largest-magnitude entry is positive, child 0 = {phi_2 < 0};
* a node whose triangle graph is disconnected (or has isolated vertices) is
  split by components first (greedy size balancing, deterministic);
* fixed depth L (equal-depth invariant); empty nodes are kept.
"""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp
import scipy.sparse.csgraph as csg
import scipy.sparse.linalg as spla

from mht_inputs.mesh import cotan_fem


def _split_components(labels, ncomp, idx):
    sizes = np.bincount(labels, minlength=ncomp)
    first = np.full(ncomp, np.iinfo(np.int64).max)
    np.minimum.at(first, labels, np.arange(labels.size))
    order = sorted(range(ncomp), key=lambda c: (-sizes[c], first[c]))
    side = np.zeros(ncomp, dtype=np.int64)
    load = [0, 0]
    for c in order:
        s = 0 if load[0] <= load[1] else 1
        side[c] = s
        load[s] += sizes[c]
    a = idx[side[labels] == 0]
    b = idx[side[labels] == 1]
    return a, b


def fiedler_split(V, F, idx):
    """Split the vertex set `idx` (sorted user indices) into two children."""
    n = idx.size
    if n <= 1:
        return idx, idx[:0]
    loc = -np.ones(V.shape[0], dtype=np.int64)
    loc[idx] = np.arange(n)
    inside = np.all(loc[F] >= 0, axis=1)
    Fs = loc[F[inside]]
    if Fs.shape[0] == 0:
        return idx[: n // 2], idx[n // 2:]
    ii = np.concatenate([Fs[:, 0], Fs[:, 1], Fs[:, 2]])
    jj = np.concatenate([Fs[:, 1], Fs[:, 2], Fs[:, 0]])
    G = sp.coo_matrix((np.ones(ii.size), (ii, jj)), shape=(n, n))
    ncomp, labels = csg.connected_components(G, directed=False)
    if ncomp > 1:
        return _split_components(labels, ncomp, idx)
    K, mass = cotan_fem(V[idx], Fs, n)
    M = sp.diags(mass)
    lam, vec = spla.eigsh(K.tocsc(), k=2, M=M.tocsc(), sigma=-1e-6, which="LM")
    phi2 = vec[:, np.argsort(lam)[1]]
    if phi2[np.argmax(np.abs(phi2))] < 0:
        phi2 = -phi2
    neg = phi2 < 0
    return idx[neg], idx[~neg]


def fiedler_tree(V, F, L: int):
    """Return (perm int32[n], sp_off int64[2^L+1]): leaves in tree order."""
    nodes = [np.arange(V.shape[0], dtype=np.int64)]
    for _ in range(L):
        nxt = []
        for idx in nodes:
            a, b = fiedler_split(V, F, idx)
            nxt += [np.sort(a), np.sort(b)]
        nodes = nxt
    perm = np.concatenate(nodes).astype(np.int32)
    sizes = np.array([x.size for x in nodes], dtype=np.int64)
    return perm, np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
