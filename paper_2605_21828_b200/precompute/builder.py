"""Row-wise butterfly factorization of Phi (host precompute, not timed).

Follows PAPER.md §2 (Alg. 1's body is missing, reading A16):

* level 0: for each frequency leaf nu, ID of the block column
  Phi(:, nu) = Phi(:, J_nu) X_nu.
* levels l = 1..L: for tau at depth l with parent p and nu at
  height l with children c1, c2, the block Phi(tau, nu) is represented through
  the previous skeletons: [U_pc1(tau,:) U_pc2(tau,:)] = Phi(tau, J_pc1 u J_pc2),
  and its column ID gives the transfer X_{tau nu} = [I T] Pi and the new
  skeleton J_{tau nu} = (J_pc1 u J_pc2)[skel].
* leaves: U_tau = Phi(tau, J_{tau, root}) stored densely.

With ID factors U_{tau nu} = Phi(tau, J_{tau nu}) is a submatrix of Phi, so only
the transfers and the leaf U_tau are stored.  Full-rank IDs are emitted as
IDENTITY blocks in natural order (SURVEY.md §0 finding 3).
"""
from __future__ import annotations

import multiprocessing as mp
import os
import time

import numpy as np

from .idecomp import column_id
from .planfile import KIND_DENSE, KIND_ID, KIND_IDENTITY, PlanWriter
from .trees import node_rows

_G = {}


def _init_worker(basis, tol):
    _G["basis"] = basis
    _G["tol"] = tol
    try:
        from threadpoolctl import threadpool_limits

        _G["tpl"] = threadpool_limits(1)
    except Exception:
        pass


def _job(task):
    stage, b, rows, Jin, seed, final = task
    basis, tol = _G["basis"], _G["tol"]
    A = basis.block(rows, Jin)
    if final:
        return b, KIND_DENSE, A.shape[0], A.shape[1], None, None, A, Jin
    k, skel, red, T = column_id(A, tol, seed=seed)
    c = len(Jin)
    if k == c:
        return b, KIND_IDENTITY, c, c, None, None, None, Jin
    return b, KIND_ID, k, c, skel, red, T, Jin[skel]


def build_plan(basis, perm, sp_off, fr_off, L, tol, path, workers=None, log=print, seed=1234, perm_k=None):
    """Factorize Phi (given by ``basis.block(rows, cols)``) and stream the plan
    to ``path``.  Returns a dict of statistics."""
    n, m = basis.n, basis.m
    nl = 1 << L
    workers = workers or max(1, os.cpu_count() or 1)
    w = PlanWriter(path, basis.dtype, n, m, L, tol, perm, sp_off, fr_off, perm_k=perm_k)
    all_rows = np.asarray(perm, dtype=np.int64)
    stats = {"stages": [], "n": n, "m": m, "L": L, "tol": tol}
    ctx = mp.get_context("fork")
    pool = ctx.Pool(workers, initializer=_init_worker, initargs=(basis, tol)) if workers > 1 else None
    if pool is None:
        _init_worker(basis, tol)

    def run(tasks):
        if pool is None:
            return map(_job, tasks)
        return pool.imap(_job, tasks, chunksize=1)

    J = None
    try:
        for s in range(L + 2):
            t0 = time.time()
            tasks = []
            if s == 0:
                for v in range(nl):
                    Jin = np.arange(fr_off[v], fr_off[v + 1], dtype=np.int64)
                    tasks.append((0, v, all_rows, Jin, seed + v, False))
            elif s <= L:
                nf, nfp = nl >> s, nl >> (s - 1)
                for b in range(nl):
                    t, v = divmod(b, nf)
                    p = t >> 1
                    Jin = np.concatenate([J[p * nfp + 2 * v], J[p * nfp + 2 * v + 1]])
                    tasks.append((s, b, node_rows(perm, sp_off, L, s, t).astype(np.int64), Jin,
                                  seed + s * nl + b, False))
            else:
                for t in range(nl):
                    tasks.append((s, t, node_rows(perm, sp_off, L, L, t).astype(np.int64), J[t], 0, True))
            w.begin_stage(s)
            Jn = [None] * nl
            for (b, kind, r_out, r_in, skel, red, T, Jout) in run(tasks):
                w.add_block(kind, r_out, r_in, skel, red, T)
                Jn[b] = Jout
            w.end_stage()
            J = Jn
            st = dict(w.stage_stats[-1])
            st["seconds"] = round(time.time() - t0, 2)
            stats["stages"].append(st)
            if log:
                log(f"[build] stage {s}: {st}")
    finally:
        if pool is not None:
            pool.close()
            pool.join()
    w.close()
    stats["entries"] = int(w.entries)
    stats["dense_entries"] = int(n) * int(m)
    stats["plan_bytes"] = int(w.body) + 256
    return stats
