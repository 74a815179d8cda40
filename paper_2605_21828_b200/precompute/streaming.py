"""Streaming butterfly factorization (§4, Alg. 3; host
precompute, not timed).

The stage-order builders (``builder.build_plan``, ``gpu_builder``) read
Phi(tau, J) for arbitrary column sets at every level, so for a stored basis
(mesh eigenvectors) they need all of Phi resident: O(n m) working memory —
the problem P:443-450 names.  Alg. 3 instead traverses the frequency tree
T_lambda in post-order ("left, right, parent"):

* at a frequency leaf nu, the next band of basis columns Phi(:, nu) (n x |nu|,
  e.g. the next eigenvectors an eigensolver delivers) is streamed in and
  compressed at once by its level-0 ID, Phi(:, nu) ~= Phi(:, J_nu) X_nu; only
  the skeleton columns Phi(:, J_nu) are kept;
* at an internal node nu of height h (both children done), for every space
  node tau at depth h with parent p, the kept skeleton columns of the two
  children restricted to tau's rows, [Phi(tau, J_{p,c1}) Phi(tau, J_{p,c2})],
  are merged and split (Fig. streaming-BF): their ID gives the
  transfer X_{tau nu} and the skeleton Phi(tau, J_{tau nu}), kept for the
  parent; the children's columns are freed;
* at the root (height L) the kept Phi(tau, J_tau) of every space leaf is the
  leaf interpolation U_tau.

Only skeleton columns of pending nodes are ever held (one per height of the
post-order stack, plus the current one), so working memory is bounded by a
small multiple of the factorization, never by Phi.  Every block gets the
same column ID (``idecomp.column_id``, reading A5) on the same submatrix
Phi(tau, J_p,c1 u J_p,c2) as the stage-order builders, so the plan is the same
factorization in the same file format (v1).

Blocks come out in post-order, not in the file's stage order: each stage's
coefficients are appended to a per-stage spool file as they are produced
(block records and index lists stay in memory: O(total rank)), and the plan
is assembled stage by stage at the end, streaming the spools.
"""
from __future__ import annotations

import os
import tempfile
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np

from .idecomp import column_id
from .planfile import KIND_DENSE, KIND_ID, KIND_IDENTITY, PlanWriter


class BandFile:
    """Basis columns on disk as Phi^T (m x n, row-major = Phi column-major),
    read band by band with explicit reads (no memory map), so Phi is never
    resident: the stand-in for an eigensolver that delivers eigenvector bands
    in eigenvalue order."""

    def __init__(self, path, n, m, dtype):
        self.path, self.n, self.m, self.dtype = path, int(n), int(m), np.dtype(dtype)

    @staticmethod
    def write(path, Phi, chunk=256):
        Phi = np.asarray(Phi)
        with open(path, "wb") as f:
            for c0 in range(0, Phi.shape[1], chunk):
                f.write(np.ascontiguousarray(Phi[:, c0:c0 + chunk].T).tobytes())
        return BandFile(path, Phi.shape[0], Phi.shape[1], Phi.dtype)

    def __call__(self, c0, c1):
        """Phi(:, c0:c1) as an (n, c1 - c0) array (user point order)."""
        with open(self.path, "rb") as f:
            f.seek(c0 * self.n * self.dtype.itemsize)
            a = np.fromfile(f, dtype=self.dtype, count=(c1 - c0) * self.n)
        return a.reshape(c1 - c0, self.n).T


class ClosedFormBands:
    """Bands of a closed-form basis (``basis.block``), evaluated on demand."""

    def __init__(self, basis):
        self.basis, self.n, self.m, self.dtype = basis, basis.n, basis.m, np.dtype(basis.dtype)

    def __call__(self, c0, c1):
        return self.basis.block(np.arange(self.n), np.arange(c0, c1))


def build_plan_streaming(bands, perm, sp_off, fr_off, L, tol, path, seed=1234, workers=None, log=print,
                         spool_dir=None, perm_k=None):
    """Alg. 3: post-order streaming factorization of Phi, whose columns come
    from ``bands(c0, c1)`` (n x (c1 - c0), rows in user point order), one
    frequency leaf at a time.  Writes the v1 plan to ``path``; returns stats
    (incl. the peak bytes of kept skeleton columns)."""
    n, m = bands.n, bands.m
    dtype = bands.dtype
    nl = 1 << L
    perm = np.asarray(perm, dtype=np.int64)
    sp_off = np.asarray(sp_off, dtype=np.int64)
    fr_off = np.asarray(fr_off, dtype=np.int64)
    sdt = np.dtype("<c16") if dtype == np.complex128 else np.dtype("<f8")
    workers = workers or max(1, min(8, os.cpu_count() or 1))
    pool = ThreadPoolExecutor(workers) if workers > 1 else None
    # parallelism comes from the block pool: single-threaded BLAS inside it
    # (nested BLAS threads would also multiply the per-thread work buffers)
    try:
        from threadpoolctl import threadpool_limits

        _tpl = threadpool_limits(1)
    except Exception:
        _tpl = None
    spool_dir = spool_dir or os.path.dirname(os.path.abspath(path))
    spools = [tempfile.NamedTemporaryFile("wb", dir=spool_dir, prefix=".bfspool", delete=False) for _ in range(L + 2)]
    ncoef = [0] * (L + 2)
    recs = [[None] * nl for _ in range(L + 2)]  # (kind, r_out, r_in, skel, red, coef_off)
    stats = {"n": n, "m": m, "L": L, "tol": tol, "builder": "streaming (post-order, Alg. 3)",
             "kept_bytes_peak": 0, "bands": nl}
    kept_bytes = 0
    t_start = time.time()

    def emit(s, b, kind, r_out, r_in, skel=None, red=None, T=None):
        off = 0
        if T is not None:
            off = ncoef[s]
            spools[s].write(np.asfortranarray(T).astype(sdt).T.tobytes())
            ncoef[s] += T.size
        recs[s][b] = (kind, r_out, r_in, skel, red, off)

    def rows_in(d, t, p_d, p):
        """Positions of space node (d, t)'s rows inside its ancestor (p_d, p)'s rows (tree order)."""
        w, wp = 1 << (L - d), 1 << (L - p_d)
        base = sp_off[p * wp]
        return slice(int(sp_off[t * w] - base), int(sp_off[(t + 1) * w] - base))

    def compress(A, sd):
        k, skel, red, T = column_id(A, tol, seed=sd)
        return k, skel, red, T

    def leaf(v):
        # Phi(:, nu) for the rows of the root, in tree order
        A = bands(int(fr_off[v]), int(fr_off[v + 1]))[perm]
        c = A.shape[1]
        k, skel, red, T = compress(A, seed + v)
        if k == c:
            emit(0, v, KIND_IDENTITY, c, c)
            return [A]
        emit(0, v, KIND_ID, k, c, skel, red, T)
        return [np.ascontiguousarray(A[:, skel])]

    def merge(h, v, left, right):
        """Node (h, v) of T_lambda: for every space node t at depth h, ID of
        [left[p](t rows), right[p](t rows)]; returns the kept skeleton columns per t."""
        nt = 1 << h

        def one(t):
            p = t >> 1
            sl = rows_in(h, t, h - 1, p)
            A = np.concatenate([left[p][sl], right[p][sl]], axis=1)
            c = A.shape[1]
            k, skel, red, T = compress(A, seed + h * nl + t * (nl >> h) + v)
            return t, A, c, k, skel, red, T

        out = [None] * nt
        res = pool.map(one, range(nt)) if pool is not None else map(one, range(nt))
        for t, A, c, k, skel, red, T in res:
            b = t * (nl >> h) + v
            if k == c:
                emit(h, b, KIND_IDENTITY, c, c)
                out[t] = A
            else:
                emit(h, b, KIND_ID, k, c, skel, red, T)
                out[t] = np.ascontiguousarray(A[:, skel])
        return out

    def nbytes(lst):
        return sum(a.nbytes for a in lst)

    # post-order traversal with an explicit stack of completed left siblings
    stack = []  # (height, v, kept)
    try:
        for v in range(nl):
            node = (0, v, leaf(v))
            kept_bytes += nbytes(node[2])
            while stack and stack[-1][0] == node[0]:
                h, vl, kl = stack.pop()
                merged = merge(h + 1, vl >> 1, kl, node[2])
                # both children and the parent's columns coexist here
                stats["kept_bytes_peak"] = max(stats["kept_bytes_peak"], kept_bytes + nbytes(merged))
                kept_bytes += nbytes(merged) - nbytes(kl) - nbytes(node[2])
                node = (h + 1, vl >> 1, merged)
            stats["kept_bytes_peak"] = max(stats["kept_bytes_peak"], kept_bytes)
            stack.append(node)
            if log and (v + 1) % max(1, nl // 8) == 0:
                log(f"[stream-build] {v + 1}/{nl} bands, kept {kept_bytes / 1e6:.1f} MB, {time.time() - t_start:.1f}s")
        assert len(stack) == 1 and stack[0][0] == L
        # leaf interpolation U_tau = Phi(tau, J_tau): the kept columns at the root
        for t, U in enumerate(stack[0][2]):
            emit(L + 1, t, KIND_DENSE, U.shape[0], U.shape[1], T=U)
    finally:
        if pool is not None:
            pool.shutdown()
        if _tpl is not None:
            _tpl.unregister()
        for f in spools:
            f.close()
    # ---- assemble the plan in stage order from the spools
    try:
        w = PlanWriter(path, dtype, n, m, L, tol, perm, sp_off, fr_off, perm_k=perm_k)
        for s in range(L + 2):
            idx, nidx, rows = [], 0, []
            for (kind, r_out, r_in, skel, red, off) in recs[s]:
                io = 0
                if kind == KIND_ID:
                    io = nidx
                    idx += [np.asarray(skel, "<i4"), np.asarray(red, "<i4")]
                    nidx += r_in
                rows.append((kind, r_out, r_in, 0, io, off))
            w.add_stage_spooled(s, spools[s].name, ncoef[s], rows, idx)
        w.close()
    finally:
        for f in spools:
            try:
                os.unlink(f.name)
            except OSError:
                pass
    stats["stages"] = w.stage_stats
    stats["entries"] = int(w.entries)
    stats["dense_entries"] = int(n) * int(m)
    stats["plan_bytes"] = int(w.body) + 256
    stats["seconds"] = round(time.time() - t_start, 2)
    return stats


def _main():
    """Build a workload's plan with the streaming builder in this process and
    report the process's peak RSS (for the comparison with the stage-order
    builder): ``python -m paper_2605_21828_b200.precompute.streaming c4 out.plan``."""
    import json
    import resource
    import sys

    import mht_inputs as mi

    from .. import workloads as W

    import threading

    import psutil

    class _Peak:
        """Resident set size sampled every 20 ms on a thread (the build's peak above
        the process's resident size just before it starts)."""

        def __init__(self):
            self.p, self.peak, self.stop_ = psutil.Process(), 0, False
            self.base = self.p.memory_info().rss
            self.t = threading.Thread(target=self.run, daemon=True)
            self.t.start()

        def run(self):
            while not self.stop_:
                self.peak = max(self.peak, self.p.memory_info().rss)
                time.sleep(0.02)

        def stop(self):
            self.stop_ = True
            self.t.join()
            self.peak = max(self.peak, self.p.memory_info().rss)
            return (self.peak - self.base) / 2**20

    name, out = sys.argv[1], sys.argv[2]
    mode = sys.argv[3] if len(sys.argv) > 3 else "streaming"  # streaming | stage | prepare (mesh band file)
    w = mi.WORKLOADS[name] if name in mi.WORKLOADS else None
    band_path = sys.argv[4] if len(sys.argv) > 4 else out + ".bands"  # mesh: the shared band file
    t0 = time.time()
    if w.family == "mesh":
        # the eigenvectors come from the eigensolver once, to a band file on disk
        # (the stand-in for a band-by-band eigensolver); both builders read that file
        from .. import mesh_setup

        if not os.path.exists(band_path):
            basis, perm, sp_off = mesh_setup.setup_mesh(w)
            np.save(band_path + ".tree.npy", np.concatenate([perm.astype(np.int64), sp_off]))
            BandFile.write(band_path, basis.Phi)
            del basis
        if mode == "prepare":
            return
        tr = np.load(band_path + ".tree.npy")
        perm, sp_off = tr[: w.n], tr[w.n:]
        bf = BandFile(band_path, w.n, w.m, np.float64)
        from .trees import freq_tree

        fr_off = freq_tree(w.m, w.L)
        rss0 = resource.getrusage(resource.RUSAGE_SELF).ru_maxrss
        t1 = time.time()
        pk = _Peak()
        if mode == "streaming":
            st = build_plan_streaming(bf, perm, sp_off, fr_off, w.L, w.tol, out, log=None)
        else:  # stage-order CPU builder on the resident Phi read from the same file
            from .basis import DenseBasis
            from .builder import build_plan

            Phi = bf(0, w.m).copy()
            st = build_plan(DenseBasis(Phi), perm, sp_off, fr_off, w.L, w.tol, out, workers=1, log=None)
    else:
        basis, perm, sp_off, fr_off, _ = W.setup(w)
        rss0 = resource.getrusage(resource.RUSAGE_SELF).ru_maxrss
        t1 = time.time()
        pk = _Peak()
        if mode == "streaming":
            st = build_plan_streaming(ClosedFormBands(basis), perm, sp_off, fr_off, w.L, w.tol, out, log=None)
        else:
            from .basis import DenseBasis
            from .builder import build_plan

            Phi = basis.block(np.arange(w.n), np.arange(w.m))
            st = build_plan(DenseBasis(Phi), perm, sp_off, fr_off, w.L, w.tol, out, workers=1, log=None)
    build_peak = pk.stop()
    rss = resource.getrusage(resource.RUSAGE_SELF).ru_maxrss
    print(json.dumps({"workload": name, "mode": mode, "seconds_build": round(time.time() - t1, 1),
                      "build_peak_rss_above_start_MB": round(build_peak, 1),
                      "seconds_total": round(time.time() - t0, 1), "peak_rss_MB": rss / 1024.0,
                      "rss_before_build_MB": rss0 / 1024.0, "entries": st["entries"],
                      "plan_bytes": st["plan_bytes"], "kept_bytes_peak": st.get("kept_bytes_peak")}))


if __name__ == "__main__":
    _main()
