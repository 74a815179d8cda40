"""Device plan builder (host precompute, outside the timed path).

Same factorization as ``builder.build_plan`` (§2), same
plan file, but the block evaluation and the interpolative decompositions run
batched on the GPU so the configs[1]/[2] plans (65,536^2, tens of GB) build in
minutes instead of hours.  The steps run in libmht's construction kernels
(include/mht_build.h, csrc/mht_build.cu): Phi blocks evaluated in-kernel
(flat) or gathered from an in-kernel harmonics table (sphere) / the stored
eigenvectors (mesh), and the batched column-pivoted QR.  torch provides the
device memory, the Gaussian sketches and the library GEMM / eigvalsh /
triangular solve; this module arranges the batches and writes the file.

Per stage, blocks are processed in canonical order in chunks of equal-shape
batches (zero-padded: zero rows leave a column ID unchanged, zero columns are
never pivoted before a non-zero one):

* tall blocks (rows >= 4 cols): the first candidate is a certified full-rank
  test on a random row subset S (|S| = 4 cols + 64): sigma_min(A) >=
  sigma_min(A(S,:)) and sigma_max(A) <= ||A||_F, so sigma_min(A(S,:)) >
  tol ||A||_F proves the block has no eps-rank deficiency -> IDENTITY.
  Otherwise a Gaussian row sketch (cols + 16 rows) is pivoted.
* all other blocks: batched Householder QR with column pivoting
  (Businger–Golub; exact trailing norms recomputed every step), rank
  k = first j with |R_jj| <= tol |R_00| (reading A5), T = R11^{-1} R12.
"""
from __future__ import annotations

import math
import time

import numpy as np

from . import devkern
from .planfile import KIND_DENSE, KIND_ID, KIND_IDENTITY, PlanWriter
from .trees import node_rows

OVERSAMPLE = 16


# ------------------------------------------------------------------ bases
class DeviceFlatBasis:
    """Flat-square basis on the device; blocks evaluated in-kernel
    (``mhtb_flat_blocks``, csrc/mht_build.cu)."""

    def __init__(self, x, k, device):
        import torch

        self.torch = torch
        self.x = torch.as_tensor(np.ascontiguousarray(x, np.float64), device=device)
        self.k = torch.as_tensor(np.ascontiguousarray(k, np.float64), device=device)
        self.n, self.m = self.x.shape[0], self.k.shape[0]
        self.dtype = np.complex128
        self.tdtype = torch.complex128

    def block_t(self, rows, cols):
        """rows (B,R) long (-1 = zero row), cols (B,C) long (-1 = zero column)
        -> At (B, C, R) with At[b, c, r] = Phi(rows[b,r], cols[b,c])."""
        return devkern.flat_blocks(self.x, self.k, rows.contiguous(), cols.contiguous())


class DeviceTableBasis:
    """Phi held on the device as a dense (n, m) table (sphere harmonics
    evaluated once in-kernel by ``sphere_table``, or stored mesh eigenvectors)."""

    def __init__(self, table, dtype):
        self.table = table  # torch (n, m)
        self.n, self.m = table.shape
        self.dtype = dtype
        self.tdtype = table.dtype

    def block_t(self, rows, cols):
        t = __import__("torch")
        B, R = rows.shape
        C = cols.shape[1]
        r = rows.clamp(min=0)
        c = cols.clamp(min=0)
        A = self.table[r[:, None, :].expand(B, C, R), c[:, :, None].expand(B, C, R)]
        mask = ((cols >= 0)[:, :, None] & (rows >= 0)[:, None, :])
        return (A * mask.to(A.dtype)).contiguous()


def sphere_table(theta, phi, lmax, device):
    """Real orthonormal SH (reading A11) at all points, (n, (lmax+1)^2) float64,
    by the normalised associated-Legendre recurrence in-kernel
    (``mhtb_sphere_table``)."""
    import torch

    th = torch.as_tensor(np.ascontiguousarray(theta, np.float64), device=device)
    ph = torch.as_tensor(np.ascontiguousarray(phi, np.float64), device=device)
    return devkern.sphere_table(th, ph, lmax)


# ------------------------------------------------------------------ CPQR
def cpqr_batched(At, tol):
    """In-place batched Householder QR with column pivoting of A = At^T on the
    device (``mhtb_cpqr``: one CTA per block).

    At: (B, C, R) contiguous.  Returns (ranks (B,), perm (B, C)); on return
    At[b, c, r] = R_b[r, c] for r < ranks[b] (the first ranks[b] rows of the
    upper-triangular factor of A_b[:, perm_b])."""
    return devkern.cpqr(At, tol)  # (raises on a non-contiguous At: the caller reads R from it)


# ------------------------------------------------------------------ builder
def _chunks(nblk_rows, nblk_cols, budget_elems):
    """Split canonical block order into chunks whose padded B x C x R fits."""
    out, cur, cmax, rmax = [], [], 0, 0
    for b, (r, c) in enumerate(zip(nblk_rows, nblk_cols)):
        nr, nc = max(rmax, r), max(cmax, c)
        if cur and (len(cur) + 1) * max(nc, 1) * max(nr, 1) > budget_elems:
            out.append(cur)
            cur, cmax, rmax = [], 0, 0
            nr, nc = r, c
        cur.append(b)
        cmax, rmax = nc, nr
    if cur:
        out.append(cur)
    return out


def build_plan_gpu(basis, perm, sp_off, fr_off, L, tol, path, device="cuda", log=print, seed=1234,
                   budget_gb=3.0, perm_k=None):
    import torch

    n, m = basis.n, basis.m
    nl = 1 << L
    w = PlanWriter(path, basis.dtype, n, m, L, tol, perm, sp_off, fr_off, perm_k=perm_k)
    perm_np = np.asarray(perm, np.int64)
    esz = 16 if basis.dtype == np.complex128 else 8
    budget = int(budget_gb * 1e9 / esz)
    gen = torch.Generator(device=device)
    gen.manual_seed(seed)
    stats = {"stages": [], "n": n, "m": m, "L": L, "tol": tol, "builder": "gpu"}
    J = None
    for s in range(L + 2):
        t0 = time.time()
        rows_l, cols_l = [], []
        if s == 0:
            for v in range(nl):
                rows_l.append(perm_np)
                cols_l.append(np.arange(fr_off[v], fr_off[v + 1], dtype=np.int64))
        elif s <= L:
            nf, nfp = nl >> s, nl >> (s - 1)
            for b in range(nl):
                t, v = divmod(b, nf)
                p = t >> 1
                rows_l.append(node_rows(perm_np, sp_off, L, s, t))
                cols_l.append(np.concatenate([J[p * nfp + 2 * v], J[p * nfp + 2 * v + 1]]))
        else:
            for t in range(nl):
                rows_l.append(node_rows(perm_np, sp_off, L, L, t))
                cols_l.append(J[t])
        final = s == L + 1
        nR = [len(r) for r in rows_l]
        nC = [len(c) for c in cols_l]
        # tall blocks only need a row subset for certification
        eff_rows = [min(r, 4 * c + 64) if (not final and r >= 4 * c) else r for r, c in zip(nR, nC)]
        w.begin_stage(s)
        Jn = [None] * nl
        for chunk in _chunks(eff_rows, nC, budget):
            results = _process_chunk(basis, rows_l, cols_l, chunk, tol, final, device, gen, budget)
            for b, (kind, r_out, r_in, skel, red, T, Jout) in zip(chunk, results):
                w.add_block(kind, r_out, r_in, skel, red, T)
                Jn[b] = Jout
        w.end_stage()
        J = Jn
        st = dict(w.stage_stats[-1])
        st["seconds"] = round(time.time() - t0, 2)
        stats["stages"].append(st)
        if log:
            log(f"[gpu-build] stage {s}: {st}")
    w.close()
    stats["entries"] = int(w.entries)
    stats["dense_entries"] = int(n) * int(m)
    stats["plan_bytes"] = int(w.body) + 256
    return stats


def _pad_idx(lists, width, device):
    import torch

    a = np.full((len(lists), max(width, 1)), -1, dtype=np.int64)
    for i, l in enumerate(lists):
        a[i, : len(l)] = l
    return torch.as_tensor(a, device=device)


def _process_chunk(basis, rows_l, cols_l, chunk, tol, final, device, gen, budget):
    import torch

    B = len(chunk)
    Cs = [len(cols_l[b]) for b in chunk]
    Rs = [len(rows_l[b]) for b in chunk]
    Cmax = max(max(Cs), 1)
    cols = _pad_idx([cols_l[b] for b in chunk], Cmax, device)
    if final:
        Rmax = max(Rs)
        At = basis.block_t(_pad_idx([rows_l[b] for b in chunk], Rmax, device), cols)
        out = []
        for i, b in enumerate(chunk):
            U = At[i, : Cs[i], : Rs[i]].T.cpu().numpy()          # (rows, r_in)
            out.append((KIND_DENSE, Rs[i], Cs[i], None, None, U, cols_l[b]))
        return out
    results = [None] * B
    tall = [Rs[i] >= 4 * Cs[i] for i in range(B)]
    # ---- certified full rank for tall blocks, from a random row subset
    todo = []
    if any(tall):
        idx_t = [i for i in range(B) if tall[i]]
        S = max(min(Rs[i], 4 * Cs[i] + 64) for i in idx_t)
        sub = []
        for i in idx_t:
            r = rows_l[chunk[i]]
            sel = torch.randperm(len(r), generator=gen, device=device)[: min(len(r), S)].cpu().numpy()
            sub.append(r[np.sort(sel)])
        Asub = basis.block_t(_pad_idx(sub, S, device), cols[idx_t])          # (Bt, C, S)
        G = torch.bmm(Asub, Asub.transpose(1, 2).conj())                        # (Bt, C, C) = A_S^H A_S (conj-symmetric)
        ev = torch.linalg.eigvalsh(G)
        for j, i in enumerate(idx_t):
            c = Cs[i]
            if c == 0:
                results[i] = (KIND_IDENTITY, 0, 0, None, None, None, cols_l[chunk[i]])
                continue
            # eigenvalues of the padded Gram include zeros for padded columns: take the
            # (Cmax - c)-th smallest onwards
            lam = ev[j, Cmax - c:]
            smin = float(lam[0].clamp(min=0).sqrt())
            fro = math.sqrt(Rs[i] * c) if isinstance(basis, DeviceFlatBasis) else None
            if fro is None:
                fro = float(_fro_norm(basis, rows_l[chunk[i]], cols_l[chunk[i]], device))
            if smin > tol * fro * 4.0:
                results[i] = (KIND_IDENTITY, c, c, None, None, None, cols_l[chunk[i]])
            else:
                todo.append(i)
    todo += [i for i in range(B) if not tall[i]]
    if not todo:
        return results
    # ---- CPQR on the block (or on a Gaussian sketch for tall blocks), in
    # sub-batches that respect the memory budget with the full row count
    groups, cur, rmax = [], [], 0
    for i in todo:
        r = max(rmax, Rs[i])
        if cur and (len(cur) + 1) * Cmax * r > budget:
            groups.append(cur)
            cur, r = [], Rs[i]
        cur.append(i)
        rmax = r
    if cur:
        groups.append(cur)
    for g in groups:
        _cpqr_group(basis, rows_l, cols_l, chunk, cols, g, Cs, Rs, tall, Cmax, tol, device, gen, results)
    return results


def _cpqr_group(basis, rows_l, cols_l, chunk, cols, todo, Cs, Rs, tall, Cmax, tol, device, gen, results):
    import torch

    Rmax = max(Rs[i] for i in todo)
    At = basis.block_t(_pad_idx([rows_l[chunk[i]] for i in todo], Rmax, device), cols[todo])
    if any(tall[i] for i in todo):
        ks = Cmax + OVERSAMPLE
        if Rmax > ks:
            shp = (len(todo), Rmax, ks)
            if At.is_complex():
                Gm = torch.complex(torch.randn(shp, generator=gen, device=device, dtype=torch.float64),
                                   torch.randn(shp, generator=gen, device=device, dtype=torch.float64))
            else:
                Gm = torch.randn(shp, generator=gen, device=device, dtype=torch.float64)
            At = torch.bmm(At, Gm)                                               # (B, C, ks): (G A)^T
            del Gm
    ranks, permc = cpqr_batched(At, tol)
    ranks = ranks.cpu().numpy()
    permc = permc.cpu().numpy()
    for jj, i in enumerate(todo):
        b = chunk[i]
        c = Cs[i]
        k = int(min(ranks[jj], c))
        pr = permc[jj]
        pr = pr[pr < c]
        if k == c:
            results[i] = (KIND_IDENTITY, c, c, None, None, None, cols_l[b])
            continue
        skel = pr[:k]
        red = pr[k:]
        if k == 0:
            T = np.zeros((0, c), dtype=basis.dtype)
        else:
            # R11 = R[:k,:k], R12 = R[:k, red positions]; At[j, col, row] holds R[row, col]
            posr = np.nonzero(permc[jj] < c)[0][k:]
            R11 = At[jj, :k, :k].transpose(0, 1)
            R12 = At[jj, torch.as_tensor(posr, device=device), :k].transpose(0, 1)
            T = torch.linalg.solve_triangular(R11, R12, upper=True).cpu().numpy()
        results[i] = (KIND_ID, k, c, skel, red, T, cols_l[b][skel])


def _fro_norm(basis, rows, cols, device):
    import torch

    r = torch.as_tensor(np.asarray(rows), device=device)
    c = torch.as_tensor(np.asarray(cols), device=device)
    A = basis.block_t(r[None, :], c[None, :])
    return torch.linalg.vector_norm(A)
