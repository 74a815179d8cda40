"""Device-accelerated plan builder (host precompute run on the GPU through torch).

Same factorization as ``builder.build_plan`` (§2), same
plan file, but the block evaluation and the interpolative decompositions run
batched on the GPU so the configs[1]/[2] plans (65,536^2, tens of GB) build in
minutes instead of hours.  Outside the timed path; the hot path never calls it.

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

from .planfile import KIND_DENSE, KIND_ID, KIND_IDENTITY, PlanWriter
from .trees import node_rows

OVERSAMPLE = 16


# ------------------------------------------------------------------ bases
class TorchFlatBasis:
    def __init__(self, x, k, device):
        import torch

        self.torch = torch
        self.x = torch.as_tensor(np.asarray(x, np.float64), device=device)
        self.k = torch.as_tensor(np.asarray(k, np.float64), device=device)
        self.n, self.m = self.x.shape[0], self.k.shape[0]
        self.dtype = np.complex128
        self.tdtype = torch.complex128

    def block_t(self, rows, cols):
        """rows (B,R) long (-1 = zero row), cols (B,C) long (-1 = zero column)
        -> At (B, C, R) with At[b, c, r] = Phi(rows[b,r], cols[b,c])."""
        t = self.torch
        kk = self.k[cols.clamp(min=0)]                     # (B, C, 2)
        xx = self.x[rows.clamp(min=0)]                     # (B, R, 2)
        ph = t.bmm(kk, xx.transpose(1, 2))                 # (B, C, R)
        A = t.complex(t.cos(ph), t.sin(ph))
        A.mul_(((cols >= 0)[:, :, None] & (rows >= 0)[:, None, :]).to(A.real.dtype))
        return A


class TorchTableBasis:
    """Phi held on the device as a dense (n, m) table (sphere harmonics
    evaluated once on the GPU, or stored mesh eigenvectors)."""

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
        return A * mask.to(A.dtype)


def sphere_table_torch(theta, phi, lmax, device, chunk=4096):
    """Real orthonormal SH (reading A11) at all points, (n, (lmax+1)^2) float64,
    by the normalised associated-Legendre recurrence vectorised on the GPU."""
    import torch

    th = torch.as_tensor(np.asarray(theta, np.float64), device=device)
    ph = torch.as_tensor(np.asarray(phi, np.float64), device=device)
    n = th.shape[0]
    M = (lmax + 1) ** 2
    out = torch.empty((n, M), dtype=torch.float64, device=device)
    ls = np.repeat(np.arange(lmax + 1), 2 * np.arange(lmax + 1) + 1)
    ms = np.arange(M) - ls * ls - ls
    am = torch.as_tensor(np.abs(ms), device=device)
    lt = torch.as_tensor(ls, device=device)
    # float64 from numpy: torch.where on two Python scalars would produce float32 (sqrt 2 to 1e-8)
    scale = torch.as_tensor(np.where(ms == 0, 1.0, math.sqrt(2.0)).astype(np.float64), device=device)
    pos = torch.as_tensor(ms >= 0, device=device)
    mvec = torch.arange(lmax + 1, dtype=torch.float64, device=device)
    for s in range(0, n, chunk):
        x = torch.cos(th[s:s + chunk])
        sn = torch.sin(th[s:s + chunk])
        npt = x.shape[0]
        P = torch.zeros((lmax + 1, lmax + 1, npt), dtype=torch.float64, device=device)
        P[0, 0] = 1.0 / math.sqrt(4.0 * math.pi)
        for mm in range(1, lmax + 1):
            P[mm, mm] = math.sqrt((2.0 * mm + 1.0) / (2.0 * mm)) * sn * P[mm - 1, mm - 1]
        for l in range(1, lmax + 1):
            P[l, l - 1] = math.sqrt(2.0 * (l - 1) + 3.0) * x * P[l - 1, l - 1]
            if l >= 2:
                m_ = mvec[: l - 1]
                a = torch.sqrt((4.0 * l * l - 1.0) / (l * l - m_ * m_))
                b = torch.sqrt(((l - 1.0) ** 2 - m_ * m_) / (4.0 * (l - 1.0) ** 2 - 1.0))
                P[l, : l - 1] = a[:, None] * (x[None, :] * P[l - 1, : l - 1] - b[:, None] * P[l - 2, : l - 1])
        val = P[lt, am, :].T                                              # (npt, M)
        mph = ph[s:s + chunk, None] * am[None, :].to(torch.float64)
        trig = torch.where(pos[None, :], torch.cos(mph), torch.sin(mph))
        out[s:s + npt] = val * scale[None, :] * trig
        del P
    return out


# ------------------------------------------------------------------ CPQR
def cpqr_batched(At, tol):
    """In-place batched Householder QR with column pivoting of A = At^T.

    At: (B, C, R) (column-contiguous).  Returns (ranks (B,), perm (B, C)); on
    return At[b, c, r] = R_b[r, c] for r <= c (the upper-triangular factor of
    A_b[:, perm_b])."""
    import torch

    B, C, R = At.shape
    kmax = min(R, C)
    dev = At.device
    bidx = torch.arange(B, device=dev)
    perm = torch.arange(C, device=dev).repeat(B, 1)
    norms = (At.real ** 2 + (At.imag ** 2 if At.is_complex() else 0)).sum(-1)
    r00 = norms.max(1).values.sqrt()
    ranks = torch.full((B,), kmax, dtype=torch.long, device=dev)
    done = torch.zeros(B, dtype=torch.bool, device=dev)
    for j in range(kmax):
        p = norms[:, j:].argmax(1) + j
        rowp = At[bidx, p].clone()
        At[bidx, p] = At[:, j].clone()  # (clone: p == j aliases the source)
        At[:, j] = rowp
        np_ = norms[bidx, p].clone()
        norms[bidx, p] = norms[:, j].clone()
        norms[:, j] = np_
        pp = perm[bidx, p].clone()
        perm[bidx, p] = perm[:, j].clone()
        perm[:, j] = pp
        rjj = norms[:, j].clamp(min=0).sqrt()
        newly = (~done) & (rjj <= tol * r00)
        ranks = torch.where(newly, torch.full_like(ranks, j), ranks)
        done = done | newly
        if (j & 15) == 15 and bool(done.all()):
            break
        x = At[:, j, j:]
        x0 = x[:, 0]
        ax0 = x0.abs()
        if At.is_complex():
            phase = torch.where(ax0 > 0, x0 / torch.where(ax0 > 0, ax0, 1.0), torch.ones_like(x0))
        else:
            phase = torch.where(x0 < 0, -1.0, 1.0).to(x0.dtype)
        alpha = -phase * rjj
        v = x.clone()
        v[:, 0] -= alpha
        vn = (v.abs() ** 2).sum(-1).sqrt()
        v = v / torch.where(vn > 0, vn, 1.0).to(v.dtype)[:, None]
        if j + 1 < C:
            Tr = At[:, j + 1:, j:]
            w = torch.bmm(Tr, v.conj().unsqueeze(-1))             # (B, C-j-1, 1)
            Tr.sub_(2.0 * w * v.unsqueeze(1))
            tail = At[:, j + 1:, j + 1:]
            norms[:, j + 1:] = (tail.real ** 2 + (tail.imag ** 2 if tail.is_complex() else 0)).sum(-1)
        At[:, j, j] = alpha
        At[:, j, j + 1:] = 0
    return ranks, perm


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
            fro = math.sqrt(Rs[i] * c) if isinstance(basis, TorchFlatBasis) else None
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
