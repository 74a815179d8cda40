"""Plan-size probe for workloads too large to factorize (configs[4]: flat,
n = m = 2^20, tol 1e-6).  SURVEY.md §8(d) "Config 5 protocol".

For each level l, sample blocks Phi(tau, nu) (tau a space node at depth l of
the median kd tree, nu a frequency node at height l spread over the annulus
radii), compute their eps-rank exactly from the eigenvalues of the Gram
matrix on the GPU (#{sigma_i > eps sigma_1}, the relative ID criterion), and
extrapolate the level's stored coefficients as

    2^L * mean(r_out * (r_in - r_out)),   r_in = 2 * mean r_out(l - 1)

(IDENTITY when r_out = r_in), plus the leaf factors U (n * r_L).  The paper
states the rank bounds of §5 only asymptotically; this
probe measures the actual ranks of this workload.

    python -m paper_2605_21828_b200.probe --workload c5 --samples 6 > probe.json
"""
from __future__ import annotations

import argparse
import json
import math
import sys
import time

import numpy as np

import mht_inputs as mi

from .precompute.trees import freq_tree, kd_tree


def eps_rank_gram(A, eps):
    import torch

    r, c = A.shape
    G = A.conj().T @ A if c <= r else A @ A.conj().T
    ev = torch.linalg.eigvalsh(G).clamp(min=0).sqrt()
    s1 = ev[-1]
    return int((ev > eps * s1).sum().item())


def probe(w: mi.Workload, samples: int = 6, seed: int = 0, device="cuda", log=print):
    import torch

    n, m, L, tol = w.n, w.m, w.L, w.tol
    x = mi.flat_points(n)
    k = mi.flat_modes(w.extra["side"])
    t0 = time.time()
    perm, sp_off = kd_tree(x, L)
    fr_off = freq_tree(m, L)
    log(f"[probe] trees in {time.time() - t0:.1f}s")
    X = torch.as_tensor(x, device=device)
    Kt = torch.as_tensor(k.astype(np.float64), device=device)
    rng = np.random.default_rng(seed)
    nl = 1 << L
    levels = []
    r_prev = 64.0
    total = 0
    for l in range(0, L + 1):
        nf = nl >> l
        w_sp = 1 << (L - l)
        vs = np.unique(np.linspace(0, nf - 1, min(samples, nf)).round().astype(int))
        ranks, shapes = [], []
        t1 = time.time()
        for v in vs:
            t = int(rng.integers(0, 1 << l))
            rows = perm[sp_off[t * w_sp]: sp_off[(t + 1) * w_sp]]
            cols = np.arange(fr_off[v * (1 << l)], fr_off[(v + 1) * (1 << l)])
            # cap the sampled block at 16k x 16k (a row subsample only lowers the rank estimate
            # when rows > 16k, where blocks are tall and full column rank anyway)
            if rows.size > 16384:
                rows = np.sort(rng.choice(rows, 16384, replace=False))
            ph = X[torch.as_tensor(rows, device=device)] @ Kt[torch.as_tensor(cols, device=device)].T
            A = torch.polar(torch.ones_like(ph), ph)
            ranks.append(eps_rank_gram(A, tol))
            shapes.append((int(rows.size), int(cols.size)))
            del A, ph
        r_out = float(np.mean(ranks))
        r_in = 64.0 if l == 0 else 2.0 * r_prev
        r_out = min(r_out, r_in)
        ident = r_out >= r_in - 0.5
        entries = 0.0 if ident else nl * r_out * (r_in - r_out)
        total += entries
        levels.append({"level": l, "blocks": nl, "block_rows": int(n >> l), "block_cols": int(64 << l),
                       "sampled_ranks": ranks, "r_out_mean": r_out, "r_in_est": r_in,
                       "identity": bool(ident), "entries_est": entries, "seconds": round(time.time() - t1, 1)})
        log(f"[probe] level {l}: ranks {ranks} -> r_out {r_out:.0f}, r_in {r_in:.0f}, entries {entries:.3g}")
        r_prev = r_out
    u_entries = n * r_prev
    total += u_entries
    sb = 16
    out = {"workload": w.name, "n": n, "m": m, "L": L, "tol": tol, "samples_per_level": samples,
           "levels": levels, "U_entries_est": u_entries, "entries_est": total,
           "plan_bytes_est": total * sb, "dense_bytes": n * m * sb,
           "fits_one_b200": total * sb < 150e9,
           "hbm_bytes": 183359 * 2**20}
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="c5")
    ap.add_argument("--samples", type=int, default=6)
    a = ap.parse_args()
    res = probe(mi.WORKLOADS[a.workload], a.samples, log=lambda s: print(s, file=sys.stderr, flush=True))
    print(json.dumps(res))


if __name__ == "__main__":
    main()
