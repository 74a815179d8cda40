"""Plan-size probe for flat workloads too large to factorize here (configs[4]:
n = m = 2^20, tol 1e-6) and for sizing the largest stand-in that fits one
B200.  SURVEY.md §8(d) "Config 5 protocol", step 1.

Per level l = 0..L the probe samples S transfer blocks (frequency nodes nu at
height l stratified over the whole eigenvalue range — the annulus radii — and
a random space node tau at depth l) and measures, with the GPU builder's own
rank criterion (gpu_builder.cpqr_batched: column-pivoted Householder QR, rank
= first j with |R_jj| <= tol |R_00|, reading A5; tall blocks on a Gaussian row
sketch of cols + 16 rows, exactly as the builder does):

    r_out = rank Phi(tau, nu),
    r_in  = rank Phi(p, c1) + rank Phi(p, c2)   (p = parent of tau, c1, c2 = children of nu),

so each sample gives the block's stored coefficients r_out (r_in - r_out)
(0 when r_out = r_in: IDENTITY).  The level's estimate is 2^L x the sample
mean; the leaf factors add sum_tau |tau| r_L(tau) ~ n x mean rank Phi(tau, all).
A row / column subset would only lower a rank, so no block is subsampled.
The paper states the rank bounds of §5 only asymptotically; the
probe measures this workload's ranks.  Validated on configs[1], whose plan is
built (profiles/r02_probe_c2.json vs the plan's stage sizes).

    python -m paper_2605_21828_b200.probe --workload c5 --samples 16 > probe.json
"""
from __future__ import annotations

import argparse
import json
import sys
import time

import numpy as np

import mht_inputs as mi

from .precompute.gpu_builder import OVERSAMPLE, DeviceFlatBasis, cpqr_batched
from .precompute.trees import freq_tree, kd_tree


def block_rank(basis, rows, cols, tol, gen):
    """The builder's rank of Phi(rows, cols) (gpu_builder._cpqr_group)."""
    import torch

    dev = basis.x.device
    r = torch.as_tensor(np.asarray(rows, np.int64), device=dev)[None, :]
    c = torch.as_tensor(np.asarray(cols, np.int64), device=dev)[None, :]
    At = basis.block_t(r, c)                                   # (1, C, R)
    C, R = At.shape[1], At.shape[2]
    if R >= 4 * C and R > C + OVERSAMPLE:
        ks = C + OVERSAMPLE
        G = torch.complex(torch.randn((1, R, ks), generator=gen, device=dev, dtype=torch.float64),
                          torch.randn((1, R, ks), generator=gen, device=dev, dtype=torch.float64))
        At = torch.bmm(At, G)
        del G
    ranks, _ = cpqr_batched(At, tol)
    out = int(min(int(ranks[0]), C))
    del At
    return out


def probe(w: mi.Workload, samples: int = 16, seed: int = 0, device="cuda", log=print):
    import torch

    n, m, L, tol = w.n, w.m, w.L, w.tol
    x = mi.flat_points(n, seed=w.extra.get("seed", mi.SEED_GEOMETRY))
    k = mi.flat_workload_modes(w)
    t0 = time.time()
    perm, sp_off = kd_tree(x, L, alternate=True)
    fr_off = freq_tree(m, L)
    log(f"[probe] trees in {time.time() - t0:.1f}s")
    basis = DeviceFlatBasis(x, k, device)
    gen = torch.Generator(device=device)
    gen.manual_seed(1234 + seed)
    rng = np.random.default_rng(seed)
    nl = 1 << L

    def rows_of(d, t):
        wd = 1 << (L - d)
        return perm[sp_off[t * wd]: sp_off[(t + 1) * wd]]

    def cols_of(h, v):
        wh = 1 << h
        return np.arange(fr_off[v * wh], fr_off[(v + 1) * wh])

    levels = []
    total = 0.0
    for l in range(0, L + 1):
        nf = nl >> l
        t1 = time.time()
        vs = np.unique(((np.arange(samples) + rng.uniform(size=samples)) * nf / samples).astype(int).clip(0, nf - 1))
        ent, r_outs, r_ins = [], [], []
        for v in vs:
            t = int(rng.integers(0, 1 << l))
            r_out = block_rank(basis, rows_of(l, t), cols_of(l, v), tol, gen)
            if l == 0:
                r_in = len(cols_of(0, v))
            else:
                p = t >> 1
                r_in = (block_rank(basis, rows_of(l - 1, p), cols_of(l - 1, 2 * v), tol, gen)
                        + block_rank(basis, rows_of(l - 1, p), cols_of(l - 1, 2 * v + 1), tol, gen))
            r_out = min(r_out, r_in)
            r_outs.append(r_out)
            r_ins.append(r_in)
            ent.append(0 if r_out == r_in else r_out * (r_in - r_out))
        lev = nl * float(np.mean(ent))
        total += lev
        levels.append({"level": l, "blocks": nl, "block_rows": int(n >> l), "block_cols": int(m >> (L - l)),
                       "samples": len(vs), "r_out": r_outs, "r_in": r_ins,
                       "r_out_mean": float(np.mean(r_outs)), "identity_fraction": float(np.mean(np.array(ent) == 0)),
                       "entries_est": lev, "entries_sem": nl * float(np.std(ent) / np.sqrt(len(ent))),
                       "seconds": round(time.time() - t1, 1)})
        log(f"[probe] level {l}: r_out mean {np.mean(r_outs):.0f} (min {min(r_outs)}, max {max(r_outs)}), "
            f"entries {lev:.3g} ({time.time() - t1:.1f}s)")
        torch.cuda.empty_cache()
    # leaf factors U_tau = Phi(tau, J_tau), r_L(tau) = rank Phi(tau, all) <= |tau|
    uts = rng.integers(0, nl, size=min(samples, nl))
    u = [len(rows_of(L, int(t))) * block_rank(basis, rows_of(L, int(t)), np.arange(m), tol, gen) for t in uts]
    u_entries = nl * float(np.mean(u))
    total += u_entries
    sb = 16
    sem = float(np.sqrt(sum(lv["entries_sem"] ** 2 for lv in levels)))
    return {"workload": w.name, "n": n, "m": m, "L": L, "tol": tol, "samples_per_level": samples,
            "rank_method": "builder CPQR (gpu_builder.cpqr_batched; tall blocks on a cols+16 Gaussian row sketch)",
            "levels": levels, "U_entries_est": u_entries, "entries_est": total, "entries_sem": sem,
            "plan_bytes_est": total * sb, "plan_bytes_sem": sem * sb, "dense_bytes": n * m * sb,
            "fits_one_b200": total * sb < 150e9, "hbm_bytes": 183359 * 2**20,
            "seconds": round(time.time() - t0, 1)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="c5")
    ap.add_argument("--samples", type=int, default=16)
    a = ap.parse_args()
    res = probe(mi.WORKLOADS[a.workload], a.samples, log=lambda s: print(s, file=sys.stderr, flush=True))
    print(json.dumps(res))


if __name__ == "__main__":
    main()
