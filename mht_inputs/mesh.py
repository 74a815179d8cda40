"""Torus-mesh inputs for configs[3] (reading A13; stand-in for
the paper's deformed-torus / mesh experiments, §6.2 P:1032-1053 and
§7, whose meshes are not available).

Geometry and the stored eigenfunction matrix are INPUTS of the transform (the
MHT takes Phi as given; P:1037-1040 computes it with an external solver), so
they live here with the other seeded generators.  Nothing here is the
method's arithmetic.

* 256 (major angle u) x 128 (minor angle v) vertex grid on the torus with
  R = 2, r = 1; each quad (i, j)-(i+1, j+1) split along that diagonal
  (V - E + F = 0); isotropic Gaussian vertex noise sigma = 0.01 (seed 0).
* P1 finite elements: cotangent stiffness K, lumped (barycentric) mass M.
* Lowest m eigenpairs of K phi = lambda M phi, M-orthonormal
  (Phi^T M Phi = I), each eigenvector's sign fixed so its largest-magnitude
  entry is positive (reading A11).  Computed through A = M^{-1/2} K M^{-1/2}:
  on a GPU for n > 8192 by Chebyshev-filtered subspace iteration on the
  sparse A (`chebyshev_subspace_eigs`, degree-64 filters: the noisy mesh's
  spectrum reaches ~4e5, degree 24 stalls; the dense eigh of the 32,768^2
  matrix took ~650 s), otherwise by a dense eigh (torch on a GPU, else scipy).
  Eigenvectors inside a degenerate eigenspace are not unique; any
  M-orthonormal basis of it is a valid input (the oracle and the plan read
  the same stored Phi).
"""
from __future__ import annotations

import os

import numpy as np
import scipy.sparse as sp

from . import SEED_GEOMETRY


def torus_mesh(nu: int = 256, nv: int = 128, R: float = 2.0, r: float = 1.0, sigma: float = 0.01,
               seed: int = SEED_GEOMETRY):
    """Return (V (n,3) float64, F (2*nu*nv, 3) int64)."""
    u = 2.0 * np.pi * np.arange(nu) / nu
    v = 2.0 * np.pi * np.arange(nv) / nv
    U, Vv = np.meshgrid(u, v, indexing="ij")
    X = np.stack([(R + r * np.cos(Vv)) * np.cos(U), (R + r * np.cos(Vv)) * np.sin(U), r * np.sin(Vv)], axis=-1)
    V = X.reshape(-1, 3)
    if sigma > 0:
        V = V + np.random.default_rng(seed).normal(0.0, sigma, size=V.shape)
    idx = lambda i, j: (i % nu) * nv + (j % nv)
    I, J = np.meshgrid(np.arange(nu), np.arange(nv), indexing="ij")
    I, J = I.ravel(), J.ravel()
    a, b, c, d = idx(I, J), idx(I + 1, J), idx(I + 1, J + 1), idx(I, J + 1)
    F = np.concatenate([np.stack([a, b, c], 1), np.stack([a, c, d], 1)]).astype(np.int64)
    return V, F


def cotan_fem(V: np.ndarray, F: np.ndarray, n: int | None = None):
    """Cotangent stiffness K (n x n, PSD) and lumped mass diagonal (n,)."""
    n = V.shape[0] if n is None else n
    i, j, k = F[:, 0], F[:, 1], F[:, 2]
    e0 = V[k] - V[j]  # opposite vertex i
    e1 = V[i] - V[k]  # opposite vertex j
    e2 = V[j] - V[i]  # opposite vertex k
    area = 0.5 * np.linalg.norm(np.cross(e2, -e1), axis=1)

    def cot(a, b):
        return np.einsum("ij,ij->i", a, b) / np.linalg.norm(np.cross(a, b), axis=1)

    # angle at vertex i is between (j - i) and (k - i), etc.
    ci = cot(e2, -e1)
    cj = cot(e0, -e2)
    ck = cot(e1, -e0)
    rows = np.concatenate([j, k, k, i, i, j])
    cols = np.concatenate([k, j, i, k, j, i])
    w = -0.5 * np.concatenate([ci, ci, cj, cj, ck, ck])
    K = sp.coo_matrix((w, (rows, cols)), shape=(n, n)).tocsr()
    K = K - sp.diags(np.asarray(K.sum(axis=1)).ravel())
    mass = np.zeros(n)
    np.add.at(mass, i, area / 3)
    np.add.at(mass, j, area / 3)
    np.add.at(mass, k, area / 3)
    return K.tocsr(), mass


def chebyshev_subspace_eigs(K, mass, m: int, device=None, oversample: int | None = None, degree: int = 64,
                            tol: float = 1e-12, maxit: int = 200, seed: int = 0, info: dict | None = None):
    """Lowest m eigenpairs of K phi = lambda M phi (M = diag(mass)) by
    Chebyshev-filtered subspace iteration on A = M^-1/2 K M^-1/2 (sparse).

    Block of p = m + oversample vectors; each sweep applies the degree-d
    Chebyshev polynomial that damps [a, b] (a = the block's largest Ritz
    value, b = a Gershgorin upper bound of the spectrum), re-orthonormalises
    (QR) and does a Rayleigh-Ritz step; stops when every one of the m wanted
    residuals ||A x - theta x|| <= tol * b.  Returns (lam (m,), Q (n, m))
    with A Q = Q diag(lam), Q orthonormal.  torch on `device` (a GPU here:
    a dense eigh of a 32,768^2 matrix takes ~10 minutes)."""
    import torch

    n = K.shape[0]
    p = m + (oversample if oversample is not None else max(64, m // 8))
    s = 1.0 / np.sqrt(mass)
    A = (K.multiply(s[:, None]).multiply(s[None, :])).tocsr()
    A = 0.5 * (A + A.T)
    A = A.tocsr()
    b = float(np.max(np.asarray(abs(A).sum(axis=1)).ravel())) * 1.01  # Gershgorin upper bound
    dev = torch.device(device) if device is not None else torch.device("cpu")
    At = torch.sparse_csr_tensor(torch.from_numpy(A.indptr.astype(np.int64)), torch.from_numpy(A.indices.astype(np.int64)),
                                 torch.from_numpy(A.data), size=A.shape, dtype=torch.float64).to(dev)
    g = torch.Generator(device="cpu").manual_seed(seed)
    X = torch.randn(n, p, generator=g, dtype=torch.float64).to(dev)
    X, _ = torch.linalg.qr(X)

    def rayleigh_ritz(X):
        AX = At @ X
        H = X.T @ AX
        w, S = torch.linalg.eigh(0.5 * (H + H.T))
        return w, X @ S, AX @ S

    w, X, AX = rayleigh_ritz(X)
    converged = False
    for it in range(maxit):
        res = torch.linalg.vector_norm(AX[:, :m] - X[:, :m] * w[None, :m], dim=0)
        if info is not None:
            info["iterations"], info["max_residual"], info["bound"] = it, float(res.max()), b
        if float(res.max()) <= tol * b:
            converged = True
            break
        a = float(w[-1])  # damp everything above the block's top Ritz value
        e, c = (b - a) / 2.0, (b + a) / 2.0
        Y0 = X
        Y1 = (At @ X - c * X) / e
        for _ in range(2, degree + 1):
            Y2 = 2.0 * (At @ Y1 - c * Y1) / e - Y0
            Y0, Y1 = Y1, Y2
        X, _ = torch.linalg.qr(Y1)
        w, X, AX = rayleigh_ritz(X)
    if not converged:
        raise RuntimeError(f"chebyshev_subspace_eigs: no convergence in {maxit} sweeps "
                           f"(max residual {float(res.max()):.3e} > {tol * b:.3e})")
    lam = w[:m].cpu().numpy()
    Q = X[:, :m].cpu().numpy()
    return lam, Q


def _eigh_lowest(A: np.ndarray, m: int):
    """Lowest m eigenpairs of a dense symmetric matrix (GPU if available)."""
    try:
        import torch

        if torch.cuda.is_available():
            At = torch.as_tensor(A, device="cuda")
            lam, Q = torch.linalg.eigh(At)
            out = lam[:m].cpu().numpy(), Q[:, :m].cpu().numpy()
            del At, lam, Q
            torch.cuda.empty_cache()
            return out
    except Exception:
        pass
    import scipy.linalg as sl

    return sl.eigh(A, subset_by_index=[0, m - 1], driver="evr")


def mesh_eigenbasis(V, F, m: int, method: str = "auto"):
    """(lam (m,), Phi (n, m) float64 M-orthonormal, mass (n,), K csr).

    method: "dense" (eigh of the dense M^-1/2 K M^-1/2), "chebyshev"
    (filtered subspace iteration, sparse), "auto" = chebyshev on a GPU for
    n > 8192, else dense."""
    n = V.shape[0]
    K, mass = cotan_fem(V, F)
    s = 1.0 / np.sqrt(mass)
    if method == "auto":
        try:
            import torch

            method = "chebyshev" if (n > 8192 and torch.cuda.is_available()) else "dense"
        except Exception:
            method = "dense"
    if method == "chebyshev":
        import torch

        lam, Q = chebyshev_subspace_eigs(K, mass, m, device="cuda" if torch.cuda.is_available() else None)
    else:
        A = (K.multiply(s[:, None]).multiply(s[None, :])).toarray()
        A = 0.5 * (A + A.T)
        lam, Q = _eigh_lowest(A, m)
    Phi = Q * s[:, None]
    # sign convention: largest-magnitude entry positive (reading A11)
    j = np.argmax(np.abs(Phi), axis=0)
    sg = np.sign(Phi[j, np.arange(m)])
    sg[sg == 0] = 1.0
    Phi = np.ascontiguousarray(Phi * sg[None, :])
    return lam, Phi, mass, K


def torus_workload_inputs(nu=256, nv=128, m=2048, cache_dir=None):
    """(V, F, lam, Phi, mass) for configs[3]; the eigen-solve is cached on disk
    (a cache only: a fresh box recomputes it)."""
    V, F = torus_mesh(nu, nv)
    cache_dir = cache_dir or os.environ.get("MHT_PLAN_DIR") or (
        "/dev/shm/mht_plans" if os.path.isdir("/dev/shm") else "/tmp/mht_plans")
    os.makedirs(cache_dir, exist_ok=True)
    path = os.path.join(cache_dir, f"torus_{nu}x{nv}_m{m}_v3.npz")
    if os.path.exists(path):
        d = np.load(path)
        return V, F, d["lam"], d["Phi"], d["mass"]
    lam, Phi, mass, _ = mesh_eigenbasis(V, F, m)
    np.savez(path + ".tmp.npz", lam=lam, Phi=Phi, mass=mass)
    os.replace(path + ".tmp.npz", path)
    return V, F, lam, Phi, mass
