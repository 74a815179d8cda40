"""Binding of the plan-construction kernels (include/mht_build.h) — argument
marshalling only: shapes, dtypes, devices, raw pointers and torch's current
stream.  Every step runs in ``libmht.so``'s kernels (csrc/mht_build.cu); there
is no fallback.  Used by ``gpu_builder``.
"""
from __future__ import annotations

import ctypes as C

from .. import mht

_bound = False


def _lib():
    global _bound
    L = mht.load_library()
    if not _bound:
        vp, i32, i64 = C.c_void_p, C.c_int, C.c_int64
        L.mhtb_flat_blocks.argtypes = [vp, vp, vp, vp, i32, i32, i32, vp, vp]
        L.mhtb_sphere_table.argtypes = [vp, vp, i64, i32, vp, vp]
        L.mhtb_cpqr.argtypes = [vp, i32, i32, i32, i32, C.c_double, vp, vp, vp]
        for nm in ("mhtb_flat_blocks", "mhtb_sphere_table", "mhtb_cpqr"):
            getattr(L, nm).restype = C.c_int
        _bound = True
    return L


def _check(st: int, what: str):
    if st != 0:
        L = mht.load_library()
        raise mht.MhtError(f"{what}: {L.mht_status_string(st).decode()} ({L.mht_last_error().decode()})")


def _dev(t, dtype, name):
    import torch

    if not t.is_cuda or t.dtype != dtype or not t.is_contiguous():
        raise mht.MhtError(f"{name}: expected a contiguous CUDA {dtype} tensor, got {t.dtype} on {t.device}")
    return C.c_void_p(t.data_ptr())


def _stream():
    import torch

    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


def flat_blocks(x, k, rows, cols):
    """x (n,2) f64, k (m,2) f64, rows (B,R) i64, cols (B,C) i64 (-1 = padding),
    all CUDA -> At (B,C,R) complex128 with At[b,c,r] = exp(i k[cols[b,c]].x[rows[b,r]])."""
    import torch

    B, R = rows.shape
    Cc = cols.shape[1]
    At = torch.empty((B, Cc, R), dtype=torch.complex128, device=rows.device)
    _check(_lib().mhtb_flat_blocks(_dev(x, torch.float64, "x"), _dev(k, torch.float64, "k"),
                                   _dev(rows, torch.int64, "rows"), _dev(cols, torch.int64, "cols"), B, R, Cc,
                                   C.c_void_p(At.data_ptr()), _stream()), "mhtb_flat_blocks")
    return At


def sphere_table(theta, phi, lmax):
    """theta, phi (n,) f64 CUDA -> Y (n, (lmax+1)^2) f64, Y[j, l^2+l+m] = Y_lm (reading A11)."""
    import torch

    n = theta.shape[0]
    Y = torch.empty((n, (lmax + 1) ** 2), dtype=torch.float64, device=theta.device)
    _check(_lib().mhtb_sphere_table(_dev(theta, torch.float64, "theta"), _dev(phi, torch.float64, "phi"), n, lmax,
                                    C.c_void_p(Y.data_ptr()), _stream()), "mhtb_sphere_table")
    return Y


def cpqr(At, tol):
    """In-place batched column-pivoted Householder QR of A_b = At[b].T
    (At (B,C,R) contiguous float64 / complex128 CUDA).  Returns (ranks (B,),
    perm (B,C)) int64 CUDA; At[b, c, r] = R_b[r, c] for r < ranks[b]."""
    import torch

    B, Cc, R = At.shape
    if At.dtype == torch.complex128:
        dt = mht.MHT_DTYPE_C128
    elif At.dtype == torch.float64:
        dt = mht.MHT_DTYPE_F64
    else:
        raise mht.MhtError(f"cpqr: unsupported dtype {At.dtype}")
    ranks = torch.empty((B,), dtype=torch.int64, device=At.device)
    perm = torch.empty((B, Cc), dtype=torch.int64, device=At.device)
    _check(_lib().mhtb_cpqr(_dev(At, At.dtype, "At"), B, Cc, R, dt, float(tol), C.c_void_p(ranks.data_ptr()),
                            C.c_void_p(perm.data_ptr()), _stream()), "mhtb_cpqr")
    return ranks, perm
