"""ORACLE — TEST INFRASTRUCTURE ONLY.

ctypes wrapper around ``oracle/oracle.c`` (plain C + OpenMP, fp64).  Only
``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this package.  The product package
``paper_2605_21828_b200`` never imports it, and it never imports the product
package: the two share only the seeded generators in ``mht_inputs``.

Functions (see oracle.c's header for the PAPER.md passages each follows):

* O1 dense sums  — ``flat_synth`` / ``flat_analysis``,
  ``sphere_synth`` / ``sphere_analysis`` / ``sphere_matrix`` (real orthonormal
  harmonics, reading A11), ``dense_synth`` / ``dense_analysis`` (stored Phi).
* O2 butterfly  — ``Plan(path).apply(c)`` / ``.adjoint(f)`` (§2, P:231-283;
  adjoint P:153-155), with its own plan-file reader.

Parity status: all pinned (tests/test_oracle_*.py); see DESIGN.md §3.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None


def build(force: bool = False) -> str:
    """Compile liboracle.so with gcc (-O2, no fast-math, OpenMP)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-fno-fast-math", "-fopenmp", "-fPIC", "-shared",
                               "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(_LIB)
        P = C.c_void_p
        i64 = C.c_int64
        L.orc_flat_synth.argtypes = [i64, i64, P, P, P, i64, P]
        L.orc_flat_analysis.argtypes = [i64, i64, P, P, P, i64, P]
        L.orc_sphere_matrix.argtypes = [i64, P, P, C.c_int, P]
        L.orc_sphere_synth.argtypes = [i64, P, P, C.c_int, P, i64, P]
        L.orc_sphere_analysis.argtypes = [i64, P, P, C.c_int, P, i64, P]
        L.orc_dense_synth.argtypes = [i64, i64, P, C.c_int, P, i64, P]
        L.orc_dense_analysis.argtypes = [i64, i64, P, C.c_int, P, i64, P]
        L.orc_plan_open.argtypes = [C.c_char_p, C.c_int]
        L.orc_plan_open.restype = P
        L.orc_plan_close.argtypes = [P]
        L.orc_plan_validate.argtypes = [P]
        L.orc_bf_apply.argtypes = [P, P, P, i64]
        L.orc_bf_adjoint.argtypes = [P, P, P, i64]
        L.orc_plan_entries.argtypes = [P]
        L.orc_plan_entries.restype = i64
        for nm in ("orc_plan_n", "orc_plan_m"):
            getattr(L, nm).argtypes = [P]
            getattr(L, nm).restype = i64
        for nm in ("orc_plan_L", "orc_plan_dtype"):
            getattr(L, nm).argtypes = [P]
            getattr(L, nm).restype = C.c_int
        L.orc_last_error.restype = C.c_char_p
        L.orc_num_threads.restype = C.c_int
        L.orc_set_threads.argtypes = [C.c_int]
        _lib = L
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


def _c2d(a) -> np.ndarray:
    """(nrhs, len) array -> contiguous 2-D."""
    a = np.asarray(a)
    if a.ndim == 1:
        a = a[None, :]
    return np.ascontiguousarray(a)


def num_threads() -> int:
    return lib().orc_num_threads()


def set_threads(t: int) -> None:
    lib().orc_set_threads(int(t))


# ------------------------------ O1 ------------------------------------------
def flat_synth(x, k, c):
    """f = Phi c with Phi_jk = exp(i k.x_j).  x (n,2), k (m,2), c (nrhs, m)."""
    x = np.ascontiguousarray(x, dtype=np.float64)
    k = np.ascontiguousarray(k, dtype=np.int64)
    c = _c2d(c).astype(np.complex128)
    n, m, r = x.shape[0], k.shape[0], c.shape[0]
    f = np.empty((r, n), dtype=np.complex128)
    lib().orc_flat_synth(n, m, _p(x), _p(k), _p(c), r, _p(f))
    return f


def flat_analysis(x, k, f):
    """c = Phi^* f.  f (nrhs, n) -> (nrhs, m)."""
    x = np.ascontiguousarray(x, dtype=np.float64)
    k = np.ascontiguousarray(k, dtype=np.int64)
    f = _c2d(f).astype(np.complex128)
    n, m, r = x.shape[0], k.shape[0], f.shape[0]
    c = np.empty((r, m), dtype=np.complex128)
    lib().orc_flat_analysis(n, m, _p(x), _p(k), _p(f), r, _p(c))
    return c


def sphere_matrix(theta, phi, lmax):
    th = np.ascontiguousarray(theta, dtype=np.float64)
    ph = np.ascontiguousarray(phi, dtype=np.float64)
    Y = np.empty((th.shape[0], (lmax + 1) ** 2))
    lib().orc_sphere_matrix(th.shape[0], _p(th), _p(ph), lmax, _p(Y))
    return Y


def sphere_synth(theta, phi, lmax, c):
    th = np.ascontiguousarray(theta, dtype=np.float64)
    ph = np.ascontiguousarray(phi, dtype=np.float64)
    c = _c2d(c).astype(np.float64)
    f = np.empty((c.shape[0], th.shape[0]))
    lib().orc_sphere_synth(th.shape[0], _p(th), _p(ph), lmax, _p(c), c.shape[0], _p(f))
    return f


def sphere_analysis(theta, phi, lmax, f):
    th = np.ascontiguousarray(theta, dtype=np.float64)
    ph = np.ascontiguousarray(phi, dtype=np.float64)
    f = _c2d(f).astype(np.float64)
    c = np.empty((f.shape[0], (lmax + 1) ** 2))
    lib().orc_sphere_analysis(th.shape[0], _p(th), _p(ph), lmax, _p(f), f.shape[0], _p(c))
    return c


def dense_synth(Phi, c):
    """f = Phi c; Phi (n, m) (any layout; stored column-major internally)."""
    cplx = np.iscomplexobj(Phi) or np.iscomplexobj(c)
    dt = np.complex128 if cplx else np.float64
    PhiF = np.asfortranarray(Phi, dtype=dt)
    c = _c2d(c).astype(dt)
    n, m = PhiF.shape
    f = np.empty((c.shape[0], n), dtype=dt)
    lib().orc_dense_synth(n, m, _p(PhiF), int(cplx), _p(c), c.shape[0], _p(f))
    return f


def dense_analysis(Phi, f):
    cplx = np.iscomplexobj(Phi) or np.iscomplexobj(f)
    dt = np.complex128 if cplx else np.float64
    PhiF = np.asfortranarray(Phi, dtype=dt)
    f = _c2d(f).astype(dt)
    n, m = PhiF.shape
    c = np.empty((f.shape[0], m), dtype=dt)
    lib().orc_dense_analysis(n, m, _p(PhiF), int(cplx), _p(f), f.shape[0], _p(c))
    return c


# ------------------------------ O2 ------------------------------------------
class Plan:
    """Independent CPU butterfly apply/adjoint over a plan file (O2)."""

    def __init__(self, path: str, verify_checksum: bool = True):
        L = lib()
        self._h = L.orc_plan_open(str(path).encode(), int(verify_checksum))
        if not self._h:
            raise ValueError("oracle plan open failed: " + L.orc_last_error().decode())
        self.n = L.orc_plan_n(self._h)
        self.m = L.orc_plan_m(self._h)
        self.L = L.orc_plan_L(self._h)
        self.dtype = np.complex128 if L.orc_plan_dtype(self._h) == 2 else np.float64

    def validate(self) -> int:
        return lib().orc_plan_validate(self._h)

    def entries(self) -> int:
        return lib().orc_plan_entries(self._h)

    def apply(self, c):
        c = _c2d(c).astype(self.dtype)
        assert c.shape[1] == self.m
        f = np.empty((c.shape[0], self.n), dtype=self.dtype)
        lib().orc_bf_apply(self._h, _p(c), _p(f), c.shape[0])
        return f

    def adjoint(self, f):
        f = _c2d(f).astype(self.dtype)
        assert f.shape[1] == self.n
        c = np.empty((f.shape[0], self.m), dtype=self.dtype)
        lib().orc_bf_adjoint(self._h, _p(f), _p(c), f.shape[0])
        return c

    def close(self):
        if self._h:
            lib().orc_plan_close(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
