"""Thin Python binding of libmht (include/mht.h) — argument marshalling only.

Every step of the transform runs in the CUDA kernels of ``libmht.so``; this
module only checks tensor shapes/dtypes/devices and passes raw pointers and
torch's current stream through ctypes.  There is no CPU fallback: if the
extension is missing or no B200 is present, the calls raise.

Names follow the C ABI: ``mht_plan_load``, ``mht_apply``, ``mht_apply_adjoint``,
``mht_apply_host``, ``mht_apply_adjoint_host``, ``mht_plan_info_get``, ...
``Plan`` wraps them for convenience.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libmht.so")

MHT_DTYPE_F64, MHT_DTYPE_C128 = 1, 2
EXPORTED = [
    "mht_plan_load", "mht_plan_info_get", "mht_plan_set_stream", "mht_reserve", "mht_apply",
    "mht_apply_adjoint", "mht_apply_host", "mht_apply_adjoint_host", "mht_apply_host_batch", "mht_apply_diag", "mht_apply_adjoint_diag", "mht_grf_sample", "mht_covariance_apply", "mht_lsqr",
    "mht_plan_load_shard", "mht_shard_info", "mht_shard_workspace", "mht_apply_shard_begin",
    "mht_apply_shard_end", "mht_apply_adjoint_shard_begin", "mht_apply_adjoint_shard_end",
    "mht_shard_export", "mht_shard_open_peers", "mht_shard_set_peers", "mht_shard_close_peers",
    "mht_set_graphs", "mht_set_fused_sums", "mht_sync",
    "mht_stage_stats", "mht_set_profiling", "mht_profile_get", "mht_profile_reset", "mht_plan_destroy",
    "mht_status_string", "mht_last_error", "mht_build_info",
]


class MhtError(RuntimeError):
    pass


class HostJob(C.Structure):
    """mht_host_job (include/mht.h)."""
    _fields_ = [("dir", C.c_int32), ("nrhs", C.c_int32), ("inp", C.c_void_p), ("out", C.c_void_p)]


class PlanInfo(C.Structure):
    _fields_ = [("n", C.c_int64), ("m", C.c_int64), ("L", C.c_int32), ("dtype", C.c_int32),
                ("tol", C.c_double), ("plan_bytes", C.c_int64), ("factor_entries", C.c_int64),
                ("device_bytes", C.c_int64), ("index_entries", C.c_int64),
                ("n_materialized", C.c_int32), ("n_alias", C.c_int32),
                ("fwd_launches", C.c_int32), ("adj_launches", C.c_int32)]


_lib = None


def load_library(path: str = LIB_PATH):
    """dlopen libmht.so (raises if it has not been built — no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise MhtError(f"{path} not found: run `python -c 'import __graft_entry__ as g; g.build()'`")
    L = C.CDLL(path)
    vp, i32, i64 = C.c_void_p, C.c_int, C.c_int64
    L.mht_plan_load.argtypes = [C.c_char_p, i32, C.POINTER(vp)]
    L.mht_plan_info_get.argtypes = [vp, C.POINTER(PlanInfo)]
    L.mht_plan_set_stream.argtypes = [vp, vp]
    L.mht_reserve.argtypes = [vp, i32]
    for nm in ("mht_apply", "mht_apply_adjoint", "mht_apply_host", "mht_apply_adjoint_host"):
        getattr(L, nm).argtypes = [vp, vp, vp, i32]
    for nm in ("mht_apply_diag", "mht_apply_adjoint_diag", "mht_grf_sample", "mht_covariance_apply"):
        getattr(L, nm).argtypes = [vp, vp, vp, vp, i32]
    L.mht_apply_host_batch.argtypes = [vp, vp, i32]
    L.mht_lsqr.argtypes = [vp, vp, vp, i32, i32, C.c_double, C.c_double, C.POINTER(C.c_int32),
                           C.POINTER(C.c_double), C.POINTER(C.c_double)]
    L.mht_plan_load_shard.argtypes = [C.c_char_p, i32, i32, i32, i32, C.POINTER(vp)]
    L.mht_shard_info.argtypes = [vp, C.POINTER(C.c_int32), C.POINTER(C.c_int32), C.POINTER(C.c_int32),
                                 C.POINTER(i64), C.POINTER(i64), C.POINTER(i64), C.POINTER(i64)]
    L.mht_shard_workspace.argtypes = [vp, i32, C.POINTER(vp)]
    for nm in ("mht_apply_shard_begin", "mht_apply_shard_end", "mht_apply_adjoint_shard_begin",
               "mht_apply_adjoint_shard_end"):
        getattr(L, nm).argtypes = [vp, vp, i32]
    L.mht_shard_export.argtypes = [vp, i32, vp, C.POINTER(i64)]
    L.mht_shard_open_peers.argtypes = [vp, i32, vp, C.POINTER(i64)]
    L.mht_shard_set_peers.argtypes = [vp, i32, C.POINTER(vp), C.POINTER(i64)]
    L.mht_shard_close_peers.argtypes = [vp]
    L.mht_set_graphs.argtypes = [vp, i32]
    L.mht_set_fused_sums.argtypes = [vp, i32]
    L.mht_sync.argtypes = [vp]
    L.mht_stage_stats.argtypes = [vp, i32, C.POINTER(i64), C.POINTER(C.c_int32), C.POINTER(C.c_int32),
                                  C.POINTER(C.c_int32)]
    L.mht_set_profiling.argtypes = [vp, i32]
    L.mht_profile_get.argtypes = [vp, i32, i32, i32, C.POINTER(C.c_double), C.POINTER(i64)]
    L.mht_profile_reset.argtypes = [vp]
    L.mht_plan_destroy.argtypes = [vp]
    L.mht_plan_destroy.restype = None
    L.mht_status_string.argtypes = [i32]
    L.mht_status_string.restype = C.c_char_p
    L.mht_last_error.restype = C.c_char_p
    L.mht_build_info.restype = C.c_char_p
    for nm in EXPORTED:
        if nm not in ("mht_plan_destroy", "mht_status_string", "mht_last_error", "mht_build_info"):
            getattr(L, nm).restype = i32
    _lib = L
    return L


def _check(st: int, what: str):
    if st != 0:
        L = load_library()
        raise MhtError(f"{what}: {L.mht_status_string(st).decode()}: {L.mht_last_error().decode()}")


# ------------------------------------------------------------ C-named calls
def mht_plan_load(path: str, device: int = 0) -> int:
    L = load_library()
    h = C.c_void_p()
    _check(L.mht_plan_load(str(path).encode(), int(device), C.byref(h)), "mht_plan_load")
    return h.value


def mht_plan_info_get(plan: int) -> PlanInfo:
    info = PlanInfo()
    _check(load_library().mht_plan_info_get(plan, C.byref(info)), "mht_plan_info_get")
    return info


def mht_plan_set_stream(plan: int, stream_ptr: int):
    _check(load_library().mht_plan_set_stream(plan, C.c_void_p(stream_ptr)), "mht_plan_set_stream")


def _dev_ptr(t, rows: int, nrhs: int, dt):
    import torch

    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise MhtError("expected a CUDA tensor")
    if t.dtype != dt or not t.is_contiguous() or t.numel() != rows * nrhs:
        raise MhtError(f"expected contiguous {dt} tensor with {rows}*{nrhs} elements, got "
                       f"{t.dtype} {tuple(t.shape)}")
    return C.c_void_p(t.data_ptr())


def mht_apply(plan: int, c, f, nrhs: int, n: int, m: int, dt):
    _check(load_library().mht_apply(plan, _dev_ptr(c, m, nrhs, dt), _dev_ptr(f, n, nrhs, dt), int(nrhs)),
           "mht_apply")


def mht_apply_adjoint(plan: int, f, c, nrhs: int, n: int, m: int, dt):
    _check(load_library().mht_apply_adjoint(plan, _dev_ptr(f, n, nrhs, dt), _dev_ptr(c, m, nrhs, dt),
                                            int(nrhs)), "mht_apply_adjoint")


def mht_plan_destroy(plan: int):
    load_library().mht_plan_destroy(plan)


# ------------------------------------------------------------ convenience
class Plan:
    """A loaded plan on one GPU.  Vectors are (nrhs, m) / (nrhs, n) tensors
    (= column-major m x nrhs / n x nrhs, the ABI layout)."""

    def __init__(self, path: str, device: int = 0):
        import torch

        self.device = torch.device("cuda", device)
        self._h = mht_plan_load(path, device)
        self.info = mht_plan_info_get(self._h)
        self.n, self.m, self.L = self.info.n, self.info.m, self.info.L
        self.is_complex = self.info.dtype == MHT_DTYPE_C128
        self.torch_dtype = torch.complex128 if self.is_complex else torch.float64
        self.np_dtype = np.complex128 if self.is_complex else np.float64
        self.scalar_bytes = 16 if self.is_complex else 8

    def _stream(self):
        import torch

        mht_plan_set_stream(self._h, torch.cuda.current_stream(self.device).cuda_stream)

    def reserve(self, nrhs: int):
        _check(load_library().mht_reserve(self._h, int(nrhs)), "mht_reserve")

    def apply(self, c, out=None):
        import torch

        c2 = c.reshape(-1, self.m) if c.dim() != 2 else c
        nrhs = c2.shape[0]
        f = out if out is not None else torch.empty((nrhs, self.n), dtype=self.torch_dtype, device=self.device)
        self._stream()
        mht_apply(self._h, c2, f, nrhs, self.n, self.m, self.torch_dtype)
        return f

    def adjoint(self, f, out=None):
        import torch

        f2 = f.reshape(-1, self.n) if f.dim() != 2 else f
        nrhs = f2.shape[0]
        c = out if out is not None else torch.empty((nrhs, self.m), dtype=self.torch_dtype, device=self.device)
        self._stream()
        mht_apply_adjoint(self._h, f2, c, nrhs, self.n, self.m, self.torch_dtype)
        return c

    # ---- applications (§7): a real coefficient-side diagonal fused
    # into the transform's own loads / stores of c (include/mht.h)
    def _diag_ptr(self, d):
        import torch

        if not isinstance(d, torch.Tensor) or not d.is_cuda or d.dtype != torch.float64 or not d.is_contiguous() \
                or d.numel() != self.m:
            raise MhtError(f"expected a contiguous CUDA float64 tensor of {self.m} entries")
        return C.c_void_p(d.data_ptr())

    def _call4(self, name, x, rows_in, d, rows_out, out):
        import torch

        x2 = x.reshape(-1, rows_in) if x.dim() != 2 else x
        nrhs = x2.shape[0]
        y = out if out is not None else torch.empty((nrhs, rows_out), dtype=self.torch_dtype, device=self.device)
        self._stream()
        _check(getattr(load_library(), name)(self._h, _dev_ptr(x2, rows_in, nrhs, self.torch_dtype), self._diag_ptr(d),
                                             _dev_ptr(y, rows_out, nrhs, self.torch_dtype), nrhs), name)
        return y

    def apply_diag(self, c, d, out=None):
        """f = Phi diag(d) c  (spectral filter F(lambda_k) = d_k, §7.1)."""
        return self._call4("mht_apply_diag", c, self.m, d, self.n, out)

    def adjoint_diag(self, f, d, out=None):
        """c = diag(d) Phi^* f."""
        return self._call4("mht_apply_adjoint_diag", f, self.n, d, self.m, out)

    def grf_sample(self, z, S, out=None):
        """y = Phi sqrt(S) z  (Karhunen-Loeve sample, §7.2; z supplied by the caller)."""
        return self._call4("mht_grf_sample", z, self.m, S, self.n, out)

    def covariance_apply(self, v, S, out=None):
        """out = Phi S Phi^* v  (covariance matvec, §7.2)."""
        return self._call4("mht_covariance_apply", v, self.n, S, self.n, out)

    def lsqr(self, b, max_iters: int, atol: float = 0.0, btol: float = 0.0, out=None):
        """Inverse MHT x = argmin ||Phi x - b|| by LSQR (§7.1).  Returns
        (x, iterations, rnorm[nrhs], arnorm[nrhs])."""
        import torch

        b2 = b.reshape(-1, self.n) if b.dim() != 2 else b
        nrhs = b2.shape[0]
        x = out if out is not None else torch.empty((nrhs, self.m), dtype=self.torch_dtype, device=self.device)
        it = C.c_int32()
        rn = (C.c_double * nrhs)()
        an = (C.c_double * nrhs)()
        self._stream()
        _check(load_library().mht_lsqr(self._h, _dev_ptr(b2, self.n, nrhs, self.torch_dtype),
                                       _dev_ptr(x, self.m, nrhs, self.torch_dtype), nrhs, int(max_iters),
                                       float(atol), float(btol), C.byref(it), rn, an), "mht_lsqr")
        return x, it.value, np.array(rn[:]), np.array(an[:])

    def _host_out(self, out, nrhs: int, rows: int):
        """A caller-supplied host output must be exactly what the C side writes:
        nrhs*rows scalars of the plan's dtype, C-contiguous and writeable (the
        device-to-host copy cannot check any of this)."""
        if out is None:
            return np.empty((nrhs, rows), dtype=self.np_dtype)
        if not isinstance(out, np.ndarray) or out.dtype != self.np_dtype or not out.flags.c_contiguous \
                or not out.flags.writeable or out.size != nrhs * rows:
            raise MhtError(f"host output must be a writeable C-contiguous {np.dtype(self.np_dtype).name} array of "
                           f"{nrhs} x {rows} entries")
        return out

    def apply_host(self, c_host: np.ndarray, f_host: np.ndarray | None = None):
        """End-to-end call from host memory (pinned for full bandwidth)."""
        c_host = np.ascontiguousarray(c_host, dtype=self.np_dtype).reshape(-1, self.m)
        nrhs = c_host.shape[0]
        f_host = self._host_out(f_host, nrhs, self.n)
        self._stream()
        _check(load_library().mht_apply_host(self._h, C.c_void_p(c_host.ctypes.data),
                                             C.c_void_p(f_host.ctypes.data), nrhs), "mht_apply_host")
        return f_host

    def adjoint_host(self, f_host: np.ndarray, c_host: np.ndarray | None = None):
        f_host = np.ascontiguousarray(f_host, dtype=self.np_dtype).reshape(-1, self.n)
        nrhs = f_host.shape[0]
        c_host = self._host_out(c_host, nrhs, self.m)
        self._stream()
        _check(load_library().mht_apply_adjoint_host(self._h, C.c_void_p(f_host.ctypes.data),
                                                     C.c_void_p(c_host.ctypes.data), nrhs),
               "mht_apply_adjoint_host")
        return c_host

    def host_batch_ptr(self, jobs):
        """mht_apply_host_batch over [(dir, nrhs, in_ptr, out_ptr), ...] (host
        pointers in the ABI layout; the caller keeps the buffers alive)."""
        arr = (HostJob * len(jobs))(*[HostJob(int(d), int(r), C.c_void_p(i), C.c_void_p(o)) for d, r, i, o in jobs])
        self._stream()
        _check(load_library().mht_apply_host_batch(self._h, arr, len(jobs)), "mht_apply_host_batch")

    def host_batch(self, jobs):
        """jobs: [(dir, host input array)] -> list of host outputs (numpy,
        pinned-or-not; checked like apply_host)."""
        ins, outs, spec = [], [], []
        for d, x in jobs:
            rows_in, rows_out = (self.m, self.n) if d == 0 else (self.n, self.m)
            x = np.ascontiguousarray(x, dtype=self.np_dtype).reshape(-1, rows_in)
            o = self._host_out(None, x.shape[0], rows_out)
            ins.append(x)
            outs.append(o)
            spec.append((d, x.shape[0], x.ctypes.data, o.ctypes.data))
        self.host_batch_ptr(spec)
        return outs

    def apply_host_ptr(self, c_ptr: int, f_ptr: int, nrhs: int):
        self._stream()
        _check(load_library().mht_apply_host(self._h, C.c_void_p(c_ptr), C.c_void_p(f_ptr), nrhs), "mht_apply_host")

    def adjoint_host_ptr(self, f_ptr: int, c_ptr: int, nrhs: int):
        self._stream()
        _check(load_library().mht_apply_adjoint_host(self._h, C.c_void_p(f_ptr), C.c_void_p(c_ptr), nrhs),
               "mht_apply_adjoint_host")

    def sync(self):
        _check(load_library().mht_sync(self._h), "mht_sync")

    def set_graphs(self, on: bool):
        _check(load_library().mht_set_graphs(self._h, int(bool(on))), "mht_set_graphs")

    def set_fused_sums(self, on: bool):
        """Adjoint group sums on the consumer's load (True, default) or as a
        separate reduce pass per stage (False); bitwise identical results."""
        _check(load_library().mht_set_fused_sums(self._h, int(bool(on))), "mht_set_fused_sums")

    def stage_stats(self):
        out = []
        for s in range(self.L + 2):
            cb = C.c_int64()
            nm, tf, ta = C.c_int32(), C.c_int32(), C.c_int32()
            _check(load_library().mht_stage_stats(self._h, s, C.byref(cb), C.byref(nm), C.byref(tf), C.byref(ta)),
                   "mht_stage_stats")
            out.append(dict(stage=s, coef_bytes=cb.value, n_mat=nm.value, fwd_tiles=tf.value, adj_tiles=ta.value))
        return out

    def set_profiling(self, on: bool):
        _check(load_library().mht_set_profiling(self._h, int(bool(on))), "mht_set_profiling")

    def profile_reset(self):
        _check(load_library().mht_profile_reset(self._h), "mht_profile_reset")

    def profile_get(self, kind: int, stage: int = -1, nrhs: int = 0):
        """(total ms, launches) of recorded launches; kind 0 fwd, 1 adj, 2 group-sum."""
        ms, n = C.c_double(), C.c_int64()
        _check(load_library().mht_profile_get(self._h, kind, stage, nrhs, C.byref(ms), C.byref(n)), "mht_profile_get")
        return ms.value, n.value

    def close(self):
        if getattr(self, "_h", None):
            mht_plan_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
