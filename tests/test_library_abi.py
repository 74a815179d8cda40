"""CPU-side checks of the boundary: libmht.so builds for sm_100a, loads, and
exports every symbol include/mht.h declares (no compute calls without a GPU)."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "mht.h")).read()
    return sorted(set(re.findall(r"\b(mht_[a-z_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def libpath():
    from paper_2605_21828_b200 import _build

    return _build.build()


def test_library_exports_every_declared_symbol(libpath):
    syms = declared_symbols()
    assert "mht_plan_load" in syms and "mht_apply" in syms and "mht_apply_adjoint" in syms
    lib = ctypes.CDLL(libpath)
    for s in syms:
        assert hasattr(lib, s), s
    out = subprocess.run(["nm", "-D", "--defined-only", libpath], capture_output=True, text=True).stdout
    for s in syms:
        assert re.search(rf"\bT {s}$", out, re.M), s


def test_binding_names_match_header():
    from paper_2605_21828_b200 import mht

    assert sorted(mht.EXPORTED) == declared_symbols()


def test_library_is_sm100a(libpath):
    out = subprocess.run(["cuobjdump", "--list-elf", libpath], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_status_strings_without_gpu(libpath):
    from paper_2605_21828_b200 import mht

    L = mht.load_library()
    assert L.mht_status_string(0) == b"MHT_OK"
    assert L.mht_status_string(2) == b"MHT_ERR_FORMAT"
    assert b"sm_100a" in L.mht_build_info()
    # invalid arguments are rejected before touching the device
    h = ctypes.c_void_p()
    assert L.mht_plan_load(None, 0, ctypes.byref(h)) == 1
    assert L.mht_apply(None, None, None, 1) == 1
    assert L.mht_apply_adjoint(None, None, None, 0) == 1
