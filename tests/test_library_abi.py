"""CPU-side checks of the boundary: libmht.so builds for sm_100a, loads, and
exports every symbol include/mht.h and include/mht_build.h declare (no compute
calls without a GPU)."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols(header="mht.h", prefix="mht_"):
    src = open(os.path.join(ROOT, "include", header)).read()
    return sorted(set(re.findall(rf"\b({prefix}[a-z_]+)\s*\(", src)))


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


def test_library_exports_build_kernels(libpath):
    """include/mht_build.h (NEXT-1 plan-construction kernels)."""
    syms = declared_symbols("mht_build.h", "mhtb_")
    assert syms == ["mhtb_cpqr", "mhtb_flat_blocks", "mhtb_sphere_table"]
    out = subprocess.run(["nm", "-D", "--defined-only", libpath], capture_output=True, text=True).stdout
    for s in syms:
        assert re.search(rf"\bT {s}$", out, re.M), s


def test_build_kernels_reject_bad_args_without_gpu(libpath):
    from paper_2605_21828_b200.precompute import devkern

    L = devkern._lib()
    assert L.mhtb_flat_blocks(None, None, None, None, -1, 1, 1, None, None) == 1
    assert L.mhtb_flat_blocks(None, None, None, None, 1, 1, 1, None, None) == 1
    assert L.mhtb_sphere_table(None, None, 4, -1, None, None) == 1
    assert L.mhtb_cpqr(None, 1, 1, 1, 7, 1e-8, None, None, None) == 1
    assert L.mhtb_cpqr(None, 1, 4, 4, 2, 1e-8, None, None, None) == 1
    # nothing to do: no device touched
    assert L.mhtb_flat_blocks(None, None, None, None, 0, 5, 5, None, None) == 0
    assert L.mhtb_cpqr(None, 0, 4, 4, 1, 1e-8, None, None, None) == 0


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
