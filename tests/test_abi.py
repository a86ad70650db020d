"""CPU-side checks of the C-ABI library: it loads without a GPU and exports
every entry point include/smp.h declares (no compute calls here)."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "smp.h")


def declared_symbols():
    txt = open(HEADER).read()
    return sorted(set(re.findall(r"SMP_API[^;(]*?\b(smp_[a-z_]+)\s*\(", txt)))


@pytest.fixture(scope="module")
def lib_path():
    from paper_1610_06656_b200 import build
    return build.build()


def test_header_declares_the_five_calls():
    syms = declared_symbols()
    for s in ["smp_sketch_init", "smp_sketch_block", "smp_finalize_norms", "smp_sample_estimate",
              "smp_waltmin"]:
        assert s in syms


def test_library_exports_every_declared_symbol(lib_path):
    lib = ctypes.CDLL(lib_path)
    for s in declared_symbols():
        assert hasattr(lib, s), s
    out = subprocess.run(["nm", "-D", "--defined-only", lib_path], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (smp_[a-z_]+)", out))
    assert set(declared_symbols()) <= exported


def test_status_strings_without_gpu(lib_path):
    from paper_1610_06656_b200 import _lib
    lib = _lib.load(lib_path)
    assert lib.smp_status_str(3) == b"SMP_EINVAL"
    assert lib.smp_status_str(6) == b"SMP_ECAPACITY"
    assert lib.smp_last_error(None) == b"null handle"


def test_init_validation_is_synchronous(lib_path):
    """Invalid descriptors are rejected before any CUDA work (no GPU needed)."""
    from paper_1610_06656_b200 import _lib
    lib = _lib.load(lib_path)
    h = ctypes.c_void_p()
    bad = [
        _lib.SketchDesc(100, 10, 10, 0, 0, 0, 0, 0, 0, 100),       # k < 1
        _lib.SketchDesc(100, 0, 10, 8, 0, 0, 0, 0, 0, 100),        # n1 < 1
        _lib.SketchDesc(100, 10, 10, 8, 0, 0, 0, 0, 50, 40),       # bad row range
        _lib.SketchDesc(100, 10, 10, 100, 2, 0, 0, 0, 0, 100),     # Hadamard, d not 2^k
        _lib.SketchDesc(128, 10, 10, 64, 2, 0, 0, 0, 0, 128),      # Hadamard, k != d
        _lib.SketchDesc(100, 10, 10, 8, 7, 0, 0, 0, 0, 100),       # unknown Π kind
    ]
    for d in bad:
        assert lib.smp_sketch_init(ctypes.byref(h), ctypes.byref(d), None) == 3


def test_kernels_are_sm100a_tensor_core_code(lib_path):
    """SASS evidence of tcgen05 (UTC*MMA), TMEM loads (LDTM) and TMA (UTMALDG)."""
    out = subprocess.run(["cuobjdump", "-sass", lib_path], capture_output=True, text=True).stdout
    assert re.search(r"UTC\w*MMA", out)
    assert "UTMALDG" in out
    assert "LDTM" in out
