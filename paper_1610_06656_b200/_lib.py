"""ctypes binding of libsmp.so (include/smp.h) — argument marshalling only.

Every step of the hot path runs in the CUDA kernels behind these entry
points.  There is deliberately no fallback: if the in-tree libsmp.so is
missing or a CUDA device is absent, loading raises.
"""
from __future__ import annotations

import ctypes
import os

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_PKG, "libsmp.so")

SMP_OK, SMP_EIO, SMP_EINVAL, SMP_ENUMERIC, SMP_ECUDA, SMP_ECAPACITY, SMP_ENOMEM = 0, 2, 3, 4, 5, 6, 7
PI_RADEMACHER, PI_GAUSSIAN, PI_HADAMARD_TEST, PI_SRHT = 0, 1, 2, 3
IN_DENSE_BF16, IN_DENSE_F32, IN_CSR_F32 = 0, 1, 2
EST_RESCALED, EST_PLAIN = 0, 1
PART_REUSE_ALL, PART_FRESH_2T1 = 0, 1
SAMPLER_BERNOULLI, SAMPLER_MULTINOMIAL = 0, 1

EXPORTS = [
    "smp_sketch_init", "smp_sketch_block", "smp_sketch_block_host", "smp_sketch_block_csr",
    "smp_sketch_partials", "smp_finalize_norms", "smp_sample_estimate", "smp_waltmin",
    "smp_sketch_reset", "smp_kernel_launches", "smp_destroy", "smp_last_error", "smp_status_str",
    "smp_set_timing", "smp_kernel_timing", "smp_sample_estimate_ex", "smp_norms_block",
    "smp_exact_entries_block", "smp_sketch_pack_partials", "smp_sketch_unpack_partials",
]


class SketchDesc(ctypes.Structure):
    _fields_ = [
        ("d_total", ctypes.c_int64), ("n1", ctypes.c_int64), ("n2", ctypes.c_int64),
        ("k", ctypes.c_int32), ("pi_kind", ctypes.c_int32), ("seed", ctypes.c_uint64),
        ("a_is_b", ctypes.c_int32), ("input", ctypes.c_int32),
        ("row_begin", ctypes.c_int64), ("row_end", ctypes.c_int64),
    ]


class WaltminDesc(ctypes.Structure):
    _fields_ = [
        ("r", ctypes.c_int32), ("T", ctypes.c_int32), ("partition", ctypes.c_int32),
        ("init_iters", ctypes.c_int32), ("trim_c", ctypes.c_double), ("ridge", ctypes.c_double),
        ("seed", ctypes.c_uint64),
    ]


class SmpError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"{msg} (status {status})")
        self.status = status


_lib = None


def load(path: str = None):
    """Load libsmp.so and declare signatures (no CUDA work happens here).
    SMP_LIB may name an alternative in-tree build (tuning experiments)."""
    global _lib
    if _lib is not None:
        return _lib
    if path is None:
        path = os.environ.get("SMP_LIB", LIB_PATH)
    if not os.path.exists(path):
        raise FileNotFoundError(
            f"{path} missing: build it with `python -m paper_1610_06656_b200.build` "
            "(there is no CPU fallback)")
    lib = ctypes.CDLL(path)
    P, i64, i32, u64, f64 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_uint64, ctypes.c_double
    H = ctypes.c_void_p
    lib.smp_sketch_init.argtypes = [ctypes.POINTER(H), ctypes.POINTER(SketchDesc), P]
    lib.smp_sketch_block.argtypes = [H, i64, i64, P, i64, P, i64]
    lib.smp_sketch_block_host.argtypes = [H, i64, i64, P, i64, P, i64, i64]
    lib.smp_sketch_block_csr.argtypes = [H, i64, i64, P, P, P, i64, P, P, P, i64]
    lib.smp_sketch_partials.argtypes = [H, ctypes.POINTER(P), ctypes.POINTER(i64),
                                        ctypes.POINTER(P), ctypes.POINTER(i64)]
    lib.smp_sketch_pack_partials.argtypes = [H, ctypes.POINTER(P), ctypes.POINTER(i64)]
    lib.smp_sketch_unpack_partials.argtypes = [H]
    lib.smp_finalize_norms.argtypes = [H, P, P, P, P, P, P, P]
    lib.smp_sample_estimate.argtypes = [H, f64, u64, i32, i64, P, P, P, P, ctypes.POINTER(i64)]
    lib.smp_sample_estimate_ex.argtypes = [H, f64, u64, i32, i32, i64, P, P, P, P, ctypes.POINTER(i64)]
    lib.smp_waltmin.argtypes = [H, P, P, P, P, i64, ctypes.POINTER(WaltminDesc), P, P]
    lib.smp_norms_block.argtypes = [H, i64, i64, P, i64, P, i64]
    lib.smp_exact_entries_block.argtypes = [H, i64, i64, P, i64, P, i64, P, P, i64, P]
    lib.smp_sketch_reset.argtypes = [H]
    lib.smp_set_timing.argtypes = [H, i32]
    lib.smp_kernel_timing.argtypes = [H, ctypes.POINTER(f64), ctypes.POINTER(i64)]
    lib.smp_kernel_launches.argtypes = [H]
    lib.smp_kernel_launches.restype = i64
    lib.smp_destroy.argtypes = [H]
    lib.smp_destroy.restype = None
    lib.smp_last_error.argtypes = [H]
    lib.smp_last_error.restype = ctypes.c_char_p
    lib.smp_status_str.argtypes = [ctypes.c_int]
    lib.smp_status_str.restype = ctypes.c_char_p
    for name in EXPORTS:
        if name not in ("smp_destroy", "smp_last_error", "smp_status_str", "smp_kernel_launches"):
            getattr(lib, name).restype = ctypes.c_int
    _lib = lib
    return lib
