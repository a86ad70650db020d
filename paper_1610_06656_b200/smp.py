"""Thin Python layer over libsmp.so: torch tensors in, torch tensors out.

PyTorch supplies device memory, streams and torch.distributed; every step of
SMP-PCA runs in the library's sm_100a kernels.  Names follow the paper
(arXiv 1610.06656): Alg. 1 — sketch (Step 1), sample_estimate
(Step 2, Eqs. 1-2), waltmin (Step 3, Alg. 2).
"""
from __future__ import annotations

import ctypes
import math

import torch

from . import _lib
from ._lib import (EST_PLAIN, EST_RESCALED, IN_CSR_F32, IN_DENSE_BF16, IN_DENSE_F32,
                   PI_GAUSSIAN, PI_HADAMARD_TEST, PI_RADEMACHER, PI_SRHT, SmpError)

__all__ = ["SMPSketch", "smp_pca", "lela", "PI_RADEMACHER", "PI_GAUSSIAN", "PI_HADAMARD_TEST", "PI_SRHT",
           "IN_DENSE_BF16", "IN_DENSE_F32", "IN_CSR_F32", "SmpError"]


class _DevArray:
    """Expose a raw device pointer to torch via __cuda_array_interface__."""

    def __init__(self, ptr, n, typestr, owner):
        self._owner = owner
        self.__cuda_array_interface__ = {
            "shape": (int(n),), "typestr": typestr, "data": (int(ptr), False), "version": 3,
            "strides": None, "stream": None,
        }


def _ptr(t):
    return ctypes.c_void_p(0 if t is None else t.data_ptr())


def _check_dense(t, name):
    if not (t.dim() == 2 and t.stride(1) == 1):
        raise ValueError(f"{name} must be a 2-D row-major tensor (stride(1) == 1)")


class SMPSketch:
    """One handle of the one-pass sketch (Alg. 1 line 2 onwards)."""

    def __init__(self, d_total, n1, n2, k, pi=PI_RADEMACHER, seed=0, a_is_b=False,
                 input=IN_DENSE_BF16, row_begin=0, row_end=None, stream=None, device=None):
        self.lib = _lib.load()
        if not torch.cuda.is_available():
            raise RuntimeError("SMP-PCA kernels need a CUDA device (no CPU fallback)")
        if device is None:
            device = torch.cuda.current_device()
        if isinstance(device, torch.device):
            device = device.index if device.index is not None else torch.cuda.current_device()
        self.device = torch.device("cuda", int(device))
        self.stream = stream if stream is not None else torch.cuda.current_stream(self.device)
        self.n1, self.n2 = int(n1), int(n1 if a_is_b else n2)
        self.k, self.a_is_b, self.input = int(k), bool(a_is_b), int(input)
        desc = _lib.SketchDesc(d_total, n1, 0 if a_is_b else n2, k, pi, seed, int(a_is_b), input,
                               row_begin, d_total if row_end is None else row_end)
        h = ctypes.c_void_p()
        with torch.cuda.device(self.device):
            st = self.lib.smp_sketch_init(ctypes.byref(h), ctypes.byref(desc),
                                          ctypes.c_void_p(self.stream.cuda_stream))
        if st != 0:
            raise SmpError(st, f"smp_sketch_init failed: {self.lib.smp_status_str(st).decode()}")
        self.h = h

    # ------------------------------------------------------------- helpers
    def _check(self, st, what):
        if st != 0:
            msg = self.lib.smp_last_error(self.h).decode()
            raise SmpError(st, f"{what}: {self.lib.smp_status_str(st).decode()}: {msg}")

    def close(self):
        if getattr(self, "h", None):
            self.lib.smp_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def reset(self):
        """Zero the accumulators for another pass over new data."""
        self._check(self.lib.smp_sketch_reset(self.h), "smp_sketch_reset")

    def set_timing(self, enable=True):
        self._check(self.lib.smp_set_timing(self.h, int(enable)), "smp_set_timing")

    def kernel_timing(self):
        """(summed K1 device ms, number of K1 launches) since the last query."""
        ms, n = ctypes.c_double(), ctypes.c_int64()
        self._check(self.lib.smp_kernel_timing(self.h, ctypes.byref(ms), ctypes.byref(n)),
                    "smp_kernel_timing")
        return ms.value, n.value

    @property
    def kernel_launches(self) -> int:
        return int(self.lib.smp_kernel_launches(self.h))

    # ------------------------------------------------------------- Step 1
    def block(self, row0, A, B=None):
        """Accumulate rows [row0, row0 + A.shape[0]) of A (and B)."""
        _check_dense(A, "A")
        if not self.a_is_b:
            _check_dense(B, "B")
        st = self.lib.smp_sketch_block(self.h, row0, A.shape[0], _ptr(A), A.stride(0),
                                       _ptr(None if self.a_is_b else B),
                                       0 if self.a_is_b else B.stride(0))
        self._check(st, "smp_sketch_block")

    def block_host(self, row0, A, B=None, chunk_rows=0):
        """Same as block() for host tensors (the library stages the copies)."""
        _check_dense(A, "A")
        if not self.a_is_b:
            _check_dense(B, "B")
        st = self.lib.smp_sketch_block_host(self.h, row0, A.shape[0], _ptr(A), A.stride(0),
                                            _ptr(None if self.a_is_b else B),
                                            0 if self.a_is_b else B.stride(0), chunk_rows)
        self._check(st, "smp_sketch_block_host")

    def norms_block(self, row0, A, B=None):
        """LELA pass 1: exact column norms of rows [row0, row0 + A.shape[0])."""
        _check_dense(A, "A")
        if not self.a_is_b:
            _check_dense(B, "B")
        st = self.lib.smp_norms_block(self.h, row0, A.shape[0], _ptr(A), A.stride(0),
                                      _ptr(None if self.a_is_b else B), 0 if self.a_is_b else B.stride(0))
        self._check(st, "smp_norms_block")

    def exact_entries_block(self, row0, A, B, I, J, acc):
        """LELA pass 2: acc[s] += Σ_t A[t, I_s] B[t, J_s] over this block."""
        _check_dense(A, "A")
        if not self.a_is_b:
            _check_dense(B, "B")
        st = self.lib.smp_exact_entries_block(self.h, row0, A.shape[0], _ptr(A), A.stride(0),
                                              _ptr(None if self.a_is_b else B),
                                              0 if self.a_is_b else B.stride(0), _ptr(I), _ptr(J),
                                              I.numel(), _ptr(acc))
        self._check(st, "smp_exact_entries_block")

    def block_csr(self, row0, rows, a_rowptr, a_col, a_val, b_rowptr=None, b_col=None, b_val=None):
        st = self.lib.smp_sketch_block_csr(
            self.h, row0, rows, _ptr(a_rowptr), _ptr(a_col), _ptr(a_val), a_col.numel(),
            _ptr(b_rowptr), _ptr(b_col), _ptr(b_val), 0 if b_col is None else b_col.numel())
        self._check(st, "smp_sketch_block_csr")

    def partials(self):
        """(fp32 unscaled sketch sums, fp64 norms²) as torch views, for one
        all-reduce across row shards."""
        sk, skn, nr, nrn = ctypes.c_void_p(), ctypes.c_int64(), ctypes.c_void_p(), ctypes.c_int64()
        self._check(self.lib.smp_sketch_partials(self.h, ctypes.byref(sk), ctypes.byref(skn),
                                                 ctypes.byref(nr), ctypes.byref(nrn)),
                    "smp_sketch_partials")
        a = torch.as_tensor(_DevArray(sk.value, skn.value, "<f4", self), device=self.device)
        b = torch.as_tensor(_DevArray(nr.value, nrn.value, "<f8", self), device=self.device)
        return a, b

    def pack_partials(self):
        """The partials as ONE fp64 device buffer [sketch sums | norms²]
        (smp_sketch_pack_partials) for a single all-reduce across row shards
        (DESIGN.md §6); enqueued on the handle's stream."""
        buf, n = ctypes.c_void_p(), ctypes.c_int64()
        self._check(self.lib.smp_sketch_pack_partials(self.h, ctypes.byref(buf), ctypes.byref(n)),
                    "smp_sketch_pack_partials")
        return torch.as_tensor(_DevArray(buf.value, n.value, "<f8", self), device=self.device)

    def unpack_partials(self):
        """Write the (all-reduced) exchange buffer back into the accumulators."""
        self._check(self.lib.smp_sketch_unpack_partials(self.h), "smp_sketch_unpack_partials")

    def finalize(self):
        dev = self.device
        A_sk = torch.empty(self.n1, self.k, dtype=torch.float32, device=dev)
        B_sk = torch.empty(self.n2, self.k, dtype=torch.float32, device=dev)
        a2 = torch.empty(self.n1, dtype=torch.float64, device=dev)
        b2 = torch.empty(self.n2, dtype=torch.float64, device=dev)
        fr = torch.empty(2, dtype=torch.float64, device=dev)
        asn = torch.empty(self.n1, dtype=torch.float32, device=dev)
        bsn = torch.empty(self.n2, dtype=torch.float32, device=dev)
        st = self.lib.smp_finalize_norms(self.h, _ptr(A_sk), _ptr(B_sk), _ptr(a2), _ptr(b2),
                                         _ptr(fr), _ptr(asn), _ptr(bsn))
        self._check(st, "smp_finalize_norms")
        return dict(A_sk=A_sk, B_sk=B_sk, a_norm2=a2, b_norm2=b2, frob2=fr, a_sknorm=asn,
                    b_sknorm=bsn)

    # ------------------------------------------------------------- Step 2
    def sample_estimate(self, m, seed, plain=False, cap=None, sampler="bernoulli"):
        """Ω (sorted by (i,j)), M̃ on Ω and q̂ (Alg. 1 lines 3-4).  sampler:
        "bernoulli" (Alg. 1 line 3) or "multinomial" (the appendix's
        row-multinomial sampler with line 3's saturation, R27:
        each drawn pair once, q̂ = its inclusion probability)."""
        smode = {"bernoulli": _lib.SAMPLER_BERNOULLI, "multinomial": _lib.SAMPLER_MULTINOMIAL}[sampler]
        if cap is None:
            cap = int(min(self.n1 * self.n2, m + 10 * math.sqrt(max(m, 1.0)) + 1024))
        dev = self.device
        while True:
            I = torch.empty(max(cap, 1), dtype=torch.int32, device=dev)
            J = torch.empty(max(cap, 1), dtype=torch.int32, device=dev)
            val = torch.empty(max(cap, 1), dtype=torch.float32, device=dev)
            qh = torch.empty(max(cap, 1), dtype=torch.float64, device=dev)
            cnt = ctypes.c_int64()
            st = self.lib.smp_sample_estimate_ex(self.h, float(m), seed,
                                                 EST_PLAIN if plain else EST_RESCALED, smode, cap,
                                                 _ptr(I), _ptr(J), _ptr(val), _ptr(qh), ctypes.byref(cnt))
            if st == _lib.SMP_ECAPACITY:
                cap = int(cnt.value)
                continue
            self._check(st, "smp_sample_estimate")
            c = int(cnt.value)
            return I[:c], J[:c], val[:c], qh[:c]

    # ------------------------------------------------------------- Step 3
    def svd_of_sketch(self, r, T=10, init_iters=30, seed=0):
        """Rank-r SVD of ÃᵀB̃ — the sketch-only baseline the paper compares
        against (Figs. 2b/4b), on the GPU through the
        same C ABI: Ω = every pair (q̂ = 1, w = 1), M̃ = ⟨Ã_i, B̃_j⟩ (the plain JL
        estimator), then WAltMin without trimming — fully observed ALS
        from a subspace-iteration start converges to (ÃᵀB̃)_r.  Returns (U, V)."""
        # q = m(α_i + β_j) >= 1 for every pair with a nonzero column (pairs of two
        # all-zero columns have (ÃᵀB̃)_ij = 0 and are not needed)
        I, J, val, qh = self.sample_estimate(1e30, seed, plain=True, cap=self.n1 * self.n2)
        return self.waltmin(I, J, val, qh, r, T, init_iters=init_iters, trim_c=0.0, seed=seed)

    def waltmin(self, I, J, val, qhat, r, T, init_iters=30, trim_c=8.0, ridge=1e-10, seed=0,
                partition="reuse_all"):
        """Alg. 2.  partition: "reuse_all" or "fresh_2t1" (line 3,
        2T+1 random subsets; R11)."""
        dev = self.device
        U = torch.empty(self.n1, r, dtype=torch.float32, device=dev)
        V = torch.empty(self.n2, r, dtype=torch.float32, device=dev)
        part = {"reuse_all": _lib.PART_REUSE_ALL, "fresh_2t1": _lib.PART_FRESH_2T1}[partition]
        w = _lib.WaltminDesc(r, T, part, init_iters, trim_c, ridge, seed)
        st = self.lib.smp_waltmin(self.h, _ptr(I), _ptr(J), _ptr(val), _ptr(qhat), I.numel(),
                                  ctypes.byref(w), _ptr(U), _ptr(V))
        self._check(st, "smp_waltmin")
        return U, V


def lela(A, B, r, m, T, seed=0, wm_seed=None, init_iters=30, trim_c=8.0, ridge=1e-10, a_is_b=False,
         partition="reuse_all", row_block=None):
    """LELA (the paper's two-pass comparison system) on
    device-resident dense A (and B), through the same C ABI: pass 1 exact
    column norms, Ω and q̂ by Eq. 1 (the SMP-PCA sampler), pass 2 exact
    entries (AᵀB)_Ω, WAltMin.  row_block streams each pass in row blocks."""
    inp = IN_DENSE_BF16 if A.dtype == torch.bfloat16 else IN_DENSE_F32
    d = A.shape[0]
    n2 = A.shape[1] if a_is_b else B.shape[1]
    sk = SMPSketch(d, A.shape[1], n2, 1, pi=PI_RADEMACHER, seed=seed, a_is_b=a_is_b, input=inp,
                   device=A.device)
    rb = d if row_block is None else int(row_block)
    try:
        for r0 in range(0, d, rb):
            sk.norms_block(r0, A[r0:r0 + rb], None if a_is_b else B[r0:r0 + rb])
        fin = sk.finalize()
        I, J, _, qh = sk.sample_estimate(m, seed)
        acc = torch.zeros(I.numel(), dtype=torch.float64, device=A.device)
        for r0 in range(0, d, rb):
            sk.exact_entries_block(r0, A[r0:r0 + rb], None if a_is_b else B[r0:r0 + rb], I, J, acc)
        val = acc.float()
        U, V = sk.waltmin(I, J, val, qh, r, T, init_iters=init_iters, trim_c=trim_c, ridge=ridge,
                          seed=seed if wm_seed is None else wm_seed, partition=partition)
        fin.update(I=I, J=J, val=val, acc=acc, qhat=qh, U=U, V=V, launches=sk.kernel_launches)
        return fin
    finally:
        sk.close()


def smp_pca(A, B, k, r, m, T, pi=PI_RADEMACHER, seed=0, omega_seed=None, wm_seed=None,
            init_iters=30, trim_c=8.0, ridge=1e-10, a_is_b=False, plain=False, row0=0,
            d_total=None, sampler="bernoulli", partition="reuse_all"):
    """Alg. 1 end to end on device-resident dense A (and B): returns a dict
    with the finalized sketch state, Ω, M̃, q̂ and the factors (U, V)."""
    inp = IN_DENSE_BF16 if A.dtype == torch.bfloat16 else IN_DENSE_F32
    d = A.shape[0] if d_total is None else d_total
    sk = SMPSketch(d, A.shape[1], A.shape[1] if a_is_b else B.shape[1], k, pi=pi, seed=seed,
                   a_is_b=a_is_b, input=inp, device=A.device)
    try:
        sk.block(row0, A, None if a_is_b else B)
        fin = sk.finalize()
        I, J, val, qh = sk.sample_estimate(m, seed if omega_seed is None else omega_seed, plain=plain,
                                           sampler=sampler)
        U, V = sk.waltmin(I, J, val, qh, r, T, init_iters=init_iters, trim_c=trim_c, ridge=ridge,
                          seed=seed if wm_seed is None else wm_seed, partition=partition)
        fin.update(I=I, J=J, val=val, qhat=qh, U=U, V=V, launches=sk.kernel_launches)
        return fin
    finally:
        sk.close()
