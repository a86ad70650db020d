"""ctypes wrapper around oracle/smp_oracle.c — TEST INFRASTRUCTURE ONLY.

Each function names the passage of PAPER.md ("P:L") it follows; the
definitions it relies on (hash, Gaussian generator, q̂ arithmetic, WAltMin
readings) are in DESIGN.md §3.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "smp_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

PI_RADEMACHER, PI_GAUSSIAN, PI_HADAMARD = 0, 1, 2
PART_REUSE_ALL, PART_FRESH_2T1 = 0, 1


def pi_srht(d: int) -> int:
    """Kind code of the SRHT Π for d rows (16 + L, 2^L >= d; R26)."""
    L = max(1, int(d - 1).bit_length())
    return 16 + L

_lib = None


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (plain -O2, no FMA contraction)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        cmd = ["gcc", "-O2", "-std=c11", "-fopenmp", "-ffp-contract=off", "-fno-fast-math",
               "-fPIC", "-shared", "-o", _LIB + ".tmp", _SRC, "-lm"]
        subprocess.check_call(cmd)
        os.replace(_LIB + ".tmp", _LIB)
    return _LIB


def _get():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_LIB)
        P = ctypes.c_void_p
        i64, i32, u64, f64 = ctypes.c_int64, ctypes.c_int32, ctypes.c_uint64, ctypes.c_double
        lib.or_philox4x32_10.argtypes = [P, P, P]
        lib.or_pi_entry.argtypes = [ctypes.c_int, u64, i64, i64]
        lib.or_pi_entry.restype = f64
        lib.or_sketch_rows.argtypes = [ctypes.c_int, u64, ctypes.c_int, i64, i64, i64, P,
                                       ctypes.c_int, i64, P, P]
        lib.or_sketch_cols.argtypes = [ctypes.c_int, u64, ctypes.c_int, i64, i64, i64, P, P,
                                       ctypes.c_int, i64, P, P]
        lib.or_sketch_csr.argtypes = [ctypes.c_int, u64, ctypes.c_int, i64, i64, i64, P, P, P,
                                      P, P]
        lib.or_sample_multinomial.argtypes = [u64, f64, i64, i64, P, P, i64, P, P, P]
        lib.or_sample_multinomial.restype = i64
        lib.or_srht_row.argtypes = [u64, ctypes.c_int, i64]
        lib.or_srht_row.restype = i64
        lib.or_srht_sign.argtypes = [u64, i64]
        lib.or_srht_sign.restype = f64
        lib.or_colnorms.argtypes = [i64, i64, P, ctypes.c_int, i64, P]
        lib.or_colnorms.restype = None
        lib.or_pairwise_sum.argtypes = [P, i64]
        lib.or_pairwise_sum.restype = f64
        lib.or_finalize.argtypes = [ctypes.c_int, i64, P, P, P, P, P]
        lib.or_alpha_beta.argtypes = [i64, i64, P, P, f64, f64, P, P]
        lib.or_qhat.argtypes = [f64, f64, f64]
        lib.or_qhat.restype = f64
        lib.or_draw.argtypes = [u64, i64, i64, f64]
        lib.or_draw.restype = ctypes.c_int
        lib.or_sample.argtypes = [u64, f64, i64, i64, P, P, i64, P, P, P]
        lib.or_sample.restype = i64
        lib.or_estimate.argtypes = [ctypes.c_int, i64, P, P, P, P, P, P, ctypes.c_int, P]
        lib.or_als_half.argtypes = [ctypes.c_int, i64, i64, P, P, P, P, P, f64, P]
        lib.or_waltmin.argtypes = [i64, i64, ctypes.c_int, ctypes.c_int, ctypes.c_int, f64, f64,
                                   u64, ctypes.c_int, i64, P, P, P, P, P, f64, P, P]
        lib.or_multinomial_draws.argtypes = [u64, f64, i64, i64, P, P, i64, P, P, P]
        lib.or_mn_rows.argtypes = [f64, i64, i64, P, P, P, P]
        lib.or_mn_rows.restype = None
        lib.or_multinomial_draws.restype = i64
        lib.or_mn_qhat.argtypes = [f64, f64, f64, f64]
        lib.or_mn_qhat.restype = f64
        lib.or_exact_entries.argtypes = [i64, P, ctypes.c_int, i64, P, ctypes.c_int, i64, i64, P, P, P]
        lib.or_exact_entries.restype = None
        lib.or_partition.argtypes = [u64, ctypes.c_int, i64, P, P, P]
        lib.or_partition.restype = None
        _lib = lib
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def _c(a, dtype):
    return np.ascontiguousarray(a, dtype=dtype)


# --------------------------------------------------------------------------
# Hash and Π (Alg. 1 line 2)
# --------------------------------------------------------------------------
def philox4x32_10(ctr, key) -> np.ndarray:
    c = _c(ctr, np.uint32)
    k = _c(key, np.uint32)
    out = np.zeros(4, np.uint32)
    _get().or_philox4x32_10(_p(c), _p(k), _p(out))
    return out


def pi_entry(kind: int, seed: int, kappa: int, t: int) -> float:
    """Unscaled Π(κ, t): ±1 (Rademacher / Hadamard) or a bf16-valued N(0,1)."""
    return _get().or_pi_entry(kind, seed, kappa, t)


def pi_matrix(kind: int, seed: int, k: int, t0: int, rows: int) -> np.ndarray:
    """Materialise unscaled Π[:, t0:t0+rows] (k x rows) — tests only."""
    lib = _get()
    out = np.empty((k, rows), np.float64)
    for kp in range(k):
        for r in range(rows):
            out[kp, r] = lib.or_pi_entry(kind, seed, kp, t0 + r)
    return out


# --------------------------------------------------------------------------
# Step 1: sketches and exact column norms in one pass
# --------------------------------------------------------------------------
def _dtype_code(X: np.ndarray) -> int:
    if X.dtype == np.float64:
        return 0
    if X.dtype == np.float32:
        return 1
    if X.dtype == np.uint16:  # raw bf16 bits
        return 2
    raise TypeError(X.dtype)


def sketch_rows(kind, seed, k, X, row0=0, sk=None, norm2=None):
    """Accumulate rows of X (rows x n, row-major) into the UNSCALED sketch sk
    (n x k, column i of Π X is sk[i]) and norm2 (n).  Returns (sk, norm2)."""
    X = np.ascontiguousarray(X)
    rows, n = X.shape
    if sk is None:
        sk = np.zeros((n, k), np.float64)
    if norm2 is None:
        norm2 = np.zeros(n, np.float64)
    _get().or_sketch_rows(kind, seed, k, row0, rows, n, _p(X), _dtype_code(X), n, _p(sk),
                          _p(norm2))
    return sk, norm2


def srht_row(seed: int, L: int, kappa: int) -> int:
    """s_κ = F_L(κ): the sampled Hadamard row of SRHT row κ (R26)."""
    return _get().or_srht_row(seed, L, kappa)


def srht_sign(seed: int, t: int) -> float:
    """D_t of the SRHT (R26)."""
    return _get().or_srht_sign(seed, t)


def colnorms(X, norm2=None):
    """norm2[c] += Σ_t X[t, c]² in fp64 (the norm half of Step 1)."""
    X = np.ascontiguousarray(X)
    rows, n = X.shape
    if norm2 is None:
        norm2 = np.zeros(n, np.float64)
    _get().or_colnorms(rows, n, _p(X), _dtype_code(X), n, _p(norm2))
    return norm2


def sketch_cols(kind, seed, k, X, cols, row0=0):
    """Unscaled sketch (len(cols) x k) and norms^2 of the selected columns of X."""
    X = np.ascontiguousarray(X)
    rows, n = X.shape
    cols = _c(cols, np.int64)
    sk = np.zeros((len(cols), k), np.float64)
    norm2 = np.zeros(len(cols), np.float64)
    _get().or_sketch_cols(kind, seed, k, row0, rows, len(cols), _p(cols), _p(X),
                          _dtype_code(X), n, _p(sk), _p(norm2))
    return sk, norm2


def sketch_csr(kind, seed, k, n, rowptr, col, val, row0=0, sk=None, norm2=None):
    rowptr = _c(rowptr, np.int64)
    col = _c(col, np.int32)
    val = _c(val, np.float32)
    rows = len(rowptr) - 1
    if sk is None:
        sk = np.zeros((n, k), np.float64)
    if norm2 is None:
        norm2 = np.zeros(n, np.float64)
    _get().or_sketch_csr(kind, seed, k, row0, rows, n, _p(rowptr), _p(col), _p(val), _p(sk),
                         _p(norm2))
    return sk, norm2


def pairwise_sum(x) -> float:
    """R5: fixed pairwise tree (power-of-two padded) sum, fp64."""
    x = _c(x, np.float64)
    return _get().or_pairwise_sum(_p(x), len(x))


def finalize(k, sk, norm2):
    """Scale by 1/sqrt(k) (N(0,1/k)); ||Ã_i||; D = ||X_i|| / ||Ã_i||.
    norm2 is flushed IN PLACE where below 2^-200 (R25) when it is a float64
    array (the caller's a2 then feeds Eq. 1 with the same zero)."""
    sk = _c(sk, np.float64)
    if not (isinstance(norm2, np.ndarray) and norm2.dtype == np.float64 and norm2.flags.c_contiguous):
        norm2 = _c(norm2, np.float64)
    n = sk.shape[0]
    out = np.empty_like(sk)
    sknorm = np.empty(n, np.float64)
    D = np.empty(n, np.float64)
    _get().or_finalize(k, n, _p(sk), _p(norm2), _p(out), _p(sknorm), _p(D))
    return out, sknorm, D


# --------------------------------------------------------------------------
# Step 2
# --------------------------------------------------------------------------
def alpha_beta(a2, b2, FA, FB):
    a2 = _c(a2, np.float64)
    b2 = _c(b2, np.float64)
    al = np.empty_like(a2)
    be = np.empty_like(b2)
    _get().or_alpha_beta(len(a2), len(b2), _p(a2), _p(b2), FA, FB, _p(al), _p(be))
    return al, be


def qhat(m, alpha_i, beta_j) -> float:
    return _get().or_qhat(m, alpha_i, beta_j)


def draw(seed, i, j, q) -> int:
    return _get().or_draw(seed, i, j, q)


def sample(seed, m, alpha, beta, cap=None):
    """Ω as (I, J, q̂), sorted by (i, j) (Alg. 1 line 3; Eq. 1)."""
    alpha = _c(alpha, np.float64)
    beta = _c(beta, np.float64)
    n1, n2 = len(alpha), len(beta)
    lib = _get()
    if cap is None:
        cap = int(min(n1 * n2, m + 10 * np.sqrt(max(m, 1.0)) + 1024))
    while True:
        I = np.empty(max(cap, 1), np.int32)
        J = np.empty(max(cap, 1), np.int32)
        q = np.empty(max(cap, 1), np.float64)
        cnt = lib.or_sample(seed, m, n1, n2, _p(alpha), _p(beta), cap, _p(I), _p(J), _p(q))
        if cnt <= cap:
            return I[:cnt].copy(), J[:cnt].copy(), q[:cnt].copy()
        cap = int(cnt)


def multinomial_draws(seed, m, alpha, beta):
    """Raw draws of the row-multinomial sampler's unsaturated part (
    R27): with replacement, sorted by (i, j), duplicates kept."""
    alpha = _c(alpha, np.float64)
    beta = _c(beta, np.float64)
    n1, n2 = len(alpha), len(beta)
    lib = _get()
    cnt = lib.or_multinomial_draws(seed, m, n1, n2, _p(alpha), _p(beta), 0, None, None, None)
    I = np.empty(max(cnt, 1), np.int32)
    J = np.empty(max(cnt, 1), np.int32)
    lib.or_multinomial_draws(seed, m, n1, n2, _p(alpha), _p(beta), cnt, _p(I), _p(J), None)
    return I[:cnt].copy(), J[:cnt].copy()


def mn_rows(m, alpha, beta):
    """(s_i, T_i) per row: saturated-prefix length and unsaturated mass (R27)."""
    alpha = _c(alpha, np.float64)
    beta = _c(beta, np.float64)
    s = np.empty(len(alpha), np.int64)
    T = np.empty(len(alpha), np.float64)
    _get().or_mn_rows(m, len(alpha), len(beta), _p(alpha), _p(beta), _p(s), _p(T))
    return s, T


def mn_qhat(m, alpha_i, beta_j, T_i) -> float:
    """Inclusion probability of (i, j) in the multinomial Ω (R27)."""
    return _get().or_mn_qhat(m, alpha_i, beta_j, T_i)


def sample_multinomial(seed, m, alpha, beta):
    """Ω by the appendix's row-multinomial sampler (R27): the SET
    of drawn pairs, sorted by (i, j), with q̂ = P((i, j) ∈ Ω)."""
    alpha = _c(alpha, np.float64)
    beta = _c(beta, np.float64)
    n1, n2 = len(alpha), len(beta)
    lib = _get()
    cap = int(m + 10 * np.sqrt(max(m, 1.0)) + 1024)
    while True:
        I = np.empty(max(cap, 1), np.int32)
        J = np.empty(max(cap, 1), np.int32)
        q = np.empty(max(cap, 1), np.float64)
        cnt = lib.or_sample_multinomial(seed, m, n1, n2, _p(alpha), _p(beta), cap, _p(I), _p(J), _p(q))
        if cnt <= cap:
            return I[:cnt].copy(), J[:cnt].copy(), q[:cnt].copy()
        cap = int(cnt)


def partition(seed, T, I, J):
    """Alg. 2 line 3 (R11 FRESH_2T1): subset id in [0, 2T+1) per sample."""
    I = _c(I, np.int32)
    J = _c(J, np.int32)
    sub = np.empty(max(len(I), 1), np.int32)
    _get().or_partition(seed, 2 * T + 1, len(I), _p(I), _p(J), _p(sub))
    return sub[:len(I)].copy()


def estimate(k, I, J, Ask, Bsk, DA, DB, plain=False):
    """Eq. 2 on Ω; plain=True gives the JL estimator."""
    I = _c(I, np.int32)
    J = _c(J, np.int32)
    Ask = _c(Ask, np.float64)
    Bsk = _c(Bsk, np.float64)
    DA = _c(DA, np.float64)
    DB = _c(DB, np.float64)
    out = np.empty(len(I), np.float64)
    _get().or_estimate(k, len(I), _p(I), _p(J), _p(Ask), _p(Bsk), _p(DA), _p(DB), int(plain),
                       _p(out))
    return out


# --------------------------------------------------------------------------
# Step 3 (Alg. 2)
# --------------------------------------------------------------------------
def als_half(r, n_out, side, other, val, w, X_other, lam=1e-10):
    side = _c(side, np.int32)
    other = _c(other, np.int32)
    val = _c(val, np.float64)
    w = _c(w, np.float64)
    X_other = _c(X_other, np.float64)
    out = np.zeros((n_out, r), np.float64)
    _get().or_als_half(r, n_out, len(side), _p(side), _p(other), _p(val), _p(w), _p(X_other),
                       lam, _p(out))
    return out


def waltmin(n1, n2, r, T, I, J, val, qhat_, a_norm, frobA, init_iters=50, trim_c=8.0,
            lam=1e-10, seed=0, partition=PART_REUSE_ALL):
    """Alg. 2; partition per R11 (REUSE_ALL or FRESH_2T1)."""
    I = _c(I, np.int32)
    J = _c(J, np.int32)
    val = _c(val, np.float64)
    qhat_ = _c(qhat_, np.float64)
    a_norm = _c(a_norm, np.float64)
    U = np.zeros((n1, r), np.float64)
    V = np.zeros((n2, r), np.float64)
    _get().or_waltmin(n1, n2, r, T, init_iters, trim_c, lam, seed, int(partition), len(I), _p(I), _p(J),
                      _p(val), _p(qhat_), _p(a_norm), frobA, _p(U), _p(V))
    return U, V


# --------------------------------------------------------------------------
# Whole pipeline (Alg. 1) on in-memory inputs (small configs only)
# --------------------------------------------------------------------------
def smp_pca(A, B, k, r, m, T, pi_kind=PI_RADEMACHER, seed=0, omega_seed=None,
            wm_seed=None, init_iters=50, trim_c=8.0, lam=1e-10, plain=False, a_is_b=False,
            sampler="bernoulli", partition=PART_REUSE_ALL):
    """Alg. 1 end to end.  Returns a dict with every intermediate."""
    omega_seed = seed if omega_seed is None else omega_seed
    wm_seed = seed if wm_seed is None else wm_seed
    skA, a2 = sketch_rows(pi_kind, seed, k, A)
    if a_is_b:
        skB, b2 = skA, a2
    else:
        skB, b2 = sketch_rows(pi_kind, seed, k, B)
    Ask, As, DA = finalize(k, skA, a2)    # flushes a2 < 2^-200 in place (R25)
    Bsk, Bs, DB = finalize(k, skB, b2)
    FA, FB = pairwise_sum(a2), pairwise_sum(b2)
    al, be = alpha_beta(a2, b2, FA, FB)
    if sampler == "multinomial":
        I, J, q = sample_multinomial(omega_seed, m, al, be)
    else:
        I, J, q = sample(omega_seed, m, al, be)
    Mt = estimate(k, I, J, Ask, Bsk, DA, DB, plain=plain)
    U, V = waltmin(len(a2), len(b2), r, T, I, J, Mt, q, np.sqrt(a2), np.sqrt(FA),
                   init_iters=init_iters, trim_c=trim_c, lam=lam, seed=wm_seed, partition=partition)
    return dict(Ask=Ask, Bsk=Bsk, a2=a2, b2=b2, FA=FA, FB=FB, As=As, Bs=Bs, DA=DA, DB=DB,
                alpha=al, beta=be, I=I, J=J, qhat=q, Mt=Mt, U=U, V=V)


# --------------------------------------------------------------------------
# LELA: the two-pass comparison system (NEXT-3)
# --------------------------------------------------------------------------
def exact_entries(A, B, I, J, out=None):
    """Pass 2 of LELA: out[s] += Σ_t A[t, I_s] B[t, J_s] over the rows of the
    block (fp64), i.e. (AᵀB)_{I_s J_s} once every row block has been seen."""
    A = np.ascontiguousarray(A)
    B = np.ascontiguousarray(B)
    I = _c(I, np.int32)
    J = _c(J, np.int32)
    if out is None:
        out = np.zeros(len(I), np.float64)
    _get().or_exact_entries(A.shape[0], _p(A), _dtype_code(A), A.shape[1], _p(B), _dtype_code(B),
                            B.shape[1], len(I), _p(I), _p(J), _p(out))
    return out


def lela(A, B, r, m, T, seed=0, wm_seed=None, init_iters=50, trim_c=8.0, lam=1e-10,
         partition=PART_REUSE_ALL):
    """LELA end to end: pass 1 exact column norms, Ω by Eq. 1 (same sampler
    and hash as SMP-PCA), pass 2 exact entries on Ω, WAltMin."""
    wm_seed = seed if wm_seed is None else wm_seed
    a2 = colnorms(A)
    b2 = colnorms(B)
    FA, FB = pairwise_sum(a2), pairwise_sum(b2)
    al, be = alpha_beta(a2, b2, FA, FB)
    I, J, q = sample(seed, m, al, be)
    M = exact_entries(A, B, I, J)
    U, V = waltmin(len(a2), len(b2), r, T, I, J, M, q, np.sqrt(a2), np.sqrt(FA), init_iters=init_iters,
                   trim_c=trim_c, lam=lam, seed=wm_seed, partition=partition)
    return dict(a2=a2, b2=b2, FA=FA, FB=FB, I=I, J=J, qhat=q, M=M, U=U, V=V)


def num_threads() -> int:
    """OpenMP threads used by the oracle (the CPU baseline's core count)."""
    lib = _get()
    lib.or_num_threads.restype = ctypes.c_int
    return int(lib.or_num_threads())
