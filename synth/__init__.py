"""Seeded synthetic inputs shaped like the paper's workloads.

This module holds NO arithmetic of the SMP-PCA method: it only produces the
matrices A and B that both the CUDA path and the CPU oracle consume.  Large
configurations are generated on the device in fixed 65,536-row generator
blocks keyed by (seed, block index), so a row-sharded run (any number of
GPUs whose shards are block aligned) sees exactly the same data.

Configurations (BASELINE.json "configs"; readings R16-R19 in DESIGN.md):
  cfg0  tiny cone, fp32, d=2000, n=100 (0.8 u + 0.6 g/sqrt(d), independent u')
  cfg1  low-rank + noise bf16, d=2^20, n=1024 (rank 20, 1/i spectrum, shared row factor)
  cfg2  cone at 30 degrees bf16, d=2^22, n=4096
  cfg3  CSR bag-of-words, Zipf(1.1) columns, zero-truncated Poisson(2) counts
  cfg4  A=B PCA fp32, d=2e6, n=2048, planted rank-10 spectrum, log-uniform column scales
"""
from __future__ import annotations

import math

import numpy as np
import torch

GEN_BLOCK = 65536

CONFIGS = {
    "cfg0": dict(d=2000, n1=100, n2=100, k=64, dtype="f32", pi="rademacher", r=5, T=10,
                 m_coef=0.3, seed=0),
    "cfg1": dict(d=1 << 20, n1=1024, n2=1024, k=256, dtype="bf16", pi="rademacher", r=5, T=10,
                 m_coef=4.0, seed=1),
    "cfg2": dict(d=1 << 22, n1=4096, n2=4096, k=1024, dtype="bf16", pi="rademacher", r=10, T=15,
                 m_coef=4.0, seed=2),
    "cfg3": dict(d=8_000_000, n1=10_000, n2=8000, k=512, dtype="csr", pi="gaussian", r=10, T=10,
                 m_coef=4.0, seed=3, nnz_a=100, nnz_b=80),
    "cfg4": dict(d=2_000_000, n1=2048, n2=2048, k=512, dtype="f32", pi="gaussian", r=10, T=15,
                 m_coef=4.0, seed=4, a_is_b=True),
}


def m_of(cfg: dict) -> float:
    """Sample budget m = c n r ln n with n = max(n1, n2) (R9/R10)."""
    n = max(cfg["n1"], cfg["n2"])
    return cfg["m_coef"] * n * cfg["r"] * math.log(n)


def _gen(seed: int, tag: int, block: int, device) -> torch.Generator:
    g = torch.Generator(device=device)
    g.manual_seed((seed * 1_000_003 + tag * 7919 + block * 104_729) % (2**63 - 1))
    return g


# ------------------------------------------------------------------ cfg0
def cone_tiny(d=2000, n=100, seed=0, c=0.8, s=0.6):
    """a_i = c u + s g_i / sqrt(d), u a fixed unit vector (BASELINE cfg0; R16).
    B is built the same way with an independent u'.  fp32, CPU tensors."""
    g = torch.Generator().manual_seed(seed)
    out = []
    for _ in range(2):
        u = torch.randn(d, 1, generator=g, dtype=torch.float64)
        u /= u.norm()
        G = torch.randn(d, n, generator=g, dtype=torch.float64)
        out.append((c * u + s * G / math.sqrt(d)).to(torch.float32))
    return out[0], out[1]


def cone_shared_axis(d, n, theta, seed=0):
    """Paper-faithful cone: y = ±(x + t), E||t|| = tan(θ/2),
    normalised; A and B share the axis x.  fp64 CPU tensors."""
    g = torch.Generator().manual_seed(seed)
    x = torch.randn(d, 1, generator=g, dtype=torch.float64)
    x /= x.norm()
    mats = []
    for _ in range(2):
        t = torch.randn(d, n, generator=g, dtype=torch.float64) * (math.tan(theta / 2) / math.sqrt(d))
        y = (x + t) * (torch.randint(0, 2, (1, n), generator=g) * 2 - 1)
        mats.append(y / y.norm(dim=0, keepdim=True))
    return mats[0], mats[1]


# ------------------------------------------------------------------ generic small
def gaussian_small(d, n, seed=0, dtype=torch.float32, scale_cols=False):
    g = torch.Generator().manual_seed(seed)
    X = torch.randn(d, n, generator=g, dtype=torch.float64)
    if scale_cols:
        X *= torch.exp(torch.randn(1, n, generator=g, dtype=torch.float64))
    return X.to(dtype)


# ------------------------------------------------------------------ cfg1
def lowrank_factors(n, rank, seed, tag, device):
    g = torch.Generator().manual_seed(seed * 31 + tag)
    Q, _ = torch.linalg.qr(torch.randn(n, rank, generator=g, dtype=torch.float64))
    return Q.to(device=device, dtype=torch.float32)


def lowrank_block(row0, rows, n, seed, VA, VB, rank=20, noise=0.01, device="cuda"):
    """Rows [row0, row0+rows) of cfg1's A and B (R17): L = G_U diag(1/i) Vᵀ
    with G_U ~ N(0,1) shared by A and B, plus N(0, noise²); bf16.
    row0 and rows must be multiples of GEN_BLOCK (or rows the remainder)."""
    assert row0 % GEN_BLOCK == 0
    A = torch.empty(rows, n, dtype=torch.bfloat16, device=device)
    B = torch.empty(rows, n, dtype=torch.bfloat16, device=device)
    sv = 1.0 / torch.arange(1, rank + 1, device=device, dtype=torch.float32)
    for b0 in range(0, rows, GEN_BLOCK):
        br = min(GEN_BLOCK, rows - b0)
        blk = (row0 + b0) // GEN_BLOCK
        g = _gen(seed, 1, blk, device)
        GU = torch.randn(br, rank, generator=g, device=device) * sv
        NA = torch.randn(br, n, generator=g, device=device)
        NB = torch.randn(br, n, generator=g, device=device)
        A[b0:b0 + br] = (GU @ VA.T + noise * NA).to(torch.bfloat16)
        B[b0:b0 + br] = (GU @ VB.T + noise * NB).to(torch.bfloat16)
    return A, B


# ------------------------------------------------------------------ cfg2
def cone_block(row0, rows, n, seed, theta_deg=30.0, device="cuda", dtype=torch.bfloat16):
    """Rows of cfg2's A and B (R16): a_i[t] = cosθ u_t + sinθ g_ti / sqrt(d)
    with u_t = z_t / sqrt(d) (a fixed, approximately unit axis), independent
    axes for A and B; d is folded into the generator scale (rows are keyed
    by global block, so any sharding gives identical data)."""
    assert row0 % GEN_BLOCK == 0
    c, s = math.cos(math.radians(theta_deg)), math.sin(math.radians(theta_deg))
    A = torch.empty(rows, n, dtype=dtype, device=device)
    B = torch.empty(rows, n, dtype=dtype, device=device)
    for b0 in range(0, rows, GEN_BLOCK):
        br = min(GEN_BLOCK, rows - b0)
        blk = (row0 + b0) // GEN_BLOCK
        g = _gen(seed, 2, blk, device)
        for X in (A, B):
            u = torch.randn(br, 1, generator=g, device=device)
            G = torch.randn(br, n, generator=g, device=device)
            X[b0:b0 + br] = (c * u + s * G).to(dtype)
    return A, B


# ------------------------------------------------------------------ cfg3
def zipf_weights(n, a=1.1):
    w = (np.arange(1, n + 1, dtype=np.float64)) ** (-a)
    return w / w.sum()


def csr_block(row0, rows, n, nnz_per_row, seed, tag, device="cuda", a=1.1, lam=2.0):
    """Rows of a cfg3 matrix (R18): exactly nnz_per_row distinct columns per
    row drawn ∝ (c+1)^-1.1 without replacement, ascending; values are
    zero-truncated Poisson(2) counts stored as fp32.  Returns (rowptr int64
    relative to the block, col int32, val fp32)."""
    w = torch.tensor(zipf_weights(n, a), device=device, dtype=torch.float32)
    cols, vals = [], []
    sub = 8192
    for b0 in range(0, rows, sub):
        br = min(sub, rows - b0)
        g = _gen(seed, 16 + tag, (row0 + b0) // sub, device)
        # Gumbel top-k == sampling without replacement ∝ w
        keys = torch.log(w)[None, :] - torch.log(-torch.log(
            torch.rand(br, n, generator=g, device=device).clamp_min(1e-30)))
        c = torch.topk(keys, nnz_per_row, dim=1).indices.sort(dim=1).values
        lamt = torch.full((br, nnz_per_row), lam, device=device)
        v = torch.poisson(lamt, generator=g)
        while bool((v == 0).any()):
            v = torch.where(v == 0, torch.poisson(lamt, generator=g), v)
        cols.append(c.to(torch.int32).reshape(-1))
        vals.append(v.to(torch.float32).reshape(-1))
    col = torch.cat(cols)
    val = torch.cat(vals)
    rowptr = torch.arange(0, rows + 1, device=device, dtype=torch.int64) * nnz_per_row
    return rowptr, col, val


# ------------------------------------------------------------------ cfg4
def pca_block(row0, rows, n, seed, W, sig, D, device="cuda"):
    """Rows of cfg4's A (R19): A = (G + Z diag(σ) Wᵀ) D, fp32."""
    assert row0 % GEN_BLOCK == 0
    A = torch.empty(rows, n, dtype=torch.float32, device=device)
    for b0 in range(0, rows, GEN_BLOCK):
        br = min(GEN_BLOCK, rows - b0)
        g = _gen(seed, 4, (row0 + b0) // GEN_BLOCK, device)
        G = torch.randn(br, n, generator=g, device=device)
        Z = torch.randn(br, W.shape[1], generator=g, device=device)
        A[b0:b0 + br] = (G + (Z * sig) @ W.T) * D
    return A


def pca_params(n, seed, rank=10, device="cuda"):
    g = torch.Generator().manual_seed(seed * 17 + 5)
    W, _ = torch.linalg.qr(torch.randn(n, rank, generator=g, dtype=torch.float64))
    sig = 10.0 / torch.arange(1, rank + 1, dtype=torch.float64)
    D = 10.0 ** (2.0 * torch.rand(n, generator=g, dtype=torch.float64))
    return (W.to(device, torch.float32), sig.to(device, torch.float32), D.to(device, torch.float32))


def bf16_bits(t: torch.Tensor) -> np.ndarray:
    """Raw bf16 bits of a tensor as numpy uint16 (oracle input format)."""
    return t.contiguous().view(torch.int16).cpu().numpy().view(np.uint16)
