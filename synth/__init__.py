"""Seeded synthetic inputs shared by the oracle side and the CUDA side.

This module holds NONE of the method's arithmetic: it only draws the test systems
(A, b) that BASELINE.json's configs describe, so that tests/ and bench.py can feed
the same bytes to oracle/ and to the product.  The paper's own benchmarks (OpenML /
scikit-learn kernel matrices) are not available offline; these spiked
systems stand in for their "few large outlying singular values over an
ill-conditioned bulk" structure, as DESIGN.md states.

Draw order (fixed): G -> U -> V (or W) -> x* -> b, from one torch.Generator seeded
with `seed` on `device`.  Values are fp64.  theta_i is log-spaced with inclusive
endpoints: theta_i = lo * (hi/lo)^((i-1)/(k-1)).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import torch


@dataclass(frozen=True)
class Config:
    name: str
    kind: str            # "kpp" (general, Kaczmarz++) or "cdpp" (PSD, CD++)
    m: int
    n: int
    k: int               # number of outlying directions
    theta_lo: float
    theta_hi: float
    bulk_scale_dim: int  # G / sqrt(bulk_scale_dim)
    consistent: bool     # b = A x* (True) or b ~ N(0, I) (False)
    s: int               # block size
    lam: float = 1e-8    # Q2: lambda = 1e-8
    max_iters: int = 0   # fixed iteration count (c1) or 0 = run to tol
    tol: float = 1e-8
    extra: dict = field(default_factory=dict)


# BASELINE.json configs[0..4]
CONFIGS = {
    "c1": Config("c1", "kpp", 256, 256, 8, 1e2, 1e4, 256, True, 32, max_iters=500, tol=0.0),
    "c2": Config("c2", "kpp", 8192, 8192, 64, 1e1, 1e3, 8192, True, 128),
    "c3": Config("c3", "kpp", 131072, 4096, 32, 1e1, 1e4, 131072, True, 256),
    "c4": Config("c4", "kpp", 4096, 131072, 32, 1e1, 1e4, 131072, False, 256),
    "c5": Config("c5", "cdpp", 65536, 65536, 100, 1e2, 1e5, 65536, False, 512,
                 extra={"shift": 2.5}),
}


def twin(name: str, m: int, n: int, s: int, k: int | None = None) -> Config:
    """A reduced-size system with the same recipe as config `name` (for oracle parity)."""
    c = CONFIGS[name]
    kk = c.k if k is None else k
    if c.kind == "cdpp":
        m = n
    scale = m if name == "c3" else n  # c3 scales the bulk by sqrt(m), the others by sqrt(n)
    return Config(f"{name}_twin_{m}x{n}_s{s}", c.kind, m, n, kk, c.theta_lo, c.theta_hi, scale,
                  c.consistent, s, c.lam, 0, c.tol, dict(c.extra))


def thetas(k: int, lo: float, hi: float) -> torch.Tensor:
    if k == 1:
        return torch.tensor([lo], dtype=torch.float64)
    i = torch.arange(k, dtype=torch.float64)
    return lo * (hi / lo) ** (i / (k - 1))


def _unit_cols(X: torch.Tensor) -> torch.Tensor:
    return X / torch.linalg.vector_norm(X, dim=0, keepdim=True)


@torch.no_grad()
def make_general(cfg: Config, seed: int = 0, device="cpu"):
    """A = G/sqrt(d) + sum_i theta_i u_i v_i^T, u_i, v_i unit Gaussian directions.
    Returns (A, b, x_star or None), fp64, on `device`."""
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    m, n = cfg.m, cfg.n
    A = torch.randn((m, n), generator=g, dtype=torch.float64, device=device)
    A.mul_(1.0 / math.sqrt(cfg.bulk_scale_dim))
    U = _unit_cols(torch.randn((m, cfg.k), generator=g, dtype=torch.float64, device=device))
    V = _unit_cols(torch.randn((n, cfg.k), generator=g, dtype=torch.float64, device=device))
    th = thetas(cfg.k, cfg.theta_lo, cfg.theta_hi).to(device)
    tile = max(1, (1 << 27) // max(n, 1))  # ~1 GiB of fp64 per tile
    for r0 in range(0, m, tile):
        r1 = min(m, r0 + tile)
        A[r0:r1].addmm_(U[r0:r1] * th, V.T)
    x_star = torch.randn((n,), generator=g, dtype=torch.float64, device=device)
    if cfg.consistent:
        b = A @ x_star
    else:
        b = torch.randn((m,), generator=g, dtype=torch.float64, device=device)
        x_star = None
    return A, b, x_star


@torch.no_grad()
def make_psd(cfg: Config, seed: int = 0, device="cpu"):
    """A = sum_i theta_i w_i w_i^T + (G + G^T)/sqrt(2n) + shift*I, bitwise symmetric.
    Returns (A, b, None)."""
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    n = cfg.n
    A = torch.randn((n, n), generator=g, dtype=torch.float64, device=device)
    W = _unit_cols(torch.randn((n, cfg.k), generator=g, dtype=torch.float64, device=device))
    th = thetas(cfg.k, cfg.theta_lo, cfg.theta_hi).to(device)
    shift = cfg.extra.get("shift", 2.5)
    sc = 1.0 / math.sqrt(2.0 * n)
    T = min(n, 4096)
    # Symmetrise tile pairs in place: A_ij <- (G_ij + G_ji^T) sc + (W_i th W_j^T + (W_j th W_i^T)^T)/2
    for i0 in range(0, n, T):
        i1 = min(n, i0 + T)
        for j0 in range(i0, n, T):
            j1 = min(n, j0 + T)
            S = (A[i0:i1, j0:j1] + A[j0:j1, i0:i1].T) * sc
            P = (W[i0:i1] * th) @ W[j0:j1].T
            Q = ((W[j0:j1] * th) @ W[i0:i1].T).T
            S += 0.5 * (P + Q)
            A[i0:i1, j0:j1] = S
            A[j0:j1, i0:i1] = S.T
    A.diagonal().add_(shift)
    b = torch.randn((n,), generator=g, dtype=torch.float64, device=device)
    return A, b, None


def make_problem(cfg: Config | str, seed: int = 0, device="cpu"):
    if isinstance(cfg, str):
        cfg = CONFIGS[cfg]
    if cfg.kind == "cdpp":
        return make_psd(cfg, seed, device)
    return make_general(cfg, seed, device)


def make_vector(n: int, seed: int, device="cpu"):
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    return torch.randn((n,), generator=g, dtype=torch.float64, device=device)


# ---------------------------------------------------------------- bell-spectrum systems (NEXT-3)
def bell_profile(k: int, effective_rank: int, tail_strength: float = 0.01) -> torch.Tensor:
    """Singular value profile of the paper's synthetic low-rank matrices (App F):
    sigma_i = (1 - ts) exp(-(i/er)^2) + ts exp(-0.1 i/er), i = 0, 1, ...  The paper prints the tail
    as ts*exp(i/er) (growing); we take the decaying form of the cited generator."""
    i = torch.arange(k, dtype=torch.float64)
    return (1.0 - tail_strength) * torch.exp(-(i / effective_rank) ** 2) + tail_strength * torch.exp(-0.1 * i / effective_rank)


@torch.no_grad()
def make_bell_psd(n: int = 4096, effective_rank: int = 25, tail_strength: float = 0.01, phi: float = 1e-3,
                  seed: int = 0, device="cpu"):
    """CD++ test system of App F: A = Phi Phi^T + phi I with Phi = U diag(sigma) V^T,
    U, V Haar-random orthogonal (QR of Gaussians, signs fixed by diag(R)), so A = U diag(sigma^2) U^T
    + phi I; b ~ N(0, I).  Symmetrised bitwise.  Returns (A, b)."""
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    G = torch.randn((n, n), generator=g, dtype=torch.float64, device=device)
    Q, R = torch.linalg.qr(G)
    Q = Q * torch.sign(torch.diagonal(R))
    sig = bell_profile(n, effective_rank, tail_strength).to(device)
    A = (Q * sig ** 2) @ Q.T
    A = 0.5 * (A + A.T)
    A.diagonal().add_(phi)
    b = torch.randn((n,), generator=g, dtype=torch.float64, device=device)
    return A, b


@torch.no_grad()
def make_bell_general(m: int = 4096, n: int = 1024, effective_rank: int = 50, tail_strength: float = 0.01,
                      seed: int = 0, device="cpu"):
    """K++ test system of App F (Fig lsqr_steps): an m x n matrix with the
    bell singular value profile, A = U diag(sigma) V^T with U (m x n, orthonormal columns) and V
    (n x n) Haar-random (QR of Gaussians, signs fixed by diag(R)); b ~ N(0, I) (inconsistent, as in
    the paper).  Returns (A, b)."""
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    U, R = torch.linalg.qr(torch.randn((m, n), generator=g, dtype=torch.float64, device=device))
    U = U * torch.sign(torch.diagonal(R))
    V, R2 = torch.linalg.qr(torch.randn((n, n), generator=g, dtype=torch.float64, device=device))
    V = V * torch.sign(torch.diagonal(R2))
    sig = bell_profile(n, effective_rank, tail_strength).to(device)
    A = (U * sig) @ V.T
    b = torch.randn((m,), generator=g, dtype=torch.float64, device=device)
    return A, b

