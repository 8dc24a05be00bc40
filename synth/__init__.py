"""Seeded synthetic inputs for RCholeskyQR -- shared by the oracle tests, the GPU parity tests and
bench.py.  Holds none of the method's arithmetic (no sketch, no QR of X, no solve).

X = G diag(sigma) W  (BASELINE.json configs; the paper's Test-1 family, with G not
orthonormalised -- DESIGN.md reading A13):
  * G: iid N(0,1), m x n;
  * sigma_j = 10^(-c j / (n-1)), j = 0..n-1, c = log10(cond) (logspaced 1 -> 10^-c);
  * W: the orthogonal factor of the QR of an n x n N(0,1) matrix (sign-fixed, diag(R_W) > 0).
X is formed in fp64 and rounded once to fp32 for the fp32 configs.  The same bytes are fed to the
GPU and to the oracle; X itself does not need to be reproducible across implementations.
"""
from __future__ import annotations

import numpy as np

CONFIGS = {
    # name: m, n, k, sketch, nnz, dtype, log10 cond
    "C1": dict(m=10_000, n=20, k=40, sketch="gaussian", nnz=8, dtype="f64", log10_cond=3),
    "C2": dict(m=1_048_576, n=100, k=200, sketch="gaussian", nnz=8, dtype="f32", log10_cond=5),
    "C3": dict(m=16_777_216, n=256, k=512, sketch="gaussian", nnz=8, dtype="f64", log10_cond=10),
    "C4": dict(m=67_108_864, n=64, k=128, sketch="sparse", nnz=8, dtype="f32", log10_cond=4),
    "C5": dict(m=4_194_304, n=1024, k=2048, sketch="gaussian", nnz=8, dtype="f64", log10_cond=12),
}

X_SEED = 0      # reading A13: X seed 0 for all configs
THETA_SEED = 0  # Theta seed 0 (domain-separated from X by construction: different generators)


def sigma(n: int, log10_cond: float) -> np.ndarray:
    if n == 1:
        return np.ones(1)
    return 10.0 ** (-log10_cond * np.arange(n) / (n - 1))


def orthogonal_W(n: int, seed: int = X_SEED) -> np.ndarray:
    rng = np.random.Generator(np.random.PCG64([seed, 4]))
    A = rng.standard_normal((n, n))
    Qw, Rw = np.linalg.qr(A)
    return Qw * np.sign(np.diag(Rw))[None, :]


def make_X(m: int, n: int, log10_cond: float, dtype: str = "f64", seed: int = X_SEED) -> np.ndarray:
    """Host (numpy) X, row-major, for sizes the oracle handles."""
    rng = np.random.Generator(np.random.PCG64([seed, 3]))
    G = rng.standard_normal((m, n))
    X = (G * sigma(n, log10_cond)[None, :]) @ orthogonal_W(n, seed)
    return np.ascontiguousarray(X if dtype == "f64" else X.astype(np.float32))


def make_X_lowrank(m: int, n: int, rank: int, log10_cond: float = 2.0, noise: float = 0.0, dtype: str = "f64",
                   seed: int = X_SEED) -> np.ndarray:
    """Numerically rank-deficient X for Alg. 7 (PAPER.md:856's third experiment, simplified):
    X = (G diag(sigma) ) B with G m x rank Gaussian, sigma graded over 10^log10_cond and B a rank x n
    Gaussian, plus noise * (an independent Gaussian m x n) / sqrt(m); columns carry norms of varying
    size (column j scaled by 2^(j mod 5 - 2)) so the normalisation D of PAPER.md:350 matters."""
    rng = np.random.Generator(np.random.PCG64([seed, 7]))
    G = rng.standard_normal((m, rank))
    B = rng.standard_normal((rank, n))
    X = (G * sigma(rank, log10_cond)[None, :]) @ B
    if noise:
        X = X + noise * rng.standard_normal((m, n)) * np.linalg.norm(X) / np.sqrt(m * n)
    X = X * (2.0 ** (np.arange(n) % 5 - 2))[None, :]
    return np.ascontiguousarray(X if dtype == "f64" else X.astype(np.float32))


CHUNK_ROWS = 1 << 18


def make_X_torch(m: int, n: int, log10_cond: float, dtype: str = "f64", seed: int = X_SEED, device="cuda",
                 row_start: int = 0):
    """Rows row_start .. row_start+m-1 of the global device X.  G is drawn per 2^18-row chunk from a
    generator seeded by (seed, chunk index), so any row range (a rank's block) is reproducible on
    its own; the fp64 product is rounded once to the storage dtype."""
    import torch
    dev = torch.device(device)
    tdt = torch.float64 if dtype == "f64" else torch.float32
    X = torch.empty((m, n), dtype=tdt, device=dev)
    Wt = torch.from_numpy(orthogonal_W(n, seed)).to(dev)
    sg = torch.from_numpy(sigma(n, log10_cond)).to(dev)
    gen = torch.Generator(device=dev)
    r = row_start
    while r < row_start + m:
        c = r // CHUNK_ROWS
        c0, c1 = c * CHUNK_ROWS, (c + 1) * CHUNK_ROWS
        gen.manual_seed((seed * 1_000_003 + 3) * 65_536 + c)
        G = torch.randn((CHUNK_ROWS, n), dtype=torch.float64, device=dev, generator=gen)
        a, b = r, min(row_start + m, c1)
        X[a - row_start:b - row_start] = ((G[a - c0:b - c0] * sg[None, :]) @ Wt).to(tdt)
        del G
        r = b
    return X


def config(name: str) -> dict:
    c = dict(CONFIGS[name])
    c["name"] = name
    return c
