"""Pins of the RRRCholeskyQR oracle (Alg. 7) against things other than itself.

* Column norms D: numpy / exact rational sums.
* RRQR (step 2, reading A21): the pivot order and R of the Businger-Golub phase equal LAPACK's
  dgeqp3 (scipy.linalg.qr(pivoting=True)); at exit the strong-RRQR conditions hold,
  rho_ij <= f (checked with scipy's triangular solve); on the Kahan matrix -- where column pivoting
  alone fails to reveal the rank -- the swaps bring |R_nn| to within sqrt(1 + f^2 (n-1)) of
  sigma_min (Gu & Eisenstat 1996, Thm 3.2), which pivoting alone misses by orders of magnitude.
* Rank rule (step 3): known exact rank r of X = G B (+ tiny noise) is found; duplicated and zero
  columns are excluded.
* Whole Alg. 7: full rank -> Alg. 2 on X[:, perm] (R to rounding); rank deficient -> cond(Q) small
  and the column-normalised residual within eq:RRRCholeskyQR21; exact metamorphic
  tests: X 2^e and power-of-two column scalings leave perm and Q bitwise unchanged (the
  normalisation P D^{-1} is exact) and scale R accordingly.
"""
from fractions import Fraction

import numpy as np
import pytest
import scipy.linalg

import oracle
import synth

U64 = 2.0**-53


def _norm_R(R):
    return np.sign(np.diag(R))[:, None] * R


def test_colnorms_matches_numpy():
    X = synth.make_X(70_001, 9, 3.0)
    d = oracle.colnorms(X)
    assert np.allclose(d, np.linalg.norm(X, axis=0), rtol=1e-13, atol=0)   # numpy: plain fp64 sums
    Xt = np.random.default_rng(4).standard_normal((17, 3))
    dt = oracle.colnorms(Xt)
    for j in range(3):
        exact = sum(Fraction(x) * Fraction(x) for x in Xt[:, j])
        assert abs(Fraction(dt[j]) ** 2 - exact) <= exact * Fraction(2.0**-50)


@pytest.mark.parametrize("k,n,seed", [(40, 20, 1), (64, 64, 2), (300, 100, 3)])
def test_pivoting_phase_matches_lapack(k, n, seed):
    P = np.random.default_rng(seed).standard_normal((k, n)) * (2.0 ** np.arange(n) % 7)[None, :]
    out = oracle.rrqr(P, tau=0.0, f=1e30)            # no truncation, no swaps: pure column pivoting
    _, Rl, piv = scipy.linalg.qr(P, pivoting=True, mode="economic")
    assert np.array_equal(out["perm"], piv)
    assert np.linalg.norm(out["R"] - _norm_R(Rl)) <= 1e-13 * np.linalg.norm(Rl)
    assert out["rank"] == n and out["swaps"] == 0


def _rho_max(R, r):
    R11, R12, R22 = R[:r, :r], R[:r, r:], R[r:, r:]
    A = scipy.linalg.solve_triangular(R11, R12)
    W = scipy.linalg.solve_triangular(R11, np.eye(r))
    inv_omega = np.linalg.norm(W, axis=1)                 # 1 / omega_i
    gamma = np.linalg.norm(R22, axis=0)
    return float(np.sqrt(np.max(A**2 + (gamma[None, :] * inv_omega[:, None]) ** 2)))


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_strong_conditions_at_exit(seed):
    rng = np.random.default_rng(seed)
    P = rng.standard_normal((60, 30)) @ np.diag(np.logspace(0, -12, 30)) @ rng.standard_normal((30, 30))
    out = oracle.rrqr(P, tau=1e-6, f=1.5)
    r = out["rank"]
    assert 0 < r < 30
    assert _rho_max(out["R"], r) <= 1.5 * (1 + 1e-12)


def _kahan(n, theta=1.2, pert=1e-10):
    c, s = np.cos(theta), np.sin(theta)
    C = np.eye(n) - c * np.triu(np.ones((n, n)), 1)
    K = np.diag(s ** np.arange(n)) @ C
    return K * ((1 - pert) ** np.arange(n))[None, :]       # QRCP then keeps the natural order


def test_kahan_matrix_needs_the_swaps():
    n = 30
    K = _kahan(n)
    smin = np.linalg.svd(K, compute_uv=False)[-1]
    qrcp = oracle.rrqr(K, tau=0.0, f=1e30, rank_fixed=n - 1)
    assert qrcp["swaps"] == 0 and np.array_equal(qrcp["perm"], np.arange(n))
    assert abs(qrcp["R"][-1, -1]) > 1e3 * smin                # column pivoting does not reveal sigma_min
    strong = oracle.rrqr(K, tau=0.0, f=1.5, rank_fixed=n - 1)
    assert strong["swaps"] > 0
    assert abs(strong["R"][-1, -1]) <= np.sqrt(1 + 1.5**2 * (n - 1)) * smin * (1 + 1e-6)
    assert _rho_max(strong["R"], n - 1) <= 1.5 * (1 + 1e-12)


@pytest.mark.parametrize("rank,noise", [(8, 1e-13), (5, 0.0), (11, 1e-14)])
def test_rank_rule_finds_the_rank(rank, noise):
    X = synth.make_X_lowrank(20_000, 12, rank, 2.0, noise)
    out = oracle.factor_rr(X, 24, tau=1e-9)
    assert out["rank"] == rank
    Q = out["Q"]
    assert Q.shape == (20_000, rank)
    assert oracle.cond(Q) <= 8.0                              # well-conditioned Q (eq:main5)


def test_full_rank_reduces_to_alg2_on_permuted_columns():
    X = synth.make_X(30_000, 16, 4.0)
    rr = oracle.factor_rr(X, 32, tau=1e-15)
    assert rr["rank"] == 16
    alg2 = oracle.factor(X[:, rr["perm"]].copy(), 32)
    assert np.linalg.norm(rr["R"] - alg2["R"]) <= 1e-13 * np.linalg.norm(alg2["R"])
    assert np.linalg.norm(rr["Q"] - alg2["Q"]) <= 10 * U64 * 1e4 * np.linalg.norm(alg2["Q"])
    Xp = X[:, rr["perm"]]
    assert np.linalg.norm(Xp - rr["Q"] @ rr["R"]) <= 10 * 16 * U64 * np.linalg.norm(X)


def test_rank_deficient_residual_bound():
    m, n, rank, tau = 20_000, 12, 8, 1e-8
    X = synth.make_X_lowrank(m, n, rank, 2.0, 1e-12)
    out = oracle.factor_rr(X, 24, tau=tau)
    p, r = out["perm"], out["rank"]
    assert r == rank
    D = out["D"][p]
    E = (X[:, p] - out["Q"] @ out["R"]) / D[None, :]          # column-normalised residual
    # eq:RRRCholeskyQR21: <= sqrt(2) (u n + 1.02 sqrt(3/2) tau) ||X_normalised||_F
    assert np.linalg.norm(E) <= np.sqrt(2) * (U64 * n + 1.02 * np.sqrt(1.5) * tau) * np.sqrt(n)
    assert np.all(np.tril(out["R"][:, :r], -1) == 0) and np.all(np.diag(out["R"][:, :r]) > 0)


def test_duplicated_and_zero_columns_are_excluded():
    X = synth.make_X(10_000, 10, 2.0)
    X[:, 6] = X[:, 2]
    X[:, 8] = 0.0
    out = oracle.factor_rr(X, 20, tau=1e-12)
    kept = set(out["perm"][: out["rank"]].tolist())
    assert out["rank"] == 8 and 8 not in kept and len(kept & {2, 6}) == 1


def test_metamorphic_power_of_two_scalings():
    X = synth.make_X_lowrank(8_000, 10, 7, 2.0, 1e-13)
    a = oracle.factor_rr(X, 20, tau=1e-9)
    b = oracle.factor_rr(X * 2.0**5, 20, tau=1e-9)
    assert np.array_equal(a["perm"], b["perm"]) and np.array_equal(a["Q"], b["Q"])
    assert np.array_equal(a["R"] * 2.0**5, b["R"])
    E = 2.0 ** np.array([0, 3, -2, 7, 1, -5, 2, 0, 4, -1], dtype=np.float64)
    c = oracle.factor_rr(X * E, 20, tau=1e-9)               # P D^{-1} is bitwise unchanged
    assert np.array_equal(a["perm"], c["perm"]) and np.array_equal(a["Q"], c["Q"])
    assert np.array_equal(a["R"] * E[a["perm"]][None, :], c["R"])


def test_rr2_orthonormal_and_consistent():
    # RRRCholeskyQR2: same rank and pivots as Alg. 7, Q orthonormal to O(r u) even for a
    # rank-deficient X, X[:, perm] = Q R to the tau bound, R = R' R1 with R' = chol(Q1^T Q1)
    m, n, rank, tau = 30_000, 14, 9, 1e-9
    X = synth.make_X_lowrank(m, n, rank, 2.0, 1e-13)
    out = oracle.factor_rr2(X, 28, tau)
    rr = oracle.factor_rr(X, 28, tau)
    assert out["rank"] == rr["rank"] == rank and np.array_equal(out["perm"], rr["perm"])
    Q, R, p = out["Q"], out["R"], out["perm"]
    assert np.linalg.norm(Q.T @ Q - np.eye(rank), 2) <= 10 * rank * U64
    assert np.linalg.cond(out["Rp"]) <= 8.0
    D = rr["D"][p]
    E = (X[:, p] - Q @ R) / D[None, :]
    assert np.linalg.norm(E) <= np.sqrt(2) * (U64 * n * 10 + 1.02 * np.sqrt(1.5) * tau) * np.sqrt(n)
    assert np.allclose(R, out["Rp"] @ rr["R"], rtol=0, atol=1e-13 * np.abs(R).max())
    assert np.all(np.tril(R[:, :rank], -1) == 0) and np.all(np.diag(R) > 0)
