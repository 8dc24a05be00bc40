"""Pins of the RCholeskyQR2 oracle (Alg. 3) against things other than itself.

* Cholesky (step 3): LAPACK's numpy.linalg.cholesky; exact small cases; SPD failure.
* Gram (step 2): exact rational arithmetic on tiny inputs; BLAS on random inputs.
* The whole algorithm: its output IS the QR factorisation of X, so R must equal LAPACK's
  Householder R of X (sign-normalised, unique for full-rank X) and Q must be orthonormal to
  O(n u) -- the property the paper adds Alg. 3 for ("orthonormal Q factor").
* Implicit form: Q = Q1 R'^{-1} with Q1 the RCholeskyQR factor and R = R' R1.
"""
from fractions import Fraction

import numpy as np
import pytest
import scipy.linalg

import oracle
import synth

U64 = 2.0**-53
U32 = 2.0**-24


@pytest.mark.parametrize("n", [1, 2, 7, 60])
def test_cholesky_matches_lapack(n):
    rng = np.random.default_rng(n)
    B = rng.standard_normal((n + 5, n))
    A = B.T @ B + 1e-3 * np.eye(n)
    Rp, st = oracle.cholesky(A)
    assert st == oracle.OK
    L = np.linalg.cholesky(A)
    assert np.allclose(Rp, L.T, rtol=1e-13, atol=1e-13 * np.abs(L).max())
    assert np.all(np.tril(Rp, -1) == 0) and np.all(np.diag(Rp) > 0)
    assert np.linalg.norm(Rp.T @ Rp - A) <= 10 * n * U64 * np.linalg.norm(A)


def test_cholesky_exact_small():
    # A = [[4, 2], [2, 5]] = R'^T R' with R' = [[2, 1], [0, 2]] exactly
    Rp, st = oracle.cholesky(np.array([[4.0, 2.0], [2.0, 5.0]]))
    assert st == oracle.OK and np.array_equal(Rp, [[2.0, 1.0], [0.0, 2.0]])


@pytest.mark.parametrize("A", [np.array([[1.0, 2.0], [2.0, 1.0]]), np.array([[0.0, 0.0], [0.0, 1.0]]),
                               np.array([[np.nan, 0.0], [0.0, 1.0]])])
def test_cholesky_not_positive_definite(A):
    _, st = oracle.cholesky(A)
    assert st == oracle.E_SINGULAR


def test_gram_exact_rational():
    rng = np.random.default_rng(3)
    Q = rng.standard_normal((37, 5))
    A = oracle.gram(Q)
    for i in range(5):
        for j in range(5):
            exact = sum(Fraction(Q[r, i]) * Fraction(Q[r, j]) for r in range(37))
            assert abs(Fraction(A[i, j]) - exact) <= abs(exact) * Fraction(2.0**-52) + Fraction(1, 2**1074)


@pytest.mark.parametrize("dt", ["f64", "f32"])
def test_gram_matches_blas(dt):
    Q = synth.make_X(70_001, 12, 2.0, dt)     # spans two 65536-row blocks
    A = oracle.gram(Q)
    Q64 = Q.astype(np.float64)
    ref = Q64.T @ Q64
    assert np.array_equal(A, A.T)
    assert np.linalg.norm(A - ref) <= 1e-13 * np.linalg.norm(ref)


def test_trmm_upper_matches_numpy():
    rng = np.random.default_rng(5)
    U, V = np.triu(rng.standard_normal((9, 9))), np.triu(rng.standard_normal((9, 9)))
    assert np.allclose(oracle.trmm_upper(U, V), U @ V, rtol=1e-14, atol=1e-14)


@pytest.mark.parametrize("m,n,c", [(20_000, 20, 3.0), (5_000, 64, 8.0), (3_000, 100, 5.0)])
def test_factor2_is_the_qr_of_x(m, n, c):
    X = synth.make_X(m, n, c)
    out = oracle.factor2(X, 2 * n)
    Q, R = out["Q"], out["R"]
    # orthonormal Q (the point of Alg. 3), residual, upper triangular R with positive diagonal
    assert np.linalg.norm(Q.T @ Q - np.eye(n), 2) <= 10 * n * U64
    assert np.linalg.norm(X - Q @ R) <= 10 * n * U64 * np.linalg.norm(X)
    assert np.all(np.tril(R, -1) == 0) and np.all(np.diag(R) > 0)
    # R is unique: LAPACK's Householder R of X, sign-normalised
    Rh = np.linalg.qr(X, mode="r")
    Rh = np.sign(np.diag(Rh))[:, None] * Rh
    # normwise: both are backward stable QRs of X and R is unique, so they agree to O(n u) ||R||
    assert np.linalg.norm(R - Rh) <= 1e3 * n * U64 * np.linalg.norm(Rh)


def test_factor2_implicit_form_and_composition():
    X = synth.make_X(8_000, 30, 6.0)
    out = oracle.factor2(X, 60)
    alg2 = oracle.factor(X, 60)
    assert np.array_equal(out["Q1"], alg2["Q"])                     # step 1 is Alg. 2 itself
    assert np.allclose(out["R"], out["Rp"] @ alg2["R"], rtol=0, atol=1e-14 * np.abs(out["R"]).max())
    Qi = scipy.linalg.solve_triangular(out["Rp"], out["Q1"].T, trans="T", lower=False).T   # Q1 R'^{-1}
    assert np.linalg.norm(Qi - out["Q"]) <= 100 * U64 * np.linalg.norm(out["Q"])
    # R' is close to the identity: Q1 is already well conditioned (cond(Q1) = cond(Theta U), A11)
    assert np.linalg.cond(out["Rp"]) <= 8.0


def test_factor2_fp32():
    X = synth.make_X(30_000, 40, 4.0, "f32")
    out = oracle.factor2(X, 80)
    Q = out["Q"].astype(np.float64)
    assert out["Q"].dtype == np.float32
    assert np.linalg.norm(Q.T @ Q - np.eye(40), 2) <= 40 * U32
    assert np.linalg.norm(X.astype(np.float64) - Q @ out["R"]) <= 40 * U32 * np.linalg.norm(X)
