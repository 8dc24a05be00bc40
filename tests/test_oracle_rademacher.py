"""Pins of the Rademacher Theta (reading A22) and of Alg. 2 with it.

* Signs come from the Philox4x32-10 words (pinned by the Random123 KATs and ATen in
  test_oracle_theta.py): bit r mod 32 of word (r mod 128) / 32 of the call (i, r / 128, domain 5).
* Distribution: balanced signs (binomial z-test), uncorrelated rows and columns, E ||Theta x||^2 =
  ||x||^2 (Rademacher is an isometry in expectation, E Theta^T Theta = I).
* Sketch: exact rational Theta X on tiny inputs; BLAS with the explicit Theta; partition invariance.
* Alg. 2 with a Rademacher Theta: R equals LAPACK's R of P; cond(Q) = cond(Theta U).
"""
from fractions import Fraction

import numpy as np
import pytest

import oracle
import synth


def test_signs_are_the_philox_bits():
    seed, k, m, ro = 123, 300, 7, 5_000_000_000
    S = oracle.theta_rademacher(seed, k, m, ro)
    for ii in range(m):
        i = ro + ii
        for q in range(3):
            w = oracle.philox4x32_10([i & 0xFFFFFFFF, i >> 32, q, 5], [seed & 0xFFFFFFFF, seed >> 32])
            for r in range(128 * q, min(k, 128 * q + 128)):
                bit = (int(w[(r % 128) // 32]) >> (r % 32)) & 1
                assert S[r, ii] == (-1 if bit else 1)


def test_sign_statistics():
    S = oracle.theta_rademacher(7, 256, 20_000).astype(np.float64)
    n = S.size
    assert abs(S.sum()) / np.sqrt(n) < 4.5                       # balanced (z-test)
    C = S @ S.T / S.shape[1]                                      # row correlations
    off = C[~np.eye(256, dtype=bool)]
    assert np.abs(off).max() < 5.0 / np.sqrt(S.shape[1]) * 1.2
    cc = np.mean(S[:, :-1] * S[:, 1:])                            # neighbouring X rows
    assert abs(cc) < 5.0 / np.sqrt(n)


def test_isometry_in_expectation():
    rng = np.random.default_rng(1)
    x = rng.standard_normal(500)
    vals = [np.sum((oracle.theta_dense(s, 64, 500, oracle.RADEMACHER) @ x) ** 2) for s in range(400)]
    assert abs(np.mean(vals) / np.dot(x, x) - 1.0) < 0.03


def test_sketch_exact_rational():
    rng = np.random.default_rng(2)
    X = rng.standard_normal((29, 3))
    P = oracle.sketch(X, 10, sketch=oracle.RADEMACHER, seed=3)
    T = oracle.theta_rademacher(3, 10, 29).astype(np.int64)
    sk = Fraction(1.0 / np.sqrt(10.0))
    for r in range(10):
        for j in range(3):
            exact = sum(int(T[r, i]) * sk * Fraction(X[i, j]) for i in range(29))
            bound = Fraction(2.0**-52) * sum(abs(sk * Fraction(X[i, j])) for i in range(29))
            assert abs(Fraction(P[r, j]) - exact) <= bound + Fraction(1, 2**1074)


@pytest.mark.parametrize("dt", ["f64", "f32"])
def test_sketch_matches_blas_and_partition(dt):
    X = synth.make_X(70_003, 7, 3.0, dt)
    P = oracle.sketch(X, 40, sketch=oracle.RADEMACHER)
    ref = oracle.theta_dense(0, 40, X.shape[0], oracle.RADEMACHER) @ X.astype(np.float64)
    assert np.linalg.norm(P - ref) <= 1e-13 * np.linalg.norm(ref)
    Pa = oracle.sketch(X[:30_000], 40, sketch=oracle.RADEMACHER)
    Pb = oracle.sketch(X[30_000:], 40, sketch=oracle.RADEMACHER, row_offset=30_000)
    assert np.allclose(Pa + Pb, P, rtol=1e-14, atol=1e-14 * np.abs(P).max())


def test_alg2_with_rademacher():
    X = synth.make_X(20_000, 16, 6.0)
    out = oracle.factor(X, 64, sketch=oracle.RADEMACHER)
    Rl = np.linalg.qr(out["P"], mode="r")
    Rl = np.sign(np.diag(Rl))[:, None] * Rl
    assert np.linalg.norm(out["R"] - Rl) <= 1e-13 * np.linalg.norm(Rl)
    U, _ = np.linalg.qr(X)
    TU = oracle.theta_dense(0, 64, X.shape[0], oracle.RADEMACHER) @ U
    assert abs(oracle.cond(out["Q"]) / oracle.cond(TU) - 1) < 1e-3
