"""Pins of the reduced RCholeskyQR oracle (Alg. 5) against things other than itself.

* Extractor Y = L X (step 1): exact rational arithmetic on tiny inputs; BLAS with an explicit L built
  from the normative draws (themselves pinned by Philox KATs, test_oracle_theta.py); the rows of L
  continue Theta's Gaussian stream (reading A20); partition invariance over global row keys.
* Z = Y R^{-1} (step 3) equals L Q for Q = X R^{-1} -- the identity the algorithm rests on
  ("first apply the extractor to X and only then compute a product with R^{-1}");
  Q from scipy's triangular solve, L explicit.
* Step 2 is Alg. 2's QR of the same P, so R and S equal Alg. 2's bit for bit.
* Exact metamorphic scaling: X 2^e -> (Z, R 2^e); X D -> (Z, R D) for a power-of-two diagonal D.
"""
from fractions import Fraction

import numpy as np
import pytest
import scipy.linalg

import oracle
import synth

U64 = 2.0**-53


def _L_dense(m, k, l, sketch=oracle.GAUSSIAN, seed=0, row_offset=0):
    l0 = oracle.extractor_row0(k, sketch)
    Z = oracle.theta_gauss_z(seed, l0 + l, m, row_offset).astype(np.float64)[l0:]
    return Z * (1.0 / np.sqrt(np.float64(l)))


def test_extract_exact_rational():
    rng = np.random.default_rng(11)
    m, n, l = 23, 3, 6
    X = rng.standard_normal((m, n))
    Y = oracle.extract(X, 8, l)
    L = _L_dense(m, 8, l)
    for j in range(l):
        for c in range(n):
            exact = sum(Fraction(L[j, i]) * Fraction(X[i, c]) for i in range(m))
            bound = Fraction(2.0**-52) * sum(abs(Fraction(L[j, i]) * Fraction(X[i, c])) for i in range(m))
            assert abs(Fraction(Y[j, c]) - exact) <= bound + Fraction(1, 2**1074)


@pytest.mark.parametrize("dt", ["f64", "f32"])
def test_extract_matches_blas(dt):
    X = synth.make_X(70_003, 9, 3.0, dt)          # spans two 65536-row blocks
    Y = oracle.extract(X, 20, 12)
    ref = _L_dense(X.shape[0], 20, 12) @ X.astype(np.float64)
    assert np.linalg.norm(Y - ref) <= 1e-13 * np.linalg.norm(ref)


def test_extractor_continues_the_gaussian_stream():
    # [Theta; L] is one (k + l)-row Gaussian draw: unscaled rows k.. of the (k + l)-row sketch are L's
    X = synth.make_X(3_000, 5, 2.0)
    k, l = 12, 8
    Pext = oracle.sketch(X, k + l) * np.sqrt(np.float64(k + l))
    Y = oracle.extract(X, k, l) * np.sqrt(np.float64(l))
    assert np.allclose(Pext[k:], Y, rtol=1e-13, atol=1e-13 * np.abs(Y).max())


def test_extract_partition_invariance():
    X = synth.make_X(10_000, 6, 3.0)
    Y = oracle.extract(X, 16, 10)
    Ya = oracle.extract(X[:4_321], 16, 10, row_offset=0)
    Yb = oracle.extract(X[4_321:], 16, 10, row_offset=4_321)
    assert np.allclose(Ya + Yb, Y, rtol=1e-14, atol=1e-14 * np.abs(Y).max())


@pytest.mark.parametrize("sk,c", [(oracle.GAUSSIAN, 3.0), (oracle.GAUSSIAN, 8.0), (oracle.SPARSE_SIGN, 4.0)])
def test_z_equals_L_times_Q(sk, c):
    m, n, k, l = 20_000, 16, 32, 24
    X = synth.make_X(m, n, c)
    out = oracle.factor_reduced(X, k, l, sketch=sk)
    Q = scipy.linalg.solve_triangular(out["R"], X.T, trans="T", lower=False).T      # X R^{-1}
    LQ = _L_dense(m, k, l, sk) @ Q
    kappa = 10.0**c
    assert np.linalg.norm(out["Z"] - LQ) <= 10 * U64 * kappa * np.linalg.norm(LQ)


def test_step2_is_alg2s_qr():
    X = synth.make_X(8_000, 12, 5.0)
    red = oracle.factor_reduced(X, 24, 7)
    alg2 = oracle.factor(X, 24)
    assert np.array_equal(red["R"], alg2["R"]) and np.array_equal(red["S"], alg2["S"])


def test_single_row_extractor_closed_form():
    X = synth.make_X(4_000, 5, 2.0)
    out = oracle.factor_reduced(X, 10, 1)
    z = scipy.linalg.solve_triangular(out["R"], out["Y"][0], trans="T", lower=False)
    assert np.allclose(out["Z"][0], z, rtol=1e-13, atol=1e-15)


def test_metamorphic_power_of_two_scaling():
    X = synth.make_X(6_000, 8, 4.0)
    a = oracle.factor_reduced(X, 16, 9)
    b = oracle.factor_reduced(X * 2.0**-7, 16, 9)
    assert np.array_equal(a["Z"], b["Z"]) and np.array_equal(a["R"] * 2.0**-7, b["R"])
    D = 2.0 ** np.array([3, -2, 0, 5, -4, 1, 2, -1], dtype=np.float64)
    c = oracle.factor_reduced(X * D, 16, 9)
    assert np.array_equal(a["Z"], c["Z"]) and np.array_equal(a["R"] * D, c["R"])


def test_fp32_x_promoted_exactly():
    X = synth.make_X(5_000, 6, 3.0, "f32")
    a = oracle.factor_reduced(X, 12, 5)
    b = oracle.factor_reduced(X.astype(np.float64), 12, 5)
    assert np.array_equal(a["Z"], b["Z"]) and np.array_equal(a["R"], b["R"])
