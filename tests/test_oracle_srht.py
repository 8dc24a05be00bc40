"""Pins of the SRHT Theta (reading A23: Theta = sqrt(m'/k) R H D, m' = 2^48).

* H is the Walsh-Hadamard matrix: for rows i < 1024 the signs equal the Sylvester construction
  H_1024 = H_2 (x) ... (x) H_2 (numpy Kronecker products, independent of the popcount formula)
  at row (s_r mod 1024), times the Philox sign d_i (pinned by the Philox KATs).
* R samples k DISTINCT rows below 2^48.
* E ||Theta x||^2 = ||x||^2 (H orthogonal, D and R unbiased); balanced signs.
* Sketch: exact rational Theta X on tiny inputs; BLAS with the explicit Theta; partition invariance.
* Alg. 2 with an SRHT Theta: R equals LAPACK's R of P; cond(Q) = cond(Theta U).
"""
from fractions import Fraction

import numpy as np

import oracle
import synth


def _sylvester(order_log2):
    H = np.array([[1]], dtype=np.int64)
    H2 = np.array([[1, 1], [1, -1]], dtype=np.int64)
    for _ in range(order_log2):
        H = np.kron(H2, H)
    return H


def _d(seed, i):
    w = oracle.philox4x32_10([i & 0xFFFFFFFF, i >> 32, 0, 6], [seed & 0xFFFFFFFF, seed >> 32])
    return -1 if int(w[0]) & 1 else 1


def test_signs_are_sylvester_hadamard_rows_times_d():
    seed, k, m = 5, 40, 1024
    H = _sylvester(10)
    s = oracle.srht_rows(seed, k)
    S = oracle.theta_srht(seed, k, m)
    d = np.array([_d(seed, i) for i in range(m)])
    for r in range(k):
        assert np.array_equal(S[r], H[int(s[r]) % 1024] * d)


def test_sampled_rows_distinct_and_in_range():
    s = oracle.srht_rows(11, 4096)
    assert len(set(s.tolist())) == 4096 and int(s.max()) < 2**48
    # the sample is not concentrated: every 4-bit prefix of the 48-bit rows occurs
    assert len(set((s >> np.uint64(44)).tolist())) == 16


def test_isometry_in_expectation_and_balance():
    rng = np.random.default_rng(3)
    x = rng.standard_normal(700)
    vals = [np.sum((oracle.theta_dense(sd, 64, 700, oracle.SRHT) @ x) ** 2) for sd in range(300)]
    assert abs(np.mean(vals) / np.dot(x, x) - 1.0) < 0.03
    S = oracle.theta_srht(2, 128, 5000, row_offset=123456789).astype(np.float64)
    assert abs(S.sum()) / np.sqrt(S.size) < 4.5


def test_sketch_exact_rational():
    rng = np.random.default_rng(4)
    X = rng.standard_normal((31, 3))
    P = oracle.sketch(X, 12, sketch=oracle.SRHT, seed=9)
    T = oracle.theta_srht(9, 12, 31).astype(np.int64)
    sk = Fraction(1.0 / np.sqrt(12.0))
    for r in range(12):
        for j in range(3):
            exact = sum(int(T[r, i]) * sk * Fraction(X[i, j]) for i in range(31))
            bound = Fraction(2.0**-52) * sum(abs(sk * Fraction(X[i, j])) for i in range(31))
            assert abs(Fraction(P[r, j]) - exact) <= bound + Fraction(1, 2**1074)


def test_sketch_matches_blas_and_partition():
    X = synth.make_X(70_003, 6, 3.0, "f32")
    P = oracle.sketch(X, 24, sketch=oracle.SRHT)
    ref = oracle.theta_dense(0, 24, X.shape[0], oracle.SRHT) @ X.astype(np.float64)
    assert np.linalg.norm(P - ref) <= 1e-13 * np.linalg.norm(ref)
    Pa = oracle.sketch(X[:40_000], 24, sketch=oracle.SRHT)
    Pb = oracle.sketch(X[40_000:], 24, sketch=oracle.SRHT, row_offset=40_000)
    assert np.allclose(Pa + Pb, P, rtol=1e-14, atol=1e-14 * np.abs(P).max())
    x = np.ascontiguousarray(X[:, 2], dtype=np.float64)
    assert abs(oracle.sketch_entry(x, 17, 24, sketch=oracle.SRHT) - P[17, 2]) <= 1e-13 * np.abs(P).max()


def test_alg2_with_srht():
    X = synth.make_X(20_000, 16, 6.0)
    out = oracle.factor(X, 64, sketch=oracle.SRHT)
    Rl = np.linalg.qr(out["P"], mode="r")
    Rl = np.sign(np.diag(Rl))[:, None] * Rl
    assert np.linalg.norm(out["R"] - Rl) <= 1e-13 * np.linalg.norm(Rl)
    U, _ = np.linalg.qr(X)
    TU = oracle.theta_dense(0, 64, X.shape[0], oracle.SRHT) @ U
    assert abs(oracle.cond(out["Q"]) / oracle.cond(TU) - 1) < 1e-3
    assert oracle.cond(out["Q"]) <= 8.0


def test_blocked_walsh_hadamard_identity():
    """The identity behind the GPU's fast transform (csrc/srht_fwht.cu; the SRHT costs
    m n log2 m): with the global row i = B h + l and s_r = B sh_r + sl_r (B a power of two),
    popcount(s_r & i) = popcount(sh_r & h) + popcount(sl_r & l), so
        (Theta X)_r sqrt(k) = sum_h (-1)^popcount(sh_r & h) Y_h[sl_r],   Y_h = H_B (d .* X)[block h],
    with blocks aligned to GLOBAL multiples of B (rows outside X are zero).  Checked in exact integer
    arithmetic against the oracle's entry-by-entry signs, with a row offset inside a block, a ragged
    last block and a Sylvester H_B built by Kronecker products (numpy only: no code of the CUDA path)."""
    B, k, m, n, ro = 64, 24, 300, 5, 2**35 + 37          # ro mod B = 37: the first block is partial
    rng = np.random.default_rng(5)
    X = rng.integers(-1000, 1000, size=(m, n)).astype(np.int64)
    S = oracle.theta_srht(3, k, m, ro).astype(np.int64)  # signs (-1)^popcount(s_r & i) d_i
    want = S @ X
    s = oracle.srht_rows(3, k)
    H = np.array([[1]], dtype=np.int64)
    while H.shape[0] < B:
        H = np.kron(np.array([[1, 1], [1, -1]], dtype=np.int64), H)   # Sylvester: H[t, l] = (-1)^popcount(t & l)
    # d_i from the oracle's own signs: row r of S is (-1)^popcount(s_r & i) d_i
    i_glob = ro + np.arange(m, dtype=np.uint64)
    par0 = np.array([bin(int(s[0] & i)).count("1") & 1 for i in i_glob])
    d = S[0] * np.where(par0 == 1, -1, 1)
    got = np.zeros((k, n), dtype=np.int64)
    h0, h1 = ro // B, (ro + m - 1) // B
    for h in range(h0, h1 + 1):
        blk = np.zeros((B, n), dtype=np.int64)
        for l in range(B):
            i = h * B + l - ro                           # local row of global row B h + l
            if 0 <= i < m:
                blk[l] = d[i] * X[i]
        Y = H @ blk                                      # the B-point Walsh-Hadamard transform of the block
        for r in range(k):
            sl, sh = int(s[r]) % B, int(s[r]) // B
            sign = -1 if bin(sh & h).count("1") & 1 else 1
            got[r] += sign * Y[sl]
    assert np.array_equal(got, want)
