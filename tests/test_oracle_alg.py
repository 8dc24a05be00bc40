"""Pins of the oracle's Algorithm 2 steps against what the paper and the
mathematics fix: exact rational arithmetic, closed forms, LAPACK/mpmath/scipy, the worked examples
of tests/golden/spec_examples.txt, the paper's bounds (eq:main1-3, Higham Thm 8.5 via PAPER.md:425),
the exact identity cond(Q) = cond(Theta U) (Cor. thm:epscond with eq:sketchedcond) and exact
power-of-two metamorphic relations.  CPU only."""
import os
from fractions import Fraction

import mpmath
import numpy as np
import pytest
import scipy.linalg as sla

import oracle
import synth

U64 = 2.0**-53
GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _spec_examples():
    out = []
    with open(os.path.join(GOLDEN, "spec_examples.txt")) as f:
        for line in f:
            if line.startswith("#") or not line.strip():
                continue
            tok = line.split()
            kind, mats, t = tok[0], {}, 1
            while t < len(tok):
                name, r, c = tok[t], int(tok[t + 1]), int(tok[t + 2])
                vals = [float(x) for x in tok[t + 3:t + 3 + r * c]]
                mats[name] = np.array(vals).reshape(r, c)
                t += 3 + r * c
            out.append((kind, mats))
    return out


# ------------------------------------------------------------------ sketch (step 1)
def test_sketch_exact_rational_tiny():
    # P = Theta X computed exactly in rationals from the same Theta, then compared with the
    # worst-case rounding bound |E1| <= m u/(1 - m u) |Theta||X|.
    rng = np.random.default_rng(0)
    for sk, zeta in [(oracle.GAUSSIAN, 8), (oracle.SPARSE_SIGN, 4)]:
        m, n, k = 37, 5, 16
        X = rng.standard_normal((m, n))
        T = oracle.theta_dense(5, k, m, sketch=sk, zeta=zeta)
        P = oracle.sketch(X, k, sketch=sk, zeta=zeta, seed=5)
        bound = (m * U64 / (1 - m * U64)) * (np.abs(T) @ np.abs(X))
        for r in range(k):
            for j in range(n):
                exact = sum(Fraction(float(T[r, i])) * Fraction(float(X[i, j])) for i in range(m))
                assert abs(Fraction(float(P[r, j])) - exact) <= Fraction(float(bound[r, j])) + Fraction(1, 10**300)


def test_sketch_n1_closed_form_and_linearity():
    rng = np.random.default_rng(1)
    m, k = 5000, 12
    x = rng.standard_normal((m, 1))
    T = oracle.theta_dense(9, k, m)
    P = oracle.sketch(x, k, seed=9)
    bound = 2 * m * U64 * (np.abs(T) @ np.abs(x[:, 0]))
    assert np.all(np.abs(P[:, 0] - T @ x[:, 0]) <= bound)
    # linearity in X: Theta(aX + bY) = a Theta X + b Theta Y with a, b powers of two
    X = rng.standard_normal((m, 3))
    Y = rng.standard_normal((m, 3))
    P1 = oracle.sketch(4.0 * X + 0.5 * Y, k, seed=9)
    P2 = 4.0 * oracle.sketch(X, k, seed=9) + 0.5 * oracle.sketch(Y, k, seed=9)
    assert np.allclose(P1, P2, rtol=1e-12, atol=1e-12 * np.abs(P2).max())


def test_sketch_partition_invariance():
    # Theta keyed by the GLOBAL row: sum of the sketches of row blocks = sketch of the whole
    # (reduction operator = addition).  The oracle's compensated sums are accurate
    # to ~1 ulp, so the parts agree with the whole to a few ulps of the largest part.
    X = synth.make_X(3 * 65536, 6, 3.0)
    P = oracle.sketch(X, 12, seed=2)
    parts = [oracle.sketch(X[b * 65536:(b + 1) * 65536], 12, seed=2, row_offset=b * 65536) for b in range(3)]
    scale = np.max(np.abs(parts), axis=0)
    assert np.all(np.abs(P - (parts[0] + parts[1] + parts[2])) <= 4 * U64 * scale)
    Pu = oracle.sketch(X[:100_000], 12, seed=2) + oracle.sketch(X[100_000:], 12, seed=2, row_offset=100_000)
    assert np.all(np.abs(P - Pu) <= 4 * U64 * scale)


def test_sketch_fp32_input_promoted_exactly():
    X = synth.make_X(20_000, 7, 2.0, dtype="f32")
    assert np.array_equal(oracle.sketch(X, 14, seed=1), oracle.sketch(X.astype(np.float64), 14, seed=1))


def test_sketch_nonfinite():
    X = np.ones((100, 3))
    X[50, 1] = np.nan
    with pytest.raises(oracle.OracleError) as e:
        oracle.sketch(X, 6)
    assert e.value.status == oracle.E_NONFINITE


# ------------------------------------------------------------------ Householder (step 2)
@pytest.mark.parametrize("case", [c for c in _spec_examples() if c[0] == "householder"])
def test_householder_spec_examples(case):
    _, M = case
    R, S, st = oracle.householder(M["P"])
    assert st == oracle.OK
    assert np.allclose(R, M["R"], atol=1e-15) and np.allclose(S, M["S"], atol=1e-15)


@pytest.mark.parametrize("k,n", [(20, 5), (40, 20), (200, 100), (10, 10), (128, 64)])
def test_householder_vs_lapack(k, n):
    rng = np.random.default_rng(k * 1000 + n)
    P = rng.standard_normal((k, n)) @ np.diag(10.0 ** -np.linspace(0, 6, n))
    R, S, st = oracle.householder(P)
    assert st == oracle.OK
    Ql, Rl = np.linalg.qr(P)
    d = np.sign(np.diag(Rl))
    Rl = d[:, None] * Rl
    Ql = Ql * d[None, :]
    assert np.all(np.diag(R) > 0)
    assert np.allclose(np.tril(R, -1), 0.0, atol=0)
    # R is unique for full-rank P: R_jl agree to O(u) relative to the column norms of P
    colnorm = np.linalg.norm(P, axis=0)
    assert np.max(np.abs(R - Rl) / colnorm[None, :]) < 50 * n * U64
    assert np.max(np.abs(S - Ql)) < 1e-9  # S is determined up to the conditioning of P
    # SPEC.md:110 invariants
    assert np.linalg.norm(S.T @ S - np.eye(n)) <= 50 * n * U64
    assert np.linalg.norm(P - S @ R) <= 50 * n * U64 * np.linalg.norm(P)


def test_householder_mpmath_50_digits():
    mpmath.mp.dps = 50
    rng = np.random.default_rng(3)
    k, n = 9, 4
    P = rng.standard_normal((k, n))
    R, _, _ = oracle.householder(P)
    # exact-arithmetic R = chol(P^T P) (unique with diag > 0), computed with 50 digits
    A = mpmath.matrix(P.tolist())
    G = A.T * A
    L = mpmath.cholesky(G)
    Rexact = np.array(L.T.tolist(), dtype=np.float64)
    assert np.max(np.abs(R - Rexact)) < 1e-14 * np.abs(Rexact).max()


def test_householder_n1_closed_form():
    p = np.array([[3.0], [-4.0], [12.0]])
    R, S, _ = oracle.householder(p)
    assert R[0, 0] == pytest.approx(13.0, rel=1e-15)
    assert np.allclose(S[:, 0], p[:, 0] / 13.0, atol=1e-16)


def test_householder_singular_and_zero_column():
    P = np.zeros((6, 3))
    P[:, 0] = 1.0
    P[:, 2] = np.arange(6)
    R, S, st = oracle.householder(P)
    assert st == oracle.E_SINGULAR and R[1, 1] == 0.0


# ------------------------------------------------------------------ substitution (step 3)
@pytest.mark.parametrize("case", [c for c in _spec_examples() if c[0] == "trisolve"])
def test_trisolve_spec_examples(case):
    _, M = case
    assert np.allclose(oracle.forward_subst(M["X"], M["R"]), M["Q"], atol=0)


def test_trisolve_identity_and_scipy():
    rng = np.random.default_rng(4)
    X = rng.standard_normal((1000, 12))
    assert np.array_equal(oracle.forward_subst(X, np.eye(12)), X)
    R = np.triu(rng.standard_normal((12, 12))) + 5 * np.eye(12)
    Q = oracle.forward_subst(X, R)
    Qs = sla.solve_triangular(R, X.T, trans="T", lower=False).T  # solve R^T Q^T = X^T
    assert np.allclose(Q, Qs, rtol=1e-12, atol=1e-12)
    # Higham Thm 8.5: each row is backward stable, |x_i - q_i R| <= 1.1 n u |q_i||R|
    E = np.abs(X - Q @ R)
    assert np.all(E <= 1.1 * 12 * U64 * (np.abs(Q) @ np.abs(R)) + 1e-300)


def test_trisolve_singular():
    R = np.eye(3)
    R[1, 1] = 0.0
    with pytest.raises(oracle.OracleError) as e:
        oracle.forward_subst(np.ones((4, 3)), R)
    assert e.value.status == oracle.E_SINGULAR


def test_trisolve_fp32_rounds_once():
    rng = np.random.default_rng(5)
    X = rng.standard_normal((500, 6)).astype(np.float32)
    R = np.triu(rng.standard_normal((6, 6))) + 4 * np.eye(6)
    Q32 = oracle.forward_subst(X, R)
    Q64 = oracle.forward_subst(X.astype(np.float64), R)
    assert np.array_equal(Q32, Q64.astype(np.float32))


# ------------------------------------------------------------------ whole Algorithm 2
@pytest.mark.parametrize("m,n,c,dt,sk", [(20_000, 20, 3, "f64", oracle.GAUSSIAN),
                                         (50_000, 32, 10, "f64", oracle.GAUSSIAN),
                                         (60_000, 16, 4, "f32", oracle.SPARSE_SIGN),
                                         (40_000, 24, 5, "f32", oracle.GAUSSIAN)])
def test_factor_paper_bounds(m, n, c, dt, sk):
    k = 2 * n
    X = synth.make_X(m, n, c, dt)
    out = oracle.factor(X, k, sketch=sk, zeta=8 if k % 8 == 0 else 4, seed=0)
    Q, R, P, S = out["Q"], out["R"], out["P"], out["S"]
    Xd = X.astype(np.float64)
    u = U64 if dt == "f64" else 2.0**-24
    # eq:main1: column residual <= 2.1 u n (fp64 solve; fp32 adds Q's rounding)
    res = oracle.col_residual(Xd, Q, R)
    assert res <= 2.1 * (U64 if dt == "f64" else u) * n, res
    # exact identity cond(Q) = cond(Theta U), U an orthonormal basis of range(X) (A11)
    Ux, _ = np.linalg.qr(Xd)
    TU = oracle.sketch(Ux, k, sketch=sk, zeta=8 if k % 8 == 0 else 4, seed=0)
    cq = oracle.cond(Q.astype(np.float64))
    assert abs(cq / oracle.cond(TU) - 1.0) < 1e-3 + 10 * u * 10**c
    # S orthonormal (eq:ass2) and P = S R
    assert oracle.orth_defect(S) < 50 * n * U64
    assert np.linalg.norm(P - S @ R) < 50 * n * U64 * np.linalg.norm(P)
    # eq:main3: ||S - Theta Q||_F <= 6.1 u n^{3/2} kappa (paper bound; rule of thumb: sqrt of it)
    TQ = oracle.sketch(Q, k, sketch=sk, zeta=8 if k % 8 == 0 else 4, seed=0)
    kappa = oracle.cond(Xd / np.linalg.norm(Xd, axis=0))
    assert np.linalg.norm(S - TQ) <= 6.1 * u * n**1.5 * kappa


def test_factor_metamorphic_power_of_two_scaling():
    # Every step is homogeneous and power-of-two scalings commute with rounding:
    # factor(X 2^e) = (Q, R 2^e) and factor(X D) = (Q, R D) BITWISE for D = diag(2^e_j).
    X = synth.make_X(30_000, 10, 6.0)
    base = oracle.factor(X, 20, seed=3)
    sc = oracle.factor(X * 2.0**7, 20, seed=3)
    assert np.array_equal(sc["Q"], base["Q"]) and np.array_equal(sc["R"], base["R"] * 2.0**7)
    D = 2.0 ** np.array([3, -2, 0, 5, -7, 1, 1, -1, 4, -3], dtype=np.float64)
    sd = oracle.factor(X * D[None, :], 20, seed=3)
    assert np.array_equal(sd["Q"], base["Q"]) and np.array_equal(sd["R"], base["R"] * D[None, :])


def test_factor_orthogonality_defect_scales_with_kappa():
    # A12: ||I - (Theta Q)^T Theta Q||_2 ~ 2 u kappa for fp64 (eq:main3), so tiny at kappa=1e3 ...
    Xa = synth.make_X(20_000, 20, 3.0)
    oa = oracle.factor(Xa, 40, seed=0)
    da = oracle.orth_defect(oracle.sketch(oa["Q"], 40, seed=0))
    assert da < 1e-12  # north-star fp64 tolerance met by the oracle at kappa = 1e3
    # ... and growing linearly with kappa (never exceeding the eq:main3-derived bound)
    Xb = synth.make_X(20_000, 20, 10.0)
    ob = oracle.factor(Xb, 40, seed=0)
    db = oracle.orth_defect(oracle.sketch(ob["Q"], 40, seed=0))
    assert 1e3 * da < db < 2 * 6.1 * U64 * 20**1.5 * 1e10


# ------------------------------------------------------------------ sketch_entry (sampled checker)
@pytest.mark.parametrize("sk,zeta", [(oracle.GAUSSIAN, 8), (oracle.SPARSE_SIGN, 8), (oracle.SPARSE_SIGN, 96)])
def test_sketch_entry_exact_rational(sk, zeta):
    # oracle_sketch_entry is the checker of the full-size GPU sketches (tests/test_gpu_parity.py).  Pin it
    # to exact rational sums of the KAT-pinned Theta (theta_dense -> oracle_theta_gauss_z /
    # oracle_theta_sparse) with a 64-bit row offset, inside the Dot2 bound (~2u |sum| + u^2 sum|terms|,
    # PAPER.md:422 with u_f ~ u^2).  zeta = 96 > 64 exercises the heap buffers (no fixed rows[64]).
    rng = np.random.default_rng(11)
    m, k, off = 45, (192 if zeta == 96 else 24), 2**35 + 3
    x = rng.standard_normal(m)
    T = oracle.theta_dense(4, k, m, sketch=sk, zeta=zeta, row_offset=off)
    for r in range(k):
        got = oracle.sketch_entry(x, r, k, sketch=sk, zeta=zeta, seed=4, row_offset=off)
        exact = sum(Fraction(float(T[r, i])) * Fraction(float(x[i])) for i in range(m))
        mag = sum(abs(Fraction(float(T[r, i])) * Fraction(float(x[i]))) for i in range(m))
        assert abs(Fraction(got) - exact) <= Fraction(2.0**-52) * abs(exact) + Fraction(2.0**-100) * mag \
            + Fraction(1, 2**1074)


@pytest.mark.parametrize("sk", [oracle.GAUSSIAN, oracle.SPARSE_SIGN, oracle.RADEMACHER])
def test_sketch_entry_equals_sketch_across_blocks(sk):
    # Same fixed 65,536-row blocks, same Dot2 order => the sampled checker reproduces the pinned
    # oracle_sketch bitwise, over several blocks and with a row offset that is not a multiple of 32.
    X = synth.make_X(2 * 65536 + 777, 5, 3.0, "f32")
    k, off = 32, 1_000_003
    P = oracle.sketch(X, k, sketch=sk, seed=7, row_offset=off)
    for r in (0, 3, 17, 31):
        for j in (0, 4):
            x = np.ascontiguousarray(X[:, j], dtype=np.float64)
            assert oracle.sketch_entry(x, r, k, sketch=sk, seed=7, row_offset=off) == P[r, j]


def test_sketch_entry_rejects_bad_arguments():
    x = np.ones(10)
    for kw in [dict(r=-1, k=8), dict(r=8, k=8), dict(r=0, k=0),
               dict(r=0, k=8, sketch=oracle.SPARSE_SIGN, zeta=0),
               dict(r=0, k=10, sketch=oracle.SPARSE_SIGN, zeta=4),
               dict(r=0, k=8, sketch=oracle.SPARSE_SIGN, zeta=9),
               dict(r=0, k=8, sketch=7)]:
        assert np.isnan(oracle.sketch_entry(x, **kw))
