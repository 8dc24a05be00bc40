"""GPU parity for the SRHT Theta (reading A23: (-1)^popcount(s_r & i) d_i / sqrt(k), m' = 2^48) through
the C ABI.

Theta signs bit-exact (rcholqr_theta_export vs oracle.theta_srht, which is pinned to a Sylvester
Hadamard matrix); P <= 1e-12 relative Frobenius vs the compensated oracle on the dense tcgen05 int8
path (n <= 64, k <= 512, row_offset % 32 == 0: Walsh masks of s_r & 31 x the ballot of d_i) and on
the DMMA path (n > 64, unaligned rows or row offsets, or RCHOLQR_RADEMACHER_DMMA); the
headroom-overflow fallback; Alg. 2 / Alg. 5 end to end.
"""
import numpy as np
import pytest
import torch

import oracle
import paper_2210_09953_b200 as rcq
import synth

pytestmark = pytest.mark.gpu
U64 = 2.0**-53
U32 = 2.0**-24


def _t(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def _np(t):
    return t.detach().cpu().numpy()


def _rel(a, b):
    a, b = np.asarray(a, dtype=np.float64), np.asarray(b, dtype=np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def _plan(n, k, dt, seed=0):
    return rcq.RCholQR(n=n, k=k, dtype=torch.float64 if dt == "f64" else torch.float32, sketch="srht",
                       seed=seed)


@pytest.mark.parametrize("k,m,ro,seed", [(300, 1000, 0, 0), (64, 777, 2**33 + 5, 99)])
def test_theta_export_bit_exact(cuda, k, m, ro, seed):
    Z = _np(rcq.theta_export(seed, k, m, sketch="srht", row_offset=ro))
    S = oracle.theta_srht(seed, k, m, ro)
    assert np.array_equal(Z, S.astype(np.float32))


@pytest.mark.parametrize("m,n,k,dt", [
    (100_003, 64, 128, "f32"),     # tcgen05 dense-E path (row_offset 32 x 777 keeps the tcgen05 path)
    (70_001, 48, 96, "f64"),       # tcgen05, fp64 digits
    (50_000, 32, 300, "f32"),      # tcgen05, three Theta tiles (Philox q = 0, 1, 2)
    (40_000, 100, 200, "f32"),     # n > 64: DMMA path drawing +-1
    (333, 17, 34, "f64"),          # fewer rows than CTAs, ragged
])
@pytest.mark.parametrize("dense", [True, False])
def test_sketch_parity(cuda, monkeypatch, m, n, k, dt, dense):
    # dense: the +-1 kernels at every k (by default k > 128 runs the fast Walsh-Hadamard transform, srht_fwht.cu)
    if dense:
        monkeypatch.setenv("RCHOLQR_SRHT_DENSE", "1")
    X = synth.make_X(m, n, 5.0, dt)
    plan = _plan(n, k, dt)
    Pg = _np(plan.sketch(_t(X), row_offset=24_864))
    assert bool(plan.last_path() & rcq.PATH_SKETCH_FWHT) == (not dense and k > 128 and (n * X.itemsize) % 16 == 0)
    Po = oracle.sketch(X, k, sketch=oracle.SRHT, row_offset=24_864)
    assert _rel(Pg, Po) <= 1e-12, _rel(Pg, Po)


def test_sketch_tc_matches_dmma(cuda, monkeypatch):
    X = _t(synth.make_X(300_000, 64, 4.0, "f32"))
    a = _np(_plan(64, 128, "f32").sketch(X))
    monkeypatch.setenv("RCHOLQR_RADEMACHER_DMMA", "1")
    b = _np(_plan(64, 128, "f32").sketch(X))
    assert _rel(a, b) <= 1e-13, _rel(a, b)


@pytest.mark.parametrize("case", ["spike", "zero-first-stage"])
def test_sketch_headroom_overflow(cuda, case):
    m, n, k = 300_000, 64, 128
    X = synth.make_X(m, n, 2.0, "f32")
    if case == "spike":
        X[1000::4099, :] *= 1e6
    else:
        X[np.arange(m) % 2048 < 64, 5] = 0.0
    Pg = _np(_plan(n, k, "f32").sketch(_t(X)))
    Po = oracle.sketch(X, k, sketch=oracle.SRHT)
    assert _rel(Pg, Po) <= 1e-12, _rel(Pg, Po)


def test_sketch_unaligned_rows_take_dmma(cuda):
    X = synth.make_X(20_000, 37, 3.0, "f32")           # 37 fp32 = 148 B rows: no bulk copies
    Pg = _np(_plan(37, 74, "f32").sketch(_t(X)))
    Po = oracle.sketch(X, 74, sketch=oracle.SRHT)
    assert _rel(Pg, Po) <= 1e-12


@pytest.mark.parametrize("dt,c", [("f32", 4), ("f64", 10)])
def test_factor_parity(cuda, dt, c):
    m, n, k = 262_144, 64, 128
    X = synth.make_X(m, n, c, dt)
    ref = oracle.factor(X, k, sketch=oracle.SRHT)
    Q, R, S = _plan(n, k, dt).factor(_t(X), want_S=True)
    assert _rel(_np(R), ref["R"]) <= (1e-10 if dt == "f64" else 1e-4)
    assert _rel(_np(Q), ref["Q"]) <= 10 * U64 * 10**c + (2 * U32 if dt == "f32" else 0)
    assert oracle.orth_defect(_np(S)) <= 1e-13


def test_unaligned_row_offset_takes_dmma(cuda):
    # the tcgen05 SRHT tile needs row_offset % 32 == 0; other offsets run the DMMA kernel
    X = synth.make_X(60_000, 32, 4.0, "f32")
    for ro in (0, 32 * 12345, 7, 2**33 + 3):
        Pg = _np(_plan(32, 64, "f32").sketch(_t(X), row_offset=ro))
        Po = oracle.sketch(X, 64, sketch=oracle.SRHT, row_offset=ro)
        assert _rel(Pg, Po) <= 1e-12, (ro, _rel(Pg, Po))


def test_reduced_with_srht(cuda):
    X = synth.make_X(100_000, 40, 4.0)
    ref = oracle.factor_reduced(X, 80, 30, sketch=oracle.SRHT)
    Z, R, _, Y = _plan(40, 80, "f64").factor_reduced(_t(X), 30, want_Y=True)
    assert _rel(_np(Y), ref["Y"]) <= 1e-12 and _rel(_np(R), ref["R"]) <= 1e-10
    assert _rel(_np(Z), ref["Z"]) <= 10 * U64 * 1e4


def test_one_plan_all_entry_points_interleaved(cuda):
    # one plan through every entry point in turn, growing workspaces (new l) in between: results equal
    # those of fresh plans and no CUDA error is left behind (regression: a workspace regrowth once
    # freed other entry points' buffers)
    X = _t(synth.make_X_lowrank(60_000, 24, 20, 2.0, 1e-13))
    plan = _plan(24, 48, "f64")
    a1 = plan.factor_reduced(X, 10)
    r1 = plan.factor_rr(X, 1e-9)
    a2 = plan.factor_reduced(X, 17)                    # regrows the reduced workspace
    r2 = plan.factor_rr(X, 1e-9)
    P = plan.sketch(X)
    q2 = plan.factor2(X)
    for got, fresh in ((a1, _plan(24, 48, "f64").factor_reduced(X, 10)),
                       (a2, _plan(24, 48, "f64").factor_reduced(X, 17))):
        assert torch.equal(got[0], fresh[0]) and torch.equal(got[1], fresh[1])
    for got in (r1, r2):
        fresh = _plan(24, 48, "f64").factor_rr(X, 1e-9)
        assert got["rank"] == fresh["rank"] == 20
        assert torch.equal(got["perm"], fresh["perm"]) and torch.equal(got["Q"], fresh["Q"])
    assert torch.equal(P, _plan(24, 48, "f64").sketch(X))
    assert torch.equal(q2[1], _plan(24, 48, "f64").factor2(X)[1])
    plan.close()
    rcq.theta_export(0, 8, 16, sketch="rademacher")    # raises if an error was left pending


def test_edge_cases_new_entry_points(cuda):
    X = synth.make_X(30_000, 20, 3.0)
    Xt = _t(X)
    # SRHT with k > 512 (beyond the tcgen05 tile limit): DMMA path, still the oracle's sketch
    Pg = _np(_plan(20, 600, "f64").sketch(Xt))
    assert _rel(Pg, oracle.sketch(X, 600, sketch=oracle.SRHT)) <= 1e-12
    # Alg. 5 with more extractor rows than sketch rows, sparse Theta
    plan = rcq.RCholQR(n=20, k=40, dtype=torch.float64, sketch="sparse", nnz_per_col=8)
    Z, R, _, Y = plan.factor_reduced(Xt, 90, want_Y=True)
    ref = oracle.factor_reduced(X, 40, 90, sketch=oracle.SPARSE_SIGN, zeta=8)
    assert _rel(_np(Y), ref["Y"]) <= 1e-12 and _rel(_np(Z), ref["Z"]) <= 1e-11
    # Alg. 7 with tau = 0 on a full-rank X: rank n, Q equals Alg. 2 on the permuted columns
    g = _plan(20, 40, "f64").factor_rr(Xt, 0.0)
    assert g["rank"] == 20
    perm = _np(g["perm"]).astype(np.int64)
    Qp, _, _ = _plan(20, 40, "f64").factor(_t(np.ascontiguousarray(X[:, perm])))
    assert _rel(_np(g["Q"]), _np(Qp)) <= 1e-12
    # RRRCholeskyQR2 at a fixed rank: orthonormal m x r Q
    g2 = _plan(20, 40, "f64").factor_rr2(Xt, 0.0, rank_fixed=7)
    Q = _np(g2["Q"])
    assert g2["rank"] == 7 and Q.shape == (30_000, 7)
    assert np.linalg.norm(Q.T @ Q - np.eye(7), 2) <= 1e-13
