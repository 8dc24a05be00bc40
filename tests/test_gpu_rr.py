"""GPU parity for the rank-revealing RCholeskyQR (Alg. 7) through the C ABI
(rcholqr_factor_rr).

Unique and compared exactly: the rank r (an integer the method decides), the selected columns
perm[:r] and the whole permutation while r = n, and the number of swaps.  Beyond the rank the
pivot order among noise-level columns is not unique (A21), so R is compared column by
ORIGINAL column index.  Bars: R <= 1e-10 relative (fp64 X) / 1e-4 (fp32 X) -- the north-star R bars;
Q <= 10 u kappa_sel relative (kappa_sel bounded by 10 n^1.5 r / tau; 1e4 used below);
Q well conditioned; the column-normalised residual within PAPER.md:743.
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


def _by_original_column(R, perm, n):
    out = np.zeros((R.shape[0], n))
    out[:, perm] = R
    return out


CASES = [
    # name, X kind, m, n, k, rank (None = full), dtype, sketch, tau, f, rank_fixed
    ("full-f64", "full", 30_000, 16, 32, None, "f64", "gaussian", 1e-15, 1.5, 0),
    ("lowrank-f64", "low", 100_000, 48, 96, 30, "f64", "gaussian", 1e-9, 1.5, 0),
    ("lowrank-f32-sparse", "low", 262_144, 64, 128, 40, "f32", "sparse", 1e-5, 1.5, 0),
    ("lowrank-f32-gauss", "low", 200_003, 100, 200, 70, "f32", "gaussian", 1e-5, 1.5, 0),
    ("C3-shape-lowrank", "low", 40_000, 256, 512, 180, "f64", "gaussian", 1e-9, 1.5, 0),
    ("swaps-fixed-rank", "full", 20_000, 24, 48, None, "f64", "gaussian", 0.0, 1.01, 12),
    ("swaps-lowrank", "low", 20_000, 24, 48, 16, "f64", "gaussian", 1e-9, 1.01, 0),
]


@pytest.mark.parametrize("name,kind,m,n,k,rank,dt,sk,tau,f,rf", CASES)
def test_factor_rr_parity(cuda, name, kind, m, n, k, rank, dt, sk, tau, f, rf):
    X = synth.make_X(m, n, 4.0, dt) if kind == "full" else synth.make_X_lowrank(m, n, rank, 2.0, 1e-13, dt)
    so = oracle.GAUSSIAN if sk == "gaussian" else oracle.SPARSE_SIGN
    ref = oracle.factor_rr(X, k, tau, f=f, rank_fixed=rf, sketch=so, zeta=8)
    plan = rcq.RCholQR(n=n, k=k, dtype=torch.float64 if dt == "f64" else torch.float32, sketch=sk, nnz_per_col=8)
    g = plan.factor_rr(_t(X), tau, f=f, rank_fixed=rf)
    # D came out of the sketch's own pass over X, not a second read: the pre-split Gaussian digit
    # split or the sparse tcgen05 sketch
    if sk in ("gaussian", "sparse"):
        assert plan.last_path() & rcq.PATH_COLSQ_FUSED, plan.last_path()
    r = g["rank"]
    perm = _np(g["perm"]).astype(np.int64)
    assert r == ref["rank"]
    if rank is not None and rf == 0:
        assert r == rank
    assert np.array_equal(perm[:r], ref["perm"][:r])
    assert sorted(perm.tolist()) == list(range(n))
    assert g["swaps"] == ref["swaps"]
    if r == n:
        assert np.array_equal(perm, ref["perm"])
    Rg = _np(g["R"])
    assert _rel(_by_original_column(Rg, perm, n), _by_original_column(ref["R"], ref["perm"], n)) <= \
        (1e-10 if dt == "f64" else 1e-4)
    assert np.all(np.tril(Rg[:, :r], -1) == 0) and np.all(np.diag(Rg[:, :r]) > 0)
    Qg = _np(g["Q"]).astype(np.float64)
    assert _rel(Qg, ref["Q"]) <= 10 * U64 * 1e4 + (2 * U32 if dt == "f32" else 0)
    assert oracle.cond(Qg) <= 10.0
    assert np.allclose(_np(g["D"]), ref["D"], rtol=1e-13 if dt == "f64" else 1e-12, atol=0)
    if rf:
        return                            # a fixed-rank truncation has no tau residual bound
    # column-normalised residual
    X64 = X.astype(np.float64)
    E = (X64[:, perm] - Qg @ Rg) / ref["D"][perm][None, :]
    u = U64 if dt == "f64" else U32
    assert np.linalg.norm(E) <= np.sqrt(2) * (u * n * 10 + 1.02 * np.sqrt(1.5) * tau) * np.sqrt(n) + 1e-12


def test_rr_column_power_of_two_scaling_is_exact(cuda):
    X = synth.make_X_lowrank(50_000, 20, 13, 2.0, 1e-13)
    plan = rcq.RCholQR(n=20, k=40, dtype=torch.float64)
    a = plan.factor_rr(_t(X), 1e-9)
    E = 2.0 ** (np.arange(20) % 9 - 4).astype(np.float64)
    b = plan.factor_rr(_t(X * E), 1e-9)
    assert a["rank"] == b["rank"] == 13
    assert torch.equal(a["perm"], b["perm"]) and torch.equal(a["Q"], b["Q"])
    pe = _np(a["perm"]).astype(np.int64)
    assert np.array_equal(_np(a["R"]) * E[pe][None, :], _np(b["R"]))


def test_rr_duplicate_and_zero_columns(cuda):
    X = synth.make_X(20_000, 10, 2.0)
    X[:, 6] = X[:, 2]
    X[:, 8] = 0.0
    plan = rcq.RCholQR(n=10, k=20, dtype=torch.float64)
    g = plan.factor_rr(_t(X), 1e-12)
    kept = set(_np(g["perm"])[: g["rank"]].tolist())
    assert g["rank"] == 8 and 8 not in kept and len(kept & {2, 6}) == 1


def test_rr_errors(cuda):
    plan = rcq.RCholQR(n=8, k=16, dtype=torch.float64)
    X = synth.make_X(2_000, 8, 2.0)
    for kw in ({"f": 1.0}, {"tau": -1.0}, {"rank_fixed": -1}):
        args = {"tau": 1e-12, **kw}
        with pytest.raises(rcq.RCholQRError) as e:
            plan.factor_rr(_t(X), **args)
        assert e.value.status == rcq.E_INVALID
    with pytest.raises(rcq.RCholQRError) as e:
        plan.factor_rr(torch.zeros((100, 8), dtype=torch.float64, device="cuda"), 1e-12)
    assert e.value.status == rcq.E_SINGULAR
    Xn = X.copy()
    Xn[5, 5] = np.inf
    with pytest.raises(rcq.RCholQRError) as e:
        plan.factor_rr(_t(Xn), 1e-12)
    assert e.value.status == rcq.E_NONFINITE


def test_rr_nccl_single_rank(cuda):
    X = _t(synth.make_X_lowrank(30_000, 24, 17, 2.0, 1e-13))
    uid = rcq.comm_unique_id()
    comm = rcq.comm_create(uid, 1, 0, 0)
    try:
        pa = rcq.RCholQR(n=24, k=48, dtype=torch.float64)
        pb = rcq.RCholQR(n=24, k=48, dtype=torch.float64, comm=comm)
        a, b = pa.factor_rr(X, 1e-9), pb.factor_rr(X, 1e-9)
        assert a["rank"] == b["rank"] == 17
        for key in ("Q", "R", "perm", "D"):
            assert torch.equal(a[key], b[key])
        pb.close()
    finally:
        rcq.comm_destroy(comm)


@pytest.mark.parametrize("m,n,k,rank,dt,sk,tau", [
    (100_000, 48, 96, 30, "f64", "gaussian", 1e-9),
    (262_144, 64, 128, 40, "f32", "sparse", 1e-5),
    (40_000, 256, 512, 180, "f64", "gaussian", 1e-9),
])
def test_factor_rr2_parity(cuda, m, n, k, rank, dt, sk, tau):
    # RRRCholeskyQR2: Alg. 7's rank and pivots, then an orthonormal Q
    X = synth.make_X_lowrank(m, n, rank, 2.0, 1e-13, dt)
    so = oracle.GAUSSIAN if sk == "gaussian" else oracle.SPARSE_SIGN
    ref = oracle.factor_rr2(X, k, tau, sketch=so, zeta=8)
    plan = rcq.RCholQR(n=n, k=k, dtype=torch.float64 if dt == "f64" else torch.float32, sketch=sk, nnz_per_col=8)
    g = plan.factor_rr2(_t(X), tau)
    r = g["rank"]
    perm = _np(g["perm"]).astype(np.int64)
    assert r == ref["rank"] == rank and np.array_equal(perm[:r], ref["perm"][:r])
    Rg = _np(g["R"])
    assert _rel(_by_original_column(Rg, perm, n), _by_original_column(ref["R"], ref["perm"], n)) <= \
        (1e-10 if dt == "f64" else 1e-4)
    Q = _np(g["Q"]).astype(np.float64)
    assert np.linalg.norm(Q.T @ Q - np.eye(r), 2) <= (1e-12 if dt == "f64" else 1e-5)
    assert _rel(Q, ref["Q"]) <= (1e-10 if dt == "f64" else 1e-5)
    assert np.linalg.cond(_np(g["Rp"])) <= 8.0
