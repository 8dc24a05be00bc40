"""GPU parity for the reduced RCholeskyQR (Alg. 5) through the C ABI
(rcholqr_factor_reduced).

Bars: Y = L X <= 1e-12 relative Frobenius vs the compensated oracle
(the sketch bar); R <= 1e-10 (fp64 X) / 1e-4 (fp32 X) (the north-star R bars); Z = Y R^{-1} (fp64)
<= 10 u kappa relative -- Z carries R^{-1}'s conditioning exactly like Q does.
"""
import numpy as np
import pytest
import torch

import oracle
import paper_2210_09953_b200 as rcq
import synth

pytestmark = pytest.mark.gpu
U64 = 2.0**-53


def _t(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def _np(t):
    return t.detach().cpu().numpy()


def _rel(a, b):
    a, b = np.asarray(a, dtype=np.float64), np.asarray(b, dtype=np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


CASES = [
    # name, m, n, k, l, dtype, sketch, log10 cond
    ("C1", 10_000, 20, 40, 30, "f64", "gaussian", 3),
    ("C2-reduced", 200_003, 100, 200, 100, "f32", "gaussian", 5),
    ("C4-reduced", 262_144, 64, 128, 64, "f32", "sparse", 4),
    ("C3-reduced", 40_000, 256, 512, 96, "f64", "gaussian", 10),
    ("ragged", 5_003, 33, 66, 7, "f64", "gaussian", 6),
    ("ragged-sparse", 4_097, 17, 32, 41, "f64", "sparse", 3),
]


@pytest.mark.parametrize("name,m,n,k,l,dt,sk,c", CASES)
def test_factor_reduced_parity(cuda, name, m, n, k, l, dt, sk, c):
    X = synth.make_X(m, n, c, dt)
    so = oracle.GAUSSIAN if sk == "gaussian" else oracle.SPARSE_SIGN
    ref = oracle.factor_reduced(X, k, l, sketch=so, zeta=8)
    plan = rcq.RCholQR(n=n, k=k, dtype=torch.float64 if dt == "f64" else torch.float32, sketch=sk, nnz_per_col=8)
    Z, R, S, Y = plan.factor_reduced(_t(X), l, want_S=True, want_Y=True)
    Z, R, S, Y = _np(Z), _np(R), _np(S), _np(Y)
    assert _rel(Y, ref["Y"]) <= 1e-12, _rel(Y, ref["Y"])
    assert _rel(R, ref["R"]) <= (1e-10 if dt == "f64" else 1e-4), _rel(R, ref["R"])
    assert np.all(np.tril(R, -1) == 0) and np.all(np.diag(R) > 0)
    assert _rel(Z, ref["Z"]) <= 10 * U64 * 10**c, _rel(Z, ref["Z"])
    assert oracle.orth_defect(S) <= 1e-13
    # the GPU's own step 3 on its own (Y, R): Z R = Y to fp64 row-wise backward error
    assert np.linalg.norm(Z @ R - Y) <= 4 * n * U64 * np.linalg.norm(np.abs(Z) @ np.abs(R))


def test_reduced_r_matches_alg2(cuda):
    # step 2 is Alg. 2's QR: the R of the one-pass (k + l)-row sketch equals Alg. 2's R to rounding
    X = _t(synth.make_X(100_000, 48, 6.0, "f32"))
    plan = rcq.RCholQR(n=48, k=96, dtype=torch.float32)
    _, R2, _ = plan.factor(X)
    _, Rr, _, _ = plan.factor_reduced(X, 50)
    assert _rel(_np(Rr), _np(R2)) <= 1e-13


def test_reduced_determinism_and_l_change(cuda):
    X = _t(synth.make_X(50_000, 32, 4.0))
    plan = rcq.RCholQR(n=32, k=64, dtype=torch.float64)
    a = plan.factor_reduced(X, 20)
    b = plan.factor_reduced(X, 45)            # workspace regrown for a new l
    c = plan.factor_reduced(X, 20)
    assert torch.equal(a[0], c[0]) and torch.equal(a[1], c[1])
    assert _rel(_np(a[1]), _np(b[1])) <= 1e-13     # same R whatever l (Theta rows are the first k)
    # L's first 20 rows are the same draws for l = 20 and l = 45 up to the 1/sqrt(l) scale
    assert _rel(_np(b[0][:20]) * np.sqrt(45.0), _np(a[0]) * np.sqrt(20.0)) <= 1e-11


def test_reduced_errors(cuda):
    plan = rcq.RCholQR(n=8, k=16, dtype=torch.float64)
    X = synth.make_X(2_000, 8, 2.0)
    with pytest.raises(rcq.RCholQRError) as e:
        plan.factor_reduced(_t(X), 0)
    assert e.value.status == rcq.E_INVALID
    Xn = X.copy()
    Xn[17, 3] = np.nan
    with pytest.raises(rcq.RCholQRError) as e:
        plan.factor_reduced(_t(Xn), 5)
    assert e.value.status == rcq.E_NONFINITE
    Xs = X.copy()
    Xs[:, 2] = 0.0
    Z = torch.full((5, 8), 7.0, dtype=torch.float64, device="cuda")
    with pytest.raises(rcq.RCholQRError) as e:
        plan.factor_reduced(_t(Xs), 5, Z=Z)
    assert e.value.status == rcq.E_SINGULAR
    assert torch.all(Z == 7.0)                # Z is not written on E_SINGULAR


def test_reduced_nccl_single_rank(cuda):
    X = _t(synth.make_X(30_000, 24, 4.0))
    uid = rcq.comm_unique_id()
    comm = rcq.comm_create(uid, 1, 0, 0)
    try:
        pa = rcq.RCholQR(n=24, k=48, dtype=torch.float64)
        pb = rcq.RCholQR(n=24, k=48, dtype=torch.float64, comm=comm)
        a, b = pa.factor_reduced(X, 30, want_Y=True), pb.factor_reduced(X, 30, want_Y=True)
        for x, y in zip(a, b):
            assert (x is None and y is None) or torch.equal(x, y)
        pb.close()
    finally:
        rcq.comm_destroy(comm)


def test_reduced_partition_emulation(cuda):
    # two row blocks with global row keys: Y sums to the whole X's extract (the multi-GPU all-reduce)
    Xh = synth.make_X(60_000, 16, 3.0)
    plan = rcq.RCholQR(n=16, k=32, dtype=torch.float64)
    _, _, _, Y = plan.factor_reduced(_t(Xh), 12, want_Y=True)
    _, _, _, Ya = plan.factor_reduced(_t(Xh[:25_001]), 12, want_Y=True)
    _, _, _, Yb = plan.factor_reduced(_t(Xh[25_001:]), 12, row_offset=25_001, want_Y=True)
    assert _rel(_np(Ya) + _np(Yb), _np(Y)) <= 1e-14
