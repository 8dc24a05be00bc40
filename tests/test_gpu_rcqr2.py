"""GPU parity for RCholeskyQR2 (Alg. 3) through the C ABI (rcholqr_factor2).

Bars: R relative Frobenius vs the oracle <= 1e-10 (fp64 X) / 1e-4
(fp32 X) (the north-star R bars); Q orthonormal: ||I - Q^T Q||_2 <= 1e-12 (fp64) / 1e-5 (fp32) --
Alg. 3's Q is orthonormal itself, not only its sketch; Q vs the oracle <= 10 u kappa (+ fp32 storage);
residual ||X - Q R|| / ||X|| <= 10 n u.  Implicit form: Q1 is Alg. 2's Q bit for bit and
Q1 R'^{-1} equals the explicit Q.
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


CASES = [
    # name, m, n, k, dtype, sketch, log10 cond
    ("C1", 10_000, 20, 40, "f64", "gaussian", 3),
    ("C2-reduced", 200_003, 100, 200, "f32", "gaussian", 5),
    ("C4-reduced", 262_144, 64, 128, "f32", "sparse", 4),
    ("C3-reduced", 40_000, 256, 512, "f64", "gaussian", 10),
    ("ragged", 5_003, 130, 260, "f64", "gaussian", 6),
]


@pytest.mark.parametrize("name,m,n,k,dt,sk,c", CASES)
def test_factor2_parity(cuda, name, m, n, k, dt, sk, c):
    X = synth.make_X(m, n, c, dt)
    so = oracle.GAUSSIAN if sk == "gaussian" else oracle.SPARSE_SIGN
    ref = oracle.factor2(X, k, sketch=so, zeta=8)
    plan = rcq.RCholQR(n=n, k=k, dtype=torch.float64 if dt == "f64" else torch.float32, sketch=sk, nnz_per_col=8)
    Qg, Rg, Rpg = plan.factor2(_t(X))
    Qg, Rg, Rpg = _np(Qg), _np(Rg), _np(Rpg)
    u = U64 if dt == "f64" else U32
    assert _rel(Rg, ref["R"]) <= (1e-10 if dt == "f64" else 1e-4), _rel(Rg, ref["R"])
    Q64 = Qg.astype(np.float64)
    orth = np.linalg.norm(Q64.T @ Q64 - np.eye(n), 2)
    assert orth <= (1e-12 if dt == "f64" else 1e-5), orth
    assert _rel(Qg, ref["Q"]) <= 10 * U64 * 10**c + (2 * U32 if dt == "f32" else 0), _rel(Qg, ref["Q"])
    assert np.linalg.norm(X.astype(np.float64) - Q64 @ Rg) <= 10 * n * u * np.linalg.norm(X)
    assert np.all(np.tril(Rg, -1) == 0) and np.all(np.diag(Rg) > 0)
    # R' = chol(Q1^T Q1) corrects each side's OWN Q1, and Q1 (Alg. 2's Q) carries the u kappa forward
    # error, so R' agrees only to that bar (the final R = R' R1 is unique and meets the R bar above)
    assert _rel(Rpg, ref["Rp"]) <= 10 * U64 * 10**c + (2 * U32 if dt == "f32" else 0)


def test_factor2_implicit_form(cuda):
    X = synth.make_X(50_000, 48, 6.0)
    plan = rcq.RCholQR(n=48, k=96, dtype=torch.float64)
    Xt = _t(X)
    Q1, R, Rp = plan.factor2(Xt, implicit=True)
    Qa, Ra, _ = plan.factor(Xt)
    assert torch.equal(Q1, Qa)                                 # step 1 is Alg. 2, same kernels
    Qe, Re, Rpe = plan.factor2(Xt)
    assert torch.equal(R, Re) and torch.equal(Rp, Rpe)
    Qi = torch.linalg.solve_triangular(Rp, Q1, upper=True, left=False)   # Q1 R'^{-1}
    assert _rel(_np(Qi), _np(Qe)) <= 1e-13


def test_factor2_singular(cuda):
    X = synth.make_X(3_000, 16, 2.0)
    X[:, 5] = 0.0
    plan = rcq.RCholQR(n=16, k=32, dtype=torch.float64)
    with pytest.raises(rcq.RCholQRError) as e:
        plan.factor2(_t(X))
    assert e.value.status == rcq.E_SINGULAR


def test_factor2_nccl_single_rank(cuda):
    X = _t(synth.make_X(30_000, 32, 4.0))
    uid = rcq.comm_unique_id()
    comm = rcq.comm_create(uid, 1, 0, 0)
    try:
        pa = rcq.RCholQR(n=32, k=64, dtype=torch.float64)
        pb = rcq.RCholQR(n=32, k=64, dtype=torch.float64, comm=comm)
        a, b = pa.factor2(X), pb.factor2(X)
        for x, y in zip(a, b):
            assert torch.equal(x, y)                         # the collective path == single-GPU path
        pb.close()
    finally:
        rcq.comm_destroy(comm)
