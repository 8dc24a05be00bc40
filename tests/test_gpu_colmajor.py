"""Column-major X and Q (rcholqr_factor_colmajor, the layout adapter of SURVEY 8(f) NEXT #4): the
factorization of a column-major X equals the row-major factorization of the same matrix BITWISE
(same kernels on the same values), for padded leading dimensions and ragged shapes; argument errors."""
import numpy as np
import pytest
import torch

import paper_2210_09953_b200 as rcq
import synth

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("m,n,k,dt,sk,pad", [
    (1_048_576, 100, 200, torch.float32, "gaussian", 0),     # the C2 shape
    (262_144, 64, 128, torch.float32, "sparse", 3),          # C4 shape, ldx = m + 3
    (40_001, 37, 74, torch.float64, "gaussian", 5),          # ragged, fp64
    (5_000, 16, 32, torch.float64, "srht", 0),
])
def test_colmajor_equals_rowmajor(cuda, m, n, k, dt, sk, pad):
    X = torch.from_numpy(synth.make_X(m, n, 4.0, "f64" if dt == torch.float64 else "f32")).cuda()
    plan = rcq.RCholQR(n=n, k=k, dtype=dt, sketch=sk)
    Q, R, S = plan.factor(X, want_S=True)
    Xt_store = torch.zeros((n, m + pad), dtype=dt, device="cuda")
    Xt_store[:, :m] = X.t()
    Qt, Rc, Sc = plan.factor_colmajor(Xt_store[:, :m], want_S=True)
    assert torch.equal(Rc, R) and torch.equal(Sc, S)
    assert torch.equal(Qt.t(), Q)


def test_colmajor_errors_and_empty(cuda):
    plan = rcq.RCholQR(n=8, k=16, dtype=torch.float64)
    Xt = torch.randn(8, 100, dtype=torch.float64, device="cuda")
    lib = rcq.load_library()
    R = torch.empty(8, 8, dtype=torch.float64, device="cuda")
    Qt = torch.empty_like(Xt)
    st = lib.rcholqr_factor_colmajor(plan._h, rcq._ptr(Xt), 100, 0, 50, rcq._ptr(Qt), 100, rcq._ptr(R), None, None)
    assert st == rcq.E_INVALID                                # ldx < m
    st = lib.rcholqr_factor_colmajor(plan._h, rcq._ptr(Xt), 100, 0, 100, rcq._ptr(Xt), 100, rcq._ptr(R), None, None)
    assert st == rcq.E_INVALID                                # Q aliases X
    with pytest.raises(rcq.RCholQRError) as e:                # m = 0: P = 0, zero pivots
        plan.factor_colmajor(torch.empty((8, 0), dtype=torch.float64, device="cuda"))
    assert e.value.status == rcq.E_SINGULAR
