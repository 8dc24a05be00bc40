"""Column-major X and Q (rcholqr_factor_colmajor): native tcgen05 kernels for
fp32 X with n <= 128 and an aligned column pitch, the layout adapter otherwise.  Either way the factorization of
a column-major X equals the row-major factorization of the same matrix BITWISE (exact digit arithmetic / the same
kernels on the same values), for padded leading dimensions and ragged shapes; argument errors."""
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


# Native column-major kernels (fp32, n <= 128, 16-byte aligned column pitch): the tcgen05 sketches and
# the tcgen05 digit solve take column-major tiles through their tensor maps.  Integer digit arithmetic is exact, so
# R, S and Q must equal the row-major path's BITWISE; rcholqr_last_path must report that no adapter ran.
@pytest.mark.parametrize("m,n,k,sk,pad", [
    (262_144, 64, 128, "sparse", 4),           # C4 shape, ldx = m + 4
    (100_003, 64, 128, "sparse", 1),           # ragged m: partial stages and tiles (ldx = 100_004)
    (70_001, 20, 40, "sparse", 3),             # n < 32: one column group, K padding
    (1_048_576, 100, 200, "gaussian", 0),      # C2 shape: pre-split Gaussian digits, 128-wide solve tiles
    (50_001, 37, 74, "gaussian", 3),           # ragged n and m
    (33_000, 128, 256, "gaussian", 0),         # n = 128
    (65_536, 48, 96, "rademacher", 0),
    (40_000, 100, 200, "rademacher", 0),       # two 64-column sketch tiles
    (65_536, 64, 128, "srht", 0),
    (517, 9, 18, "sparse", 3),                 # fewer rows than CTAs
])
def test_colmajor_native_bitwise(cuda, m, n, k, sk, pad):
    X0 = torch.from_numpy(synth.make_X(m, n, 4.0, "f32")).cuda()
    X = torch.zeros((m, (n + 3) // 4 * 4), dtype=torch.float32, device="cuda")[:, :n]   # 16-byte row pitch: tcgen05 row-major path
    X.copy_(X0)
    plan = rcq.RCholQR(n=n, k=k, dtype=torch.float32, sketch=sk, nnz_per_col=(8 if k % 8 == 0 else 2))
    Q = torch.zeros((m, (n + 3) // 4 * 4), dtype=torch.float32, device="cuda")[:, :n]
    Q, R, S = plan.factor(X, want_S=True, Q=Q)
    assert plan.last_path() & rcq.PATH_SKETCH_TC and plan.last_path() & rcq.PATH_SOLVE_TC
    Xt_store = torch.full((n, m + pad), float("nan"), dtype=torch.float32, device="cuda")   # the pitch padding is never read
    Xt_store[:, :m] = X.t()
    Qt_store = torch.full((n, m + pad), 7.0, dtype=torch.float32, device="cuda")
    Qt, Rc, Sc = plan.factor_colmajor(Xt_store[:, :m], want_S=True, Qt=Qt_store[:, :m])
    path = plan.last_path()
    assert path & rcq.PATH_COLMAJOR_NATIVE, hex(path)
    assert not path & (rcq.PATH_SKETCH_FALLBACK | rcq.PATH_SKETCH_CUDA_CORE | rcq.PATH_SOLVE_DMMA), hex(path)
    assert torch.equal(Rc, R) and torch.equal(Sc, S)
    assert torch.equal(Qt.t(), Q)
    assert torch.all(Qt_store[:, m:] == 7.0)                  # the padding of the column pitch is not written


def test_colmajor_native_overflow_takes_adapter(cuda):
    """A spike far above the first stage's column maximum raises the sketch's headroom flag; the native call must
    notice it and redo the factorization through the adapter (same result as the row-major path)."""
    m, n, k = 200_000, 64, 128
    X = torch.from_numpy(synth.make_X(m, n, 2.0, "f32")).cuda()
    X[150_000, 5] = 1.0e6
    plan = rcq.RCholQR(n=n, k=k, dtype=torch.float32, sketch="sparse", nnz_per_col=8)
    Q, R, _ = plan.factor(X)
    assert plan.last_path() & rcq.PATH_SKETCH_FALLBACK
    Qt, Rc, _ = plan.factor_colmajor(X.t().contiguous())
    assert not plan.last_path() & rcq.PATH_COLMAJOR_NATIVE
    assert torch.equal(Rc, R) and torch.equal(Qt.t(), Q)


def test_colmajor_native_status(cuda):
    """Zero column -> E_SINGULAR, NaN -> E_NONFINITE through the native kernels, Q untouched."""
    m, n, k = 50_000, 32, 64
    X = torch.from_numpy(synth.make_X(m, n, 2.0, "f32")).cuda()
    plan = rcq.RCholQR(n=n, k=k, dtype=torch.float32, sketch="sparse", nnz_per_col=8)
    Xz = X.clone(); Xz[:, 3] = 0
    Qt = torch.full((n, m), 5.0, dtype=torch.float32, device="cuda")
    with pytest.raises(rcq.RCholQRError) as e:
        plan.factor_colmajor(Xz.t().contiguous(), Qt=Qt)
    assert e.value.status == rcq.E_SINGULAR and torch.all(Qt == 5.0)
    Xn = X.clone(); Xn[123, 4] = float("nan")
    with pytest.raises(rcq.RCholQRError) as e:
        plan.factor_colmajor(Xn.t().contiguous(), Qt=Qt)
    assert e.value.status == rcq.E_NONFINITE


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
