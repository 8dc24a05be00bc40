"""The rest of the C ABI on the GPU: the asynchronous factorization and its status query, the library
timing events, the launch-count introspection, and non-default CUDA streams."""
import numpy as np
import pytest
import torch

import paper_2210_09953_b200 as rcq
import synth

pytestmark = pytest.mark.gpu


def test_async_factor_and_query_status(cuda):
    X = torch.from_numpy(synth.make_X(50_000, 24, 4.0)).cuda()
    plan = rcq.RCholQR(n=24, k=48, dtype=torch.float64)
    Qs, Rs, _ = plan.factor(X)
    Qa, Ra, _ = plan.factor(X, sync=False)               # rcholqr_factor_async: returns before completion
    assert plan.query_status() == rcq.OK
    assert torch.equal(Qa, Qs) and torch.equal(Ra, Rs)
    Xs = X.clone()
    Xs[:, 7] = 0.0                                       # numerically singular: reported by the query
    plan.factor(Xs, sync=False)
    assert plan.query_status() == rcq.E_SINGULAR
    plan.factor(X, sync=False)                           # the status word is reset per call
    assert plan.query_status() == rcq.OK


def test_timing_events(cuda):
    X = torch.from_numpy(synth.make_X(1 << 20, 100, 5.0, "f32")).cuda()
    plan = rcq.RCholQR(n=100, k=200, dtype=torch.float32)
    plan.factor(X)
    plan.set_timing(True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    plan.factor(X)
    e1.record()
    torch.cuda.synchronize()
    t = plan.last_timings()
    plan.set_timing(False)
    assert set(t) == {"sketch", "reduce", "allreduce", "small_qr", "tri_prep", "solve"}
    assert all(v >= 0.0 for v in t.values())
    total = e0.elapsed_time(e1)
    assert 0.5 * total <= sum(t.values()) <= 1.05 * total + 0.05
    assert t["sketch"] > t["small_qr"] > 0.0                     # the sketch dominates C2


@pytest.mark.parametrize("n,k,dt,sk,expect_min", [(100, 200, torch.float32, "gaussian", 6),
                                                  (64, 128, torch.float32, "sparse", 5),
                                                  (256, 512, torch.float64, "gaussian", 6)])
def test_launches_per_factor(cuda, n, k, dt, sk, expect_min):
    plan = rcq.RCholQR(n=n, k=k, dtype=dt, sketch=sk)
    m = 1 << 20
    cnt = plan.launches_per_factor(m)
    assert expect_min <= cnt <= 64
    assert plan.launches_per_factor(0) < cnt                      # no sketch / solve kernels for m = 0


def test_non_default_stream(cuda):
    X = torch.from_numpy(synth.make_X(80_000, 32, 3.0, "f32")).cuda()
    plan = rcq.RCholQR(n=32, k=64, dtype=torch.float32)
    Q0, R0, _ = plan.factor(X)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        Q1, R1, _ = plan.factor(X, stream=s)
    s.synchronize()
    assert torch.equal(Q1, Q0) and torch.equal(R1, R0)
    Z0 = plan.factor_reduced(X, 10)[0]
    with torch.cuda.stream(s):
        Z1 = plan.factor_reduced(X, 10, stream=s)[0]
    s.synchronize()
    assert torch.equal(Z0, Z1)
    assert np.isfinite(Q1.cpu().numpy()).all()
