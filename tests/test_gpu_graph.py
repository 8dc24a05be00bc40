"""rcholqr_factor_graph (include/rcholqr.h): Alg. 2's kernel chain replayed from a CUDA graph for launch-bound
problems (BASELINE C1).  The replay must give the plain call's Q, R, S BITWISE (same kernels, same launch
configurations), follow changes of the buffers' contents, re-capture on new buffers, and report status."""
import pytest
import torch

import paper_2210_09953_b200 as rcq
import synth

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name,m,n,k,dt,sk", [
    ("C1", 10_000, 20, 40, torch.float64, "gaussian"),
    ("C2-shape", 60_000, 100, 200, torch.float32, "gaussian"),
    ("C4-shape", 50_000, 64, 128, torch.float32, "sparse"),
    ("wide fp64", 5_000, 300, 600, torch.float64, "gaussian"),      # blocked QR + streamed solve: many launches
])
def test_graph_replay_bitwise(cuda, name, m, n, k, dt, sk):
    f = "f64" if dt == torch.float64 else "f32"
    X = torch.from_numpy(synth.make_X(m, n, 3.0, f)).cuda()
    plan = rcq.RCholQR(n=n, k=k, dtype=dt, sketch=sk)
    Q0, R0, S0 = plan.factor(X, want_S=True)
    path0 = plan.last_path()
    Q, R, S = torch.empty_like(Q0), torch.empty_like(R0), torch.empty_like(S0)
    for it in range(3):                                     # 1st: direct + capture; 2nd, 3rd: replays
        Q.fill_(float("nan")); R.fill_(float("nan")); S.fill_(float("nan"))
        plan.factor(X, Q=Q, R=R, S=S, graph=True)
        assert torch.equal(Q, Q0) and torch.equal(R, R0) and torch.equal(S, S0), (name, it)
        assert plan.last_path() == path0
    # new contents in the same buffers: the replay reads them
    X2 = torch.from_numpy(synth.make_X(m, n, 2.0, f, seed=7)).cuda()
    Q2, R2, _ = plan.factor(X2)
    X.copy_(X2)
    plan.factor(X, Q=Q, R=R, S=S, graph=True)
    assert torch.equal(Q, Q2) and torch.equal(R, R2)
    # other buffers: re-captured, then replayed
    Xb, Qb, Rb = X2.clone(), torch.empty_like(Q0), torch.empty_like(R0)
    for _ in range(2):
        plan.factor(Xb, Q=Qb, R=Rb, graph=True)
        assert torch.equal(Qb, Q2) and torch.equal(Rb, R2)


def test_graph_status(cuda):
    m, n, k = 10_000, 20, 40
    X = torch.from_numpy(synth.make_X(m, n, 3.0, "f64")).cuda()
    plan = rcq.RCholQR(n=n, k=k, dtype=torch.float64)
    Q, R = torch.empty_like(X), torch.empty((n, n), dtype=torch.float64, device="cuda")
    plan.factor(X, Q=Q, R=R, graph=True)
    plan.factor(X, Q=Q, R=R, graph=True)
    X[:, 3] = 0                                            # replay on a rank-deficient X: E_SINGULAR from the graph's kernels
    with pytest.raises(rcq.RCholQRError) as e:
        plan.factor(X, Q=Q, R=R, graph=True)
    assert e.value.status == rcq.E_SINGULAR
    X[:, 3] = 1.0; X[5, 3] = 2.0; X[77, 2] = float("inf")
    with pytest.raises(rcq.RCholQRError) as e:
        plan.factor(X, Q=Q, R=R, graph=True)
    assert e.value.status == rcq.E_NONFINITE


def test_graph_survives_workspace_regrowth(cuda):
    """A larger plain call regrows the plan's lazily sized workspaces (the pre-split digit buffer, the streamed
    solve's T buffer): a graph captured before that holds freed pointers and must be re-captured, not replayed."""
    for n, k, dt in ((100, 200, torch.float32), (300, 600, torch.float64)):
        f = "f64" if dt == torch.float64 else "f32"
        Xs = torch.from_numpy(synth.make_X(30_000, n, 3.0, f)).cuda()
        Xl = torch.from_numpy(synth.make_X(90_000, n, 3.0, f, seed=3)).cuda()
        plan = rcq.RCholQR(n=n, k=k, dtype=dt)
        Q0, R0, _ = plan.factor(Xs)
        Q, R = torch.empty_like(Q0), torch.empty_like(R0)
        plan.factor(Xs, Q=Q, R=R, graph=True)
        plan.factor(Xs, Q=Q, R=R, graph=True)                # replay
        Ql, Rl, _ = plan.factor(Xl)                           # three times the rows: workspaces regrown
        Q.fill_(0); R.fill_(0)
        plan.factor(Xs, Q=Q, R=R, graph=True)
        assert torch.equal(Q, Q0) and torch.equal(R, R0)
        plan.factor(Xs, Q=Q, R=R, graph=True)
        assert torch.equal(Q, Q0) and torch.equal(R, R0)
        Q2, R2, _ = plan.factor(Xl)
        assert torch.equal(Q2, Ql) and torch.equal(R2, Rl)
