"""The N > 1 product path on real GPUs (S3): one process per GPU, X row-partitioned with a global-row
offset, the library-owned NCCL communicator (rcholqr_comm_create) and the in-factor ncclAllReduce of the k x n
sketch, R computed redundantly, Q solved locally -- checked against the CPU oracle's factorization of the WHOLE X.

Needs at least two visible CUDA devices; the boxes this project builds on expose one, so these tests are SKIPPED
there (the same partition / all-reduce / redundant-R logic runs on CPU with gloo in tests/test_dist_cpu.py, and the
one-rank communicator and rank-partition sums run in tests/test_gpu_parity.py).  No torch.distributed here: the parent
creates the ncclUniqueId and hands it to the spawned ranks."""
import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

import oracle
import synth
from paper_2210_09953_b200.partition import row_block

pytestmark = pytest.mark.gpu


def _rank(rank, world, uid, m, n, k, dt, sketch, c, algo, out_q):
    import paper_2210_09953_b200 as rcq
    try:
        torch.cuda.set_device(rank)
        comm = rcq.comm_create(uid, world, rank, rank)
        X = synth.make_X(m, n, c, dt)
        ro, ml = row_block(m, world, rank)
        Xl = torch.from_numpy(np.ascontiguousarray(X[ro:ro + ml])).cuda(rank)
        plan = rcq.RCholQR(n=n, k=k, dtype=Xl.dtype, sketch=sketch, nnz_per_col=8, device=rank, comm=comm)
        if algo == "rcholqr":
            Q, R, S = plan.factor(Xl, row_offset=ro, want_S=True)
            out = (Q.cpu().numpy(), R.cpu().numpy(), S.cpu().numpy())
        else:                                              # Alg. 3: + the Gram all-reduce
            Q, R, Rp = plan.factor2(Xl, row_offset=ro)
            out = (Q.cpu().numpy(), R.cpu().numpy(), Rp.cpu().numpy())
        torch.cuda.synchronize()
        plan.close()
        rcq.comm_destroy(comm)
        out_q.put((rank, ro, None) + out)
    except Exception as e:                                 # report instead of hanging the parent's queue.get
        out_q.put((rank, -1, repr(e), None, None, None))


def _run(world, m, n, k, dt, sketch, c, algo):
    import paper_2210_09953_b200 as rcq
    uid = rcq.comm_unique_id()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_rank, args=(r, world, uid, m, n, k, dt, sketch, c, algo, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=600) for _ in range(world)], key=lambda t: t[0])
    for p in procs:
        p.join(timeout=120)
    for r in res:
        assert r[2] is None, r[2]
    return res


def _rel(a, b):
    return float(np.linalg.norm(np.asarray(a, dtype=np.float64) - b) / max(np.linalg.norm(b), 1e-300))


@pytest.mark.parametrize("m,n,k,dt,sketch,c", [
    (262_147, 64, 128, "f32", "sparse", 4),        # C4 shape, ragged split (row offsets not multiples of 32)
    (100_001, 100, 200, "f32", "gaussian", 5),     # C2 shape
    (40_001, 40, 80, "f64", "gaussian", 8),
    (50_000, 24, 200, "f64", "srht", 6),           # SRHT by the fast transform: blocks straddle the rank boundary
])
def test_multi_gpu_factor_vs_oracle(cuda, m, n, k, dt, sketch, c):
    world = min(torch.cuda.device_count(), 4)
    if world < 2:
        pytest.skip("needs >= 2 CUDA devices")
    so = {"gaussian": oracle.GAUSSIAN, "sparse": oracle.SPARSE_SIGN, "srht": oracle.SRHT}[sketch]
    X = synth.make_X(m, n, c, dt)
    ref = oracle.factor(X, k, sketch=so, zeta=8, want_S=True)
    res = _run(world, m, n, k, dt, sketch, c, "rcholqr")
    u = 2.0**-53
    for rank, ro, _, Q, R, S in res:
        assert np.array_equal(R, res[0][4])                   # R bit-identical on every rank (redundant, deterministic QR)
        assert np.array_equal(S, res[0][5])
        assert _rel(R, ref["R"]) <= (1e-10 if dt == "f64" else 1e-4)
        ml = Q.shape[0]
        assert _rel(Q, ref["Q"][ro:ro + ml]) <= 10 * u * 10**c + (2 * 2.0**-24 if dt == "f32" else 0)
    assert sum(r[3].shape[0] for r in res) == m
    assert oracle.orth_defect(res[0][5]) <= 1e-13


def test_multi_gpu_factor2_vs_oracle(cuda):
    world = min(torch.cuda.device_count(), 4)
    if world < 2:
        pytest.skip("needs >= 2 CUDA devices")
    m, n, k, c = 60_001, 32, 64, 6
    X = synth.make_X(m, n, c, "f64")
    ref = oracle.factor2(X, k)
    res = _run(world, m, n, k, "f64", "gaussian", c, "rcholqr2")
    Q = np.concatenate([r[3] for r in res])
    for r in res:
        assert np.array_equal(r[4], res[0][4])
        assert _rel(r[4], ref["R"]) <= 1e-10
    assert np.linalg.norm(np.eye(n) - Q.T @ Q, 2) <= 1e-12    # Alg. 3's Q itself is orthonormal
