"""The N>1 path on CPU with the gloo backend (world_size 2): row partition with global-row-keyed
Theta, ONE all-reduce (sum) of the k x n sketch, R computed redundantly on every
rank, Q solved locally -- equals the single-process factorization of the whole X.  The arithmetic
is the oracle's; what is tested is the partition / reduction / redundancy logic the GPU path uses."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import synth
from paper_2210_09953_b200.partition import row_block, weak_block


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, m, n, k, sketch, c, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        X = synth.make_X(m, n, c, "f64")
        ro, ml = row_block(m, world, rank)
        Xl = X[ro:ro + ml]
        so = oracle.GAUSSIAN if sketch == "gaussian" else oracle.SPARSE_SIGN
        P = torch.from_numpy(oracle.sketch(Xl, k, sketch=so, zeta=8, row_offset=ro))
        dist.all_reduce(P, op=dist.ReduceOp.SUM)          # the method's one global synchronisation
        R, _, st = oracle.householder(P.numpy(), want_S=False)
        Rs = [torch.zeros_like(torch.from_numpy(R)) for _ in range(world)]
        dist.all_gather(Rs, torch.from_numpy(R))
        same_R = all(torch.equal(Rs[0], r) for r in Rs)
        Ql = oracle.forward_subst(Xl, R)
        out_q.put((rank, ro, P.numpy(), R, Ql, same_R, st))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("m,n,k,sketch,c", [(70_001, 12, 24, "gaussian", 6), (131_075, 8, 16, "sparse", 4)])
def test_two_rank_factorization_equals_single(m, n, k, sketch, c):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, m, n, k, sketch, c, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=300) for _ in range(world)], key=lambda t: t[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    X = synth.make_X(m, n, c, "f64")
    so = oracle.GAUSSIAN if sketch == "gaussian" else oracle.SPARSE_SIGN
    full = oracle.factor(X, k, sketch=so, zeta=8, want_S=False)
    P0, R0 = res[0][2], res[0][3]
    assert all(r[5] for r in res), "R must be bit-identical on every rank"
    assert np.array_equal(P0, res[1][2])
    assert np.all(np.abs(P0 - full["P"]) <= 4 * 2.0**-53 * np.abs(full["P"]).max())
    assert np.linalg.norm(R0 - full["R"]) <= 1e-13 * np.linalg.norm(full["R"])
    Q = np.concatenate([r[4] for r in res])
    # both Q's carry the u*kappa forward error of the solve (eq:stab3)
    assert np.linalg.norm(Q - full["Q"]) <= 10 * 2.0**-53 * 10**c * np.linalg.norm(full["Q"])


def test_partition_helpers():
    assert row_block(10, 3, 0) == (0, 4) and row_block(10, 3, 1) == (4, 3) and row_block(10, 3, 2) == (7, 3)
    offs = [row_block(1_000_003, 8, r) for r in range(8)]
    assert sum(ml for _, ml in offs) == 1_000_003
    assert all(offs[r][0] + offs[r][1] == offs[r + 1][0] for r in range(7))
    assert weak_block(100, 4, 3) == (300, 100, 400)
    with pytest.raises(ValueError):
        row_block(5, 2, 2)


def _worker_alg(rank, world, port, algo, m, n, k, out_q):
    """Alg. 5 / Alg. 7 / Alg. 3 on 2 ranks: one all-reduce of the stacked small matrices each needs
    ([P; Y], [P; D^2]; Alg. 3 adds the Gram all-reduce), everything after it redundant per rank."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        if algo == "rr":
            X = synth.make_X_lowrank(m, n, n - 4, 2.0, 1e-13)
        else:
            X = synth.make_X(m, n, 5.0, "f64")
        ro, ml = row_block(m, world, rank)
        Xl = X[ro:ro + ml]
        P = oracle.sketch(Xl, k, row_offset=ro)
        if algo == "reduced":
            l = 9
            Y = oracle.extract(Xl, oracle.extractor_row0(k), l, row_offset=ro)
            buf = torch.from_numpy(np.concatenate([P, Y]))
            dist.all_reduce(buf, op=dist.ReduceOp.SUM)
            P, Y = buf.numpy()[:k], buf.numpy()[k:]
            R, _, _ = oracle.householder(P, want_S=False)
            out = {"R": R, "Z": oracle.forward_subst(Y, R)}
        elif algo == "rr":
            d2 = np.sum(Xl.astype(np.float64) ** 2, axis=0)
            buf = torch.from_numpy(np.concatenate([P, d2[None, :]]))
            dist.all_reduce(buf, op=dist.ReduceOp.SUM)
            P, D = buf.numpy()[:k], np.sqrt(buf.numpy()[k])
            rq = oracle.rrqr(P / D[None, :], 1e-9)
            r, perm = rq["rank"], rq["perm"]
            Rf = rq["R"][:r] * D[perm][None, :]
            out = {"rank": r, "perm": perm, "R": Rf,
                   "Q": oracle.forward_subst(np.ascontiguousarray(Xl[:, perm[:r]]), Rf[:, :r].copy())}
        else:   # rcqr2
            Pt = torch.from_numpy(P)
            dist.all_reduce(Pt, op=dist.ReduceOp.SUM)
            R1, _, _ = oracle.householder(Pt.numpy(), want_S=False)
            Q1 = oracle.forward_subst(Xl, R1)
            A = torch.from_numpy(oracle.gram(Q1))
            dist.all_reduce(A, op=dist.ReduceOp.SUM)            # the second all-reduce of Alg. 3
            Rp, _ = oracle.cholesky(A.numpy())
            out = {"R": oracle.trmm_upper(Rp, R1), "Q": oracle.forward_subst(Q1, Rp)}
        out_q.put((rank, out))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("algo", ["reduced", "rr", "rcqr2"])
def test_two_rank_variants_equal_single(algo):
    m, n, k, world = 70_001, 12, 24, 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_alg, args=(r, world, port, algo, m, n, k, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    a, b = res[0], res[1]
    assert np.array_equal(a["R"], b["R"])                       # redundant small steps agree bitwise
    if algo == "reduced":
        full = oracle.factor_reduced(synth.make_X(m, n, 5.0, "f64"), k, 9, want_S=False)
        assert np.array_equal(a["Z"], b["Z"])
        assert np.linalg.norm(a["Z"] - full["Z"]) <= 1e-10 * np.linalg.norm(full["Z"])
        assert np.linalg.norm(a["R"] - full["R"]) <= 1e-13 * np.linalg.norm(full["R"])
    elif algo == "rr":
        full = oracle.factor_rr(synth.make_X_lowrank(m, n, n - 4, 2.0, 1e-13), k, 1e-9)
        assert a["rank"] == b["rank"] == full["rank"] == n - 4
        assert np.array_equal(a["perm"][: a["rank"]], full["perm"][: full["rank"]])
        Q = np.concatenate([a["Q"], b["Q"]])
        assert np.linalg.norm(Q - full["Q"]) <= 1e-10 * np.linalg.norm(full["Q"])
    else:
        full = oracle.factor2(synth.make_X(m, n, 5.0, "f64"), k)
        assert np.linalg.norm(a["R"] - full["R"]) <= 1e-12 * np.linalg.norm(full["R"])
        Q = np.concatenate([a["Q"], b["Q"]])
        assert np.linalg.norm(Q.T @ Q - np.eye(n), 2) <= 1e-13
