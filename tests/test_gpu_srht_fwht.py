"""SRHT by the blocked fast Walsh-Hadamard transform (srht_fwht.cu; the SRHT costs m n log2 m):
P <= 1e-12 relative Frobenius vs the compensated oracle (reading A23, Theta_ri = (-1)^popcount(s_r & i) d_i / sqrt(k))
for every accumulator variant (k <= 128, 256, 512, 1024), ragged m and n, row offsets that are not multiples of
the 1024-row transform block (a rank's first block is partial: negative TMA start row), several blocks per CTA;
agreement with the dense +-1 kernels; the row-partition sum; Alg. 2 end to end."""
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


@pytest.fixture(autouse=True)
def _force_fwht(monkeypatch):
    monkeypatch.setenv("RCHOLQR_SRHT_FWHT", "1")         # by default the transform serves k > 128 only


def _plan(n, k, dt, seed=0):
    return rcq.RCholQR(n=n, k=k, dtype=torch.float64 if dt == "f64" else torch.float32, sketch="srht", seed=seed)


@pytest.mark.parametrize("m,n,k,dt,ro", [
    (100_003, 64, 128, "f32", 0),               # C4 shape: KU = 4, 98 blocks, ragged last block
    (70_001, 48, 96, "f64", 24_864),            # fp64 in-place stages, row offset inside a block
    (50_000, 32, 300, "f32", 7),                # KU = 16, odd offset
    (40_000, 100, 200, "f32", 2**33 + 3),       # n not a multiple of 8 (13 column tiles, the last one clipped), huge offset
    (30_000, 20, 512, "f64", 1024 * 5),         # KU = 16, block-aligned offset
    (20_000, 12, 1000, "f64", 1023),            # KU = 32 (250 registers), first block holds one row
    (9_000, 12, 1024, "f32", 511),              # k = 1024
    (6_000, 8, 2500, "f64", 77),                # k > 1024: three launches of <= 1024 sketch rows
    (333, 18, 36, "f64", 900),                  # fewer rows than one block, straddling a block boundary
    (1, 8, 16, "f32", 5),                       # single row
    (120_000, 256, 512, "f64", 0),              # C3 shape: 32 column tiles x 9 splits, 14 blocks per CTA (ring wraps)
])
def test_fwht_sketch_parity(cuda, m, n, k, dt, ro):
    X = synth.make_X(m, n, 5.0, dt)
    plan = _plan(n, k, dt)
    Pg = _np(plan.sketch(_t(X), row_offset=ro))
    assert plan.last_path() & rcq.PATH_SKETCH_FWHT, plan.last_path()
    Po = oracle.sketch(X, k, sketch=oracle.SRHT, row_offset=ro)
    assert _rel(Pg, Po) <= 1e-12, _rel(Pg, Po)


def test_fwht_matches_dense(cuda, monkeypatch):
    X = _t(synth.make_X(300_000, 64, 4.0, "f32"))
    a = _np(_plan(64, 128, "f32").sketch(X))
    monkeypatch.delenv("RCHOLQR_SRHT_FWHT")
    plan = _plan(64, 128, "f32")                          # k <= 128: the dense tcgen05 kernel by default
    b = _np(plan.sketch(X))
    assert not plan.last_path() & rcq.PATH_SKETCH_FWHT and plan.last_path() & rcq.PATH_SKETCH_TC
    assert _rel(a, b) <= 1e-13, _rel(a, b)


def test_fwht_strided_and_unaligned(cuda):
    # a 16-byte aligned row pitch larger than n goes through the tensor map; an unaligned pitch takes the dense kernels
    X = synth.make_X(20_000, 37, 3.0, "f32")
    Po = oracle.sketch(X, 74, sketch=oracle.SRHT)
    plan = _plan(37, 74, "f32")
    Xp = torch.zeros((20_000, 40), dtype=torch.float32, device="cuda")
    Xp[:, :37] = _t(X)
    Pg = _np(plan.sketch(Xp[:, :37]))
    assert plan.last_path() & rcq.PATH_SKETCH_FWHT
    assert _rel(Pg, Po) <= 1e-12
    Pg = _np(plan.sketch(_t(X)))                          # 148-byte rows
    assert not plan.last_path() & rcq.PATH_SKETCH_FWHT
    assert _rel(Pg, Po) <= 1e-12


def test_fwht_rank_partition_sum(cuda):
    # blocks are aligned to GLOBAL multiples of 1024 rows: the partial sketches of any row partition add up to the
    # sketch of the whole X (the method's single all-reduce)
    m, n, k = 50_000, 24, 48
    X = synth.make_X(m, n, 4.0, "f64")
    Po = oracle.sketch(X, k, sketch=oracle.SRHT, row_offset=100)
    plan = _plan(n, k, "f64")
    cuts = [0, 1, 1500, 20_001, 49_999, m]
    tot = np.zeros((k, n))
    for a, b in zip(cuts[:-1], cuts[1:]):
        tot += _np(plan.sketch(_t(X[a:b]), row_offset=100 + a)) * 1.0
    assert _rel(tot, Po) <= 1e-12, _rel(tot, Po)


@pytest.mark.parametrize("dt,c", [("f32", 4), ("f64", 10)])
def test_fwht_factor_parity(cuda, dt, c):
    m, n, k = 262_144, 64, 128
    X = synth.make_X(m, n, c, dt)
    ref = oracle.factor(X, k, sketch=oracle.SRHT)
    plan = _plan(n, k, dt)
    Q, R, S = plan.factor(_t(X), want_S=True)
    assert plan.last_path() & rcq.PATH_SKETCH_FWHT
    assert _rel(_np(R), ref["R"]) <= (1e-10 if dt == "f64" else 1e-4), _rel(_np(R), ref["R"])
    assert _rel(_np(Q), ref["Q"]) <= 10 * U64 * 10**c + (2 * U32 if dt == "f32" else 0)
    assert oracle.orth_defect(_np(S)) <= 1e-13


def test_fwht_nonfinite(cuda):
    X = synth.make_X(30_000, 16, 2.0, "f32")
    X[12_345, 3] = np.inf
    plan = _plan(16, 32, "f32")
    with pytest.raises(rcq.RCholQRError) as e:
        plan.factor(_t(X))
    assert e.value.status == rcq.E_NONFINITE
