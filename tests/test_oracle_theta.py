"""Pins of the oracle's Theta (readings A1-A4) against things
other than itself: published Philox known answers, ATen's independent Philox, fp64 libm,
distribution tests, structural invariants.  CPU only."""
import os
import subprocess

import numpy as np
import pytest
import scipy.stats as ss

import oracle

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _kat():
    rows = []
    with open(os.path.join(GOLDEN, "philox4x32_10_kat.txt")) as f:
        for line in f:
            if line.startswith("#") or not line.strip():
                continue
            w = [int(x, 16) for x in line.split()]
            rows.append((w[0:4], w[4:6], w[6:10]))
    return rows


@pytest.mark.parametrize("ctr,key,out", _kat())
def test_philox_known_answers(ctr, key, out):
    # Random123 kat_vectors (Salmon et al. SC'11), tests/golden/philox4x32_10_kat.txt
    assert oracle.philox4x32_10(ctr, key).tolist() == out


@pytest.fixture(scope="module")
def aten_philox(tmp_path_factory):
    """ATen's PhiloxRNGEngine (an implementation independent of ours), compiled test-only."""
    import torch.utils.cpp_extension as ce
    d = tmp_path_factory.mktemp("aten")
    src = d / "p.cpp"
    src.write_text(
        "#include <ATen/core/PhiloxRNGEngine.h>\n#include <cstdio>\n#include <cstdlib>\n"
        "int main(int c, char** v){ for (int a = 1; a + 2 < c; a += 3) {"
        " at::Philox4_32 e(strtoull(v[a],0,0), strtoull(v[a+2],0,0), strtoull(v[a+1],0,0));"
        " for (int i = 0; i < 4; ++i) printf(\"%u \", e()); printf(\"\\n\"); } }\n")
    exe = d / "p"
    inc = ce.include_paths()[0]
    subprocess.check_call(["g++", "-std=c++17", "-O1", "-I" + inc, str(src), "-o", str(exe)])
    return str(exe)


def test_philox_matches_aten(aten_philox):
    # ATen: key = seed, counter = (offset lo, offset hi, subsequence lo, subsequence hi).
    rng = np.random.default_rng(7)
    cases = [(int(rng.integers(0, 2**64, dtype=np.uint64)), int(rng.integers(0, 2**64, dtype=np.uint64)),
              int(rng.integers(0, 2**64, dtype=np.uint64))) for _ in range(64)]
    cases += [(0, 0, 0), (2**64 - 1, 2**64 - 1, 2**64 - 1), (0, 123456789, (1 << 32) | 5)]
    args = []
    for seed, off, sub in cases:
        args += [str(seed), str(off), str(sub)]
    out = subprocess.check_output([aten_philox] + args, text=True).split("\n")
    for (seed, off, sub), line in zip(cases, out):
        ctr = [off & 0xFFFFFFFF, off >> 32, sub & 0xFFFFFFFF, sub >> 32]
        key = [seed & 0xFFFFFFFF, seed >> 32]
        assert oracle.philox4x32_10(ctr, key).tolist() == [int(x) for x in line.split()]


def test_ln32_exhaustive_vs_libm():
    # every uniform the transform can see: a = 1 - j 2^-23, j = 0..2^23-1 (reading A1)
    a = (1.0 - np.arange(0, 2**23, dtype=np.float64) * 2.0**-23).astype(np.float32)
    got = oracle.ln32(a).astype(np.float64)
    ref = np.log(a.astype(np.float64))
    ulp = np.spacing(np.abs(ref).astype(np.float32)).astype(np.float64)
    ulp[ref == 0] = np.spacing(np.float32(0))
    err = np.abs(got - ref) / ulp
    assert err.max() <= 2.0, err.max()      # measured 1.5 ulp
    assert got[0] == 0.0                     # ln(1) = 0 exactly
    assert np.all(np.diff(got) <= 0)         # monotone (a decreasing)


def test_sincos2pi_j_exhaustive_vs_libm():
    j = np.arange(0, 2**23, dtype=np.uint32)
    s, c = oracle.sincos2pi_j(j)
    ang = 2.0 * np.pi * j.astype(np.float64) * 2.0**-23
    es = np.abs(s - np.sin(ang))
    ec = np.abs(c - np.cos(ang))
    assert es.max() <= 1.6 * 2.0**-24 and ec.max() <= 1.6 * 2.0**-24, (es.max(), ec.max())
    # exact special angles
    assert s[0] == 0.0 and c[0] == 1.0
    q = 2**21  # j 2^-23 = 1/4, 1/2, 3/4
    assert (s[q], c[q]) == (1.0, 0.0) and (s[2 * q], c[2 * q]) == (0.0, -1.0) and (s[3 * q], c[3 * q]) == (-1.0, 0.0)
    assert np.all(np.abs(s.astype(np.float64) ** 2 + c.astype(np.float64) ** 2 - 1) < 4e-7)


def test_gauss4_box_muller_definition():
    # z = sqrt(-2 ln ua) (cos 2 pi ub, sin 2 pi ub), ua = 1 - (wa >> 9) 2^-23, ub = (wb >> 9) 2^-23,
    # checked against fp64 libm.
    for (seed, i, q) in [(0, 0, 0), (0, 12345, 7), (2**63 + 5, 2**40 + 3, 99), (17, 2**32 + 1, 2**20)]:
        z = oracle.gauss4(seed, i, q).astype(np.float64)
        ctr = [i & 0xFFFFFFFF, i >> 32, q, 1]
        w = oracle.philox4x32_10(ctr, [seed & 0xFFFFFFFF, seed >> 32]).astype(np.uint64)
        for p in range(2):
            ua = 1.0 - (w[2 * p] >> 9) * 2.0**-23
            ub = (w[2 * p + 1] >> 9) * 2.0**-23
            rho = np.sqrt(-2.0 * np.log(ua))
            assert abs(z[2 * p] - rho * np.cos(2 * np.pi * ub)) <= 8e-7 * max(1.0, rho)
            assert abs(z[2 * p + 1] - rho * np.sin(2 * np.pi * ub)) <= 8e-7 * max(1.0, rho)


def test_gaussian_distribution():
    Z = oracle.theta_gauss_z(0, 64, 200_000).astype(np.float64).ravel()
    n = Z.size
    assert abs(Z.mean()) < 4.0 / np.sqrt(n)
    assert abs(Z.var() - 1.0) < 4.0 * np.sqrt(2.0 / n)
    assert abs(ss.skew(Z)) < 4.0 * np.sqrt(6.0 / n)
    assert abs(ss.kurtosis(Z)) < 4.0 * np.sqrt(24.0 / n)
    assert ss.kstest(Z[:2_000_000], "norm").pvalue > 1e-4
    # mean of Theta^2 = 1/k within 3%
    k = 64
    assert abs(np.mean((Z / np.sqrt(k)) ** 2) * k - 1.0) < 0.03


def test_gaussian_isometry_in_expectation():
    # E ||Theta x||^2 = ||x||^2 (rescaled Gaussian), 500 seeds within 5%
    rng = np.random.default_rng(1)
    x = rng.standard_normal(300)
    k = 40
    vals = []
    for seed in range(500):
        T = oracle.theta_dense(seed, k, x.size)
        vals.append(np.sum((T @ x) ** 2))
    assert abs(np.mean(vals) / np.sum(x * x) - 1.0) < 0.05


def test_theta_keyed_by_global_row():
    Z = oracle.theta_gauss_z(3, 12, 100, row_offset=0)
    Z2 = oracle.theta_gauss_z(3, 12, 60, row_offset=40)
    assert np.array_equal(Z[:, 40:], Z2)
    Z3 = oracle.theta_gauss_z(4, 12, 100, row_offset=0)
    assert not np.array_equal(Z, Z3)


@pytest.mark.parametrize("k,zeta", [(128, 8), (64, 8), (96, 12), (40, 4), (16, 16)])
def test_sparse_sign_structure(k, zeta):
    m = 50_000
    rows, signs = oracle.theta_sparse(11, k, zeta, m)
    beta = k // zeta
    blocks = rows // beta
    assert np.array_equal(blocks, np.broadcast_to(np.arange(zeta), rows.shape))   # one row per block
    assert np.all((rows >= 0) & (rows < k))
    assert np.all(np.abs(signs) == 1)
    # uniformity of the within-block row and of the sign (chi^2)
    within = (rows % beta).ravel()
    cnt = np.bincount(within, minlength=beta)
    if beta > 1:
        assert ss.chisquare(cnt).pvalue > 1e-4
    assert abs(np.mean(signs == 1) - 0.5) < 4 * 0.5 / np.sqrt(signs.size)
    T = oracle.theta_dense(11, k, 64, sketch=oracle.SPARSE_SIGN, zeta=zeta)
    assert np.all(np.count_nonzero(T, axis=0) == zeta)
    assert np.allclose(np.abs(T[T != 0]), 1 / np.sqrt(zeta), rtol=0, atol=0)
