"""CPU fp64 oracle for RCholeskyQR (Balabanov, arXiv 2210.09953, Algorithm 2).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this package.  It shares no code with
``paper_2210_09953_b200`` (the CUDA product path) and never imports it.

The arithmetic lives in ``oracle/oracle.c`` (plain C, fp64, -ffp-contract=off); this module is
ctypes marshalling plus the stability *metrics* the paper defines (PAPER.md:773, 797:
cond(Q), ||I - (Theta Q)^T Theta Q||, column residuals), written with numpy/LAPACK.

Parity status of each oracle function ("Oracle pins"):
  philox4x32_10      pinned: Random123 known-answer vectors + ATen's independent Philox
  ln32 / sincos2pi_j pinned: exhaustive 2^23-input comparison against fp64 libm
  gauss4 / theta     pinned: moments, KS test vs N(0,1), E||Theta x||^2 = ||x||^2
  sparse_col         pinned: structural invariants (one row per block, +-1/sqrt(zeta)), chi^2
  sketch             pinned: exact rational Theta X on tiny inputs, n=1 closed form, linearity,
                     partition invariance
  sketch_entry       pinned: exact rational sums (Gaussian, sparse-sign incl. zeta > 64, Rademacher,
                     SRHT), bitwise equal to sketch across 65,536-row blocks, NaN on bad arguments
  householder        pinned: SPEC examples, LAPACK QR (sign-normalised), mpmath 50-digit QR
  forward_subst      pinned: SPEC examples, R = I, scipy solve_triangular, Higham Thm 8.5 bound
  factor             pinned: cond(Q) = cond(Theta U) identity, eq:main1 residual, metamorphic
                     power-of-two scaling (bitwise)
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None

OK, E_INVALID, E_SHAPE, E_NONFINITE, E_SINGULAR, E_NOMEM = 0, 1, 2, 3, 4, 7
GAUSSIAN, SPARSE_SIGN, RADEMACHER, SRHT = 0, 1, 2, 3
F64, F32 = 0, 1


def build(force: bool = False) -> str:
    """Compile oracle.c into liboracle.so (gcc, -O2 -fopenmp -ffp-contract=off, no fast-math)."""
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(_SRC):
        tmp = _LIB_PATH + ".tmp%d" % os.getpid()
        cmd = ["gcc", "-O2", "-std=c11", "-fPIC", "-shared", "-fopenmp", "-ffp-contract=off",
               "-fno-fast-math", "-Wall", "-o", tmp, _SRC, "-lm"]
        subprocess.check_call(cmd)
        os.replace(tmp, _LIB_PATH)
    return _LIB_PATH


def _L():
    global _lib
    with _lock:
        if _lib is None:
            build()
            lib = ctypes.CDLL(_LIB_PATH)
            P, I64, I32, U64, U32 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_uint64, ctypes.c_uint32
            lib.oracle_philox4x32_10.argtypes = [P, P, P]
            lib.oracle_ln32.argtypes = [ctypes.c_float]
            lib.oracle_ln32.restype = ctypes.c_float
            lib.oracle_ln32_batch.argtypes = [P, P, I64]
            lib.oracle_sincos2pi_j_batch.argtypes = [P, P, P, I64]
            lib.oracle_gauss4.argtypes = [U64, U64, U32, P]
            lib.oracle_theta_gauss.argtypes = [U64, I32, U64, I32]
            lib.oracle_theta_gauss.restype = ctypes.c_double
            lib.oracle_theta_gauss_z.argtypes = [U64, I32, I64, I64, P]
            lib.oracle_theta_sparse.argtypes = [U64, I32, I32, I64, I64, P, P]
            lib.oracle_theta_rademacher.argtypes = [U64, I32, I64, I64, P]
            lib.oracle_theta_srht.argtypes = [U64, I32, I64, I64, P]
            lib.oracle_srht_rows.argtypes = [U64, I32, P]
            lib.oracle_srht_sign.argtypes = [U64, U64, U64]
            lib.oracle_srht_sign.restype = I32
            lib.oracle_rademacher_sign.argtypes = [U64, U64, I32]
            lib.oracle_rademacher_sign.restype = I32
            lib.oracle_sketch.argtypes = [P, I32, I64, I32, I64, I64, I32, I32, I32, U64, P]
            lib.oracle_sketch.restype = I32
            lib.oracle_householder.argtypes = [P, I32, I32, P, P]
            lib.oracle_householder.restype = I32
            lib.oracle_forward_subst.argtypes = [P, I32, I64, I32, I64, P, P, I64]
            lib.oracle_forward_subst.restype = I32
            lib.oracle_factor.argtypes = [P, I32, I64, I32, I64, I64, I32, I32, I32, U64, P, I64, P, P, P]
            lib.oracle_factor.restype = I32
            lib.oracle_num_threads.restype = I32
            lib.oracle_gram.argtypes = [P, I32, I64, I32, I64, P]
            lib.oracle_gram.restype = I32
            lib.oracle_cholesky.argtypes = [P, I32, P]
            lib.oracle_cholesky.restype = I32
            lib.oracle_trmm_upper.argtypes = [P, P, I32, P]
            lib.oracle_factor2.argtypes = [P, I32, I64, I32, I64, I64, I32, I32, I32, U64, P, I64, P, P, P]
            lib.oracle_factor2.restype = I32
            lib.oracle_extract.argtypes = [P, I32, I64, I32, I64, I64, I32, I32, U64, P]
            lib.oracle_extract.restype = I32
            lib.oracle_factor_reduced.argtypes = [P, I32, I64, I32, I64, I64, I32, I32, I32, U64, I32, P, P, P, P]
            lib.oracle_factor_reduced.restype = I32
            lib.oracle_colnorms.argtypes = [P, I32, I64, I32, I64, P]
            lib.oracle_colnorms.restype = I32
            lib.oracle_rrqr.argtypes = [P, I32, I32, ctypes.c_double, ctypes.c_double, I32, P, P, P, P, P]
            lib.oracle_rrqr.restype = I32
            lib.oracle_factor_rr.argtypes = [P, I32, I64, I32, I64, I64, I32, I32, I32, U64, ctypes.c_double,
                                             ctypes.c_double, I32, P, I64, P, P, P, P, P, P]
            lib.oracle_factor_rr.restype = I32
            lib.oracle_sketch_entry.argtypes = [P, I64, I64, I32, I32, I32, U64, I32]
            lib.oracle_sketch_entry.restype = ctypes.c_double
            _lib = lib
    return _lib


def _ptr(a):
    return None if a is None else ctypes.c_void_p(a.ctypes.data)


def _dtype_code(X):
    if X.dtype == np.float64:
        return F64
    if X.dtype == np.float32:
        return F32
    raise TypeError("X must be float64 or float32")


def num_threads() -> int:
    return int(_L().oracle_num_threads())


class OracleError(RuntimeError):
    def __init__(self, status: int, where: str):
        super().__init__(f"oracle {where}: status {status}")
        self.status = status


# ---------------------------------------------------------------- Theta (reading A1-A4)
def philox4x32_10(ctr, key) -> np.ndarray:
    c = np.ascontiguousarray(ctr, dtype=np.uint32)
    k = np.ascontiguousarray(key, dtype=np.uint32)
    out = np.zeros(4, dtype=np.uint32)
    _L().oracle_philox4x32_10(_ptr(c), _ptr(k), _ptr(out))
    return out


def ln32(a) -> np.ndarray:
    a = np.ascontiguousarray(a, dtype=np.float32)
    out = np.empty_like(a)
    _L().oracle_ln32_batch(_ptr(a), _ptr(out), a.size)
    return out


def sincos2pi_j(j):
    """sin, cos of 2 pi j 2^-23 for integer j in [0, 2^23) (fp32, normative transform)."""
    j = np.ascontiguousarray(j, dtype=np.uint32)
    s = np.empty(j.shape, dtype=np.float32)
    c = np.empty(j.shape, dtype=np.float32)
    _L().oracle_sincos2pi_j_batch(_ptr(j), _ptr(s), _ptr(c), j.size)
    return s, c


def gauss4(seed: int, i: int, q: int) -> np.ndarray:
    z = np.zeros(4, dtype=np.float32)
    _L().oracle_gauss4(seed, i, q, _ptr(z))
    return z


def theta_gauss_z(seed: int, k: int, m: int, row_offset: int = 0) -> np.ndarray:
    """Unscaled N(0,1) fp32 draws z_ri, shape (k, m), columns = global rows row_offset..+m."""
    Z = np.empty((k, m), dtype=np.float32)
    _L().oracle_theta_gauss_z(seed, k, row_offset, m, _ptr(Z))
    return Z


def theta_sparse(seed: int, k: int, zeta: int, m: int, row_offset: int = 0):
    """Sparse-sign columns: rows (m, zeta) int32 and signs (m, zeta) int8."""
    rows = np.empty((m, zeta), dtype=np.int32)
    signs = np.empty((m, zeta), dtype=np.int8)
    _L().oracle_theta_sparse(seed, k, zeta, row_offset, m, _ptr(rows), _ptr(signs))
    return rows, signs


def theta_rademacher(seed: int, k: int, m: int, row_offset: int = 0) -> np.ndarray:
    """Rademacher signs (k, m) int8 (unscaled; Theta = signs / sqrt(k), reading A22)."""
    S = np.empty((k, m), dtype=np.int8)
    _L().oracle_theta_rademacher(seed, k, row_offset, m, _ptr(S))
    return S


def srht_rows(seed: int, k: int) -> np.ndarray:
    """The k sampled Hadamard rows s_r (uint64, < 2^48) of the SRHT Theta (reading A23)."""
    s = np.empty(k, dtype=np.uint64)
    _L().oracle_srht_rows(seed, k, _ptr(s))
    return s


def theta_srht(seed: int, k: int, m: int, row_offset: int = 0) -> np.ndarray:
    """SRHT signs (k, m) int8 (unscaled; Theta = signs / sqrt(k), reading A23)."""
    S = np.empty((k, m), dtype=np.int8)
    _L().oracle_theta_srht(seed, k, row_offset, m, _ptr(S))
    return S


def theta_dense(seed: int, k: int, m: int, sketch: int = GAUSSIAN, zeta: int = 8,
                row_offset: int = 0) -> np.ndarray:
    """Explicit fp64 Theta (k x m) -- for tiny test inputs only."""
    if sketch == GAUSSIAN:
        Z = theta_gauss_z(seed, k, m, row_offset).astype(np.float64)
        return Z * (1.0 / np.sqrt(np.float64(k)))
    if sketch == RADEMACHER:
        return theta_rademacher(seed, k, m, row_offset).astype(np.float64) * (1.0 / np.sqrt(np.float64(k)))
    if sketch == SRHT:
        return theta_srht(seed, k, m, row_offset).astype(np.float64) * (1.0 / np.sqrt(np.float64(k)))
    rows, signs = theta_sparse(seed, k, zeta, m, row_offset)
    T = np.zeros((k, m), dtype=np.float64)
    v = 1.0 / np.sqrt(np.float64(zeta))
    for i in range(m):
        for t in range(zeta):
            T[rows[i, t], i] = v if signs[i, t] > 0 else -v
    return T


# ---------------------------------------------------------------- Algorithm 2 steps
def sketch(X: np.ndarray, k: int, sketch: int = GAUSSIAN, zeta: int = 8, seed: int = 0,
           row_offset: int = 0) -> np.ndarray:
    """Step 1, P = Theta X."""
    X = np.ascontiguousarray(X)
    m, n = X.shape
    P = np.empty((k, n), dtype=np.float64)
    st = _L().oracle_sketch(_ptr(X), _dtype_code(X), m, n, n, row_offset, k, sketch, zeta, seed, _ptr(P))
    if st != OK:
        raise OracleError(st, "sketch")
    return P


def sketch_entry(x_col: np.ndarray, r: int, k: int, sketch: int = GAUSSIAN, zeta: int = 8, seed: int = 0,
                 row_offset: int = 0) -> float:
    """P_rj = sum_i Theta_ri x_ij for one column x (fp64) -- sampled full-size sketch checks."""
    x = np.ascontiguousarray(x_col, dtype=np.float64)
    return float(_L().oracle_sketch_entry(_ptr(x), x.size, row_offset, k, sketch, zeta, seed, r))


def householder(P: np.ndarray, want_S: bool = True):
    """Step 2, [R, S] = QR(P) by Householder; diag(R) >= 0.

    Returns (R, S, status); status E_SINGULAR is returned, not raised."""
    P = np.ascontiguousarray(P, dtype=np.float64)
    k, n = P.shape
    R = np.empty((n, n), dtype=np.float64)
    S = np.empty((k, n), dtype=np.float64) if want_S else None
    st = _L().oracle_householder(_ptr(P), k, n, _ptr(R), _ptr(S))
    if st not in (OK, E_SINGULAR):
        raise OracleError(st, "householder")
    return R, S, st


def forward_subst(X: np.ndarray, R: np.ndarray) -> np.ndarray:
    """Step 3, Q = X R^{-1} by row-wise forward substitution."""
    X = np.ascontiguousarray(X)
    R = np.ascontiguousarray(R, dtype=np.float64)
    m, n = X.shape
    Q = np.empty_like(X)
    st = _L().oracle_forward_subst(_ptr(X), _dtype_code(X), m, n, n, _ptr(R), _ptr(Q), n)
    if st != OK:
        raise OracleError(st, "forward_subst")
    return Q


def factor(X: np.ndarray, k: int, sketch: int = GAUSSIAN, zeta: int = 8, seed: int = 0,
           row_offset: int = 0, want_S: bool = True) -> dict:
    """Whole Algorithm 2: returns dict(Q, R, P, S)."""
    X = np.ascontiguousarray(X)
    m, n = X.shape
    Q = np.empty_like(X)
    R = np.empty((n, n), dtype=np.float64)
    P = np.empty((k, n), dtype=np.float64)
    S = np.empty((k, n), dtype=np.float64) if want_S else None
    st = _L().oracle_factor(_ptr(X), _dtype_code(X), m, n, n, row_offset, k, sketch, zeta, seed,
                            _ptr(Q), n, _ptr(R), _ptr(P), _ptr(S))
    if st != OK:
        raise OracleError(st, "factor")
    return {"Q": Q, "R": R, "P": P, "S": S}


def gram(Q: np.ndarray) -> np.ndarray:
    """A = Q^T Q, compensated (Alg. 3 step 2)."""
    Q = np.ascontiguousarray(Q)
    m, n = Q.shape
    A = np.empty((n, n), dtype=np.float64)
    st = _L().oracle_gram(_ptr(Q), _dtype_code(Q), m, n, n, _ptr(A))
    if st != OK:
        raise OracleError(st, "gram")
    return A


def cholesky(A: np.ndarray):
    """R' upper triangular with A = R'^T R' (Alg. 3 step 3); returns (R', status)."""
    A = np.ascontiguousarray(A, dtype=np.float64)
    n = A.shape[0]
    Rp = np.empty((n, n), dtype=np.float64)
    st = _L().oracle_cholesky(_ptr(A), n, _ptr(Rp))
    if st not in (OK, E_SINGULAR):
        raise OracleError(st, "cholesky")
    return Rp, st


def trmm_upper(U: np.ndarray, V: np.ndarray) -> np.ndarray:
    U = np.ascontiguousarray(U, dtype=np.float64)
    V = np.ascontiguousarray(V, dtype=np.float64)
    out = np.empty_like(U)
    _L().oracle_trmm_upper(_ptr(U), _ptr(V), U.shape[0], _ptr(out))
    return out


def factor2(X: np.ndarray, k: int, sketch: int = GAUSSIAN, zeta: int = 8, seed: int = 0,
            row_offset: int = 0) -> dict:
    """Whole Algorithm 3 (RCholeskyQR2): dict(Q, R, Q1, Rp) with Q = Q1 Rp^{-1}."""
    X = np.ascontiguousarray(X)
    m, n = X.shape
    Q = np.empty_like(X)
    Q1 = np.empty_like(X)
    R = np.empty((n, n), dtype=np.float64)
    Rp = np.empty((n, n), dtype=np.float64)
    st = _L().oracle_factor2(_ptr(X), _dtype_code(X), m, n, n, row_offset, k, sketch, zeta, seed,
                             _ptr(Q), n, _ptr(R), _ptr(Q1), _ptr(Rp))
    if st != OK:
        raise OracleError(st, "factor2")
    return {"Q": Q, "R": R, "Q1": Q1, "Rp": Rp}


def extractor_row0(k: int, sketch: int = GAUSSIAN) -> int:
    """First Gaussian-stream row of the Alg. 5 extractor L (reading A20): k after a Gaussian Theta, else 0."""
    return k if sketch == GAUSSIAN else 0


def extract(X: np.ndarray, l0: int, l: int, seed: int = 0, row_offset: int = 0) -> np.ndarray:
    """Y = L X with L_ji = z(seed, i, l0 + j) / sqrt(l) (Alg. 5 step 1)."""
    X = np.ascontiguousarray(X)
    m, n = X.shape
    Y = np.empty((l, n), dtype=np.float64)
    st = _L().oracle_extract(_ptr(X), _dtype_code(X), m, n, n, row_offset, l0, l, seed, _ptr(Y))
    if st != OK:
        raise OracleError(st, "extract")
    return Y


def factor_reduced(X: np.ndarray, k: int, l: int, sketch: int = GAUSSIAN, zeta: int = 8, seed: int = 0,
                   row_offset: int = 0, want_S: bool = True) -> dict:
    """Whole Algorithm 5 (reduced RCholeskyQR): dict(Z, R, Y, S), Z = Y R^{-1} = L Q."""
    X = np.ascontiguousarray(X)
    m, n = X.shape
    Z = np.empty((l, n), dtype=np.float64)
    Y = np.empty((l, n), dtype=np.float64)
    R = np.empty((n, n), dtype=np.float64)
    S = np.empty((k, n), dtype=np.float64) if want_S else None
    st = _L().oracle_factor_reduced(_ptr(X), _dtype_code(X), m, n, n, row_offset, k, sketch, zeta, seed, l,
                                    _ptr(Z), _ptr(R), _ptr(Y), _ptr(S))
    if st != OK:
        raise OracleError(st, "factor_reduced")
    return {"Z": Z, "R": R, "Y": Y, "S": S}


def colnorms(X: np.ndarray) -> np.ndarray:
    """D = diag(||X(:, j)||_2), compensated (Alg. 7 normalisation)."""
    X = np.ascontiguousarray(X)
    m, n = X.shape
    d = np.empty(n, dtype=np.float64)
    st = _L().oracle_colnorms(_ptr(X), _dtype_code(X), m, n, n, _ptr(d))
    if st != OK:
        raise OracleError(st, "colnorms")
    return d


def rrqr(P: np.ndarray, tau: float, f: float = 1.5, rank_fixed: int = 0, want_S: bool = False) -> dict:
    """Strong RRQR of P (Alg. 7 steps 2-3, reading A21): dict(perm, R (n x n of P[:, perm]), rank, swaps, S)."""
    P = np.ascontiguousarray(P, dtype=np.float64)
    k, n = P.shape
    perm = np.empty(n, dtype=np.int32)
    R = np.empty((n, n), dtype=np.float64)
    S = np.empty((k, n), dtype=np.float64) if want_S else None
    rank = ctypes.c_int(0)
    swaps = ctypes.c_int(0)
    st = _L().oracle_rrqr(_ptr(P), k, n, float(tau), float(f), int(rank_fixed), _ptr(perm), _ptr(R), _ptr(S),
                          ctypes.byref(rank), ctypes.byref(swaps))
    if st not in (OK, E_SINGULAR):
        raise OracleError(st, "rrqr")
    return {"perm": perm, "R": R, "rank": rank.value, "swaps": swaps.value, "S": S, "status": st}


def factor_rr(X: np.ndarray, k: int, tau: float, f: float = 1.5, rank_fixed: int = 0, sketch: int = GAUSSIAN,
              zeta: int = 8, seed: int = 0, row_offset: int = 0, want_S: bool = False) -> dict:
    """Whole Algorithm 7 (RRRCholeskyQR): dict(Q (m x r), R (r x n), perm, rank, D, S, swaps)
    with X[:, perm] ~= Q R."""
    X = np.ascontiguousarray(X)
    m, n = X.shape
    Q = np.zeros_like(X)
    R = np.empty((n, n), dtype=np.float64)
    perm = np.empty(n, dtype=np.int32)
    D = np.empty(n, dtype=np.float64)
    S = np.empty((k, n), dtype=np.float64) if want_S else None
    rank = ctypes.c_int(0)
    swaps = ctypes.c_int(0)
    st = _L().oracle_factor_rr(_ptr(X), _dtype_code(X), m, n, n, row_offset, k, sketch, zeta, seed, float(tau),
                               float(f), int(rank_fixed), _ptr(Q), n, _ptr(R), _ptr(perm), ctypes.byref(rank),
                               _ptr(D), _ptr(S), ctypes.byref(swaps))
    if st != OK:
        raise OracleError(st, "factor_rr")
    r = rank.value
    return {"Q": Q[:, :r].copy(), "R": R[:r].copy(), "perm": perm, "rank": r, "D": D,
            "S": None if S is None else S[:, :r].copy(), "swaps": swaps.value}


def factor_rr2(X: np.ndarray, k: int, tau: float, f: float = 1.5, rank_fixed: int = 0, sketch: int = GAUSSIAN,
               zeta: int = 8, seed: int = 0, row_offset: int = 0) -> dict:
    """RRRCholeskyQR2 (RRRCholeskyQR "augmented with the classical CholeskyQR in exactly the
    same way as done in RCholeskyQR2"): Alg. 7 gives (Q1, R1, perm, r); then A = Q1^T Q1, R' = chol(A),
    R = R' R1 (r x n, upper trapezoidal), Q = Q1 R'^{-1}.  Returns dict(Q, R, Rp, Q1, perm, rank, swaps)."""
    rr = factor_rr(X, k, tau, f=f, rank_fixed=rank_fixed, sketch=sketch, zeta=zeta, seed=seed,
                   row_offset=row_offset)
    Q1 = np.ascontiguousarray(rr["Q"])
    A = gram(Q1)
    Rp, st = cholesky(A)
    if st != OK:
        raise OracleError(st, "factor_rr2 cholesky")
    R = np.triu(Rp @ rr["R"])          # (r x r upper) (r x n upper trapezoidal); exact zeros kept below
    Q = forward_subst(Q1, Rp)
    return {"Q": Q, "R": R, "Rp": Rp, "Q1": Q1, "perm": rr["perm"], "rank": rr["rank"], "swaps": rr["swaps"]}


# ---------------------------------------------------------------- metrics
def orth_defect(S: np.ndarray) -> float:
    """||I - S^T S||_2 (fp64)."""
    S = np.asarray(S, dtype=np.float64)
    G = S.T @ S
    return float(np.linalg.norm(np.eye(G.shape[0]) - G, 2))


def cond(A: np.ndarray) -> float:
    s = np.linalg.svd(np.asarray(A, dtype=np.float64), compute_uv=False)
    return float(s[0] / s[-1]) if s[-1] > 0 else float("inf")


def cond_from_gram(G: np.ndarray) -> float:
    """cond(Q) from its fp64 Gram matrix Q^T Q (valid while cond(Q)^2 u << 1)."""
    w = np.linalg.eigvalsh(np.asarray(G, dtype=np.float64))
    return float(np.sqrt(w[-1] / w[0])) if w[0] > 0 else float("inf")


def col_residual(X: np.ndarray, Q: np.ndarray, R: np.ndarray) -> float:
    """max_j ||X_j - (Q R)_j|| / ||X_j||  (eq:main1)."""
    Xd = np.asarray(X, dtype=np.float64)
    E = Xd - np.asarray(Q, dtype=np.float64) @ R
    return float(np.max(np.linalg.norm(E, axis=0) / np.linalg.norm(Xd, axis=0)))
