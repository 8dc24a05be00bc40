"""B200-native direct randomized Cholesky QR (RCholeskyQR, Balabanov arXiv 2210.09953, Alg. 2).

Thin Python binding of the C ABI declared in ``include/rcholqr.h`` (argument marshalling only --
every step of the factorization runs in the CUDA kernels of ``lib/librcholqr.so``).  PyTorch is
used for device memory, streams and process groups.  There is no CPU fallback: importing works
anywhere, but any call that needs the library raises if it is missing or no GPU is present.

    plan = RCholQR(n=100, k=200, dtype=torch.float32, sketch="gaussian", seed=0)
    Q, R, _ = plan.factor(X)            # X: (m, n) CUDA tensor, row-major
"""
from __future__ import annotations

import ctypes
import os
import threading
from typing import Optional, Tuple

__all__ = ["RCholQR", "RCholQRError", "load_library", "library_path", "theta_export",
           "comm_unique_id", "comm_create", "comm_destroy", "strerror", "version",
           "OK", "E_INVALID", "E_SHAPE", "E_NONFINITE", "E_SINGULAR", "E_CUDA", "E_NCCL", "E_NOMEM",
           "GAUSSIAN", "SPARSE_SIGN", "RADEMACHER", "SRHT"]

_PKG = os.path.dirname(os.path.abspath(__file__))
# RCHOLQR_ABLATION_LIB=1 (kernel experiments under tools/ only) loads the build with the role ablation switches
# compiled in (python -m paper_2210_09953_b200.build --ablation); the product path always loads librcholqr.so
_LIB_PATH = os.path.join(_PKG, "lib", "librcholqr_ablation.so" if os.environ.get("RCHOLQR_ABLATION_LIB") else "librcholqr.so")
_lock = threading.Lock()
_lib = None

OK, E_INVALID, E_SHAPE, E_NONFINITE, E_SINGULAR, E_CUDA, E_NCCL, E_NOMEM = range(8)
GAUSSIAN, SPARSE_SIGN, RADEMACHER, SRHT = 0, 1, 2, 3
F64, F32 = 0, 1

# exported symbols (checked by tests/test_abi.py against include/rcholqr.h)
SYMBOLS = ["rcholqr_create", "rcholqr_destroy", "rcholqr_factor", "rcholqr_factor_async", "rcholqr_factor_graph",
           "rcholqr_query_status", "rcholqr_factor_host", "rcholqr_sketch", "rcholqr_small_qr",
           "rcholqr_tri_solve", "rcholqr_theta_export", "rcholqr_comm_unique_id",
           "rcholqr_comm_create", "rcholqr_comm_destroy", "rcholqr_strerror", "rcholqr_version",
           "rcholqr_launches_per_factor", "rcholqr_set_timing", "rcholqr_last_timings", "rcholqr_factor2",
           "rcholqr_factor_reduced", "rcholqr_factor_rr", "rcholqr_factor_colmajor",
           "rcholqr_factor_rr2", "rcholqr_last_path"]

# rcholqr_last_path bits (include/rcholqr.h)
PATH_SKETCH_TC, PATH_SKETCH_PRESPLIT, PATH_SKETCH_CUDA_CORE, PATH_SKETCH_FALLBACK = 1, 2, 4, 8
PATH_SOLVE_TC, PATH_SOLVE_DMMA, PATH_COLSQ_FUSED, PATH_COLMAJOR_NATIVE, PATH_SKETCH_FWHT = 16, 32, 64, 128, 256


class _Desc(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int32), ("k", ctypes.c_int32), ("dtype", ctypes.c_int32),
                ("sketch", ctypes.c_int32), ("nnz_per_col", ctypes.c_int32), ("device", ctypes.c_int32),
                ("seed", ctypes.c_uint64), ("nccl_comm", ctypes.c_void_p)]


class RCholQRError(RuntimeError):
    def __init__(self, status: int, where: str):
        super().__init__(f"{where}: {strerror(status)} (status {status})")
        self.status = status


def library_path() -> str:
    return _LIB_PATH


def load_library():
    """Load lib/librcholqr.so (built by ``__graft_entry__.build()`` / ``python -m
    paper_2210_09953_b200.build``).  Raises if it is missing -- there is no fallback."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(_LIB_PATH):
            raise RuntimeError(f"CUDA library not built: {_LIB_PATH} (run python -m paper_2210_09953_b200.build)")
        lib = ctypes.CDLL(_LIB_PATH)
        V, I32, I64, U64 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_uint64
        sig = {
            "rcholqr_create": ([ctypes.POINTER(_Desc), ctypes.POINTER(V)], I32),
            "rcholqr_destroy": ([V], I32),
            "rcholqr_factor": ([V, V, I64, I64, I64, V, I64, V, V, V], I32),
            "rcholqr_factor_async": ([V, V, I64, I64, I64, V, I64, V, V, V], I32),
            "rcholqr_factor_graph": ([V, V, I64, I64, I64, V, I64, V, V, V], I32),
            "rcholqr_query_status": ([V, V], I32),
            "rcholqr_factor_host": ([V, V, I64, I64, I64, V, I64, V, V, V], I32),
            "rcholqr_factor2": ([V, V, I64, I64, I64, V, I64, V, V, I32, V], I32),
            "rcholqr_factor_reduced": ([V, V, I64, I64, I64, I32, V, V, V, V, V], I32),
            "rcholqr_factor_colmajor": ([V, V, I64, I64, I64, V, I64, V, V, V], I32),
            "rcholqr_factor_rr2": ([V, V, I64, I64, I64, ctypes.c_double, ctypes.c_double, I32, V, I64, V, V, V, V,
                                    ctypes.POINTER(I32), ctypes.POINTER(I32), V], I32),
            "rcholqr_factor_rr": ([V, V, I64, I64, I64, ctypes.c_double, ctypes.c_double, I32, V, I64, V, V, V, V,
                                   ctypes.POINTER(I32), ctypes.POINTER(I32), V], I32),
            "rcholqr_sketch": ([V, V, I64, I64, I64, V, V], I32),
            "rcholqr_small_qr": ([V, V, V, V, V], I32),
            "rcholqr_tri_solve": ([V, V, I64, I64, V, V, I64, V], I32),
            "rcholqr_theta_export": ([U64, I32, I32, I32, I64, I64, V, V, V, V], I32),
            "rcholqr_comm_unique_id": ([V], I32),
            "rcholqr_comm_create": ([V, I32, I32, I32, ctypes.POINTER(V)], I32),
            "rcholqr_comm_destroy": ([V], I32),
            "rcholqr_strerror": ([I32], ctypes.c_char_p),
            "rcholqr_version": ([], I32),
            "rcholqr_launches_per_factor": ([V, I64], I32),
            "rcholqr_set_timing": ([V, I32], I32),
            "rcholqr_last_timings": ([V, V], I32),
            "rcholqr_last_path": ([V, ctypes.POINTER(ctypes.c_uint32), V], I32),
        }
        for name, (argt, rest) in sig.items():
            f = getattr(lib, name)
            f.argtypes, f.restype = argt, rest
        _lib = lib
        return lib


def strerror(status: int) -> str:
    try:
        return load_library().rcholqr_strerror(status).decode()
    except Exception:  # noqa: BLE001 - message only
        return f"status {status}"


def version() -> int:
    return int(load_library().rcholqr_version())


def _check(st: int, where: str):
    if st != OK:
        raise RCholQRError(st, where)


def _torch():
    import torch
    return torch


def _stream_ptr(stream) -> Optional[int]:
    torch = _torch()
    if stream is None:
        stream = torch.cuda.current_stream()
    return ctypes.c_void_p(stream.cuda_stream)


def _ptr(t) -> ctypes.c_void_p:
    return ctypes.c_void_p(0 if t is None else t.data_ptr())


class RCholQR:
    """A plan (``rcholqr_create``) for m x n matrices X with fixed n, k, dtype, sketch and seed."""

    def __init__(self, n: int, k: int, dtype=None, sketch: str = "gaussian", nnz_per_col: int = 8,
                 seed: int = 0, device: int = 0, comm: Optional[int] = None):
        torch = _torch()
        if not torch.cuda.is_available():
            raise RuntimeError("RCholQR needs a CUDA device (no CPU fallback)")
        dtype = torch.float64 if dtype is None else dtype
        if dtype not in (torch.float64, torch.float32):
            raise TypeError("dtype must be torch.float64 or torch.float32")
        self.n, self.k, self.dtype, self.seed, self.device = int(n), int(k), dtype, int(seed), int(device)
        self.sketch_kind = {"gaussian": GAUSSIAN, "sparse": SPARSE_SIGN, "sparse_sign": SPARSE_SIGN,
                            "rademacher": RADEMACHER, "srht": SRHT}[sketch]
        self.nnz_per_col = int(nnz_per_col)
        self._lib = load_library()
        d = _Desc(self.n, self.k, F64 if dtype == torch.float64 else F32, self.sketch_kind, self.nnz_per_col,
                  self.device, self.seed, ctypes.c_void_p(comm or 0))
        h = ctypes.c_void_p()
        _check(self._lib.rcholqr_create(ctypes.byref(d), ctypes.byref(h)), "rcholqr_create")
        self._h = h

    # -- lifecycle
    def close(self):
        if getattr(self, "_h", None) and self._h.value:
            self._lib.rcholqr_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    # -- helpers
    def _dev(self):
        return _torch().device("cuda", self.device)

    def _check_out(self, t, name, rows, cols, dtype, cuda=True, exact=False):
        """Validate a caller-supplied output buffer before its raw pointer reaches the C ABI: device
        (the plan's CUDA device, or CPU for the host entry point), dtype, 2-D, at least rows x cols,
        stride(1) == 1 (exact=True: exactly rows x cols and contiguous -- buffers without a leading
        dimension in the ABI).  Returns its leading dimension."""
        if t is None:
            return cols
        ok_dev = (t.is_cuda and t.device.index == self.device) if cuda else (not t.is_cuda)
        if not ok_dev or t.dtype != dtype or t.dim() != 2:
            where = f"cuda:{self.device}" if cuda else "cpu"
            raise ValueError(f"{name} must be a 2-D {dtype} tensor on {where}")
        if exact:
            if tuple(t.shape) != (rows, cols) or not t.is_contiguous():
                raise ValueError(f"{name} must be a contiguous ({rows}, {cols}) tensor")
            return cols
        if t.shape[0] < rows or t.shape[1] < cols or (rows > 0 and t.stride(1) != 1):
            raise ValueError(f"{name} must have shape >= ({rows}, {cols}) with stride(1) == 1")
        return max(t.stride(0), cols) if rows > 1 else cols

    def _check_x(self, X):
        torch = _torch()
        if not (X.is_cuda and X.device.index == self.device and X.dtype == self.dtype and X.dim() == 2
                and X.shape[1] == self.n):
            raise ValueError(f"X must be a cuda:{self.device} {self.dtype} tensor of shape (m, {self.n})")
        if X.stride(1) != 1:
            raise ValueError("X must be row-major (stride(1) == 1)")
        return X.shape[0], max(X.stride(0), self.n) if X.shape[0] > 1 else self.n

    # -- Algorithm 2
    def factor(self, X, row_offset: int = 0, want_S: bool = False, Q=None, R=None, S=None,
               stream=None, sync: bool = True, graph: bool = False) -> Tuple:
        """Q, R (and S) of X.  ``sync=False`` uses rcholqr_factor_async (status via query_status);
        ``graph=True`` uses rcholqr_factor_graph (the chain replayed from a CUDA graph when X, Q, R, S
        are the same buffers as in the previous call)."""
        torch = _torch()
        m, ldx = self._check_x(X)
        Q = torch.empty((m, self.n), dtype=self.dtype, device=X.device) if Q is None else Q
        R = torch.empty((self.n, self.n), dtype=torch.float64, device=X.device) if R is None else R
        if want_S and S is None:
            S = torch.empty((self.k, self.n), dtype=torch.float64, device=X.device)
        ldq = self._check_out(Q, "Q", m, self.n, self.dtype)
        self._check_out(R, "R", self.n, self.n, torch.float64, exact=True)
        self._check_out(S, "S", self.k, self.n, torch.float64, exact=True)
        fn = self._lib.rcholqr_factor_graph if graph else (self._lib.rcholqr_factor if sync else self._lib.rcholqr_factor_async)
        st = fn(self._h, _ptr(X), m, row_offset, ldx, _ptr(Q), ldq, _ptr(R), _ptr(S), _stream_ptr(stream))
        _check(st, "rcholqr_factor")
        if graph and sync:
            _check(self.query_status(stream), "rcholqr_factor_graph")
        return Q, R, S

    def factor_colmajor(self, Xt, row_offset: int = 0, want_S: bool = False, Qt=None, R=None, S=None, stream=None):
        """Alg. 2 on column-major X given as its transpose Xt (n, m) row-major CUDA tensor -- i.e. the
        column-major buffer itself; returns (Qt (n, m), R, S) with Qt the column-major Q."""
        torch = _torch()
        if not (Xt.is_cuda and Xt.dtype == self.dtype and Xt.dim() == 2 and Xt.shape[0] == self.n and Xt.stride(1) == 1):
            raise ValueError(f"Xt must be a CUDA {self.dtype} tensor of shape ({self.n}, m), stride(1) == 1")
        m = Xt.shape[1]
        ldx = max(Xt.stride(0), m, 1)
        Qt = torch.empty((self.n, m), dtype=self.dtype, device=Xt.device) if Qt is None else Qt
        R = torch.empty((self.n, self.n), dtype=torch.float64, device=Xt.device) if R is None else R
        if want_S and S is None:
            S = torch.empty((self.k, self.n), dtype=torch.float64, device=Xt.device)
        st = self._lib.rcholqr_factor_colmajor(self._h, _ptr(Xt), m, row_offset, ldx, _ptr(Qt), max(Qt.stride(0), m, 1),
                                               _ptr(R), _ptr(S), _stream_ptr(stream))
        _check(st, "rcholqr_factor_colmajor")
        return Qt, R, S

    def factor2(self, X, row_offset: int = 0, Q=None, R=None, Rprime=None, implicit: bool = False,
                stream=None) -> Tuple:
        """RCholeskyQR2 (Alg. 3): Q (orthonormal; with ``implicit`` RCholeskyQR's Q1), R, R'."""
        torch = _torch()
        m, ldx = self._check_x(X)
        Q = torch.empty((m, self.n), dtype=self.dtype, device=X.device) if Q is None else Q
        R = torch.empty((self.n, self.n), dtype=torch.float64, device=X.device) if R is None else R
        if Rprime is None:
            Rprime = torch.empty((self.n, self.n), dtype=torch.float64, device=X.device)
        ldq = self._check_out(Q, "Q", m, self.n, self.dtype)
        self._check_out(R, "R", self.n, self.n, torch.float64, exact=True)
        self._check_out(Rprime, "Rprime", self.n, self.n, torch.float64, exact=True)
        st = self._lib.rcholqr_factor2(self._h, _ptr(X), m, row_offset, ldx, _ptr(Q), ldq, _ptr(R), _ptr(Rprime),
                                       int(bool(implicit)), _stream_ptr(stream))
        _check(st, "rcholqr_factor2")
        return Q, R, Rprime

    def factor_reduced(self, X, l: int, row_offset: int = 0, want_S: bool = False, want_Y: bool = False, Z=None,
                       R=None, S=None, Y=None, stream=None) -> Tuple:
        """Reduced RCholeskyQR (Alg. 5): Z = L Q (l x n) without forming Q; returns (Z, R, S, Y)."""
        torch = _torch()
        m, ldx = self._check_x(X)
        f64 = dict(dtype=torch.float64, device=X.device)
        Z = torch.empty((l, self.n), **f64) if Z is None else Z
        R = torch.empty((self.n, self.n), **f64) if R is None else R
        if want_S and S is None:
            S = torch.empty((self.k, self.n), **f64)
        if want_Y and Y is None:
            Y = torch.empty((l, self.n), **f64)
        for t, name, rows in ((Z, "Z", l), (R, "R", self.n), (S, "S", self.k), (Y, "Y", l)):
            self._check_out(t, name, rows, self.n, torch.float64, exact=True)
        st = self._lib.rcholqr_factor_reduced(self._h, _ptr(X), m, row_offset, ldx, int(l), _ptr(Z), _ptr(R),
                                              _ptr(S), _ptr(Y), _stream_ptr(stream))
        _check(st, "rcholqr_factor_reduced")
        return Z, R, S, Y

    def factor_rr(self, X, tau: float, f: float = 1.5, rank_fixed: int = 0, row_offset: int = 0,
                  want_S: bool = False, Q=None, R=None, stream=None) -> dict:
        """Rank-revealing RCholeskyQR (Alg. 7): dict(Q (m x r view), R (r x n view), perm, rank, D, S, swaps)
        with X[:, perm] ~= Q R."""
        torch = _torch()
        m, ldx = self._check_x(X)
        Q = torch.empty((m, self.n), dtype=self.dtype, device=X.device) if Q is None else Q
        R = torch.empty((self.n, self.n), dtype=torch.float64, device=X.device) if R is None else R
        perm = torch.empty(self.n, dtype=torch.int32, device=X.device)
        D = torch.empty(self.n, dtype=torch.float64, device=X.device)
        S = torch.empty((self.k, self.n), dtype=torch.float64, device=X.device) if want_S else None
        ldq = self._check_out(Q, "Q", m, self.n, self.dtype)
        self._check_out(R, "R", self.n, self.n, torch.float64, exact=True)
        rank, swaps = ctypes.c_int32(0), ctypes.c_int32(0)
        st = self._lib.rcholqr_factor_rr(self._h, _ptr(X), m, row_offset, ldx, float(tau), float(f), int(rank_fixed),
                                         _ptr(Q), ldq, _ptr(R), _ptr(perm), _ptr(D),
                                         _ptr(S), ctypes.byref(rank), ctypes.byref(swaps), _stream_ptr(stream))
        _check(st, "rcholqr_factor_rr")
        r = rank.value
        return {"Q": Q[:, :r], "R": R[:r], "perm": perm, "rank": r, "D": D,
                "S": None if S is None else S[:, :r], "swaps": swaps.value}

    def factor_rr2(self, X, tau: float, f: float = 1.5, rank_fixed: int = 0, row_offset: int = 0, Q=None,
                   stream=None) -> dict:
        """RRRCholeskyQR2: dict(Q (m x r, orthonormal), R (r x n), Rp (r x r), perm, rank, D, swaps)."""
        torch = _torch()
        m, ldx = self._check_x(X)
        Q = torch.empty((m, self.n), dtype=self.dtype, device=X.device) if Q is None else Q
        f64 = dict(dtype=torch.float64, device=X.device)
        R = torch.empty((self.n, self.n), **f64)
        Rp = torch.empty((self.n * self.n,), **f64)
        perm = torch.empty(self.n, dtype=torch.int32, device=X.device)
        D = torch.empty(self.n, **f64)
        rank, swaps = ctypes.c_int32(0), ctypes.c_int32(0)
        ldq = self._check_out(Q, "Q", m, self.n, self.dtype)
        st = self._lib.rcholqr_factor_rr2(self._h, _ptr(X), m, row_offset, ldx, float(tau), float(f), int(rank_fixed),
                                          _ptr(Q), ldq, _ptr(R), _ptr(Rp), _ptr(perm),
                                          _ptr(D), ctypes.byref(rank), ctypes.byref(swaps), _stream_ptr(stream))
        _check(st, "rcholqr_factor_rr2")
        r = rank.value
        return {"Q": Q[:, :r], "R": R[:r], "Rp": Rp[: r * r].view(r, r), "perm": perm, "rank": r, "D": D,
                "swaps": swaps.value}

    def query_status(self, stream=None) -> int:
        return int(self._lib.rcholqr_query_status(self._h, _stream_ptr(stream)))

    def factor_host(self, X_host, row_offset: int = 0, want_S: bool = False, Q_host=None, R_host=None,
                    S_host=None, stream=None):
        """End-to-end call with host (preferably pinned) CPU tensors; copies are inside the call."""
        torch = _torch()
        if X_host.is_cuda or X_host.dtype != self.dtype or X_host.shape[1] != self.n or X_host.stride(1) != 1:
            raise ValueError("X_host must be a row-major CPU tensor of the plan's dtype")
        m = X_host.shape[0]
        Q_host = torch.empty((m, self.n), dtype=self.dtype, pin_memory=True) if Q_host is None else Q_host
        R_host = torch.empty((self.n, self.n), dtype=torch.float64, pin_memory=True) if R_host is None else R_host
        if want_S and S_host is None:
            S_host = torch.empty((self.k, self.n), dtype=torch.float64, pin_memory=True)
        ldq = self._check_out(Q_host, "Q_host", m, self.n, self.dtype, cuda=False)
        self._check_out(R_host, "R_host", self.n, self.n, torch.float64, cuda=False, exact=True)
        self._check_out(S_host, "S_host", self.k, self.n, torch.float64, cuda=False, exact=True)
        st = self._lib.rcholqr_factor_host(self._h, _ptr(X_host), m, row_offset, max(X_host.stride(0), self.n),
                                           _ptr(Q_host), ldq, _ptr(R_host), _ptr(S_host), _stream_ptr(stream))
        _check(st, "rcholqr_factor_host")
        return Q_host, R_host, S_host

    # -- step-level entry points
    def sketch(self, X, row_offset: int = 0, P=None, stream=None):
        torch = _torch()
        m, ldx = self._check_x(X)
        P = torch.empty((self.k, self.n), dtype=torch.float64, device=X.device) if P is None else P
        self._check_out(P, "P", self.k, self.n, torch.float64, exact=True)
        _check(self._lib.rcholqr_sketch(self._h, _ptr(X), m, row_offset, ldx, _ptr(P), _stream_ptr(stream)),
               "rcholqr_sketch")
        return P

    def small_qr(self, P, want_S: bool = True, stream=None):
        """Returns (R, S, status) -- E_SINGULAR is returned, not raised (R is still written)."""
        torch = _torch()
        P = P.contiguous()
        R = torch.empty((self.n, self.n), dtype=torch.float64, device=P.device)
        S = torch.empty((self.k, self.n), dtype=torch.float64, device=P.device) if want_S else None
        st = self._lib.rcholqr_small_qr(self._h, _ptr(P), _ptr(R), _ptr(S), _stream_ptr(stream))
        if st not in (OK, E_SINGULAR):
            _check(st, "rcholqr_small_qr")
        return R, S, int(st)

    def tri_solve(self, X, R, Q=None, stream=None):
        torch = _torch()
        m, ldx = self._check_x(X)
        R = R.contiguous()
        Q = torch.empty((m, self.n), dtype=self.dtype, device=X.device) if Q is None else Q
        ldq = self._check_out(Q, "Q", m, self.n, self.dtype)
        self._check_out(R, "R", self.n, self.n, torch.float64, exact=True)
        _check(self._lib.rcholqr_tri_solve(self._h, _ptr(X), m, ldx, _ptr(R), _ptr(Q), ldq,
                                           _stream_ptr(stream)), "rcholqr_tri_solve")
        return Q

    # -- introspection
    def launches_per_factor(self, m: int) -> int:
        return int(self._lib.rcholqr_launches_per_factor(self._h, m))

    def last_path(self, stream=None) -> int:
        """RCHOLQR_PATH_* bits of the kernels that served the last call (rcholqr_last_path)."""
        out = ctypes.c_uint32(0)
        _check(self._lib.rcholqr_last_path(self._h, ctypes.byref(out), _stream_ptr(stream)), "rcholqr_last_path")
        return int(out.value)

    def set_timing(self, enable: bool = True):
        _check(self._lib.rcholqr_set_timing(self._h, int(enable)), "rcholqr_set_timing")

    def last_timings(self) -> dict:
        out = (ctypes.c_float * 6)()
        _check(self._lib.rcholqr_last_timings(self._h, out), "rcholqr_last_timings")
        keys = ["sketch", "reduce", "allreduce", "small_qr", "tri_prep", "solve"]
        return {k: float(v) for k, v in zip(keys, out)}


def theta_export(seed: int, k: int, m: int, sketch: str = "gaussian", nnz_per_col: int = 8,
                 row_offset: int = 0, device: int = 0, stream=None):
    """GPU-generated Theta for global rows row_offset..+m (test export, rcholqr_theta_export).

    Gaussian / Rademacher -> Z (k, m) float32 unscaled draws / signs; sparse -> (rows (m, nnz) int32,
    signs (m, nnz) int8)."""
    torch = _torch()
    lib = load_library()
    dev = torch.device("cuda", device)
    if sketch in ("gaussian", "rademacher", "srht"):
        Z = torch.empty((k, m), dtype=torch.float32, device=dev)
        kind = {"gaussian": GAUSSIAN, "rademacher": RADEMACHER, "srht": SRHT}[sketch]
        _check(lib.rcholqr_theta_export(seed, k, kind, 0, row_offset, m, _ptr(Z), None, None,
                                        _stream_ptr(stream)), "rcholqr_theta_export")
        return Z
    rows = torch.empty((m, nnz_per_col), dtype=torch.int32, device=dev)
    signs = torch.empty((m, nnz_per_col), dtype=torch.int8, device=dev)
    _check(lib.rcholqr_theta_export(seed, k, SPARSE_SIGN, nnz_per_col, row_offset, m, None, _ptr(rows),
                                    _ptr(signs), _stream_ptr(stream)), "rcholqr_theta_export")
    return rows, signs


def comm_unique_id() -> bytes:
    buf = (ctypes.c_uint8 * 128)()
    _check(load_library().rcholqr_comm_unique_id(buf), "rcholqr_comm_unique_id")
    return bytes(buf)


def comm_create(uid: bytes, nranks: int, rank: int, device: int) -> int:
    buf = (ctypes.c_uint8 * 128).from_buffer_copy(uid)
    out = ctypes.c_void_p()
    _check(load_library().rcholqr_comm_create(buf, nranks, rank, device, ctypes.byref(out)), "rcholqr_comm_create")
    return int(out.value)


def comm_destroy(comm: int):
    _check(load_library().rcholqr_comm_destroy(ctypes.c_void_p(comm)), "rcholqr_comm_destroy")
