"""The C-ABI library builds for sm_100a, loads without a GPU, exports every symbol include/rcholqr.h
declares, and the Python binding mirrors those names.  No compute calls (CPU only)."""
import ctypes
import os
import re
import subprocess

import pytest

import paper_2210_09953_b200 as rcq
from paper_2210_09953_b200 import build as rbuild

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "rcholqr.h")


def _declared():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(rcholqr_[a-z0-9_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib():
    rbuild.build()
    return ctypes.CDLL(rbuild.LIB)


def test_header_declares_the_boundary():
    names = _declared()
    for must in ["rcholqr_create", "rcholqr_factor", "rcholqr_destroy", "rcholqr_strerror"]:
        assert must in names
    assert set(names) == set(rcq.SYMBOLS)


def test_library_exports_every_declared_symbol(lib):
    out = subprocess.check_output(["nm", "-D", "--defined-only", rbuild.LIB], text=True)
    exported = {l.split()[-1] for l in out.splitlines() if " T " in l}
    for name in _declared():
        assert name in exported, name
        assert hasattr(lib, name)


def test_library_is_sm100a(lib):
    out = subprocess.check_output(["cuobjdump", "--list-elf", rbuild.LIB], text=True)
    assert "sm_100a" in out
    sass = subprocess.check_output(["cuobjdump", "-sass", rbuild.LIB], text=True)
    assert "DMMA" in sass  # FP64 tensor-core MMA in the sketch and the tall solve


def test_no_fast_math_in_theta_source():
    # bit-exact Theta needs IEEE round-to-nearest fp32 ops (reading A1)
    flags = " ".join(rbuild.ARCH)
    assert "use_fast_math" not in open(rbuild.__file__).read()
    assert "compute_100a" in flags


def test_strerror_and_version_without_gpu(lib):
    lib.rcholqr_strerror.restype = ctypes.c_char_p
    lib.rcholqr_strerror.argtypes = [ctypes.c_int]
    assert lib.rcholqr_strerror(4).decode().startswith("R has a zero")
    assert lib.rcholqr_version() == 100


def test_create_validates_before_touching_the_device(lib):
    d = rcq._Desc(0, 10, 0, 0, 8, 0, 0, None)   # n < 1
    h = ctypes.c_void_p()
    lib.rcholqr_create.argtypes = [ctypes.POINTER(rcq._Desc), ctypes.POINTER(ctypes.c_void_p)]
    assert lib.rcholqr_create(ctypes.byref(d), ctypes.byref(h)) == rcq.E_SHAPE and not h.value
    d = rcq._Desc(10, 5, 0, 0, 8, 0, 0, None)   # k < n
    assert lib.rcholqr_create(ctypes.byref(d), ctypes.byref(h)) == rcq.E_SHAPE
    d = rcq._Desc(10, 20, 7, 0, 8, 0, 0, None)  # bad dtype
    assert lib.rcholqr_create(ctypes.byref(d), ctypes.byref(h)) == rcq.E_INVALID
    d = rcq._Desc(10, 20, 0, 1, 3, 0, 0, None)  # sparse: k % nnz != 0
    assert lib.rcholqr_create(ctypes.byref(d), ctypes.byref(h)) == rcq.E_SHAPE
    assert lib.rcholqr_create(None, ctypes.byref(h)) == rcq.E_INVALID
    assert lib.rcholqr_destroy(None) == rcq.OK


def test_product_path_has_no_oracle_or_fallback():
    pkg = os.path.join(ROOT, "paper_2210_09953_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt and "liboracle" not in txt, f
                assert "numpy.linalg" not in txt and "np.linalg" not in txt, f


def test_binding_fails_loudly_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(RuntimeError):
        rcq.RCholQR(n=4, k=8)


def test_header_is_plain_c_and_the_c_example_links(lib, tmp_path):
    """include/rcholqr.h compiles as C99 with no CUDA or C++ headers, and examples/factor_host.c links against the
    in-tree library (the program itself needs a GPU: tests/test_gpu_c_example.py runs it)."""
    probe = tmp_path / "probe.c"
    probe.write_text('#include "rcholqr.h"\nint main(void) { rcholqr_desc d = {1, 2, RCHOLQR_F64, RCHOLQR_GAUSSIAN, 8, 0, 0, 0}; '
                     'return (int)sizeof(d) == 0; }\n')
    subprocess.run(["gcc", "-std=c99", "-pedantic", "-Werror", "-I" + os.path.join(ROOT, "include"), "-fsyntax-only",
                    str(probe)], check=True)
    libdir = os.path.dirname(rbuild.LIB)
    subprocess.run(["gcc", "-O1", "-Wall", "-Werror", "-I" + os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "examples", "factor_host.c"), "-L" + libdir, "-lrcholqr", "-Wl,-rpath," + libdir,
                    "-lm", "-o", str(tmp_path / "factor_host")], check=True)


def test_tcgen05_and_tma_in_sass(lib):
    """The tensor-core paths are Blackwell-native: tcgen05 MMAs (UTCIMMA), TMEM loads (LDTM) and TMA tensor loads /
    stores (UTMALDG / UTMASTG) are in the library's SASS."""
    sass = subprocess.check_output(["cuobjdump", "-sass", rbuild.LIB], text=True)
    for mnemonic in ("UTCIMMA", "LDTM", "UTMALDG", "UTMASTG"):
        assert mnemonic in sass, mnemonic
