"""The C ABI used from plain C (examples/factor_host.c): compiled with gcc against include/rcholqr.h and the in-tree
librcholqr.so, no CUDA headers and no Python in the program; it factors a host matrix with three sketches through
rcholqr_factor_host and checks X = QR, the shape of R and the conditioning of Q itself."""
import os
import subprocess

import pytest

import paper_2210_09953_b200 as rcq

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_c_example_builds_and_runs(cuda, tmp_path):
    rcq.load_library()                                   # builds the library if needed
    lib = os.path.join(ROOT, "paper_2210_09953_b200", "lib")
    exe = str(tmp_path / "factor_host")
    subprocess.run(["gcc", "-O2", "-Wall", "-I" + os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "examples", "factor_host.c"), "-L" + lib, "-lrcholqr",
                    "-Wl,-rpath," + lib, "-lm", "-o", exe], check=True)
    out = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "c abi example ok" in out.stdout, out.stdout
