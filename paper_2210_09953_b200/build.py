"""Build the in-tree CUDA library ``lib/librcholqr.so`` for sm_100a (nvcc, no JIT cache).

Staleness is decided by CONTENT, not mtimes: a SHA-256 over the sources, headers and the nvcc command
is written next to the library (``lib/librcholqr.so.sha256``) and the library is rebuilt whenever it
differs -- so a prebuilt .so shipped with a snapshot is reused only if it was built from exactly these
sources.  ``build()`` returns the path; ``last_build_info()`` says whether this process rebuilt it.
Translation units compile in parallel (one nvcc per .cu) and are linked once.
"""
from __future__ import annotations

import concurrent.futures as cf
import glob
import hashlib
import os
import shutil
import subprocess
import sys
import tempfile

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
LIB = os.path.join(PKG, "lib", "librcholqr.so")
STAMP = LIB + ".sha256"
SRCS = sorted(glob.glob(os.path.join(PKG, "csrc", "*.cu")))
HDRS = sorted(glob.glob(os.path.join(PKG, "csrc", "*.cuh"))) + [os.path.join(ROOT, "include", "rcholqr.h")]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-std=c++20", *ARCH, "-lineinfo", "-Xcompiler", "-fPIC"]
_info = {"rebuilt": False, "hash": None}


def _nccl_include() -> str:
    import importlib.util
    spec = importlib.util.find_spec("nvidia.nccl")
    for p in (spec.submodule_search_locations if spec else []) or []:
        inc = os.path.join(p, "include")
        if os.path.exists(os.path.join(inc, "nccl.h")):
            return inc
    for inc in ("/usr/include", "/usr/local/cuda/include"):
        if os.path.exists(os.path.join(inc, "nccl.h")):
            return inc
    raise RuntimeError("nccl.h not found (needed for the multi-GPU all-reduce types)")


def _lib(ablation: bool) -> str:
    return LIB.replace("librcholqr.so", "librcholqr_ablation.so") if ablation else LIB


def _ablation_flags() -> list:
    # kernel experiments (tools/ only): extra -D switches for the ablation library, never for the product build
    return ["-DRCHOLQR_ABLATION"] + os.environ.get("RCHOLQR_EXTRA_NVCC_FLAGS", "").split()


def source_hash(ablation: bool = False) -> str:
    h = hashlib.sha256()
    h.update(" ".join(FLAGS + (_ablation_flags() if ablation else [])).encode())
    for f in SRCS + HDRS:
        h.update(os.path.basename(f).encode())
        with open(f, "rb") as fh:
            h.update(fh.read())
    return h.hexdigest()


def _stale(digest: str, lib: str) -> bool:
    stamp = lib + ".sha256"
    if not os.path.exists(lib) or not os.path.exists(stamp):
        return True
    with open(stamp) as f:
        return f.read().strip() != digest


def build(force: bool = False, verbose: bool = False, ablation: bool = False) -> str:
    """ablation=True: a separate library (lib/librcholqr_ablation.so) with the kernels' role-ablation switches
    (RCHOLQR_*_DEBUG) compiled in, for the experiments under tools/; never loaded by the product path."""
    LIB = _lib(ablation)
    STAMP = LIB + ".sha256"
    digest = source_hash(ablation)
    if not ablation:
        _info["hash"] = digest
    if not force and not _stale(digest, LIB):
        return LIB
    os.makedirs(os.path.dirname(LIB), exist_ok=True)
    nvcc = os.path.join(os.environ.get("CUDA_HOME", "/usr/local/cuda"), "bin", "nvcc")
    inc = ["-I" + os.path.join(ROOT, "include"), "-I" + _nccl_include()]
    extra = ["-Xptxas=-v"] if verbose else []
    tmpdir = tempfile.mkdtemp(prefix="rcholqr_build_")
    try:
        def obj(src):
            o = os.path.join(tmpdir, os.path.basename(src) + ".o")
            subprocess.check_call([nvcc, *FLAGS, *extra, *(_ablation_flags() if ablation else []), *inc, "-c", "-o", o, src])
            return o
        with cf.ThreadPoolExecutor(max_workers=min(len(SRCS), os.cpu_count() or 4)) as ex:
            objs = list(ex.map(obj, SRCS))
        tmp = LIB + ".tmp%d" % os.getpid()
        subprocess.check_call([nvcc, *ARCH, "-shared", "-o", tmp, *objs, "-ldl"])
        os.replace(tmp, LIB)
        with open(STAMP, "w") as f:
            f.write(digest + "\n")
    finally:
        shutil.rmtree(tmpdir, ignore_errors=True)
    if not ablation:
        _info["rebuilt"] = True
    return LIB


def last_build_info() -> dict:
    """{"rebuilt": did this process compile the library, "hash": the source hash it matches}."""
    return dict(_info)


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv, ablation="--ablation" in sys.argv))
