"""Per-role timeline of CTA 0 of the tcgen05 tall solve (ablation build: RCHOLQR_ABLATION_LIB=1), C4-shaped.
Prints per-tile event times (clock64, relative) for the MMA issuer, loader, drain sets and the first digit warp,
and the steady-state averages of each wait and each phase."""
import argparse
import ctypes
import json
import os
import sys

os.environ["RCHOLQR_ABLATION_LIB"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2210_09953_b200 as rcq  # noqa: E402
import synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C4")
ap.add_argument("--m", type=int, default=16 * 1024 * 1024)
ap.add_argument("--which", type=int, default=0, help="0: solve, 1: sparse sketch")
a = ap.parse_args()
cfg = synth.config(a.config)
X = synth.make_X_torch(a.m, cfg["n"], cfg["log10_cond"], cfg["dtype"])
plan = rcq.RCholQR(n=cfg["n"], k=cfg["k"], dtype=X.dtype, sketch=cfg["sketch"], nnz_per_col=cfg["nnz"])
lib = rcq.load_library()
lib.rcholqr_trace_read.argtypes = [ctypes.c_int32, ctypes.c_void_p, ctypes.c_size_t]
buf = np.zeros(8 * 64 * 8, dtype=np.int64)
P = plan.sketch(X)
R, _, _ = plan.small_qr(P, want_S=False)
Q = torch.empty_like(X)
for _ in range(2):
    if a.which == 0:
        plan.tri_solve(X, R, Q=Q)
    else:
        plan.sketch(X)
    torch.cuda.synchronize()
    lib.rcholqr_trace_read(a.which, buf.ctypes.data, buf.nbytes)
T = buf.reshape(8, 64, 8).astype(np.float64)
t0 = T[T > 0].min()
T = np.where(T > 0, T - t0, np.nan)
names = {0: "mma", 1: "load", 2: "drain0", 3: "drain1", 4: "digit"} if a.which == 0 else \
    {0: "mma", 1: "load", 2: "bgrp0", 3: "bgrp1", 4: "egrp0", 5: "egrp1"}
out = {}
for r, nm in names.items():
    ev = T[r]
    if np.all(np.isnan(ev)):
        continue
    d = np.diff(ev, axis=1)                 # event-to-event durations per tile
    out[nm] = {"per_tile_start_delta": float(np.nanmean(np.diff(ev[8:48, 0]))),
               "phase_means": [None if np.all(np.isnan(d[8:48, e])) else float(np.nanmean(d[8:48, e])) for e in range(7)]}
print(json.dumps(out, indent=1))
np.set_printoptions(linewidth=200, suppress=True)
for r, nm in names.items():
    print(nm, T[r, 10:14, :6].astype(np.int64) if not np.all(np.isnan(T[r])) else "-")
