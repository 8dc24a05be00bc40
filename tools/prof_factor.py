"""Run a few factorizations of one BASELINE config (for ncu / compute-sanitizer captures)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2210_09953_b200 as rcq  # noqa: E402
import synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C2")
ap.add_argument("--iters", type=int, default=3)
ap.add_argument("--m", type=int, default=0, help="override m (smaller runs)")
ap.add_argument("--sketch", default="", help="another Theta on the same shape")
a = ap.parse_args()
cfg = synth.config(a.config)
if a.sketch:
    cfg["sketch"] = a.sketch
m = a.m or cfg["m"]
X = synth.make_X_torch(m, cfg["n"], cfg["log10_cond"], cfg["dtype"])
plan = rcq.RCholQR(n=cfg["n"], k=cfg["k"], dtype=X.dtype, sketch=cfg["sketch"], nnz_per_col=cfg["nnz"])
for _ in range(a.iters):
    Q, R, _ = plan.factor(X)
torch.cuda.synchronize()
print("ok", a.config, m, float(R[0, 0]))
