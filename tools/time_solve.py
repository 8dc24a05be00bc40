"""Time plan.tri_solve (tri prep + tall solve) for one BASELINE config with CUDA events (kernel experiments)."""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2210_09953_b200 as rcq  # noqa: E402
import synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C4")
ap.add_argument("--m", type=int, default=0)
ap.add_argument("--iters", type=int, default=5)
a = ap.parse_args()
cfg = synth.config(a.config)
m = a.m or cfg["m"]
X = synth.make_X_torch(m, cfg["n"], cfg["log10_cond"], cfg["dtype"])
plan = rcq.RCholQR(n=cfg["n"], k=cfg["k"], dtype=X.dtype, sketch=cfg["sketch"], nnz_per_col=cfg["nnz"])
P = plan.sketch(X)
R, _, _ = plan.small_qr(P, want_S=False)
Q = torch.empty_like(X)
plan.tri_solve(X, R, Q=Q)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(a.iters):
    plan.tri_solve(X, R, Q=Q)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / a.iters
nbytes = 2 * X.numel() * X.element_size()
print(json.dumps({"config": a.config, "m": m, "env": {k: v for k, v in os.environ.items() if k.startswith("RCHOLQR")},
                  "ms": ms, "GBps_rw": nbytes / ms / 1e6}))
