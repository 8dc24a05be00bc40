"""Time plan.small_qr (step 2) on the sketch of one BASELINE config with CUDA events (kernel experiments)."""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2210_09953_b200 as rcq  # noqa: E402
import synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C2")
ap.add_argument("--iters", type=int, default=20)
a = ap.parse_args()
cfg = synth.config(a.config)
X = synth.make_X_torch(min(cfg["m"], 1 << 20), cfg["n"], cfg["log10_cond"], cfg["dtype"])
plan = rcq.RCholQR(n=cfg["n"], k=cfg["k"], dtype=X.dtype, sketch=cfg["sketch"], nnz_per_col=cfg["nnz"])
P = plan.sketch(X)
R, _, _ = plan.small_qr(P, want_S=False)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(a.iters):
    plan.small_qr(P, want_S=False)
e1.record()
torch.cuda.synchronize()
print(json.dumps({"config": a.config, "env": {k: v for k, v in os.environ.items() if k.startswith("RCHOLQR")},
                  "ms": e0.elapsed_time(e1) / a.iters, "R00": float(R[0, 0])}))
