"""One Alg. 7 factorization of a BASELINE config (for an ncu launch list of its kernels)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2210_09953_b200 as rcq  # noqa: E402
import synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C2")
ap.add_argument("--tau", type=float, default=2e-7)
ap.add_argument("--reps", type=int, default=2)
a = ap.parse_args()
cfg = synth.config(a.config)
X = synth.make_X_torch(cfg["m"], cfg["n"], cfg["log10_cond"], cfg["dtype"])
plan = rcq.RCholQR(n=cfg["n"], k=cfg["k"], dtype=X.dtype, sketch=cfg["sketch"], nnz_per_col=cfg["nnz"])
for _ in range(a.reps):
    out = plan.factor_rr(X, a.tau)
torch.cuda.synchronize()
print("rank", out["rank"], "swaps", out["swaps"])
