"""Split RCholeskyQR2's time (Alg. 3) into Alg. 2, the Gram + Cholesky + R'R1 part and the second solve.

factor (Alg. 2), factor2(implicit) (Alg. 2 + steps 2-3) and factor2 (all four steps) are timed with
CUDA events on the current stream; the differences are the added steps.  Kernel experiments only.
"""
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
ap.add_argument("--m", type=int, default=0)
ap.add_argument("--iters", type=int, default=5)
a = ap.parse_args()
cfg = synth.config(a.config)
m = a.m or cfg["m"]
X = synth.make_X_torch(m, cfg["n"], cfg["log10_cond"], cfg["dtype"])
plan = rcq.RCholQR(n=cfg["n"], k=cfg["k"], dtype=X.dtype, sketch=cfg["sketch"], nnz_per_col=cfg["nnz"])
Q = torch.empty_like(X)
n = cfg["n"]
R = torch.empty(n, n, dtype=torch.float64, device=X.device)
Rp = torch.empty_like(R)


def timed(fn):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(a.iters):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / a.iters


t_alg2 = timed(lambda: plan.factor(X, Q=Q, R=R))
t_impl = timed(lambda: plan.factor2(X, Q=Q, R=R, Rprime=Rp, implicit=True))
t_expl = timed(lambda: plan.factor2(X, Q=Q, R=R, Rprime=Rp))
print(json.dumps({"config": a.config, "m": m, "env": {k: v for k, v in os.environ.items() if k.startswith("RCHOLQR")},
                  "alg2_ms": t_alg2, "gram_chol_trmm_ms": t_impl - t_alg2, "second_solve_ms": t_expl - t_impl,
                  "factor2_ms": t_expl}))
