"""Sustained timing of the sketch and the tall solve of one BASELINE config with SM clock and power samples (NVML),
for A/B runs of kernel variants (RCHOLQR_ABLATION_LIB=1 loads lib/librcholqr_ablation.so built with
RCHOLQR_EXTRA_NVCC_FLAGS).  Each kernel: warm-up iterations, then `iters` timed back to back (CUDA events)."""
import argparse
import json
import os
import sys
import threading
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2210_09953_b200 as rcq  # noqa: E402
import synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C4")
ap.add_argument("--m", type=int, default=0)
ap.add_argument("--iters", type=int, default=40)
ap.add_argument("--warm", type=int, default=15)
ap.add_argument("--what", default="solve,sketch")
ap.add_argument("--tag", default="")
ap.add_argument("--sketch", default="")
a = ap.parse_args()
cfg = synth.config(a.config)
m = a.m or cfg["m"]
if a.sketch:
    cfg["sketch"] = a.sketch
X = synth.make_X_torch(m, cfg["n"], cfg["log10_cond"], cfg["dtype"])
plan = rcq.RCholQR(n=cfg["n"], k=cfg["k"], dtype=X.dtype, sketch=cfg["sketch"], nnz_per_col=cfg["nnz"])
P = plan.sketch(X)
R, _, _ = plan.small_qr(P, want_S=False)
Q = torch.empty_like(X)


class Smp:
    def __init__(self):
        import pynvml
        pynvml.nvmlInit()
        self.nv, self.h = pynvml, pynvml.nvmlDeviceGetHandleByIndex(0)
        self.clk, self.pw, self.stop = [], [], threading.Event()

    def run(self):
        while not self.stop.is_set():
            self.clk.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
            self.pw.append(self.nv.nvmlDeviceGetPowerUsage(self.h) / 1000.0)
            time.sleep(0.003)


def timed(fn):
    for _ in range(a.warm):
        fn()
    torch.cuda.synchronize()
    s = Smp()
    th = threading.Thread(target=s.run)
    th.start()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(a.iters):
        fn()
    e1.record()
    torch.cuda.synchronize()
    s.stop.set()
    th.join()
    c = sorted(s.clk)
    return {"ms": round(e0.elapsed_time(e1) / a.iters, 4), "sm_mhz_med": c[len(c) // 2] if c else None,
            "power_w_max": round(max(s.pw), 1) if s.pw else None}


out = {"tag": a.tag, "config": a.config, "m": m, "sketch": cfg["sketch"]}
for w in a.what.split(","):
    if w == "solve":
        out["solve"] = timed(lambda: plan.tri_solve(X, R, Q=Q))
    elif w == "sketch":
        out["sketch_ms"] = timed(lambda: plan.sketch(X))
        out["sketch_ms"]["path"] = plan.last_path()
    elif w == "factor":
        out["factor"] = timed(lambda: plan.factor(X, Q=Q))
    elif w == "factor_cm":                               # column-major X and Q (native kernels when applicable)
        Xt = X.t().contiguous()
        del X
        Qt = Q.view(Xt.shape)
        out["factor_cm"] = timed(lambda: plan.factor_colmajor(Xt, Qt=Qt))
        out["factor_cm"]["native"] = bool(plan.last_path() & rcq.PATH_COLMAJOR_NATIVE)
print(json.dumps(out))
