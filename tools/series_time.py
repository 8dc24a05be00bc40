"""Per-iteration device times of back-to-back sketch / solve / factor calls with NVML SM + memory clocks, power and
throttle reasons sampled alongside: shows how the sustained rate differs from an isolated launch."""
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
ap.add_argument("--iters", type=int, default=60)
ap.add_argument("--what", default="sketch")
ap.add_argument("--sleep", type=float, default=0.0, help="host sleep between iterations (isolated launches)")
a = ap.parse_args()
cfg = synth.config(a.config)
X = synth.make_X_torch(cfg["m"], cfg["n"], cfg["log10_cond"], cfg["dtype"])
plan = rcq.RCholQR(n=cfg["n"], k=cfg["k"], dtype=X.dtype, sketch=cfg["sketch"], nnz_per_col=cfg["nnz"])
P = plan.sketch(X)
R, _, _ = plan.small_qr(P, want_S=False)
Q = torch.empty_like(X)
fn = {"sketch": lambda: plan.sketch(X), "solve": lambda: plan.tri_solve(X, R, Q=Q), "factor": lambda: plan.factor(X, Q=Q)}[a.what]
import pynvml as nv  # noqa: E402
nv.nvmlInit()
h = nv.nvmlDeviceGetHandleByIndex(0)
smp, stop = [], threading.Event()


def run():
    t0 = time.time()
    while not stop.is_set():
        smp.append((round(time.time() - t0, 3), nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM),
                    nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_MEM), round(nv.nvmlDeviceGetPowerUsage(h) / 1000.0),
                    hex(nv.nvmlDeviceGetCurrentClocksEventReasons(h)), nv.nvmlDeviceGetTemperature(h, 0)))
        time.sleep(0.01)


torch.cuda.synchronize()
time.sleep(1.0)
th = threading.Thread(target=run)
th.start()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(a.iters + 1)]
ev[0].record()
for i in range(a.iters):
    fn()
    ev[i + 1].record()
    if a.sleep:
        torch.cuda.synchronize()
        time.sleep(a.sleep)
        ev[i + 1].record()
torch.cuda.synchronize()
stop.set()
th.join()
if a.sleep:
    ms = None
else:
    ms = [round(ev[i].elapsed_time(ev[i + 1]), 3) for i in range(a.iters)]
print(json.dumps({"what": a.what, "sleep": a.sleep, "ms": ms, "samples": smp[:: max(1, len(smp) // 40)]}))
