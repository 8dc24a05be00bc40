#!/usr/bin/env python
"""Benchmark: RandCholQR factor throughput (GB/s of X, rows/s) on B200 (BASELINE.json metric).

One step = one whole Algorithm 2 factorization (sketch + reduce [+ all-reduce] + Householder QR +
R^-1 + tall solve) of the workload's X, inputs resident in HBM.  The default workload is BASELINE.json
C4 (m = 2^26, n = 64, k = 128, sparse-sign Theta, fp32 X, cond 1e4), one of the metric's 1/2/4/8-GPU
configs: with N GPUs (torchrun, one process per GPU) the full C4 matrix is row-partitioned across the
ranks with one NCCL all-reduce of the 128 x 64 sketch ("strong" scaling; C3 / C5 likewise).  C1 / C2
(single-GPU configs) stay available with --config; at N > 1 they give each rank its own block ("weak").

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C4] [--impl reference]
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import synth  # noqa: E402

DMMA_PEAK_DERIVED = 37.2   # 148 SMs x 64 FP64 FMA/clk x 2 x 1.965 GHz (fallback only)
L2_BYTES = 126 * 2**20
DEFAULT_CONFIG = "C4"


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except OSError:
        return {}


def _unit_peaks():
    """Measured FP64 (DMMA) and tcgen05 kind::i8 peaks of this pool's B200s from
    profiles/peaks_r2.jsonl (tools/measure_peaks.sh: tools/micro/peaks.cu and tc_rate.cu on all SMs,
    with the SM clock sampled under load).  Falls back to the derived DMMA figure when absent."""
    out = {"dmma_tflops": DMMA_PEAK_DERIVED, "dmma_source": "derived 148 SM x 64 FMA/clk x 2 x 1.965 GHz",
           "i8_tops": None, "i8_source": None}
    try:
        rows = [json.loads(x) for x in open(os.path.join(ROOT, "profiles", "peaks_r2.jsonl")) if x.strip()]
    except OSError:
        return out
    dm = [r["tflops"] for r in rows if str(r.get("kernel", "")).startswith("dmma")]
    if dm:
        out["dmma_tflops"] = max(dm)
        out["dmma_source"] = "measured: max DMMA (mma.sync f64) rate, profiles/peaks_r2.jsonl"
    i8 = [r for r in rows if r.get("kind") == "i8" and "tops_chip" in r]
    if i8:
        best = max(i8, key=lambda r: r["tops_chip"])
        out["i8_tops"] = best["tops_chip"]
        out["i8_source"] = (f"measured: tcgen05.mma kind::i8 M=128 N={best['N']}, {best['mac_per_cyc']:.0f} MAC/clk/SM "
                            f"x 148 SM x 2 x {best['sm_mhz']} MHz, profiles/peaks_r2.jsonl")
    return out


class ClockSampler:
    """SM clocks + throttle reasons sampled with NVML during the timed region."""

    def __init__(self, dev_index: int):
        self.samples, self.reasons, self._stop = [], set(), threading.Event()
        self.max_mhz = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self._nv = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(dev_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM)
        except Exception:  # noqa: BLE001
            self._nv = None

    def _run(self):
        nv = self._nv
        names = {
            "hw_slowdown": getattr(nv, "nvmlClocksEventReasonHwSlowdown", 0x8),
            "sw_thermal_slowdown": getattr(nv, "nvmlClocksEventReasonSwThermalSlowdown", 0x20),
            "hw_thermal_slowdown": getattr(nv, "nvmlClocksEventReasonHwThermalSlowdown", 0x40),
            "sw_power_cap": getattr(nv, "nvmlClocksEventReasonSwPowerCap", 0x4),
            "hw_power_brake_slowdown": getattr(nv, "nvmlClocksEventReasonHwPowerBrakeSlowdown", 0x80),
        }
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self._h)
                for k, bit in names.items():
                    if r & bit:
                        self.reasons.add(k)
            except Exception:  # noqa: BLE001
                pass
            time.sleep(0.005)

    def __enter__(self):
        if self._nv:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self._nv:
            self._t.join()

    def summary(self):
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons), "samples": len(self.samples)}


def _dist():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def _workload(cfg_name: str, ws: int, rank: int):
    from paper_2210_09953_b200.partition import row_block, weak_block
    cfg = synth.config(cfg_name)
    if cfg_name in ("C1", "C2"):           # single-GPU configs: weak scaling, one block per rank
        ro, m_local, m_global = weak_block(cfg["m"], ws, rank)
        scaling = "weak"
    else:                                  # BASELINE multi-GPU configs: row-partition the full X
        m_global = cfg["m"]
        ro, m_local = row_block(m_global, ws, rank)
        scaling = "strong"
    return cfg, m_local, m_global, ro, scaling


def _cpu_sample_rate(X_dev, cfg, target_s: float, algo: str = "rcholqr", l: int = 0, tau: float = 0.0):
    """Time the oracle (as it stands, all host cores) on a bounded leading sample of X."""
    import oracle
    so = {"gaussian": oracle.GAUSSIAN, "sparse": oracle.SPARSE_SIGN, "rademacher": oracle.RADEMACHER,
          "srht": oracle.SRHT}[cfg["sketch"]]
    if algo == "rcholqr2":
        run = lambda A: oracle.factor2(A, cfg["k"], sketch=so, zeta=cfg["nnz"])  # noqa: E731
    elif algo == "rcholqr_rr":
        run = lambda A: oracle.factor_rr(A, cfg["k"], tau, sketch=so, zeta=cfg["nnz"])  # noqa: E731
    elif algo == "rcholqr_rr2":
        run = lambda A: oracle.factor_rr2(A, cfg["k"], tau, sketch=so, zeta=cfg["nnz"])  # noqa: E731
    elif algo == "rcholqr_reduced":
        run = lambda A: oracle.factor_reduced(A, cfg["k"], l, sketch=so, zeta=cfg["nnz"], want_S=False)  # noqa: E731
    else:
        run = lambda A: oracle.factor(A, cfg["k"], sketch=so, zeta=cfg["nnz"], want_S=False)  # noqa: E731
    m = X_dev.shape[0]
    rows = min(m, 4096)
    while True:
        Xs = X_dev[:rows].cpu().numpy()
        t0 = time.perf_counter()
        run(Xs)
        dt = time.perf_counter() - t0
        if dt >= target_s * 0.5 or rows >= m:
            return rows, dt, oracle.num_threads()
        rows = min(m, int(rows * max(2.0, 0.8 * target_s / max(dt, 1e-3))))


def _host_X(cfg: dict, rows: int):
    """The workload's X (its leading `rows` rows) on the host: generated on the GPU when one is present
    (the same bytes bench.py's own arm factors, synth.make_X_torch), else by the host generator."""
    try:
        import torch
        if torch.cuda.is_available():
            Xd = synth.make_X_torch(rows, cfg["n"], cfg["log10_cond"], cfg["dtype"], seed=synth.X_SEED)
            X = Xd.cpu().numpy()
            del Xd
            torch.cuda.empty_cache()
            return X
    except Exception:  # noqa: BLE001 - fall back to the host generator
        pass
    return synth.make_X(rows, cfg["n"], cfg["log10_cond"], cfg["dtype"])


def run_reference(args):
    """--impl reference: the CPU fp64 oracle timed as it stands (this tier's reference arm) on the host
    cores.  The sample is the WHOLE workload when the --steps/--warmup run fits the time budget
    (then the line's config equals our arm's), else the leading rows -- never fewer than
    cores x 65,536, so every OpenMP thread has one of the oracle's fixed 65,536-row blocks."""
    ws, rank, _ = _dist()
    if rank != 0:
        return 0
    import oracle
    cfg = synth.config(args.config)
    if args.sketch:
        cfg["sketch"] = args.sketch
    so = {"gaussian": oracle.GAUSSIAN, "sparse": oracle.SPARSE_SIGN, "rademacher": oracle.RADEMACHER,
          "srht": oracle.SRHT}[cfg["sketch"]]
    s_x = 8 if cfg["dtype"] == "f64" else 4
    cores = oracle.num_threads()
    m = cfg["m"]
    run = lambda A: oracle.factor(A, cfg["k"], sketch=so, zeta=cfg["nnz"], want_S=False)  # noqa: E731
    budget_s = args.ref_budget_s                       # whole warm-up + timed run
    per_step_s = budget_s / (args.steps + args.warmup)
    rows = min(m, cores * 65536)
    X = _host_X(cfg, rows)                             # leading rows of the workload's X
    t0 = time.perf_counter()
    run(X)                                             # calibration (also the first warm-up step)
    dt = time.perf_counter() - t0
    if rows < m:
        rate = rows / max(dt, 1e-6)                    # rows per second of this oracle on these cores
        want = max(rows, min(m, int(rate * per_step_s)))
        want = m if want >= 0.98 * m else want // 65536 * 65536 or want
        if want > rows:
            rows = want
            del X
            X = _host_X(cfg, rows)
    Xs = X
    for _ in range(max(0, args.warmup - 1)):
        run(Xs)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        run(Xs)
    el = time.perf_counter() - t0
    ms = el / args.steps * 1e3
    gbs = rows * cfg["n"] * s_x / (ms * 1e-3) / 1e9
    whole = rows == m
    sample = (f"the whole {args.config} X ({m} rows)" if whole else
              f"{rows} leading rows of {args.config} (m={m}; the whole X does not fit the {budget_s:.0f} s budget)") + \
        f" per step, oracle.factor (fp64 C, OpenMP over fixed 65,536-row blocks, {cores} threads)"
    line = {"metric": "RandCholQR factor throughput (GB/s of X)", "value": gbs, "unit": "GB/s",
            "impl": "reference", "n_gpus": ws, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "rows_per_s": rows / (ms * 1e-3), "higher_is_better": True, "scaling": "strong" if whole else "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": _config_dict(args.config, cfg, rows, s_x),
            "cpu_baseline": {"value": gbs, "unit": "GB/s", "cores": cores, "kind": "oracle", "sample": sample},
            "e2e": {"value": gbs, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def _path_names(rcq, bits: int) -> dict:
    """rcholqr_last_path of the timed loop's last step, decoded: which kernels served the factorization."""
    names = [("sketch_tcgen05", rcq.PATH_SKETCH_TC), ("sketch_presplit_digits", rcq.PATH_SKETCH_PRESPLIT),
             ("sketch_cuda_core_or_dmma", rcq.PATH_SKETCH_CUDA_CORE), ("sketch_overflow_fallback", rcq.PATH_SKETCH_FALLBACK),
             ("solve_tcgen05", rcq.PATH_SOLVE_TC), ("solve_dmma", rcq.PATH_SOLVE_DMMA),
             ("colnorms_fused", rcq.PATH_COLSQ_FUSED), ("colmajor_native", rcq.PATH_COLMAJOR_NATIVE),
             ("sketch_srht_fwht", rcq.PATH_SKETCH_FWHT)]
    return {"bits": bits, "kernels": [n for n, b in names if bits & b]}


def _config_dict(name: str, cfg: dict, m_global: int, s_x: int) -> dict:
    """The workload description both arms print (identical keys and values for the same workload, so
    the driver can match the reference arm's line to ours)."""
    return {"workload": name, "m": m_global, "n": cfg["n"], "k": cfg["k"], "sketch": cfg["sketch"],
            "x_dtype": cfg["dtype"], "cond": 10.0 ** cfg["log10_cond"],
            "l2": "inputs larger than L2 (per-rank X > 126 MiB), no flush" if m_global * cfg["n"] * s_x > 8 * L2_BYTES
                  else "flushed: 4 x L2 written between timed steps, each step its own device event pair"}


def _i8_macs(cfg: dict, m: int, k: int) -> float:
    """int8 MACs the pre-split tcgen05 Gaussian sketch issues for m rows (sketch_gtc.cu): X digit b (DX of
    them) times the Theta digit prefix of min(LK - b, 6) digits, over the padded tile (k up to KT rows,
    n up to 128 columns)."""
    f32 = cfg["dtype"] == "f32"
    dx, lk, kt = (6, 8, 40) if f32 else (8, 9, 48)
    pairs = sum(min(lk - b, 6) for b in range(dx))
    kpad = -(-k // kt) * kt
    npad = -(-cfg["n"] // 128) * 128
    return float(pairs) * kpad * npad * m


def run(args):
    import torch
    import torch.distributed as dist

    import paper_2210_09953_b200 as rcq

    up = _unit_peaks()
    DMMA_PEAK_TFLOPS = up["dmma_tflops"]

    ws, rank, local = _dist()
    if ws != args.gpus and "WORLD_SIZE" in os.environ:
        print(f"warning: --gpus {args.gpus} but WORLD_SIZE={ws}", file=sys.stderr)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    comm = None
    if ws > 1:
        dist.init_process_group("nccl", device_id=dev)
        obj = [rcq.comm_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        comm = rcq.comm_create(obj[0], ws, rank, local)

    cfg, m_local, m_global, ro, scaling = _workload(args.config, ws, rank)
    if args.sketch:                          # experiments: another Theta on the same workload shape
        cfg["sketch"] = args.sketch
    n, k, dt = cfg["n"], cfg["k"], cfg["dtype"]
    s_x = 8 if dt == "f64" else 4
    # each rank generates exactly its own rows of the global X (reproducible per row range)
    X = synth.make_X_torch(m_local, n, cfg["log10_cond"], dt, seed=synth.X_SEED, device=dev, row_start=ro)
    plan = rcq.RCholQR(n=n, k=k, dtype=X.dtype, sketch=cfg["sketch"], nnz_per_col=cfg["nnz"], seed=synth.THETA_SEED,
                       device=local, comm=comm)
    Q = torch.empty_like(X)
    R = torch.empty((n, n), dtype=torch.float64, device=dev)
    stream = torch.cuda.current_stream()

    Rp = torch.empty((n, n), dtype=torch.float64, device=dev)
    l_red = args.l or k                     # Alg. 5: rows of the extractor L (default: as many as Theta)
    Z = torch.empty((l_red, n), dtype=torch.float64, device=dev) if args.algo == "rcholqr_reduced" else None

    # Alg. 7: the paper's truncation tolerances (4e-15 in fp64; 2e-7 in fp32)
    tau_rr = args.tau if args.tau > 0 else (4e-15 if dt == "f64" else 2e-7)
    rr_last = {}

    # launch-bound configs (X fits in L2: C1): the chain is replayed from a CUDA graph (rcholqr_factor_graph) and
    # L2 is flushed between timed steps, each step timed by its own event pair
    small = m_local * n * s_x <= 8 * L2_BYTES
    use_graph = args.algo == "rcholqr" and ws == 1 and (args.graph == "on" or (args.graph == "auto" and small))
    flush = torch.empty(4 * L2_BYTES, dtype=torch.uint8, device=dev) if small else None

    def step():
        if args.algo == "rcholqr_rr":   # Alg. 7: synchronous (rank and swap decisions on the host)
            rr_last.update(plan.factor_rr(X, tau_rr, row_offset=ro, Q=Q, R=R, stream=stream))
        elif args.algo == "rcholqr_rr2":   # RRRCholeskyQR2: Alg. 7 + one CholeskyQR pass
            rr_last.update(plan.factor_rr2(X, tau_rr, row_offset=ro, Q=Q, stream=stream))
        elif args.algo == "rcholqr2":   # Alg. 3: synchronous (status read inside the call)
            plan.factor2(X, row_offset=ro, Q=Q, R=R, Rprime=Rp, stream=stream)
        elif args.algo == "rcholqr_reduced":   # Alg. 5: synchronous
            plan.factor_reduced(X, l_red, row_offset=ro, Z=Z, R=R, stream=stream)
        else:
            plan.factor(X, row_offset=ro, Q=Q, R=R, stream=stream, sync=False, graph=use_graph)

    def barrier():
        if ws > 1:
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        step()
    st = plan.query_status()
    if st != rcq.OK:
        raise rcq.RCholQRError(st, "warm-up factor")

    # ---- timed region (device events on the launching stream; inputs > L2, no flush needed)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        barrier()
        if small:      # per-step event pairs; a write of 4 x L2 between steps evicts X, Q and the workspaces
            evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
            for a, b in evs:
                flush.fill_(1)
                a.record(stream)
                step()
                b.record(stream)
            barrier()
            ms_local = sum(a.elapsed_time(b) for a, b in evs) / args.steps
        else:
            e0.record(stream)
            for _ in range(args.steps):
                step()
            e1.record(stream)
            barrier()
            ms_local = e0.elapsed_time(e1) / args.steps
    st = plan.query_status()
    if st != rcq.OK:
        raise rcq.RCholQRError(st, "timed factor")
    path_bits = plan.last_path()
    t = torch.tensor([ms_local], dtype=torch.float64, device=dev)
    if ws > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())

    # ---- per-kernel times (library-recorded CUDA events on the same stream), separate pass.  The plan owns ONE set
    # of events, so a measured step is followed by a synchronize; two un-synchronized steps run in front of each
    # measured one so that it sees the timed loop's steady state (back-to-back steps: clocks under the power cap,
    # L2 full of the previous step's Q) and not an idle GPU
    plan.set_timing(True)
    per = {}
    lead = 0 if small else int(os.environ.get("RCHOLQR_BENCH_LEAD_STEPS", "2"))
    for _ in range(max(3, min(args.steps, 20))):
        for _ in range(lead):
            step()
        step()
        plan.query_status()
        for kk, v in plan.last_timings().items():
            per.setdefault(kk, []).append(v)
    plan.set_timing(False)
    per_ms = {kk: statistics.median(v) for kk, v in per.items()}

    # ---- end-to-end through the public API with host buffers (H2D + D2H inside the timed region)
    e2e = None
    if not args.no_e2e and args.algo == "rcholqr":
        Xh = X.cpu().pin_memory()
        Qh = torch.empty_like(Xh).pin_memory()
        Rh = torch.empty((n, n), dtype=torch.float64).pin_memory()
        plan.factor_host(Xh, row_offset=ro, Q_host=Qh, R_host=Rh, stream=stream)
        ke = max(2, min(args.steps, 10))
        barrier()
        h0, h1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        h0.record(stream)
        for _ in range(ke):
            plan.factor_host(Xh, row_offset=ro, Q_host=Qh, R_host=Rh, stream=stream)
        h1.record(stream)
        barrier()
        te = torch.tensor([h0.elapsed_time(h1) / ke], dtype=torch.float64, device=dev)
        if ws > 1:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        e2e_ms = float(te.item())
        e2e = {"value": m_global * n * s_x / (e2e_ms * 1e-3) / 1e9, "unit": "GB/s", "ms_per_step": e2e_ms,
               "h2d_bytes_per_step": m_local * n * s_x, "d2h_bytes_per_step": m_local * n * s_x + n * n * 8}
        del Xh, Qh

    # ---- rooflines: every heavy kernel against its own bound, algorithmic
    # work per launch / its library-event time on the launching stream; "roofline" = the dominant one.
    gbs = m_global * n * s_x / (ms * 1e-3) / 1e9
    peaks = _peaks()
    hbm = peaks.get("hbm_gbs", 6545.0)
    roofs = {}
    reduced = args.algo == "rcholqr_reduced"
    rr = args.algo in ("rcholqr_rr", "rcholqr_rr2")
    r_rr = rr_last.get("rank", n)
    k_sk = k + l_red if reduced else k      # Alg. 5 with a Gaussian Theta: one (k + l)-row sketch
    if cfg["sketch"] == "gaussian":
        # exact int8 digit-product sketch (sketch_gtc.cu); its algorithmic work is the method's 2kmn
        # fp64 flops, so it is measured against the FP64 tensor (DMMA) peak it replaces.
        flops = 2.0 * k_sk * m_local * n
        ach = flops / (per_ms["sketch"] * 1e-3) / 1e12
        roofs["sketch"] = {"kernel": "xdig_split_kernel + sketch_gauss_tcp_kernel", "bound": "tensor",
                           "achieved": ach, "peak": DMMA_PEAK_TFLOPS, "unit": "TFLOP/s", "frac": ach / DMMA_PEAK_TFLOPS,
                           "peak_source": up["dmma_source"] + ": fp64-equivalent view of the exact int8 digit emulation",
                           "algorithmic": f"2*{'(k+l)' if reduced else 'k'}*m*n = {flops:.4g} flop per launch",
                           "traffic": None}
        if flops < 2e7:      # launch-bound sizes (C1) run the single DMMA kernel (sketch.cu, gauss_tc_min_work)
            roofs["sketch"]["kernel"] = "sketch_gauss_kernel"
            roofs["sketch"]["peak_source"] = up["dmma_source"]
        elif up["i8_tops"]:    # the unit that actually does the work: executed int8 MACs vs the tcgen05 i8 rate
            i8 = 2.0 * _i8_macs(cfg, m_local, k_sk) / (per_ms["sketch"] * 1e-3) / 1e12
            roofs["sketch"]["int8_view"] = {"achieved": i8, "peak": up["i8_tops"], "unit": "TOP/s",
                                            "frac": i8 / up["i8_tops"], "peak_source": up["i8_source"],
                                            "executed": "2 x int8 MACs issued incl. tile padding (sketch_gtc.cu)"}
    elif reduced:
        # sparse Theta: P by the sparse tcgen05 sketch (one HBM pass), then Y = L X by the Gaussian
        # one; the Gaussian extract's 2 l m n fp64-equivalent flops dominate both passes' time
        flops = 2.0 * l_red * m_local * n
        ach = flops / (per_ms["sketch"] * 1e-3) / 1e12
        roofs["sketch"] = {"kernel": "xdig_split_kernel + sketch_gauss_tcp_kernel", "bound": "tensor", "achieved": ach,
                           "peak": DMMA_PEAK_TFLOPS, "unit": "TFLOP/s", "frac": ach / DMMA_PEAK_TFLOPS,
                           "peak_source": up["dmma_source"] + " (fp64-equivalent view of the exact int8 digits)",
                           "algorithmic": f"2*l*m*n = {flops:.4g} flop (Gaussian extract; the time includes "
                                          "the sparse sketch pass)", "traffic": None}
    elif cfg["sketch"] == "srht" and k > 128:
        # blocked fast Walsh-Hadamard transform (srht_fwht.cu): one read of X, 10 + k/1024 fp64 adds per element
        byts = m_local * n * s_x
        ach = byts / (per_ms["sketch"] * 1e-3) / 1e9
        roofs["sketch"] = {"kernel": "srht_fwht_kernel", "bound": "hbm", "achieved": ach, "peak": hbm,
                           "unit": "GB/s", "frac": ach / hbm, "peak_source": "MEASURED_PEAKS.json hbm_gbs",
                           "algorithmic": f"m*n*s_x = {byts:.4g} B per launch (one read of X)", "traffic": None}
    elif cfg["sketch"] in ("rademacher", "srht") and n > 64:
        flops = 2.0 * k * m_local * n
        ach = flops / (per_ms["sketch"] * 1e-3) / 1e12
        roofs["sketch"] = {"kernel": f"sketch_gauss_kernel ({cfg['sketch']} draws)", "bound": "tensor", "achieved": ach,
                           "peak": DMMA_PEAK_TFLOPS, "unit": "TFLOP/s", "frac": ach / DMMA_PEAK_TFLOPS,
                           "peak_source": up["dmma_source"], "algorithmic": f"2*k*m*n = {flops:.4g} flop",
                           "traffic": None}
    else:   # sparse-sign, or Rademacher on the dense-E tcgen05 kernel: one read of X per Theta tile
        byts = m_local * n * s_x
        ach = byts / (per_ms["sketch"] * 1e-3) / 1e9
        roofs["sketch"] = {"kernel": "sketch_sparse_tc_kernel", "bound": "hbm", "achieved": ach, "peak": hbm,
                           "unit": "GB/s", "frac": ach / hbm, "peak_source": "MEASURED_PEAKS.json hbm_gbs",
                           "algorithmic": f"m*n*s_x = {byts:.4g} B per launch (one read of X)", "traffic": None}
    if reduced:
        pass                                 # step 3 is the tiny l x n substitution (rowsub_kernel)
    elif rr:
        # Alg. 7: column norms (one read of X), gather of the r kept columns, solve with r columns
        byts = m_local * n * s_x
        if plan.last_path() & rcq.PATH_COLSQ_FUSED:
            # D came out of the sketch's own pass over X: no separate kernel, nothing to rate
            roofs["colnorms"] = {"kernel": "fused into the sketch pass (RCHOLQR_PATH_COLSQ_FUSED)", "bound": "hbm",
                                 "achieved": None, "peak": hbm, "unit": "GB/s", "frac": None,
                                 "algorithmic": "0 B (no second read of X)", "traffic": None}
        else:
            ach = byts / (max(per_ms["reduce"], 1e-6) * 1e-3) / 1e9
            roofs["colnorms"] = {"kernel": "colsq_kernel", "bound": "hbm", "achieved": ach, "peak": hbm, "unit": "GB/s",
                                 "frac": ach / hbm, "peak_source": "MEASURED_PEAKS.json hbm_gbs",
                                 "algorithmic": f"m*n*s_x = {byts:.4g} B (one read of X)", "traffic": None}
        byts = 2.0 * m_local * r_rr * s_x
        ach = byts / (per_ms["tri_prep"] * 1e-3) / 1e9
        roofs["gather"] = {"kernel": "gather_x_kernel", "bound": "hbm", "achieved": ach, "peak": hbm, "unit": "GB/s",
                           "frac": ach / hbm, "peak_source": "MEASURED_PEAKS.json hbm_gbs",
                           "algorithmic": f"2*m*r*s_x = {byts:.4g} B (read r columns, write them packed)",
                           "traffic": None}
        if dt == "f32" and r_rr <= 128 and not os.environ.get("RCHOLQR_SOLVE_DMMA"):
            byts = 2.0 * m_local * r_rr * s_x
            ach = byts / (per_ms["solve"] * 1e-3) / 1e9
            roofs["solve"] = {"kernel": "solve_tc_kernel, r columns", "bound": "hbm", "achieved": ach, "peak": hbm,
                              "unit": "GB/s", "frac": ach / hbm, "peak_source": "MEASURED_PEAKS.json hbm_gbs",
                              "algorithmic": f"2*m*r*s_x = {byts:.4g} B (read the packed columns, write Q)",
                              "traffic": None}
        else:
            flops = float(m_local) * r_rr * r_rr
            ach = flops / (per_ms["solve"] * 1e-3) / 1e12
            roofs["solve"] = {"kernel": "blocked substitution (fp64 DMMA), r columns", "bound": "tensor",
                              "achieved": ach, "peak": DMMA_PEAK_TFLOPS, "unit": "TFLOP/s",
                              "frac": ach / DMMA_PEAK_TFLOPS, "peak_source": up["dmma_source"],
                              "algorithmic": f"m*r^2 = {flops:.4g} flop", "traffic": None}
        per_ms = {"sketch": per_ms["sketch"], "colnorms": per_ms["reduce"], "allreduce": per_ms["allreduce"],
                  "rrqr": per_ms["small_qr"], "gather": per_ms["tri_prep"], "solve": per_ms["solve"]}
    elif dt == "f32" and n <= 128 and not os.environ.get("RCHOLQR_SOLVE_DMMA"):   # tcgen05 digit solve
        byts = 2.0 * m_local * n * s_x
        ach = byts / (per_ms["solve"] * 1e-3) / 1e9
        roofs["solve"] = {"kernel": "solve_tc_kernel", "bound": "hbm", "achieved": ach, "peak": hbm, "unit": "GB/s",
                          "frac": ach / hbm, "peak_source": "MEASURED_PEAKS.json hbm_gbs",
                          "algorithmic": f"2*m*n*s_x = {byts:.4g} B per launch (read X, write Q)", "traffic": None}
    else:
        flops = float(m_local) * n * n
        ach = flops / (per_ms["solve"] * 1e-3) / 1e12
        roofs["solve"] = {"kernel": "blocked substitution (fp64 DMMA)", "bound": "tensor", "achieved": ach,
                          "peak": DMMA_PEAK_TFLOPS, "unit": "TFLOP/s", "frac": ach / DMMA_PEAK_TFLOPS,
                          "peak_source": up["dmma_source"], "algorithmic": f"m*n^2 = {flops:.4g} flop per solve",
                          "traffic": None}
    try:   # DRAM bytes per launch from one `ncu --set full` capture of the same workload (tools/ncu_traffic.py)
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            tr = json.load(f).get(args.config) or {}
    except OSError:
        tr = {}
    try:   # issue / SM / tensor-pipe utilisation of the same capture (the kernels' native bound, e.g. the
        #   Gaussian sketch's instruction issue behind its fp64-equivalent tensor view)
        with open(os.path.join(ROOT, "profiles", "issue.json")) as f:
            iss = json.load(f).get(args.config) or {}
    except OSError:
        iss = {}
    for r_ in roofs.values():
        names = [x.strip() for x in r_["kernel"].split("+")]
        if ws == 1 and any(x in iss for x in names):
            r_["ncu_utilisation"] = {x: iss[x] for x in names if x in iss}
        tb = sum(tr[x] for x in names) if all(x in tr for x in names) else None
        if tb is not None and ws == 1:
            r_["traffic"] = tb
            r_["traffic_source"] = "ncu --set full: dram__bytes_read.sum + dram__bytes_write.sum per launch"
    dom = max(roofs, key=lambda kk: per_ms.get(kk, 0.0))
    roof = dict(roofs[dom])
    roof["share_of_step"] = per_ms.get(dom, 0.0) / ms
    # north-star roofline for the whole factorization
    t_hbm = 3.0 * m_local * n * s_x / (hbm * 1e9)
    t_flop = m_local * n * n / (DMMA_PEAK_TFLOPS * 1e12)
    ns = {"t_hbm_ms": t_hbm * 1e3, "t_solve_fp64_ms": t_flop * 1e3, "roofline_ms": max(t_hbm, t_flop) * 1e3,
          "frac": max(t_hbm, t_flop) * 1e3 / ms,
          "sketch_inclusive_roofline_ms": max(t_hbm, (m_local * n * n + 2.0 * k * m_local * n) /
                                               (DMMA_PEAK_TFLOPS * 1e12)) * 1e3}

    line = {"metric": "RandCholQR factor throughput (GB/s of X)", "value": gbs, "unit": "GB/s",
            "rows_per_s": m_global / (ms * 1e-3), "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms, "higher_is_better": True, "scaling": scaling, "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": _config_dict(args.config, cfg, m_global, s_x),
            "partition": {"m_local": m_local, "row_offset": ro, "parallelism": f"row-partition x{ws}, 1 all-reduce"},
            "per_kernel_ms": per_ms, "roofline": roof, "kernel_rooflines": roofs, "northstar_roofline": ns,
            "gpu_launches": plan.launches_per_factor(m_local) * args.steps,
            "clocks": clk.summary(), "e2e": e2e, "cuda_graph": use_graph, "path": _path_names(rcq, path_bits)}

    if args.algo == "rcholqr2":
        # split Alg. 3's own steps by differences of device-timed calls on the same stream:
        # factor (Alg. 2) | factor2(implicit) (+ Gram, Cholesky, R'R1) | factor2 (+ the second solve)
        def _avg(fn, reps):
            fn()
            torch.cuda.synchronize()
            a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a0.record(stream)
            for _ in range(reps):
                fn()
            a1.record(stream)
            torch.cuda.synchronize()
            return a0.elapsed_time(a1) / reps
        reps = max(3, min(args.steps, 10))
        t2 = _avg(lambda: plan.factor(X, row_offset=ro, Q=Q, R=R, stream=stream), reps)
        ti = _avg(lambda: plan.factor2(X, row_offset=ro, Q=Q, R=R, Rprime=Rp, implicit=True, stream=stream), reps)
        te = _avg(lambda: plan.factor2(X, row_offset=ro, Q=Q, R=R, Rprime=Rp, stream=stream), reps)
        per_ms.update({"gram_cholesky": ti - t2, "second_solve": te - ti})
        line["per_kernel_ms"] = per_ms
        flops = float(m_local) * n * (n + 1)          # upper triangle of Q1^T Q1 (incl. the diagonal)
        ach = flops / ((ti - t2) * 1e-3) / 1e12
        roofs["gram"] = {"kernel": ("gram_small_kernel" if n <= 128 else "gram_kernel") +
                                   " + sketch_reduce_kernel + cholesky_kernel", "bound": "tensor",
                         "achieved": ach, "peak": DMMA_PEAK_TFLOPS, "unit": "TFLOP/s", "frac": ach / DMMA_PEAK_TFLOPS,
                         "peak_source": up["dmma_source"],
                         "algorithmic": f"m*n*(n+1) = {flops:.4g} flop (time: factor2(implicit) - factor)",
                         "traffic": None}
        dom = max(roofs, key=lambda kk: {"gram": ti - t2}.get(kk, per_ms.get(kk, 0.0)))
        roof = dict(roofs[dom])
        roof["share_of_step"] = (ti - t2 if dom == "gram" else per_ms.get(dom, 0.0)) / ms
        line["roofline"] = roof
        line["kernel_rooflines"] = roofs
        # Alg. 3 = Alg. 2 + Gram (reads Q1) + Cholesky + second solve (reads Q1, writes Q): 6 passes
        # over an m x n matrix and 2 m n^2 (solves) + m n^2 (Gram, both triangles) fp64 flops
        t_hbm2 = 6.0 * m_local * n * s_x / (hbm * 1e9)
        t_flop2 = 3.0 * m_local * n * n / (DMMA_PEAK_TFLOPS * 1e12)
        line["metric"] = "RandCholQR2 factor throughput (GB/s of X)"
        line["config"]["algo"] = "rcholqr2 (Alg. 3, explicit Q)"
        line["northstar_roofline"] = {"t_hbm_ms": t_hbm2 * 1e3, "t_fp64_ms": t_flop2 * 1e3,
                                      "roofline_ms": max(t_hbm2, t_flop2) * 1e3,
                                      "frac": max(t_hbm2, t_flop2) * 1e3 / ms,
                                      "note": "Alg. 3 accounting: 6 passes over m x n, 3 m n^2 fp64 flops"}
        line["gpu_launches"] = (plan.launches_per_factor(m_local) + 4 + 2) * args.steps
        line["e2e"] = None   # the host-buffer entry point is Alg. 2's
    if reduced:
        # Alg. 5 reads X once: max(one pass at HBM, the (k + l)-row sketch's 2 (k + l) m n fp64 flops)
        t_hbm5 = 1.0 * m_local * n * s_x / (hbm * 1e9)
        t_flop5 = 2.0 * (k_sk if cfg["sketch"] == "gaussian" else l_red) * m_local * n / (DMMA_PEAK_TFLOPS * 1e12)
        if cfg["sketch"] != "gaussian":
            t_hbm5 *= 2.0            # sparse Theta: P and Y are two passes over X
        line["metric"] = "Reduced RandCholQR throughput (GB/s of X)"
        line["config"]["algo"] = f"rcholqr_reduced (Alg. 5, Gaussian extractor l = {l_red})"
        line["config"]["l"] = l_red
        line["northstar_roofline"] = {"t_hbm_ms": t_hbm5 * 1e3, "t_fp64_ms": t_flop5 * 1e3,
                                      "roofline_ms": max(t_hbm5, t_flop5) * 1e3,
                                      "frac": max(t_hbm5, t_flop5) * 1e3 / ms,
                                      "note": "Alg. 5 accounting: 1 pass over X, 2 (k+l) m n fp64-equivalent flops"}
        # Alg. 2's launches minus its solve (prep + solve) plus the Z substitution
        line["gpu_launches"] = (plan.launches_per_factor(m_local) - 1) * args.steps
        line["e2e"] = None
    if rr:
        # Alg. 7 passes: sketch + column norms (2 reads of X), gather (r/n read + write), solve (r/n read + write);
        # RRRCholeskyQR2 adds the Gram (r/n read) and a second solve (r/n read + write) and 2 m r^2 flops
        two = args.algo == "rcholqr_rr2"
        t_hbm7 = (2.0 + (7.0 if two else 4.0) * r_rr / n) * m_local * n * s_x / (hbm * 1e9)
        t_flop7 = (3.0 if two else 1.0) * float(m_local) * r_rr * r_rr / (DMMA_PEAK_TFLOPS * 1e12)
        line["metric"] = ("RRRCholQR2" if two else "RRRCholQR") + " factor throughput (GB/s of X)"
        line["config"]["algo"] = f"{args.algo} ({'PAPER.md:397' if two else 'Alg. 7'}, tau = {tau_rr:g}, f = 1.5)"
        line["config"]["rank"] = r_rr
        line["config"]["swaps"] = rr_last.get("swaps")
        line["northstar_roofline"] = {"t_hbm_ms": t_hbm7 * 1e3, "t_fp64_ms": t_flop7 * 1e3,
                                      "roofline_ms": max(t_hbm7, t_flop7) * 1e3,
                                      "frac": max(t_hbm7, t_flop7) * 1e3 / ms,
                                      "note": "Alg. 7 accounting: (2 + 4 r/n) passes over m x n, m r^2 fp64 flops"
                                              + ("; RRRCholeskyQR2: + 3 r/n passes, + 2 m r^2 flops" if two else "")}
        # sketch launches + colsq (2) + normalize + qrcp + gather + QR + rank + strong + finalize + gather_x
        # + check_diag + solve
        line["gpu_launches"] = (plan.launches_per_factor(m_local) + 10) * args.steps
        line["e2e"] = None
    if rank == 0 and not args.no_cpu_baseline:   # rank 0's host cores (the other ranks wait below)
        rows, dt_s, cores = _cpu_sample_rate(X, cfg, args.cpu_seconds, args.algo, l_red, tau_rr)
        fn = {"rcholqr2": "factor2", "rcholqr_reduced": "factor_reduced", "rcholqr_rr": "factor_rr",
              "rcholqr_rr2": "factor_rr2"}.get(args.algo,
                                                                                                       "factor")
        line["cpu_baseline"] = {"value": rows * n * s_x / dt_s / 1e9, "unit": "GB/s", "cores": cores,
                                "kind": "oracle", "seconds": dt_s,
                                "sample": f"oracle.{fn} on the leading {rows} rows of rank 0's block of the same X "
                                          f"(measured after the timed region)"}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if ws > 1:
        dist.barrier()
    plan.close()
    if comm is not None:
        rcq.comm_destroy(comm)
    if ws > 1:
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default=DEFAULT_CONFIG, choices=sorted(synth.CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--graph", default="auto", choices=["auto", "on", "off"],
                    help="Alg. 2 through rcholqr_factor_graph (auto: configs whose X fits in L2, i.e. C1)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--ref-budget-s", type=float, default=240.0,
                    help="--impl reference: wall-clock budget of the whole warm-up + timed oracle run")
    ap.add_argument("--algo", default="rcholqr",
                    choices=["rcholqr", "rcholqr2", "rcholqr_reduced", "rcholqr_rr", "rcholqr_rr2"],
                    help="Alg. 2 (default, the north star), Alg. 3 RCholeskyQR2 (orthonormal Q) or Alg. 5 "
                         "reduced RCholeskyQR (Z = L Q)")
    ap.add_argument("--l", type=int, default=0, help="Alg. 5: rows of the extractor L (default k)")
    ap.add_argument("--sketch", default="", choices=["", "gaussian", "sparse", "rademacher", "srht"],
                    help="override the config's Theta (the BASELINE metric is quoted on the config's own)")
    ap.add_argument("--tau", type=float, default=0.0,
                    help="Alg. 7: truncation tolerance (default: the paper's 4e-15 fp64 / 2e-7 fp32)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        return run_reference(args)
    return run(args)


if __name__ == "__main__":
    sys.exit(main())
