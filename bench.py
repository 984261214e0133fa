"""Benchmark of the B200 mixed-precision Paterson-Stockmeyer hot path.

Default workload (BASELINE.json configs[1], the metric's single-GPU
config): Taylor approximant of exp, m=30, s=6, a batch of 64 real matrices
n=256, X ~ N(0,1) rescaled to ||X||_1 = 1 (seeded), double-double working
precision with the planner's lower-precision levels.  One step = one
mixed-precision PS evaluation of the whole batch (powers, blocks + norms,
host planner, mixed Horner) through the public API.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Multi-GPU (torchrun): every rank evaluates its own 64-matrix batch (batch
sharding, no data-path collective) -> weak scaling; the JSON line reports
the whole-job evals/s with the max-over-ranks device time.

``--impl reference`` times the reference algorithm's CPU implementation
(the oracle port in oracle/, a C restatement of the reference's MPFR
arithmetic; the reference itself is pure Python over gmpy2, absent from this
image) on the host cores, on one matrix of the same workload per step.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    "cfg1": dict(workload="cfg1: Taylor exp m=16 s=4, one n=32 matrix, ||X||_1=0.5, fp64 working (fp32 levels)",
                 batch=1, n=32, m=16, digits=15, norm=0.5, kind="exp"),
    "cfg2": dict(workload="cfg2: Taylor exp m=30 s=6, batch 64 x n=256, ||X||_1=1, dd working (mixed dd/fp64/fp32 levels)",
                 batch=64, n=256, m=30, digits=31, norm=1.0, kind="exp"),
    "cfg3": dict(workload="cfg3: scaling-and-squaring exp, PS Taylor m=42 s=7 + l=extra_squarings dd squarings, "
                          "batch 16 x n=1024, ||A||_1 log-uniform [1e-2,1e3], dd working",
                 batch=16, n=1024, m=42, digits=31, norm=None, kind="expm"),
    "cfg4": dict(workload="cfg4: Pade [26/26] numerator+denominator by mixed PS at qd, one n=2048 matrix, ||X||_1=2",
                 batch=1, n=2048, m=26, digits=63, norm=2.0, kind="pade"),
    "cfg5": dict(workload="cfg5: cos Taylor deg 24 in Z=X^2 (s=5), one n=8192 matrix, ||X||_1=1 (X~N(0,1)/sqrt(n)), "
                          "dd working, 2-D block SUMMA over NCCL",
                 batch=1, n=8192, m=24, digits=31, norm=1.0, kind="summa_cos"),
}
CFG = dict(CONFIGS["cfg2"])
METRIC = "matrix-polynomial evals/sec"


def synth(n, target, seed):
    G = np.random.default_rng(seed).standard_normal((n, n))
    return G * (target / np.abs(G).sum(axis=0).max())


def make_batch(rank, batch, n, norm):
    return np.stack([synth(n, norm, rank * batch + i) for i in range(batch)])


# ----------------------------------------------------------------- clocks
class ClockSampler:
    """SM clocks and clock-event (throttle) reasons sampled DURING the timed
    region: an NVML polling thread (~0.5 ms period, so even a few-ms region
    gets many samples); nvidia-smi -lms 200 when NVML is unavailable."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    NAMES = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []
        self.nvml = None
        self.samples = []
        self.running = False

    def start(self):
        try:
            import pynvml as nv
            nv.nvmlInit()
            self.nvml = nv
            self.hdl = nv.nvmlDeviceGetHandleByIndex(self.index)
            self.smax = float(nv.nvmlDeviceGetMaxClockInfo(self.hdl, nv.NVML_CLOCK_SM))
            get = getattr(nv, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
                nv.nvmlDeviceGetCurrentClocksThrottleReasons
            self.bits = (nv.nvmlClocksThrottleReasonHwSlowdown, nv.nvmlClocksThrottleReasonHwThermalSlowdown,
                         nv.nvmlClocksThrottleReasonSwThermalSlowdown, nv.nvmlClocksThrottleReasonSwPowerCap)
            self.running = True

            def poll():
                while self.running:
                    try:
                        self.samples.append((float(nv.nvmlDeviceGetClockInfo(self.hdl, nv.NVML_CLOCK_SM)),
                                             int(get(self.hdl))))
                    except Exception:
                        pass
                    time.sleep(0.0005)
            self.thread = threading.Thread(target=poll, daemon=True)
            self.thread.start()
            return
        except Exception:
            self.nvml = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.nvml is not None:
            self.running = False
            self.thread.join(timeout=2)
            sm = [c for c, _ in self.samples]
            reasons = {nm for _, r in self.samples for nm, bit in zip(self.NAMES, self.bits) if r & bit}
            return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": self.smax,
                    "reasons": sorted(reasons), "samples": len(sm), "source": "nvml"}
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, smax, reasons = [], None, set()
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                smax = float(parts[1])
            except ValueError:
                continue
            for nm, v in zip(self.NAMES, parts[4:8]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm), "source": "nvidia-smi"}


# ------------------------------------------------------------- peaks
def measure_peaks(torch, h):
    """FP64 / FP32 FMA pipe peaks on this GPU (2 flops per FMA): the
    per-precision roofline denominators (MEASURED_PEAKS.json has only HBM and
    bf16).  Peak_dd / Peak_qd follow SURVEY 8(d): Peak_fp64 / k with
    k_dd = 15 and k_qd = 115 FP64-pipe instructions per canonical MAC."""
    out = {}
    scratch = torch.zeros(16, dtype=torch.float64, device="cuda")
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    for fmt, name, iters in ((15, "fp64", 4096), (7, "fp32", 16384)):
        blocks = sms * 8
        h.probe_fma(fmt, blocks, 64, scratch)  # warm
        best = 0.0
        for _ in range(3):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            h.probe_fma(fmt, blocks, iters, scratch)
            b.record()
            torch.cuda.synchronize()
            sec = a.elapsed_time(b) * 1e-3
            best = max(best, blocks * 256 * 16.0 * iters / sec)
        out[name] = best / 1e12
    out["dd"] = out["fp64"] / 15.0
    out["qd"] = out["fp64"] / 115.0
    # INT8 tensor pipe (tcgen05 kind::i8), the bound of the tensor-core GEMMs
    iters = 4096
    h.probe_i8mma(sms, 64, scratch)
    best = 0.0
    for _ in range(3):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        h.probe_i8mma(sms, iters, scratch)
        b.record()
        torch.cuda.synchronize()
        best = max(best, sms * 2.0 * 128 * 256 * 32 * iters / (a.elapsed_time(b) * 1e-3))
    out["int8_tops"] = best / 1e12
    # global -> shared ingest (TMA bulk copies, one CTA per SM, L2-resident
    # 48 MiB source): the per-SM fill rate that bounds the tensor-core GEMMs
    src = torch.zeros(48 << 20, dtype=torch.uint8, device="cuda")
    iters = 2048
    h.probe_ingest(sms, 64, src)
    best = 0.0
    for _ in range(3):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        h.probe_ingest(sms, iters, src)
        b.record()
        torch.cuda.synchronize()
        best = max(best, sms * iters * 16384.0 / (a.elapsed_time(b) * 1e-3))
    out["ingest_tbps"] = best / 1e12
    return out


def honest_gemms(plan):
    """GEMMs the device executes per evaluation, by lattice format: s-1
    powers at the working format + one per Horner level, except the K3 top
    level when m mod s == 0 (B_r = b_m I -> elementwise)."""
    from paper_2312_17396_b200.precision import FORMAT_NAME
    fm = plan.level_formats
    counts = {}
    w = FORMAT_NAME[fm[0]]
    counts[w] = counts.get(w, 0) + plan.s - 1
    top_scalar = (CFG["m"] % plan.s == 0)
    for j in range(1, plan.r + 1):
        if j == plan.r and top_scalar:
            continue
        f = FORMAT_NAME[fm[j]]
        counts[f] = counts.get(f, 0) + 1
    return counts


# ---------------------------------------------------------- reference
def run_reference(args, rank, world):
    """The reference algorithm's CPU path (oracle port) on host cores."""
    if rank != 0:
        return
    import oracle
    from paper_2312_17396_b200.coefficients import taylor_exp_coeffs
    oracle.build()
    cores = os.cpu_count() or 1
    os.environ.setdefault("OMP_NUM_THREADS", str(cores))
    n, m, d = CFG["n"], CFG["m"], CFG["digits"]
    coeffs = taylor_exp_coeffs(m).coeffs
    X = [synth(n, CFG["norm"], i) for i in range(args.warmup + args.steps)]
    for i in range(args.warmup):
        oracle.ps_eval(X[i], coeffs, d)
    t0 = time.perf_counter()
    for i in range(args.steps):
        oracle.ps_eval(X[args.warmup + i], coeffs, d)
    sec = time.perf_counter() - t0
    v = args.steps / sec
    line = {"metric": METRIC, "value": v, "unit": "evals/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * sec / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "mpfr-103bit (per-op rounded, reference semantics)",
            "data": "synthetic (seeded N(0,1), ||X||_1=1)", "impl": "reference",
            "config": {"workload": CFG["workload"], "batch": CFG["batch"], "n": n, "m": m, "digits": d},
            "cpu_baseline": {"value": v, "unit": "evals/s", "cores": cores, "kind": "port",
                             "sample": f"1 matrix (n={n}) of the 64-matrix batch per step, full mixed PS "
                                       "evaluation in the C MPFR restatement (oracle/mpfr_oracle.c), "
                                       "OpenMP over GEMM rows"},
            "e2e": {"value": v, "unit": "evals/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def pcie_rates(torch, h2d_bytes: int, d2h_bytes: int, reps: int = 5):
    """Plain pinned-host <-> device copy rates of one step's input / result
    sizes in this process (the ceiling of the e2e stream; the host memory
    placement of a VM makes it differ between processes)."""
    try:
        hb = torch.empty(max(h2d_bytes, d2h_bytes) // 8, dtype=torch.float64).pin_memory()
        db = torch.empty_like(hb, device="cuda")
        out = {}
        for name, nbytes, dst, src in (("h2d", h2d_bytes, db, hb), ("d2h", d2h_bytes, hb, db)):
            k = nbytes // 8
            dst[:k].copy_(src[:k], non_blocking=True)
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(reps):
                dst[:k].copy_(src[:k], non_blocking=True)
            b.record()
            b.synchronize()
            out[name] = reps * nbytes / (a.elapsed_time(b) * 1e-3) / 1e9
        return out
    except Exception as e:  # diagnostics only
        return {"error": str(e)[:120]}


def cpu_baseline_sample(cores_hint=None):
    if _ORIG_AFFINITY:      # the CPU baseline uses every host core, not the GPU-local ones
        os.sched_setaffinity(0, _ORIG_AFFINITY)
    import oracle
    from paper_2312_17396_b200.coefficients import taylor_exp_coeffs
    oracle.build()
    n, m, d = CFG["n"], CFG["m"], CFG["digits"]
    X = synth(n, CFG["norm"], 0)
    t0 = time.perf_counter()
    oracle.ps_eval(X, taylor_exp_coeffs(m).coeffs, d)
    sec = time.perf_counter() - t0
    return {"value": 1.0 / sec, "unit": "evals/s", "cores": os.cpu_count() or 1, "kind": "port",
            "sample": f"1 matrix (n={n}, seed 0) of the cfg2 batch, full mixed PS in the C MPFR "
                      f"restatement of the reference (oracle/), OpenMP over GEMM rows, {sec:.1f} s"}


# ---------------------------------------------------------------- ours
class Workload:
    """One benchmark config: device-resident inputs, a step through the
    public API, an end-to-end step from pinned host buffers, and the honest
    GEMM count per unit."""

    def __init__(self, name, rank, world, torch, mp):
        self.name, self.cfg = name, CONFIGS[name]
        self.rank, self.world, self.torch, self.mp = rank, world, torch, mp
        c = self.cfg
        self.ctx = mp.PrecisionCtx(c["digits"])
        self.n, self.B, self.m = c["n"], c["batch"], c["m"]
        self.kind = c["kind"]
        self.scaling = "strong" if self.kind == "summa_cos" else "weak"
        self.grid = None
        if self.kind == "expm":
            rng = np.random.default_rng(1000 + rank)
            targets = 10.0 ** rng.uniform(-2, 3, size=self.B)
            self.Xh = np.stack([synth(self.n, t, rank * self.B + i) for i, t in enumerate(targets)])
        elif self.kind == "summa_cos":
            from paper_2312_17396_b200 import summa
            pr, pc = summa.ProcessGrid.for_world(world)
            self.grid = summa.ProcessGrid(pr, pc) if world > 1 else None
            X = np.random.default_rng(0).standard_normal((self.n, self.n)) / np.sqrt(self.n)
            X *= c["norm"] / np.abs(X).sum(axis=0).max()
            if self.grid is None:
                self.Xh = X
            else:
                r0, mr, c0, nc = self.grid.block(self.n)
                self.Xh = np.ascontiguousarray(X[r0:r0 + mr, c0:c0 + nc])
            self.parallelism = f"SUMMA {pr}x{pc}"
        else:
            self.Xh = make_batch(rank, self.B, self.n, c["norm"])
            if self.B == 1:
                self.Xh = self.Xh[0]
        if self.kind != "summa_cos":
            self.parallelism = f"batch-sharded x{world}" if world > 1 else "single GPU"
        self.Xd = torch.from_numpy(self.Xh).cuda()
        self.Xpin = torch.from_numpy(self.Xh).pin_memory()

    def _summa(self, X):
        from paper_2312_17396_b200 import summa
        from paper_2312_17396_b200.precision import MatBatch
        torch = self.torch
        grid = self.grid
        if grid is None:
            grid = summa.ProcessGrid.__new__(summa.ProcessGrid)
            grid.pr = grid.pc = 1
            grid.rank = grid.I = grid.J = 0
            grid.row_group = grid.col_group = None
        if X.device.type == "cpu":
            X = X.to("cuda", non_blocking=True)
        blk = MatBatch(X.reshape(1, 1, *X.shape), 15)
        ops = summa.DeviceOps()
        Z = summa.cos_argument_dist(blk, self.ctx, grid, ops)
        return summa.ps_mixed_dist(Z, self.mp.taylor_cos_coeffs(self.m), self.ctx, grid, ops)

    def step(self, X):
        mp, ctx, m = self.mp, self.ctx, self.m
        if self.kind == "exp":
            return mp.ps_mixed_exp(X, m, ctx, timing=False)
        if self.kind == "expm":
            return mp.expm_ss(X, ctx, m, timing=False)
        if self.kind == "pade":
            return mp.ps_mixed_pade(X, m, ctx, timing=False)
        return self._summa(X)

    def results(self, rep):
        """Device tensors holding the step's result(s)."""
        if self.kind == "pade":
            return [r.result.data for r in rep]
        if self.kind == "summa_cos":
            return [rep.block.data]
        return [rep.result.data]

    def plans(self, rep):
        if self.kind == "pade":
            return [rep[0].plan, rep[1].plan]
        if self.kind == "summa_cos":
            return [rep.plan(self.ctx)]
        if hasattr(rep, "plan"):
            return [rep.plan]
        return [rep[0].plan]

    def formats(self, rep):
        if self.kind == "summa_cos":
            from paper_2312_17396_b200.precision import FORMAT_NAME
            return [FORMAT_NAME[f] for f in self.plans(rep)[0].level_formats]
        r0 = rep[0] if self.kind == "pade" or not hasattr(rep, "diagnostics") else rep
        return r0.diagnostics["level_formats"]

    def gemms(self, rep):
        """Honest device GEMMs per step, by format (whole local step)."""
        from paper_2312_17396_b200.precision import FORMAT_NAME
        counts = {}

        def add(f, c):
            counts[f] = counts.get(f, 0) + c

        plans = self.plans(rep)
        for i, p in enumerate(plans):
            fm = p.level_formats
            if not (self.kind == "pade" and i > 0):
                add(FORMAT_NAME[fm[0]], p.s - 1)           # powers (shared by the Pade pair)
            for j in range(1, p.r + 1):
                if j == p.r and self.m % p.s == 0:
                    continue                                # K3: elementwise
                add(FORMAT_NAME[fm[j]], 1)
        mult = self.B if self.kind in ("exp", "expm") else 1
        counts = {k: v * mult for k, v in counts.items()}
        if self.kind == "summa_cos":
            add("dd", 1)                                    # Z = X X
        if self.kind == "expm":
            ells = [r.diagnostics["squarings"] for r in (rep if not hasattr(rep, "plan") else [rep])]
            add("dd", sum(ells))
        return counts

    def units(self):
        return self.B if self.kind in ("exp", "expm") else 1

    def flop_scale(self):
        """GEMM flops are 2 n^3 per (global) GEMM; for SUMMA each rank does
        1/world of every GEMM."""
        return 2.0 * self.n ** 3 / (self.world if self.kind == "summa_cos" else 1)


def run_ours(args, rank, world, local_rank):
    import torch
    import paper_2312_17396_b200 as mp
    from paper_2312_17396_b200 import _lib

    torch.cuda.set_device(local_rank)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    wl = Workload(args.config, rank, world, torch, mp)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
    h = _lib.handle_for()

    for _ in range(args.warmup):
        rep = wl.step(wl.Xd)
    torch.cuda.synchronize()
    gem = wl.gemms(rep)
    plans = wl.plans(rep)
    # long-lived objects (graphs, buffers, the workload) out of the collector's
    # generations: no multi-ms gen-2 pause inside a timed region
    import gc
    gc.collect()
    gc.freeze()

    def barrier():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    # ---- device-resident timed region (value) ----
    clocks = ClockSampler(local_rank) if (rank == 0 and not args.no_clocks) else None
    barrier()
    if clocks:
        clocks.start()
    from paper_2312_17396_b200 import graphs as _graphs
    l0 = _lib.total_launches()
    total = 0.0
    for _ in range(args.steps):
        flush.zero_()  # 256 MiB write between steps: L2 (126 MB) flushed
        barrier()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        rep = wl.step(wl.Xd)
        b.record()
        b.synchronize()
        total += a.elapsed_time(b) * 1e-3
    barrier()
    if _graphs.enabled() and _graphs.last_launches():
        launches = float(_graphs.last_launches())      # kernels per graphed evaluation
    else:
        launches = (_lib.total_launches() - l0) / args.steps
    clk = clocks.stop() if clocks else None

    # ---- roofline pass: the same K steps eagerly (graphs off) with a CUDA
    # event pair around every GEMM launch on the launching stream ----
    probe = None
    if not args.no_probe:
        was = _graphs.enabled()
        _graphs.set_enabled(False)
        h = _lib.handle_for()
        wl.step(wl.Xd)
        torch.cuda.synchronize()
        h.probe = {}
        for _ in range(args.steps):
            flush.zero_()
            barrier()
            wl.step(wl.Xd)
        torch.cuda.synchronize()
        probe, h.probe = h.probe, None
        _graphs.set_enabled(was)

    # ---- end-to-end through the public API with host buffers ----
    # batched exp configs: paper_2312_17396_b200.pipeline.evaluate_host (H2D of
    # chunk c+1 and D2H of chunk c-1 overlap the evaluation of chunk c)
    from paper_2312_17396_b200 import pipeline as _pl
    outs = None
    e2e_total = 0.0
    # 4 chunks alternating over two compute streams (pipeline.evaluate_host):
    # each chunk's kernels fill the other's tails; its copies and host
    # planning overlap the other chunks' evaluation
    if wl.kind == "exp" and wl.B >= 16:
        chunks = [wl.B // 2, wl.B - wl.B // 2]
    else:
        chunks = 1
    e2e_streams = 2 if chunks != 1 else 1
    e2e_mode = "per step"
    if chunks != 1:
        # the K steps as one host stream (K x B matrices, pinned): chunks of
        # every step flow through a window of graph slots, so the copies
        # of step i overlap the evaluation of step i+1; every step's H2D
        # and D2H stay inside the one timed region
        W = {15: 1, 31: 2, 63: 4}[wl.cfg["digits"]]
        Xbig = wl.Xpin.repeat(args.steps, 1, 1).pin_memory()
        outs = [torch.empty((W,) + tuple(Xbig.shape), dtype=torch.float64).pin_memory()]
        sizes = list(chunks) * args.steps
        sub = _pl.mixed_exp(wl.m, wl.ctx, timing=False)
        win = 6    # tools/e2e_sweep.py: [32, 32] x window 6 ~ [16]*4 x 12 > [16]*4 x 8 > [64] x 3
        _pl.evaluate_host(sub, Xbig, outs[0], sizes, streams=e2e_streams, window=win)   # warm-up / capture
        flush.zero_()
        barrier()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        _pl.evaluate_host(sub, Xbig, outs[0], sizes, streams=e2e_streams, window=win)
        b.record()
        b.synchronize()
        e2e_total = a.elapsed_time(b) * 1e-3
        e2e_mode = f"{args.steps} steps streamed in one call (window {win} chunk slots)"
        # per-step bytes: one step's input and result
        outs = [torch.empty((W,) + tuple(wl.Xpin.shape), dtype=torch.float64)]
    for i in range(args.steps + 1 if chunks == 1 else 0):
        flush.zero_()
        barrier()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        if chunks != 1:
            if outs is None:
                W = {15: 1, 31: 2, 63: 4}[wl.cfg["digits"]]
                outs = [torch.empty((W,) + tuple(wl.Xpin.shape), dtype=torch.float64).pin_memory()]
            _pl.evaluate_host(_pl.mixed_exp(wl.m, wl.ctx, timing=False), wl.Xpin, outs[0], chunks,
                              streams=e2e_streams)
        else:
            rep = wl.step(wl.Xpin)
            res = wl.results(rep)
            if outs is None:
                outs = [torch.empty(r.shape, dtype=r.dtype).pin_memory() for r in res]
            for o, r in zip(outs, res):
                o.copy_(r, non_blocking=True)
        b.record()
        b.synchronize()
        if i > 0:
            e2e_total += a.elapsed_time(b) * 1e-3
    h2d = wl.Xh.nbytes
    d2h = sum(o.numel() * o.element_size() for o in outs)
    link = pcie_rates(torch, h2d, d2h)

    t = torch.tensor([total, e2e_total], dtype=torch.float64, device="cuda")
    if dist is not None:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    total, e2e_total = float(t[0]), float(t[1])
    if rank != 0:
        dist.destroy_process_group()
        return
    per_step_units = wl.units() * (world if wl.scaling == "weak" else 1)
    value = per_step_units * args.steps / total
    e2e = per_step_units * args.steps / e2e_total

    # ---- roofline of the dominant kernel (timed live over the timed region) ----
    peaks = measure_peaks(torch, h)
    by_key = {}
    for key, evs in (probe or {}).items():
        durs = [x.elapsed_time(y) * 1e-3 for x, y in evs]
        by_key[key] = (len(durs), sum(durs))
    names = {7: "fp32", 15: "fp64", 31: "dd", 63: "qd"}
    if not by_key:
        by_key[("none", 31, 31, 1, 1, 1, 1, 0, 0)] = (1, 1.0)
    dom = max(by_key.items(), key=lambda kv: kv[1][1])
    (kind, fin, fout, M, N, K, nb, S_used, db_used), (cnt, sec) = dom
    eager_step = None
    fname = names[fin]
    logical = 2.0 * M * N * K * nb / (sec / cnt) / 1e12       # logical TFLOP/s of the format
    step_time = total / args.steps
    fs = wl.flop_scale()
    t_ideal = sum(fs * c / (peaks[f] * 1e12) for f, c in gem.items())
    eff_gflops = sum(fs * c for c in gem.values()) * world * args.steps / total / 1e9
    plan0 = plans[0]
    if kind.endswith("_tc"):
        # INT8 tensor-core GEMM by exact digit-plane splitting: the hardware
        # bound is the INT8 tensor pipe; algorithmic ops per launch =
        # 2 M N K x (S(S+1)/2 plane pairs); S = 4/8/16/31 (7-bit digits) or
        # 4/8/14/28 (8-bit) for fp32/fp64/dd/qd, recorded per launch
        S = S_used or {7: 4, 15: 8, 31: 16, 63: 31}[fin]
        achieved = logical * S * (S + 1) / 2
        S7 = {7: 4, 15: 8, 31: 16, 63: 31}[fin]
        roof = {"bound": "tensor (int8)", "achieved": achieved, "peak": peaks["int8_tops"],
                "unit": "TOPS (int8)", "frac": achieved / peaks["int8_tops"],
                "frac_7bit_equivalent": logical * S7 * (S7 + 1) / 2 / peaks["int8_tops"],
                "frac_note": "frac counts the S(S+1)/2 plane-pair products per output this launch executed; "
                             "8-bit digits need fewer (dd 105 vs 136) for the same product, so "
                             "frac_7bit_equivalent rates the same logical throughput in 7-bit plane pairs",
                "logical_tflops": logical, "logical_frac_of_format_peak": logical / peaks[fname],
                "peak_source": f"tcgen05 kind::i8 probe in bench.py on this GPU ({peaks['int8_tops']:.0f} TOPS); "
                               f"format peaks from DFMA/FFMA probes (fp64 {peaks['fp64']:.2f} TF/s, "
                               f"Peak_dd = Peak_fp64/15, Peak_qd = Peak_fp64/115, SURVEY 8d); "
                               "MEASURED_PEAKS.json holds only HBM and bf16"}
    else:
        roof = {"bound": "fp64-pipe" if fname != "fp32" else "fp32-pipe", "achieved": logical, "peak": peaks[fname],
                "unit": "TFLOP/s (logical)", "frac": logical / peaks[fname],
                "peak_source": "FMA pipe microbenchmark in bench.py on this GPU "
                               f"(fp64 {peaks['fp64']:.2f} TF/s, fp32 {peaks['fp32']:.2f} TF/s); "
                               "Peak_dd = Peak_fp64/15, Peak_qd = Peak_fp64/115 (SURVEY 8d); "
                               "MEASURED_PEAKS.json holds only HBM and bf16"}
    if kind.endswith("_tc"):
        # global->shared bytes the kernel moves per launch: every 128-row x
        # NT-column output tile streams all S digit planes of its A rows and
        # B columns over K (NT = 32, 16 for qd)
        NT = 16 if S > 16 else 32      # 14 planes (8-bit dd) still use NT = 32
        tiles = nb * (-(-M // 128)) * (-(-N // NT))
        ingest = tiles * (-(-K // 32)) * S * (128 + NT) * 32.0
        ach = ingest / (sec / cnt) / 1e12
        roof["ingest"] = {"achieved": ach, "peak": peaks["ingest_tbps"], "unit": "TB/s", "frac": ach / peaks["ingest_tbps"],
                          "bytes_per_launch": ingest,
                          "note": "digit-plane bytes moved global->shared per launch (128-row x NT tiles, "
                                  "all S planes of A and B over K) and their rate vs the bulk-copy ingest probe "
                                  "(one CTA per SM, L2-resident 16 KB copies) run in this bench; with 32-byte K "
                                  "boxes the L2 slices run at ~64% of peak (ncu lts__throughput, n=1024) and the "
                                  "tensor pipe at ~62% -- DESIGN 5.1"}
    kkey = f"{kind} {fname}->{names[fout]} {M}x{N}x{K} x{nb}"
    if kind.endswith("_tc"):
        roof["digit_planes"] = S
        roof["digit_bits"] = db_used
    traffic, tsrc = None, None
    try:   # committed ncu --set full capture of this kernel at this shape (profiles/traffic.json)
        tr = json.load(open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", "traffic.json")))
        if kkey in tr:
            traffic = tr[kkey]["dram_bytes_per_launch"]
            tsrc = f"{tr[kkey]['capture']} ({tr[kkey]['kernel']}), bytes per launch"
    except Exception:
        pass
    roof.update({"kernel": kkey, "traffic": traffic, "traffic_source": tsrc,
                 "share_of_step": sec / args.steps / step_time, "launches_per_step": cnt / args.steps,
                 "eval_frac": t_ideal / step_time,
                 "measured_in": "a second timed pass of the same K steps run eagerly (the value pass "
                                "replays CUDA graphs, whose kernels cannot be bracketed by events)"})
    line = {
        "metric": METRIC, "value": value, "unit": "evals/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * step_time, "higher_is_better": True,
        "scaling": wl.scaling, "vs_baseline": None, "dtype": names[plan0.level_formats[0]],
        "data": "synthetic (seeded N(0,1) rescaled to the config's ||X||_1; BASELINE configs have no dataset)",
        "config": {"workload": wl.cfg["workload"], "name": args.config, "units_per_gpu_step": wl.units(),
                   "n": wl.n, "m": wl.m, "digits": wl.cfg["digits"],
                   "schedule_digits": [list(p.level_digits) for p in plans],
                   "level_formats": wl.formats(rep), "gemms_per_step_per_gpu": gem,
                   "gemm_engine": __import__("paper_2312_17396_b200.gemm_engine", fromlist=["x"]).engine(),
                   "parallelism": wl.parallelism,
                   "host_affinity": (f"{len(CFG['numa_cpus'])} GPU-local CPUs (NVML affinity)"
                                     if CFG.get("numa_cpus") else "unbound"),
                   "l2": "256 MiB buffer written between timed steps (L2 flushed)"},
        "gflops_effective": eff_gflops,
        "roofline": roof,
        "peaks_tflops": peaks,
        "e2e": {"value": e2e, "unit": "evals/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                "path": ("paper_2312_17396_b200.pipeline.evaluate_host(ps_mixed_exp, pinned host stream of the "
                         f"{args.steps} steps' batches, chunks {chunks} per step over {e2e_streams} compute streams, "
                         "a window of 6 chunk slots: copies and host planning overlap compute, also across steps; "
                         "no L2 flush inside the stream, per-step working set ~1 GB > L2)") if chunks != 1 else
                        "public API on a pinned host batch, result copied back to pinned host memory",
                "mode": e2e_mode,
                "link_gbs": link},
        "gpu_launches": launches,
        "clocks": clk,
    }
    if world == 1 and not args.no_cpu_baseline and args.config == "cfg2":
        try:
            line["cpu_baseline"] = cpu_baseline_sample()
        except Exception as e:  # the baseline is reported, never required
            line["cpu_baseline"] = {"value": None, "error": str(e)[:200]}
    print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()


_ORIG_AFFINITY = []


def bind_to_gpu_numa(local_rank: int):
    """Pin this rank's host threads to the CPUs NVML reports as local to its
    GPU, so the pinned host buffers of the e2e stream are first-touched on
    the GPU's NUMA node (a far node measured 20-25K instead of 35K evals/s
    on the cfg2 host stream).  Returns the CPU list or None."""
    try:
        import pynvml as nv
        nv.nvmlInit()
        hdl = nv.nvmlDeviceGetHandleByIndex(local_rank)
        ncpu = os.cpu_count() or 1
        words = nv.nvmlDeviceGetCpuAffinity(hdl, (ncpu + 63) // 64)
        cpus = [w * 64 + b for w, m in enumerate(words) for b in range(64) if (int(m) >> b) & 1 and w * 64 + b < ncpu]
        if cpus:
            _ORIG_AFFINITY[:] = sorted(os.sched_getaffinity(0))
            os.sched_setaffinity(0, cpus)
            return cpus
    except Exception:
        return None
    return None


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--config", default="cfg2", choices=sorted(CONFIGS))
    ap.add_argument("--no-probe", action="store_true", help="diagnostic: no per-launch events")
    ap.add_argument("--no-clocks", action="store_true", help="diagnostic: no nvidia-smi sampling")
    args = ap.parse_args()
    CFG.clear()
    CFG.update(CONFIGS[args.config])
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl != "reference":
        CFG["numa_cpus"] = bind_to_gpu_numa(local_rank)
    if args.impl == "reference":
        run_reference(args, rank, world)
    else:
        run_ours(args, rank, world, local_rank)


if __name__ == "__main__":
    main()
