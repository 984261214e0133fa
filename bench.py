"""Benchmark of the B200 mixed-precision Paterson-Stockmeyer hot path.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config cfgX ...] [--scaling weak|strong]

With no --config the run prints two JSON lines: cfg2 (BASELINE configs[1],
64 x n=256 Taylor exp at dd) and then, LAST, the headline cfg5 (the largest
single-GPU config: Taylor cosine of degree 24 in Z = X^2, one n=8192 matrix,
dd working).  One step = one mixed-precision PS evaluation of the config's
unit (the whole batch, or the one matrix) through the public API: powers,
blocks + norms, host planner, mixed Horner.

Inputs: seeded synthetic matrices of the BASELINE shapes (the
configs have no dataset).  Every timed step reads a different input batch
(a pool of distinct seeded batches, cycled when one step's input is larger
than ~1 GB), so the speculative Horner graph can miss; the line reports
graphs.speculation_stats().

Multi-GPU: ``--gpus N`` without torchrun re-executes itself under
``torch.distributed.run`` (one rank per GPU, NCCL).  Batched configs shard
their matrices over the ranks with no data-path collective (``--scaling
weak``: every rank evaluates its own B matrices, the default; ``strong``:
one B-matrix batch split B/N per rank); cfg5 at N > 1 runs the 2-D block
SUMMA (summa.py).  Device time is the max over ranks.

``--impl reference`` times the reference algorithm's CPU path (the oracle
port: the C MPFR restatement of the reference's arithmetic in oracle/; the
reference itself is pure Python over gmpy2, absent from this image) on all
host cores, on the same config dicts: cfg1/cfg2 run whole evaluations of
one matrix per step; cfg3/4/5 cannot finish on a CPU (hours to weeks), so
each step times the port's mat_mul at every precision the config's GEMM
list needs on an n=256 sample and extrapolates the evaluation as
sum_g n^3 t_MAC(bits_g), labelled "extrapolated".
"""

from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
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
                          "dd working; 2-D block SUMMA over NCCL at N>1",
                 batch=1, n=8192, m=24, digits=31, norm=1.0, kind="cos"),
}
DEFAULT_CONFIGS = ("cfg2", "cfg5")      # the last line is the headline
METRIC = "matrix-polynomial evals/sec"
POOL_BYTES = 1 << 30                    # distinct inputs kept per run (device + pinned host)
WARM_SECONDS = 1.0                      # untimed warm-up lasts at least this long (and at least --warmup steps)
E2E_PASSES = 3                          # timed passes of the host-stream e2e measurement (median reported)


def synth(n, target, seed, cos=False):
    """SURVEY 8d generator (tests/_util.synth): X = G target/||G||_1,
    G ~ N(0,1) from default_rng(seed) (/sqrt(n) first for the cosine)."""
    G = np.random.default_rng(seed).standard_normal((n, n))
    if cos:
        G = G / np.sqrt(n)
    return G * (target / np.abs(G).sum(axis=0).max())


def config_dict(name, world, scaling):
    """The `config` object of BOTH arms (identical for the same run)."""
    c = CONFIGS[name]
    if c["kind"] == "cos":
        par = "single GPU" if world == 1 else "2-D block SUMMA over %dx%d ranks" % _grid_shape(world)
    elif world == 1:
        par = "single GPU"
    elif scaling == "strong":
        par = f"batch-sharded {c['batch']}/{world} matrices per GPU (strong)"
    else:
        par = f"batch-sharded, {c['batch']} matrices per GPU (weak)"
    return {"workload": c["workload"], "name": name, "batch": c["batch"], "n": c["n"], "m": c["m"],
            "digits": c["digits"], "parallelism": par,
            "l2": "256 MiB buffer written between timed steps (L2 flushed); inputs distinct per step"}


def _grid_shape(world):
    from paper_2312_17396_b200 import summa
    return summa.ProcessGrid.for_world(world)


# ----------------------------------------------------------------- clocks
_SAMPLER_SRC = r"""
import sys, time
period = float(sys.argv[2])
try:
    import pynvml as nv
    nv.nvmlInit()
    hdl = nv.nvmlDeviceGetHandleByIndex(int(sys.argv[1]))
    get = getattr(nv, "nvmlDeviceGetCurrentClocksEventReasons", None) or nv.nvmlDeviceGetCurrentClocksThrottleReasons
    bits = (nv.nvmlClocksThrottleReasonHwSlowdown, nv.nvmlClocksThrottleReasonHwThermalSlowdown,
            nv.nvmlClocksThrottleReasonSwThermalSlowdown, nv.nvmlClocksThrottleReasonSwPowerCap)
    print("max", float(nv.nvmlDeviceGetMaxClockInfo(hdl, nv.NVML_CLOCK_SM)), flush=True)
    while True:
        r = int(get(hdl))
        print(time.monotonic(), float(nv.nvmlDeviceGetClockInfo(hdl, nv.NVML_CLOCK_SM)),
              "".join("1" if r & b else "0" for b in bits), flush=True)
        time.sleep(period)
except Exception as e:
    print("error", repr(e)[:200], flush=True)
"""


class ClockSampler:
    """SM clocks and clock-event (throttle) reasons sampled DURING the timed
    region by a separate process polling NVML (1 ms period; CLOCK_MONOTONIC
    timestamps, the bench keeps the samples inside [start, stop]).  A polling
    thread inside this process made the device-resident cfg2 loop bimodal
    (57K or 27-35K evals/s from run to run: its NVML calls and the GIL
    hand-overs delay the step's graph launches; 8 of 8 runs at 57-58K
    without it), hence the process."""

    NAMES = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")

    def __init__(self, index, period=0.001):
        self.t0 = self.t1 = None
        try:
            import tempfile
            # samples go to a file, not a pipe: a full pipe would block the sampler mid-run
            self.log = tempfile.NamedTemporaryFile("w+", prefix="mpps_clocks_", suffix=".txt", delete=False)
            self.proc = subprocess.Popen([sys.executable, "-c", _SAMPLER_SRC, str(index), str(period)],
                                         stdout=self.log, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None

    def start(self):
        self.t0 = time.monotonic()

    def stop(self):
        self.t1 = time.monotonic()
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["clock sampler unavailable"]}
        time.sleep(0.005)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        try:
            self.log.flush()
            out = open(self.log.name).read()
            self.log.close()
            os.unlink(self.log.name)
        except Exception:
            out = ""
        smax, sm, reasons, err = None, [], set(), None
        for ln in out.splitlines():
            parts = ln.split()
            if not parts:
                continue
            if parts[0] == "max":
                smax = float(parts[1])
            elif parts[0] == "error":
                err = " ".join(parts[1:])
            elif len(parts) == 3:
                try:
                    t, c = float(parts[0]), float(parts[1])
                except ValueError:
                    continue
                if self.t0 <= t <= self.t1:
                    sm.append(c)
                    reasons.update(nm for nm, bit in zip(self.NAMES, parts[2]) if bit == "1")
        if err and not sm:
            return {"sm_mhz": None, "sm_max_mhz": smax, "reasons": [f"clock sampler: {err}"]}
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": smax, "reasons": sorted(reasons),
                "samples": len(sm), "source": "nvml (separate process, 1 ms period)"}


# ------------------------------------------------------------- peaks
def measure_peaks(torch, h):
    """FP64 / FP32 FMA pipe peaks on this GPU (2 flops per FMA): the
    per-precision roofline denominators (MEASURED_PEAKS.json has only HBM and
    bf16).  Peak_dd / Peak_qd follow SURVEY 8(d): Peak_fp64 / k with
    k_dd = 15 and k_qd = 115 FP64-pipe instructions per canonical MAC.
    Plus the INT8 tcgen05 pipe (the tensor-core GEMMs' bound) and the
    global->shared ingest rate."""
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
    # sustained: the same probe (pseudo-random operands) back to back for
    # ~3 s -- the clock settles under the power cap, as in a long step; the
    # rate of the last second
    one = sms * 2.0 * 128 * 256 * 32 * iters
    t_end = time.perf_counter() + 3.0
    evs = []
    while time.perf_counter() < t_end:
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(8):
            h.probe_i8mma(sms, iters, scratch)
        b.record()
        b.synchronize()
        evs.append((time.perf_counter(), a.elapsed_time(b) * 1e-3))
    tail = [sec for t, sec in evs if t >= evs[-1][0] - 1.0] or [evs[-1][1]]
    out["int8_tops_sustained"] = 8 * one * len(tail) / sum(tail) / 1e12
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


# ---------------------------------------------------------- reference arm
def _all_cores():
    if _ORIG_AFFINITY:      # the CPU baseline uses every host core, not the GPU-local ones
        os.sched_setaffinity(0, _ORIG_AFFINITY)
    cores = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 1)
    os.environ["OMP_NUM_THREADS"] = str(cores)
    return cores


def _ref_gemm_list(name):
    """(bits, count) per evaluation of the oracle composition (SURVEY 8c:
    powers/blocks at the working bits, Horner levels at the snapped digits'
    bits) for the configs the port cannot finish, from the committed
    full-size plan fixture (tests/golden/fullsize_plans.json, written by
    oracle/make_fullsize_plans.py with the oracle's planner)."""
    import oracle
    c = CONFIGS[name]
    fx = json.load(open(os.path.join(ROOT, "tests", "golden", "fullsize_plans.json")))[name]
    wb = oracle.bits_of(c["digits"])
    counts = {}

    def add(bits, k):
        counts[bits] = counts.get(bits, 0) + k
    for ent in fx["plans"]:
        s, r, m = ent["s"], ent["r"], ent["m"]
        if not ent.get("shared_powers_with_previous"):
            add(wb, s - 1)                       # X^2..X^s (form_powers; shared by the Pade pair)
        for j, dj in enumerate(ent["snapped"], start=1):
            if j == r and m % s == 0:
                continue                         # B_r = b_m I: no product
            add(oracle.bits_of(dj), 1)
        add(wb, ent.get("squarings", 0))
        add(wb, ent.get("argument_gemms", 0))    # cosine Z = X X
    per_unit = fx.get("units", 1)
    return counts, per_unit


def reference_step_extrapolated(name, n_s=256):
    """One bounded step of the reference arm for cfg3/4/5: the port's
    mat_mul timed at each precision of the GEMM list on an n_s sample (all
    cores); returns (extrapolated seconds per unit, detail)."""
    import oracle
    c = CONFIGS[name]
    counts, units = _ref_gemm_list(name)
    A = synth(n_s, 1.0, 7)
    Bm = synth(n_s, 1.0, 8)
    t_mac = {}
    for bits in sorted(counts):
        t0 = time.perf_counter()
        oracle.matmul(A, Bm, bits)
        t_mac[bits] = (time.perf_counter() - t0) / n_s ** 3
    total = sum(c["n"] ** 3 * t_mac[b] * k for b, k in counts.items())
    return total / units, {"t_mac_ns": {str(b): 1e9 * t for b, t in t_mac.items()},
                           "gemms_per_unit": {str(b): k / units for b, k in counts.items()}}


def reference_step_full(name, seed):
    """One bounded step for cfg1/cfg2: a whole mixed evaluation of one
    matrix of the config in the port; returns seconds."""
    import oracle
    from paper_2312_17396_b200.coefficients import taylor_exp_coeffs
    c = CONFIGS[name]
    X = synth(c["n"], c["norm"], seed)
    t0 = time.perf_counter()
    oracle.ps_eval(X, taylor_exp_coeffs(c["m"]).coeffs, c["digits"])
    return time.perf_counter() - t0


def reference_sample(name, steps, warmup):
    """(value evals/s, cpu_baseline dict) of the port on this config."""
    import oracle
    oracle.build()
    cores = _all_cores()
    kind = CONFIGS[name]["kind"]
    full = kind == "exp"
    for i in range(warmup):
        (reference_step_full(name, 10_000 + i) if full else reference_step_extrapolated(name))
    total, detail = 0.0, None
    t0 = time.perf_counter()
    for i in range(steps):
        if full:
            total += reference_step_full(name, i)
        else:
            sec, detail = reference_step_extrapolated(name)
            total += sec
    wall = time.perf_counter() - t0
    v = steps / total
    n = CONFIGS[name]["n"]
    if full:
        sample = (f"{steps} whole mixed PS evaluations of one n={n} matrix each (seeds 0..{steps - 1}) in the C "
                  f"MPFR restatement of the reference (oracle/), OpenMP over GEMM rows, {wall:.1f} s")
    else:
        sample = (f"extrapolated: each of {steps} steps times the port's mat_mul (precision.py:160-184 "
                  f"restated) at every precision of the config's GEMM list on an n=256 sample "
                  f"(t_MAC ns per precision bits {({k: round(x, 2) for k, x in detail['t_mac_ns'].items()})}), "
                  f"evaluation = sum_g n^3 t_MAC(bits_g) over {detail['gemms_per_unit']} GEMMs per unit; "
                  f"O(n^2) terms omitted; {wall:.1f} s of CPU time")
    cb = {"value": v, "unit": "evals/s", "cores": cores, "kind": "port", "sample": sample}
    if not full:
        cb["extrapolated"] = True
    return v, cb


def run_reference(name, args, rank, world):
    if rank != 0:
        return
    v, cb = reference_sample(name, args.steps, args.warmup)
    line = {"metric": METRIC, "value": v, "unit": "evals/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 / v, "higher_is_better": True,
            "scaling": _scaling(name, args), "vs_baseline": None,
            "dtype": f"mpfr {_bits_note(name)} (per-op rounded, reference semantics)",
            "data": "synthetic (seeded N(0,1) rescaled to the config's ||X||_1; BASELINE configs have no dataset)",
            "impl": "reference", "config": config_dict(name, world, args.scaling),
            "cpu_baseline": cb,
            "e2e": {"value": v, "unit": "evals/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def _bits_note(name):
    import oracle
    return f"{oracle.bits_of(CONFIGS[name]['digits'])}-bit working"


def _scaling(name, args):
    return "strong" if (CONFIGS[name]["kind"] == "cos" or args.scaling == "strong") else "weak"


def pcie_rates(torch, h2d_bytes: int, d2h_bytes: int, reps: int = 5):
    """Plain pinned-host <-> device copy rates of one step's input / result
    sizes in this process (the ceiling of the e2e stream)."""
    try:
        hb = torch.empty(max(h2d_bytes, d2h_bytes) // 8, dtype=torch.float64).pin_memory()
        db = torch.empty_like(hb, device="cuda")
        out = {}
        for nm, nbytes, dst, src in (("h2d", h2d_bytes, db, hb), ("d2h", d2h_bytes, hb, db)):
            k = nbytes // 8
            dst[:k].copy_(src[:k], non_blocking=True)
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(reps):
                dst[:k].copy_(src[:k], non_blocking=True)
            b.record()
            b.synchronize()
            out[nm] = reps * nbytes / (a.elapsed_time(b) * 1e-3) / 1e9
        return out
    except Exception as e:  # diagnostics only
        return {"error": str(e)[:120]}


# ---------------------------------------------------------------- ours
class Workload:
    """One benchmark config on this rank: a pool of distinct device-resident
    (and pinned host) inputs, a step through the public API, and the honest
    GEMM count per unit."""

    def __init__(self, name, rank, world, torch, mp, scaling, steps, warmup):
        self.name, self.cfg = name, CONFIGS[name]
        self.rank, self.world, self.torch, self.mp = rank, world, torch, mp
        c = self.cfg
        self.ctx = mp.PrecisionCtx(c["digits"])
        self.n, self.m = c["n"], c["m"]
        self.kind = c["kind"]
        self.scaling = "strong" if (self.kind == "cos" or scaling == "strong") else "weak"
        self.grid = None
        if self.kind == "cos" and world > 1:
            from paper_2312_17396_b200 import summa
            pr, pc = summa.ProcessGrid.for_world(world)
            self.grid = summa.ProcessGrid(pr, pc)
        B = c["batch"]
        if self.kind in ("exp", "expm") and self.scaling == "strong" and world > 1:
            from paper_2312_17396_b200.sharding import shard_bounds
            lo, hi = shard_bounds(B, world, rank)
            self.members = list(range(lo, hi))
        else:
            self.members = list(range(B))
        self.B = len(self.members)
        step_bytes = self.B * self.n * self.n * 8
        self.pool = max(2, min(steps + warmup + 1, POOL_BYTES // step_bytes))
        self.Xh = [self._make(t) for t in range(self.pool)]
        self.Xd = [torch.from_numpy(x).cuda() for x in self.Xh]
        self.Xpin = [torch.from_numpy(x).pin_memory() for x in self.Xh]

    def _make(self, t):
        """Input of pool slot t on this rank: seeds never repeat across
        slots or ranks (slot 0 of rank 0 is the parity tests' seed set)."""
        c, n, B = self.cfg, self.n, self.cfg["batch"]
        from paper_2312_17396_b200.sharding import batch_id
        gid = batch_id(t, self.world, self.rank, self.scaling == "strong")
        if self.kind == "exp":
            X = np.stack([synth(n, c["norm"], gid * B + i) for i in self.members])
            return X[0] if c["batch"] == 1 else X
        if self.kind == "expm":
            rng = np.random.default_rng(1000 + gid)
            targets = 10.0 ** rng.uniform(-2, 3, size=B)
            return np.stack([synth(n, targets[i], gid * B + i) for i in self.members])
        if self.kind == "pade":
            return synth(n, c["norm"], gid)
        X = synth(n, c["norm"], t, cos=True)                    # cosine: one matrix per step
        if self.grid is not None:
            r0, mr, c0, nc = self.grid.block(n)
            X = np.ascontiguousarray(X[r0:r0 + mr, c0:c0 + nc])
        return X

    def _summa(self, X):
        from paper_2312_17396_b200 import summa
        from paper_2312_17396_b200.precision import MatBatch
        if X.device.type == "cpu":
            X = X.to("cuda", non_blocking=True)
        blk = MatBatch(X.reshape(1, 1, *X.shape), 15)
        ops = summa.DeviceOps()
        Z = summa.cos_argument_dist(blk, self.ctx, self.grid, ops)
        return summa.ps_mixed_dist(Z, self.mp.taylor_cos_coeffs(self.m), self.ctx, self.grid, ops)

    def step(self, X):
        mp, ctx, m = self.mp, self.ctx, self.m
        if self.kind == "exp":
            return mp.ps_mixed_exp(X, m, ctx, timing=False)
        if self.kind == "expm":
            return mp.expm_ss(X, ctx, m, timing=False)
        if self.kind == "pade":
            return mp.ps_mixed_pade(X, m, ctx, timing=False)
        if self.grid is not None:
            return self._summa(X)
        Z = mp.cos_argument(X, ctx)
        return mp.ps_mixed_general(Z, mp.taylor_cos_coeffs(m), ctx, timing=False)

    def results(self, rep):
        """Device tensors holding the step's result(s)."""
        if self.kind == "pade":
            return [r.result.data for r in rep]
        if self.grid is not None:
            return [rep.block.data]
        return [rep.result.data]

    def plans(self, rep):
        if self.kind == "pade":
            return [rep[0].plan, rep[1].plan]
        if self.grid is not None:
            return [rep.plan(self.ctx)]
        if hasattr(rep, "plan"):
            return [rep.plan]
        return [r.plan for r in rep]

    def formats(self, rep):
        from paper_2312_17396_b200.precision import FORMAT_NAME
        return [[FORMAT_NAME[f] for f in p.level_formats] for p in self.plans(rep)[:4]]

    def _schedules(self, rep):
        """(s, r, working format, level formats) of every matrix/polynomial
        of a step, from the executed digits (no exact plan records)."""
        from paper_2312_17396_b200.planner import default_block_size, formats_of_digits
        wf = 15 if self.cfg["digits"] <= 15 else self.cfg["digits"]
        s = default_block_size(self.m)
        r = self.m // s
        if self.grid is not None:
            return [(s, r, wf, formats_of_digits(rep.digits))]
        reps = list(rep) if isinstance(rep, (list, tuple)) else [rep]
        out = []
        for r_ in reps:
            ex = getattr(r_, "_executed", None)
            if ex is not None:
                fm = formats_of_digits(ex[0])
            else:
                fm = r_.plan.level_formats[1:]
            out.append((s, r, wf, tuple(fm)))
        return out

    def gemms(self, rep):
        """Honest device GEMMs per step on this rank, by format."""
        from paper_2312_17396_b200.precision import FORMAT_NAME
        counts = {}

        def add(f, c):
            counts[f] = counts.get(f, 0) + c

        for i, (s, r, wf, fm) in enumerate(self._schedules(rep)):
            if not (self.kind == "pade" and i > 0):
                add(FORMAT_NAME[wf], s - 1)                 # powers (shared by the Pade pair)
            for j in range(1, r + 1):
                if j == r and self.m % s == 0:
                    continue                                # K3: elementwise
                add(FORMAT_NAME[fm[j - 1]], 1)
        if self.kind == "cos":
            add("dd", 1)                                    # Z = X X
        if self.kind == "expm":
            reps = rep if not hasattr(rep, "plan") else [rep]
            add("dd", sum(r._diag_extra.get("squarings", 0) for r in reps))
        return counts

    def units(self):
        return self.B if self.kind in ("exp", "expm") else 1

    def flop_scale(self):
        """GEMM flops are 2 n^3 per (global) GEMM; for SUMMA each rank does
        1/world of every GEMM."""
        return 2.0 * self.n ** 3 / (self.world if self.grid is not None else 1)


def run_ours(name, args, rank, world, local_rank, dist):
    import torch
    import paper_2312_17396_b200 as mp
    from paper_2312_17396_b200 import _lib, graphs as _graphs

    # the clock sampler process starts now, so that it is polling by the time the warm-up is over
    clocks = ClockSampler(local_rank) if (rank == 0 and not args.no_clocks) else None
    wl = Workload(name, rank, world, torch, mp, args.scaling, args.steps, args.warmup)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
    h = _lib.handle_for()
    P = wl.pool

    # W untimed warm-up steps, and for millisecond steps as many more as fill WARM_SECONDS: five
    # 1 ms steps leave the host (clock governor, allocator, page cache of a fresh box) cold and
    # the first process on a box measured 53-55K evals/s at cfg2 against 58K for every later one
    t_warm = time.perf_counter()
    warm_run = 0
    # (SUMMA steps hold collectives: every rank must run the same count, so only W there)
    while warm_run < args.warmup or (wl.grid is None and time.perf_counter() - t_warm < WARM_SECONDS
                                     and warm_run < 2000):
        rep = wl.step(wl.Xd[(args.steps + warm_run) % P])
        warm_run += 1
        if warm_run >= args.warmup:
            torch.cuda.synchronize()
    torch.cuda.synchronize()
    import gc
    gc.collect()
    gc.freeze()
    # the collection walks the whole heap and leaves the host caches cold: timed step 0 was the
    # slowest of every run (cfg1: 0.28 ms against a median of 0.103) -- one more untimed step
    # (run exactly like a timed step: L2 flushed first)
    flush.zero_()
    torch.cuda.synchronize()
    rep = wl.step(wl.Xd[(args.steps + warm_run) % P])
    warm_run += 1
    torch.cuda.synchronize()

    def barrier():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    # ---- device-resident timed region (value): step t reads input t ----

    spec0 = _graphs.speculation_stats()
    barrier()
    if clocks:
        clocks.start()
    l0 = _lib.total_launches()
    total = 0.0
    step_times = []
    gem = {}
    gc.disable()       # no collector pause inside a timed step (a serving loop would tune it too)
    # one pair of timing events, created (torch creates them lazily at the first record) before the
    # loop: the creation of the end event used to fall inside timed step 0
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    b.record()
    b.synchronize()
    for t in range(args.steps):
        flush.zero_()  # 256 MiB write between steps: L2 (126 MB) flushed
        barrier()
        a.record()
        rep = wl.step(wl.Xd[t % P])
        b.record()
        b.synchronize()
        step_times.append(a.elapsed_time(b))
        total += step_times[-1] * 1e-3
        # honest GEMM counts of every timed step, from the executed schedules
        # (cheap; the exact plan records are built lazily, below, once)
        for f, c in wl.gemms(rep).items():
            gem[f] = gem.get(f, 0) + c
        # the report kept for the plan / format fields is the LAST step's: holding an earlier one
        # pins its result buffer, the next steps then need a third 64 MiB block and the caching
        # allocator's cudaMalloc lands inside a timed step (always timed step 2: 1.9 ms instead of
        # 1.06, and 7-108 ms in one run of four on this pool's VMs -- 57K evals/s read 19-23K)
        if t == args.steps - 1:
            rep0 = rep
    gc.enable()
    barrier()
    plans, fmts = wl.plans(rep0), wl.formats(rep0)
    del rep0
    clk = clocks.stop() if clocks else None
    spec1 = _graphs.speculation_stats()
    eager_launches = _lib.total_launches() - l0
    if eager_launches == 0 and _graphs.enabled() and _graphs.last_launches() and wl.kind == "exp":
        per_step = float(_graphs.last_launches())      # kernels per graphed evaluation (captured count)
        launches = per_step * args.steps
    else:
        launches = float(eager_launches)
        per_step = launches / args.steps
    gem = {k: v / args.steps for k, v in gem.items()}

    # ---- roofline pass: the same K steps eagerly (graphs off) with a CUDA
    # event pair around every GEMM launch on the launching stream ----
    probe = None
    if not args.no_probe:
        was = _graphs.enabled()
        _graphs.set_enabled(False)
        h = _lib.handle_for()
        wl.step(wl.Xd[0])
        torch.cuda.synchronize()
        h.probe = {}
        for t in range(args.steps):
            flush.zero_()
            barrier()
            wl.step(wl.Xd[t % P])
        torch.cuda.synchronize()
        probe, h.probe = h.probe, None
        _graphs.set_enabled(was)

    # ---- end-to-end through the public API with host buffers ----
    from paper_2312_17396_b200 import pipeline as _pl
    W = {15: 1, 31: 2, 63: 4}[wl.cfg["digits"]]
    e2e_total = 0.0
    if wl.kind == "exp" and wl.B >= 16:
        # the K steps' batches as one pinned host stream through
        # pipeline.evaluate_host: chunks of every step flow through a window
        # of graph slots, so the copies of step t overlap the evaluation of
        # step t+1; every step's H2D and D2H stay inside the timed region
        chunks = [wl.B // 2, wl.B - wl.B // 2]
        Xbig = torch.cat([wl.Xpin[t % P] for t in range(args.steps)]).pin_memory()
        out = torch.empty((W,) + tuple(Xbig.shape), dtype=torch.float64).pin_memory()
        sizes = list(chunks) * args.steps
        sub = _pl.mixed_exp(wl.m, wl.ctx, timing=False)
        win = 6    # tools/e2e_sweep.py: [32, 32] x window 6 ~ [16]*4 x 12 > [16]*4 x 8 > [64] x 3
        Xwarm = torch.cat([wl.Xpin[(args.steps + t) % P] for t in range(args.steps)]).pin_memory()
        _pl.evaluate_host(sub, Xwarm, out, sizes, streams=2, window=win)   # warm-up / capture
        del Xwarm
        # the K-step stream lasts ~30 ms, so one host hiccup is a third of it (one pass in ~20
        # measured 31.9K evals/s between passes at 46K): the median of E2E_PASSES timed passes
        passes = []
        for _ in range(E2E_PASSES):
            flush.zero_()
            barrier()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            _pl.evaluate_host(sub, Xbig, out, sizes, streams=2, window=win)
            b.record()
            b.synchronize()
            passes.append(a.elapsed_time(b) * 1e-3)
        e2e_total = sorted(passes)[len(passes) // 2]
        e2e_path = ("paper_2312_17396_b200.pipeline.evaluate_host(ps_mixed_exp, pinned host stream of the "
                    f"{args.steps} steps' distinct batches, chunks {chunks} per step over 2 compute streams, a "
                    f"window of {win} chunk slots: copies and host planning overlap compute, also across steps; "
                    f"no L2 flush inside the stream, per-step working set ~1 GB > L2; median of {E2E_PASSES} "
                    f"timed passes of the K steps: {[round(args.steps * wl.B / p) for p in passes]} evals/s)")
        h2d = wl.Xh[0].nbytes
        d2h = W * wl.Xh[0].nbytes
    elif wl.kind == "exp" or os.environ.get("MPPS_BENCH_E2E_STREAM") == "0":
        # one call per step through the public API, the result copied back
        # to pinned memory, each step synchronised (cfg1: one small matrix
        # per step; nothing to overlap).
        outs = None
        for i in range(args.steps + 1):
            X = wl.Xpin[(i + P - 1) % P]
            flush.zero_()
            barrier()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            rep = wl.step(X)
            res = wl.results(rep)
            if outs is None:
                outs = [torch.empty(r.shape, dtype=r.dtype).pin_memory() for r in res]
            for o, r in zip(outs, res):
                o.copy_(r, non_blocking=True)
            b.record()
            b.synchronize()
            if i > 0:            # the first call is a warm-up of the host-input path
                e2e_total += a.elapsed_time(b) * 1e-3
        e2e_path = "public API on a pinned host input, result copied back to pinned host memory, per step"
        h2d = wl.Xh[0].nbytes
        d2h = sum(o.numel() * o.element_size() for o in outs)
    else:
        # the K steps' inputs as one pinned host stream through
        # pipeline.evaluate_stream: H2D of step t+1 and D2H of step t-1
        # overlap the evaluation of step t; every copy is inside the region
        rep = wl.step(wl.Xpin[0])             # warm-up of the host-input path
        torch.cuda.synchronize()
        outs = [[torch.empty(r.shape, dtype=r.dtype).pin_memory() for r in wl.results(rep)] for _ in range(2)]
        del rep
        Xs = [wl.Xpin[t % P] for t in range(args.steps)]
        outl = [outs[t % 2] for t in range(args.steps)]
        # one untimed pass over the distinct inputs of the pool: every plan
        # structure of the stream has its Horner graph captured before the
        # timed region (as the warm-up pass of the batched host stream above)
        _pl.evaluate_stream(wl.step, Xs[:min(args.steps, P)], outl[:min(args.steps, P)], wl.results,
                            keep_reports=False)
        torch.cuda.synchronize()
        flush.zero_()
        barrier()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        _pl.evaluate_stream(wl.step, Xs, outl, wl.results, keep_reports=False)
        b.record()
        b.synchronize()
        e2e_total = a.elapsed_time(b) * 1e-3
        e2e_path = ("paper_2312_17396_b200.pipeline.evaluate_stream(public API per step, pinned host inputs of the "
                    f"{args.steps} steps): H2D of step t+1 and D2H of step t-1 overlap step t; all copies inside "
                    "the timed region")
        h2d = wl.Xh[0].nbytes
        d2h = sum(o.numel() * o.element_size() for o in outs[0])
    link = pcie_rates(torch, h2d, d2h)

    tt = torch.tensor([total, e2e_total], dtype=torch.float64, device="cuda")
    if dist is not None:
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    total, e2e_total = float(tt[0]), float(tt[1])
    if rank != 0:
        return
    per_step_units = wl.units() * (world if wl.scaling == "weak" else 1)
    if wl.scaling == "strong" and wl.kind in ("exp", "expm"):
        per_step_units = wl.cfg["batch"]
    value = per_step_units * args.steps / total
    e2e = per_step_units * args.steps / e2e_total

    # ---- roofline of the dominant kernel (timed live over the K steps) ----
    peaks = measure_peaks(torch, h)
    by_key = {}
    for key, evs in (probe or {}).items():
        durs = [x.elapsed_time(y) * 1e-3 for x, y in evs]
        by_key[key] = (len(durs), sum(durs))
    names = {7: "fp32", 15: "fp64", 31: "dd", 63: "qd"}
    small = not by_key          # K5 path (n <= 32): no GEMM launches to bracket
    if small:
        by_key[("none", 31, 31, 1, 1, 1, 1, 0, 0)] = (1, 1.0)
    dom = max(by_key.items(), key=lambda kv: kv[1][1])
    (kind, fin, fout, M, N, K, nb, S_used, db_used), (cnt, sec) = dom
    fname = names[fin]
    logical = 2.0 * M * N * K * nb / (sec / cnt) / 1e12       # logical TFLOP/s of the format
    step_time = total / args.steps
    fs = wl.flop_scale()
    t_ideal = sum(fs * c / (peaks[f] * 1e12) for f, c in gem.items())
    eff_gflops = sum(fs * c for c in gem.values()) * (world if wl.scaling == "weak" or wl.grid is not None else 1) \
        * args.steps / total / 1e9
    if kind.endswith("_tc"):
        # INT8 tensor-core GEMM by exact digit-plane splitting: algorithmic
        # ops per launch = 2 M N K x S(S+1)/2 plane-pair products (S planes
        # recorded per launch: 4/8/14/28 for fp32/fp64/dd/qd with 8-bit
        # digits, 4/8/16/31 with 7-bit)
        S = S_used or {7: 4, 15: 8, 31: 16, 63: 31}[fin]
        pairs = S * (S + 1) / 2
        achieved = logical * pairs
        S7 = {7: 4, 15: 8, 31: 16, 63: 31}[fin]
        # the sustained probe peak for a kernel timed inside a long run (the
        # K steps last >= 1 s: the clock sits under the power cap, as in the
        # sustained probe); the burst peak otherwise (B200_PROFILING rule)
        long_run = total >= 1.0
        pk = peaks["int8_tops_sustained"] if long_run else peaks["int8_tops"]
        roof = {"bound": "tensor", "pipe": "int8 (tcgen05.mma kind::i8)", "achieved": achieved,
                "peak": pk, "peak_kind": "sustained (3 s back-to-back probe)" if long_run else "burst",
                "unit": "TOPS (int8)", "frac": achieved / pk,
                "frac_of_burst_peak": achieved / peaks["int8_tops"],
                "frac_7bit_equivalent": logical * S7 * (S7 + 1) / 2 / pk,
                "algorithmic_ops_per_launch": 2.0 * M * N * K * nb * pairs,
                "mean_launch_s": sec / cnt,
                "frac_note": "frac counts the S(S+1)/2 plane-pair products per output this launch executed; "
                             "frac_7bit_equivalent rates the same logical throughput in 7-bit plane pairs",
                "logical_tflops": logical, "logical_frac_of_format_peak": logical / peaks[fname],
                "peak_source": f"tcgen05 kind::i8 probe in bench.py on this GPU (burst {peaks['int8_tops']:.0f}, "
                               f"sustained {peaks['int8_tops_sustained']:.0f} TOPS; "
                               "MEASURED_PEAKS.json has no INT8 figure); format peaks from DFMA/FFMA probes "
                               f"(fp64 {peaks['fp64']:.2f} TF/s, Peak_dd = Peak_fp64/15, SURVEY 8d)"}
        NT = 16 if S > 16 else 32
        tiles = nb * (-(-M // 128)) * (-(-N // NT))
        ingest = tiles * (-(-K // 32)) * S * (128 + NT) * 32.0
        ach = ingest / (sec / cnt) / 1e12
        roof["ingest"] = {"achieved": ach, "peak": peaks["ingest_tbps"], "unit": "TB/s",
                          "frac": ach / peaks["ingest_tbps"], "bytes_per_launch": ingest}
        roof["digit_planes"] = S
        roof["digit_bits"] = db_used
    else:
        roof = {"bound": "fp64-pipe" if fname != "fp32" else "fp32-pipe", "achieved": logical, "peak": peaks[fname],
                "unit": "TFLOP/s (logical)", "frac": logical / peaks[fname], "mean_launch_s": sec / cnt,
                "peak_source": "FMA pipe microbenchmark in bench.py on this GPU"}
    if small:
        # the fused small-matrix evaluation: two launches around the host
        # planner, one CTA per matrix -- a latency-bound step; rated as the
        # evaluation's logical GEMM flops over the step against the fp64 pipe
        flops = sum(fs * c for c in gem.values())
        roof = {"bound": "latency", "achieved": flops / step_time / 1e12, "peak": peaks["fp64"],
                "unit": "TFLOP/s (logical fp64)", "frac": flops / step_time / 1e12 / peaks["fp64"],
                "mean_launch_s": None,
                "note": "K5 (csrc/small_ps.cuh): small_prepare_kernel + small_horner_kernel, one CTA per matrix, "
                        "operands in shared memory; one n = 32 matrix occupies one SM, so the step is launch / "
                        "host latency, not a pipe or HBM bound (DESIGN 6)",
                "peak_source": "FMA pipe microbenchmark in bench.py on this GPU"}
    kkey = (f"{kind} {fname}->{names[fout]} {M}x{N}x{K} x{nb}" if not small
            else "small_prepare_kernel + small_horner_kernel (fused PS, n <= 32)")
    traffic, tsrc = None, None
    try:   # committed ncu --set full capture of this kernel at this shape (profiles/traffic.json)
        tr = json.load(open(os.path.join(ROOT, "profiles", "traffic.json")))
        if kkey in tr:
            traffic = tr[kkey]["dram_bytes_per_launch"]
            tsrc = f"{tr[kkey]['capture']} ({tr[kkey]['kernel']}), bytes per launch"
    except Exception:
        pass
    roof.update({"kernel": kkey, "traffic": traffic, "traffic_source": tsrc,
                 "share_of_step": None if small else sec / args.steps / step_time,
                 "launches_per_step": per_step if small else cnt / args.steps,
                 "eval_frac": t_ideal / step_time,
                 "measured_in": "a second timed pass of the same K steps run eagerly (the value pass "
                                "replays CUDA graphs, whose kernels cannot be bracketed by events)"})
    spec = {k: spec1[k] - spec0[k] for k in spec1}
    line = {
        "metric": METRIC, "value": value, "unit": "evals/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "warmup_steps_run": warm_run, "ms_per_step": 1e3 * step_time,
        "step_ms": {"min": min(step_times), "median": float(np.median(step_times)), "max": max(step_times),
                    "slowest_step": int(np.argmax(step_times))},
        "higher_is_better": True,
        "scaling": wl.scaling, "vs_baseline": None, "dtype": names[plans[0].level_formats[0]],
        "data": "synthetic (seeded N(0,1) rescaled to the config's ||X||_1; BASELINE configs have no dataset)",
        "config": config_dict(name, world, args.scaling),
        "inputs": f"{P} distinct seeded input batches in HBM, step t reads batch t mod {P}",
        "plan": {"schedule_digits": [list(p.level_digits) for p in plans[:4]], "level_formats": fmts,
                 "gemms_per_step_per_gpu": gem, "speculation": spec,
                 "host_affinity": (f"{len(_NUMA_CPUS)} GPU-local CPUs (NVML affinity)" if _NUMA_CPUS else "unbound")},
        "gflops_effective": eff_gflops,
        "roofline": roof,
        "peaks_tflops": peaks,
        "e2e": {"value": e2e, "unit": "evals/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                "path": e2e_path, "link_gbs": link},
        "gpu_launches": launches,
        "gpu_launches_per_step": per_step,
        "clocks": clk,
    }
    if world == 1 and not args.no_cpu_baseline:
        try:
            _, line["cpu_baseline"] = reference_sample(name, 1, 0)
        except Exception as e:  # the baseline is reported, never required
            line["cpu_baseline"] = {"value": None, "error": str(e)[:200]}
        finally:
            if _NUMA_CPUS:
                os.sched_setaffinity(0, _NUMA_CPUS)
    print(json.dumps(line), flush=True)
    # release this config's pools before the next config
    wl = rep = None
    gc.unfreeze()
    gc.collect()
    torch.cuda.empty_cache()


_ORIG_AFFINITY = []
_NUMA_CPUS = []


def bind_to_gpu_numa(local_rank: int):
    """Pin this rank's host threads to the CPUs NVML reports as local to its
    GPU, so the pinned host buffers of the e2e stream are first-touched on
    the GPU's NUMA node (a far node measured 20-25K instead of 35K evals/s
    on the cfg2 host stream)."""
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
            _NUMA_CPUS[:] = cpus
    except Exception:
        pass


def _relaunch_under_torchrun(gpus: int) -> int:
    """`bench.py --gpus N` outside torchrun: one rank per GPU on this node."""
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", action="append", choices=sorted(CONFIGS),
                    help="config(s) to run, in order (default: cfg2 then the headline cfg5)")
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"],
                    help="batched configs at N>1: B matrices per rank (weak) or B/N (strong)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-probe", action="store_true", help="diagnostic: no per-launch events")
    ap.add_argument("--no-clocks", action="store_true", help="diagnostic: no nvidia-smi sampling")
    args = ap.parse_args()
    if args.warmup < 3:
        ap.error("--warmup must be >= 3")
    world = int(os.environ.get("WORLD_SIZE", "0"))
    if world == 0 and args.gpus > 1:
        sys.exit(_relaunch_under_torchrun(args.gpus))
    world = max(world, 1)
    if world != args.gpus:
        ap.error(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    names = args.config or list(DEFAULT_CONFIGS)
    if args.impl == "reference":
        for name in names:
            run_reference(name, args, rank, world)
        return
    bind_to_gpu_numa(local_rank)
    import torch
    torch.cuda.set_device(local_rank)
    dist = None
    if world > 1:
        os.environ.setdefault("NCCL_DEBUG", "INFO")          # communicator rank counts in the log
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    for name in names:
        run_ours(name, args, rank, world, local_rank, dist)
    if dist is not None:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
