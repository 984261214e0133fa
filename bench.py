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

CFG = dict(workload="cfg2: Taylor exp m=30 s=6, batch 64 x n=256, ||X||_1=1, dd working (mixed dd/fp64/fp32 levels)",
           batch=64, n=256, m=30, digits=31, norm=1.0)
METRIC = "matrix-polynomial evals/sec"


def synth(n, target, seed):
    G = np.random.default_rng(seed).standard_normal((n, n))
    return G * (target / np.abs(G).sum(axis=0).max())


def make_batch(rank, batch, n, norm):
    return np.stack([synth(n, norm, rank * batch + i) for i in range(batch)])


# ----------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
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
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                smax = float(parts[1])
            except ValueError:
                continue
            for nm, v in zip(names, parts[4:8]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm)}


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


def cpu_baseline_sample(cores_hint=None):
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
def run_ours(args, rank, world, local_rank):
    import torch
    import paper_2312_17396_b200 as mp
    from paper_2312_17396_b200 import _lib
    from paper_2312_17396_b200.precision import MatBatch

    torch.cuda.set_device(local_rank)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    ctx = mp.PrecisionCtx(CFG["digits"])
    B, n, m = CFG["batch"], CFG["n"], CFG["m"]
    Xh = make_batch(rank, B, n, CFG["norm"])
    Xd = torch.from_numpy(Xh).cuda()
    Xpin = torch.from_numpy(Xh).pin_memory()
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
    h = _lib.handle_for()

    def step(X):
        return mp.ps_mixed_exp(X, m, ctx, timing=False)

    for _ in range(args.warmup):
        rep = step(Xd)
    torch.cuda.synchronize()
    plan0 = rep[0].plan
    gem = honest_gemms(plan0)

    def barrier():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    # ---- device-resident timed region (value) ----
    clocks = ClockSampler(local_rank) if rank == 0 else None
    barrier()
    if clocks:
        clocks.start()
    h.probe = {}
    l0 = h.launches
    total = 0.0
    for _ in range(args.steps):
        flush.zero_()  # 256 MiB write between steps: L2 (126 MB) flushed
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        rep = step(Xd)
        b.record()
        b.synchronize()
        total += a.elapsed_time(b) * 1e-3
    barrier()
    launches = (h.launches - l0 - 0) / args.steps
    probe = h.probe
    h.probe = None
    clk = clocks.stop() if clocks else None
    # flush.zero_ is a torch kernel, not ours; launches counts libmpps kernels only

    # ---- end-to-end through the public API with host buffers ----
    out_host = torch.empty((2, B, n, n), dtype=torch.float64).pin_memory()
    e2e_total = 0.0
    for i in range(args.steps + 1):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        rep = step(Xpin)
        out_host.copy_(rep.result.data, non_blocking=True)
        b.record()
        b.synchronize()
        if i > 0:
            e2e_total += a.elapsed_time(b) * 1e-3
    h2d = Xh.nbytes
    d2h = out_host.numel() * 8

    t = torch.tensor([total, e2e_total], dtype=torch.float64, device="cuda")
    if dist is not None:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    total, e2e_total = float(t[0]), float(t[1])
    if rank != 0:
        dist.destroy_process_group()
        return
    evals = B * world * args.steps
    value = evals / total
    e2e = B * world * args.steps / e2e_total

    # ---- roofline of the dominant kernel (dd power GEMM, batch 64) ----
    peaks = measure_peaks(torch, h)
    by_key = {}
    for key, evs in probe.items():
        durs = [x.elapsed_time(y) * 1e-3 for x, y in evs]
        by_key[key] = (len(durs), sum(durs))
    dom = max(by_key.items(), key=lambda kv: kv[1][1])
    (kind, fin, fout, M, N, K, nb), (cnt, sec) = dom
    fname = {7: "fp32", 15: "fp64", 31: "dd", 63: "qd"}[fin]
    flops_per_launch = 2.0 * M * N * K * nb
    achieved = flops_per_launch / (sec / cnt) / 1e12
    peak = peaks[fname]
    step_time = total / args.steps
    dom_share = sec / args.steps / step_time
    # whole-evaluation roofline: T_ideal = sum_P 2n^3 #GEMM_P / Peak_P
    t_ideal = sum(2.0 * n ** 3 * c * B / (peaks[f] * 1e12) for f, c in gem.items())
    eff_gflops = sum(2.0 * n ** 3 * c for c in gem.values()) * B * world * args.steps / total / 1e9

    line = {
        "metric": METRIC, "value": value, "unit": "evals/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * step_time, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "dd",
        "data": "synthetic (seeded N(0,1) rescaled to ||X||_1=1, seeds rank*64+i)",
        "config": {"workload": CFG["workload"], "batch_per_gpu": B, "n": n, "m": m, "digits": CFG["digits"],
                   "schedule_digits": list(plan0.level_digits),
                   "level_formats": rep[0].diagnostics["level_formats"],
                   "gemms_per_eval": gem, "parallelism": f"batch-sharded x{world}",
                   "l2": "256 MiB buffer written between timed steps (L2 flushed)"},
        "gflops_effective": eff_gflops,
        "roofline": {"bound": "fp64-pipe", "kernel": f"{kind} {fname}->{ {7: 'fp32', 15: 'fp64', 31: 'dd', 63: 'qd'}[fout]} "
                                                     f"{M}x{N}x{K} x{nb}",
                     "achieved": achieved, "peak": peak, "unit": "TFLOP/s (logical)",
                     "frac": achieved / peak, "traffic": None, "share_of_step": dom_share,
                     "launches_per_step": cnt / args.steps,
                     "peak_source": "FMA pipe microbenchmark in bench.py on this GPU "
                                    f"(fp64 {peaks['fp64']:.2f} TF/s, fp32 {peaks['fp32']:.2f} TF/s); "
                                    "Peak_dd = Peak_fp64/15 (SURVEY 8d k_dd=15); MEASURED_PEAKS.json "
                                    "holds only HBM and bf16",
                     "eval_frac": t_ideal / step_time},
        "peaks_tflops": peaks,
        "e2e": {"value": e2e, "unit": "evals/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h},
        "gpu_launches": launches,
        "clocks": clk,
    }
    if world == 1 and not args.no_cpu_baseline:
        try:
            line["cpu_baseline"] = cpu_baseline_sample()
        except Exception as e:  # the baseline is reported, never required
            line["cpu_baseline"] = {"value": None, "error": str(e)[:200]}
    print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
    else:
        run_ours(args, rank, world, local_rank)


if __name__ == "__main__":
    main()
