"""e2e (pinned host in -> pinned host out) time of cfg2 vs chunk count."""
import sys, time
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_2312_17396_b200 as m
from paper_2312_17396_b200 import pipeline

B, n = 64, 256
rng = np.random.default_rng(0)
X = rng.standard_normal((B, n, n))
X /= np.abs(X).sum(axis=1).max(axis=1)[:, None, None]
Xh = torch.from_numpy(X).pin_memory()
out = torch.empty((2, B, n, n), dtype=torch.float64).pin_memory()
ctx = m.PrecisionCtx(31)
fn = pipeline.mixed_exp(30, ctx, timing=False)
cases = [([32, 32], 1, False)] + [(c, 2, True) for c in ([16] * 4, [24, 20, 12, 8], [20, 20, 16, 8], [16, 16, 16, 8, 8],
                                                    [8, 16, 16, 16, 8], [12, 16, 16, 12, 8], [20, 16, 16, 12])]
for chunks, streams, ahead in cases:
    for _ in range(3):
        pipeline.evaluate_host(fn, Xh, out, chunks, streams=streams, ahead=ahead)
    torch.cuda.synchronize()
    ts = []
    for _ in range(10):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); pipeline.evaluate_host(fn, Xh, out, chunks, streams=streams, ahead=ahead); b.record(); b.synchronize()
        ts.append(a.elapsed_time(b))
    print(f"chunks={chunks} streams={streams} ahead={ahead} median {np.median(ts):.3f} ms  min {min(ts):.3f}  -> {B/np.median(ts)*1e3:.0f} evals/s", flush=True)

import time as _t
for chunks, streams, ahead in (([16] * 4, 2, True), ([24, 20, 12, 8], 2, True)):
    pipeline.evaluate_host(fn, Xh, out, chunks, streams=streams, ahead=ahead)
    torch.cuda.synchronize()
    tr = []
    a = torch.cuda.Event(enable_timing=True); a.record()
    h0 = _t.perf_counter()
    pipeline.evaluate_host(fn, Xh, out, chunks, trace=tr, streams=streams, ahead=ahead)
    h1 = _t.perf_counter()
    b = torch.cuda.Event(enable_timing=True); b.record(); b.synchronize()
    print(f"--- chunks={chunks} total {a.elapsed_time(b):.3f} ms, host returned at {(h1-h0)*1e3:.3f} ms")
    print("  " + "  ".join(f"{l}:{a.elapsed_time(e):.2f}" for l, e, _ in tr))
    print("  host " + "  ".join(f"{l}:{(t - h0) * 1e3:.2f}" for l, _, t in tr))

# correctness: every (chunks, streams) gives the same bits
ref = out.clone()
pipeline.evaluate_host(fn, Xh, out, 1)
torch.cuda.synchronize()
ref = out.clone()
for chunks, streams, ahead in cases:
    out.zero_()
    pipeline.evaluate_host(fn, Xh, out, chunks, streams=streams, ahead=ahead)
    torch.cuda.synchronize()
    print(f"bitwise equal chunks={chunks} streams={streams} ahead={ahead}: {bool(torch.equal(out, ref))}")
