"""cProfile of the host side of pipeline.evaluate_host (cfg2, [32, 32])."""
import cProfile, pstats, sys, time
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
chunks = [32, 32] if len(sys.argv) < 2 else eval(sys.argv[1])
streams = 1 if len(sys.argv) < 3 else int(sys.argv[2])
for _ in range(5):
    pipeline.evaluate_host(fn, Xh, out, chunks, streams=streams)
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
t0 = time.perf_counter()
for _ in range(20):
    pipeline.evaluate_host(fn, Xh, out, chunks, streams=streams)
    torch.cuda.synchronize()
t1 = time.perf_counter()
pr.disable()
print(f"{(t1-t0)/20*1e3:.3f} ms per call (profiled)")
pstats.Stats(pr).sort_stats("tottime").print_stats(22)
