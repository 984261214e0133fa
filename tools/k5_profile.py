"""Dev tool: host-side profile of the cfg1 (K5) evaluation."""
import cProfile
import pstats
import sys
import time
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_2312_17396_b200 as mp
sys.path.insert(0, "tests")
from _util import synth

X = torch.from_numpy(synth(32, 0.5, 0)).cuda()
ctx = mp.PrecisionCtx(15)
for _ in range(20):
    mp.ps_mixed_exp(X, 16, ctx, timing=False)
torch.cuda.synchronize()
t = time.perf_counter()
N = 200
for _ in range(N):
    mp.ps_mixed_exp(X, 16, ctx, timing=False)
torch.cuda.synchronize()
print(f"wall per eval {1e6 * (time.perf_counter() - t) / N:.1f} us")
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
mp.ps_mixed_exp(X, 16, ctx, timing=False)
b.record()
b.synchronize()
print(f"event-timed eval {1e3 * a.elapsed_time(b):.1f} us")
pr = cProfile.Profile()
pr.enable()
for _ in range(N):
    mp.ps_mixed_exp(X, 16, ctx, timing=False)
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(25)
