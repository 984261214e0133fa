"""Dev tool: spread of the cfg2 e2e stream throughput over repeated calls."""
import os, sys, gc
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
import paper_2312_17396_b200 as mp
from paper_2312_17396_b200 import pipeline as pl

wl = bench.Workload("cfg2", 0, 1, torch, mp, "weak", 10, 0)
K = 10
Xbig = torch.cat([wl.Xpin[t % wl.pool] for t in range(K)]).pin_memory()
out = torch.empty((2,) + tuple(Xbig.shape), dtype=torch.float64).pin_memory()
sub = pl.mixed_exp(wl.m, wl.ctx, timing=False)
sizes = [32, 32] * K
pl.evaluate_host(sub, Xbig, out, sizes, streams=2, window=6)
torch.cuda.synchronize()
if len(sys.argv) > 1 and sys.argv[1] == "freeze":
    gc.collect()
    gc.freeze()
vals = []
for _ in range(20):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    pl.evaluate_host(sub, Xbig, out, sizes, streams=2, window=6)
    b.record(); b.synchronize()
    vals.append(64 * K / (a.elapsed_time(b) * 1e-3))
print(" ".join(f"{v/1e3:.1f}K" for v in vals))
