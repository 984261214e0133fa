"""Dev tool: cfg2 e2e host stream, chunk sizes x streams x window (after the persistent kernels)."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
import paper_2312_17396_b200 as mp
from paper_2312_17396_b200 import pipeline as pl

K = 20
wl = bench.Workload("cfg2", 0, 1, torch, mp, "weak", K, 0)
Xbig = torch.cat([wl.Xpin[t % wl.pool] for t in range(K)]).pin_memory()
out = torch.empty((2,) + tuple(Xbig.shape), dtype=torch.float64).pin_memory()
sub = pl.mixed_exp(wl.m, wl.ctx, timing=False)
cases = [([64] * K, 1, 3), ([64] * K, 1, 4), ([64] * K, 2, 4), ([32, 32] * K, 2, 6), ([32, 32] * K, 1, 6),
         ([32, 32] * K, 2, 8), ([64] * K, 1, 6)]
for sizes, streams, win in cases:
    pl.evaluate_host(sub, Xbig, out, sizes, streams=streams, ahead=True, window=win)
    torch.cuda.synchronize()
    best = []
    for _ in range(3):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        pl.evaluate_host(sub, Xbig, out, sizes, streams=streams, ahead=True, window=win)
        b.record(); b.synchronize()
        best.append(64 * K / (a.elapsed_time(b) * 1e-3))
    print(sizes[:2], "streams", streams, "window", win, " ".join(f"{v:.0f}" for v in best), flush=True)
