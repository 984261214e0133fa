"""Dev tool: e2e (host stream) throughput of cfg2 for chunk sizes / windows."""
import os, sys
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
for chunks, win in (([16] * 4, 8), ([16] * 4, 12), ([32, 32], 4), ([32, 32], 6), ([64], 2), ([64], 3),
                    ([24, 24, 16], 6)):
    sizes = chunks * K
    pl.evaluate_host(sub, Xbig, out, sizes, streams=2, window=win)
    torch.cuda.synchronize()
    best = 0
    for _ in range(2):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        pl.evaluate_host(sub, Xbig, out, sizes, streams=2, window=win)
        b.record(); b.synchronize()
        best = max(best, 64 * K / (a.elapsed_time(b) * 1e-3))
    print(chunks, win, f"{best:.0f} evals/s", flush=True)
