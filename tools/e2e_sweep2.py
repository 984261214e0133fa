"""Dev tool: cfg2 e2e host stream with tapered chunk lists (small chunks at
the head and tail of the stream, full batches in the middle)."""
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
cases = [
    ([64] * K, 3),
    ([16, 48] + [64] * (K - 2) + [48, 16], 3),
    ([16, 48] + [64] * (K - 2) + [48, 16], 4),
    ([32, 32] + [64] * (K - 2) + [32, 32], 3),
    ([16, 16, 32] + [64] * (K - 2) + [32, 16, 16], 4),
    ([32, 32] * K, 6),
    ([64] * K, 4),
    ([64] * K, 6),
    ([16] * (4 * K), 12),
]
for sizes, win in cases:
    assert sum(sizes) == 64 * K
    pl.evaluate_host(sub, Xbig, out, sizes, streams=2, window=win)
    torch.cuda.synchronize()
    best = []
    for _ in range(3):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        pl.evaluate_host(sub, Xbig, out, sizes, streams=2, window=win)
        b.record(); b.synchronize()
        best.append(64 * K / (a.elapsed_time(b) * 1e-3))
    print(sizes[:4], "...", win, " ".join(f"{v:.0f}" for v in best), flush=True)
