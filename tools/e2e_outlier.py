"""Dev tool: find the stall in slow cfg2 e2e host-stream calls: the largest
host-side gaps between consecutive pipeline marks."""
import os, sys, time, gc
import numpy as np
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
gcs = []
gc.callbacks.append(lambda phase, info: gcs.append((phase, info.get("generation"), time.perf_counter())))
for it in range(20):
    tr = []
    gcs.clear()
    t0 = time.perf_counter()
    pl.evaluate_host(sub, Xbig, out, sizes, streams=2, window=6, trace=tr)
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) * 1e3
    hs = [h for _, _, h in tr]
    gaps = sorted(((hs[i + 1] - hs[i]) * 1e3, tr[i][0], tr[i + 1][0]) for i in range(len(hs) - 1))[-3:]
    ngc = [(p, g, round((t - t0) * 1e3, 2)) for p, g, t in gcs]
    print(f"{it:2d} {dt:7.2f} ms  host gaps {[(round(a, 2), b, c) for a, b, c in gaps]}  gc {ngc}", flush=True)
