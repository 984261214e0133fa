"""Dev tool: event timeline of the cfg2 e2e host stream (K steps, [32, 32]
chunks, window 6): per-chunk upload / pre / post / download intervals and
the busy fraction of each engine."""
import os, sys
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
sizes = [64] * K if "full" in sys.argv else [32, 32] * K
ST = 1 if "full" in sys.argv else 2
WIN = 4 if "full" in sys.argv else 6
for _ in range(2):
    pl.evaluate_host(sub, Xbig, out, sizes, streams=ST, ahead=True, window=WIN)
torch.cuda.synchronize()
tr = []
t0 = torch.cuda.Event(enable_timing=True)
t0.record()
th0 = __import__('time').perf_counter()
pl.evaluate_host(sub, Xbig, out, sizes, streams=ST, ahead=True, window=WIN, trace=tr)
th1 = __import__('time').perf_counter()
t1 = torch.cuda.Event(enable_timing=True)
t1.record()
torch.cuda.synchronize()
total = t0.elapsed_time(t1)
ev = {lab: (t0.elapsed_time(e), host) for lab, e, host in tr}
h0 = min(h for _, h in ev.values())
rows = []
for c in range(len(sizes)):
    g = lambda k: (ev.get(f"{k}{c}<", (np.nan, 0))[0], ev.get(f"{k}{c}>", (np.nan, 0))[0])
    rows.append((c,) + g("up") + g("pre") + g("post") + g("down") + ((ev[f"post{c}<"][1] - h0) * 1e3,))
print(f"total {total:.3f} ms for {K} steps -> {64 * K / total * 1e3:.0f} evals/s; host returned after {(th1-th0)*1e3:.3f} ms")
print("chunk  up[<,>]  pre[<,>] post[<,>] down[<,>]  host_post_issue(ms)")
for r in rows[:12] + rows[-4:]:
    print(" ".join(f"{x:7.3f}" if isinstance(x, float) else f"{x:3d}" for x in r))
down = sum(r[8] - r[7] for r in rows)
up = sum(r[2] - r[1] for r in rows)
print(f"download busy {down:.3f} ms, upload busy {up:.3f} ms of {total:.3f}")
