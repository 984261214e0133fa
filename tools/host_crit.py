"""Dev tool: host time of the post-norm critical path of a graphed cfg2 step
(norms ready -> result enqueued), per phase, with perf_counter."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench
import paper_2312_17396_b200 as mp
from paper_2312_17396_b200 import engine, graphs, planner

wl = bench.Workload("cfg2", 0, 1, torch, mp, "weak", 10, 0)
for _ in range(4):
    wl.step(wl.Xd)
torch.cuda.synchronize()
T = {}
def wrap(mod, name):
    f = getattr(mod, name)
    def g(*a, **k):
        t = time.perf_counter(); r = f(*a, **k); T[name] = T.get(name, 0) + time.perf_counter() - t; return r
    setattr(mod, name, g)
for mod, name in ((engine, "plan_digits_batch"), (engine, "_structure"), (engine, "_selections"),
                  (engine, "_graphed_reports"), (graphs, "finish"), (graphs, "submit")):
    wrap(mod, name)
N = 20
t0 = time.perf_counter()
for _ in range(N):
    wl.step(wl.Xd)
torch.cuda.synchronize()
tot = (time.perf_counter() - t0) / N
print(f"wall per step {tot*1e6:.0f} us; " + ", ".join(f"{k} {v/N*1e6:.0f} us" for k, v in T.items()))
