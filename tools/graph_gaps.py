"""GPU-side timeline of a graphed cfg2 evaluation: pre graph, host planning
gap, Horner graph (events around CUDAGraph.replay)."""
import os, sys, time
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
import paper_2312_17396_b200 as mp

name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
wl = bench.Workload(name, 0, 1, torch, mp, "weak", 12, 0)
for i in range(3):
    wl.step(wl.Xd[i])
torch.cuda.synchronize()
orig = torch.cuda.CUDAGraph.replay
marks = []


def timed(self):
    a = torch.cuda.Event(enable_timing=True); a.record()
    orig(self)
    b = torch.cuda.Event(enable_timing=True); b.record()
    marks.append((a, b))


torch.cuda.CUDAGraph.replay = timed
rows = []
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
for i in range(10):
    marks.clear()
    flush.zero_(); torch.cuda.synchronize()
    s = torch.cuda.Event(enable_timing=True); s.record()
    rep = wl.step(wl.Xd[3 + i % 9])
    e = torch.cuda.Event(enable_timing=True); e.record(); e.synchronize()
    t = [(s.elapsed_time(a), s.elapsed_time(b)) for a, b in marks]
    rows.append([s.elapsed_time(e)] + [x for ab in t for x in ab])
r = np.median(np.array(rows), axis=0)
print(f"{name}: total {r[0]:.3f} ms; pre graph {r[1]:.3f}->{r[2]:.3f} ms; post graph {r[3]:.3f}->{r[4]:.3f} ms; "
      f"GPU gap (host planning) {r[3]-r[2]:.3f} ms; tail after post {r[0]-r[4]:.3f} ms")
