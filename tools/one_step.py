"""Run K eager steps of a bench config (for ncu launch lists and
compute-sanitizer): MPPS_GRAPHS=0 python tools/one_step.py cfg2 4 [batch]"""
import sys
import torch
sys.path.insert(0, ".")
import bench
import paper_2312_17396_b200 as mp

name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
k = int(sys.argv[2]) if len(sys.argv) > 2 else 4
if len(sys.argv) > 3:                      # smaller batch (sanitizer runs)
    bench.CONFIGS[name] = dict(bench.CONFIGS[name], batch=int(sys.argv[3]))
wl = bench.Workload(name, 0, 1, torch, mp, "weak", k, 0)
for t in range(k):
    wl.step(wl.Xd[t % wl.pool])
torch.cuda.synchronize()
print("ok")
