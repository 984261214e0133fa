"""Run K eager steps of a bench config (for ncu launch lists):
MPPS_GRAPHS=0 python tools/one_step.py cfg2 4"""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import bench
import paper_2312_17396_b200 as mp

name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
k = int(sys.argv[2]) if len(sys.argv) > 2 else 4
wl = bench.Workload(name, 0, 1, torch, mp)
for _ in range(k):
    wl.step(wl.Xd)
torch.cuda.synchronize()
print("ok")
