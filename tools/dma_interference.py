"""Dev tool: device-resident cfg2 steps alone and with concurrent pinned H2D / D2H copies of the
e2e stream's sizes on other streams (does DMA traffic slow the kernels?)."""
import os, sys, threading
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
import paper_2312_17396_b200 as mp

K = 20
wl = bench.Workload("cfg2", 0, 1, torch, mp, "weak", K, 0)
for i in range(4):
    wl.step(wl.Xd[i])
torch.cuda.synchronize()
hu = torch.empty(32 << 17, dtype=torch.float64).pin_memory(); du = torch.empty_like(hu, device="cuda")
hd = torch.empty(64 << 17, dtype=torch.float64).pin_memory(); dd = torch.empty_like(hd, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()

def steps(copies):
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for t in range(K):
        if copies & 1:
            with torch.cuda.stream(s1): du.copy_(hu, non_blocking=True)
        if copies & 2:
            with torch.cuda.stream(s2): hd.copy_(dd, non_blocking=True)
        wl.step(wl.Xd[t % wl.pool])
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / K

for c, lab in ((0, "no copies"), (1, "H2D 32 MiB per step"), (2, "D2H 64 MiB per step"), (3, "both")):
    print(f"{lab}: {steps(c):.3f} ms per step", flush=True)
