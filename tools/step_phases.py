"""Dev tool: per-step wall time and CUDA-event phase buckets for cfg2."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2312_17396_b200 as mp
torch.cuda.set_device(0)
def synth(n, t, seed):
    G = np.random.default_rng(seed).standard_normal((n, n)); return G * (t / np.abs(G).sum(0).max())
X = torch.from_numpy(np.stack([synth(256, 1.0, i) for i in range(64)])).cuda()
ctx = mp.PrecisionCtx(31)
for i in range(15):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    rep = mp.ps_mixed_exp(X, 30, ctx, timing=True)
    torch.cuda.synchronize(); t1 = time.perf_counter()
    print(i, f"{(t1-t0)*1e3:.2f} ms", {k: round(v*1e3, 2) for k, v in rep.seconds.items()}, flush=True)
