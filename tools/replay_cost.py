"""Host cost of CUDAGraph.replay for the cfg2 graphs (idle GPU vs busy GPU)."""
import sys, time
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_2312_17396_b200 as m
from paper_2312_17396_b200 import graphs

B, n = 64, 256
rng = np.random.default_rng(0)
X = rng.standard_normal((B, n, n))
X /= np.abs(X).sum(axis=1).max(axis=1)[:, None, None]
Xd = torch.from_numpy(X).cuda()
ctx = m.PrecisionCtx(31)
for _ in range(3):
    m.ps_mixed_exp(Xd, 30, ctx, timing=False)
torch.cuda.synchronize()
g = next(iter(graphs._CACHE.values()))
post = next(iter(g.post.values()))[0]
for label, gr in (("pre", g.pre), ("post", post)):
    torch.cuda.synchronize()
    t = []
    for _ in range(10):
        torch.cuda.synchronize()
        t0 = time.perf_counter(); gr.replay(); t.append(time.perf_counter() - t0)
    torch.cuda.synchronize()
    print(f"{label}: idle-GPU replay host cost median {np.median(t)*1e6:.1f} us")
    t = []
    torch.cuda.synchronize()
    for _ in range(10):
        t0 = time.perf_counter(); gr.replay(); t.append(time.perf_counter() - t0)
    torch.cuda.synchronize()
    print(f"{label}: back-to-back replay host cost " + " ".join(f"{x*1e6:.0f}" for x in t))
big = torch.empty(1 << 28, dtype=torch.uint8, device="cuda")
t = []
for _ in range(10):
    torch.cuda._sleep(2_000_000)
    t0 = time.perf_counter(); g.pre.replay(); t.append(time.perf_counter() - t0)
torch.cuda.synchronize()
print("pre replay behind a busy stream: " + " ".join(f"{x*1e6:.0f}" for x in t))
s2 = torch.cuda.Stream()
t = []
for _ in range(5):
    with torch.cuda.stream(s2):
        g.pre.replay()
    t0 = time.perf_counter(); post.replay(); t.append(time.perf_counter() - t0)
torch.cuda.synchronize()
print("post replay while pre runs on another stream: " + " ".join(f"{x*1e6:.0f}" for x in t))

from paper_2312_17396_b200 import pipeline
Xh = torch.from_numpy(X).pin_memory()
out = torch.empty((2, B, n, n), dtype=torch.float64).pin_memory()
fn = pipeline.mixed_exp(30, ctx, timing=False)
orig = torch.cuda.CUDAGraph.replay
log = []
T0 = [0.0]
def timed(self):
    t0 = time.perf_counter(); orig(self); log.append((id(self) % 10000, (t0 - T0[0]) * 1e3, (time.perf_counter() - t0) * 1e6))
torch.cuda.CUDAGraph.replay = timed
origsync = torch.cuda.Event.synchronize
def tsync(self):
    t0 = time.perf_counter(); origsync(self); log.append(("evsync", (t0 - T0[0]) * 1e3, (time.perf_counter() - t0) * 1e6))
torch.cuda.Event.synchronize = tsync
for chunks in ([32, 32], [32, 32], [32, 32]):
    torch.cuda.synchronize()
    log.clear()
    T0[0] = time.perf_counter()
    pipeline.evaluate_host(fn, Xh, out, chunks)
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(f"host {(t1-T0[0])*1e3:.2f} ms, sync done {(t2-T0[0])*1e3:.2f}: " + "  ".join(f"{a}@{b:.2f}:{c:.0f}us" for a, b, c in log))
