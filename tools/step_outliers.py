"""Dev tool: where a rare slow cfg2 step spends its time (host wall clock between the phases of
graphs.submit / finish next to the step's CUDA-event time)."""
import gc, os, sys, time
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
import paper_2312_17396_b200 as mp
from paper_2312_17396_b200 import graphs

N = int(sys.argv[1]) if len(sys.argv) > 1 else 3000
wl = bench.Workload("cfg2", 0, 1, torch, mp, "weak", 20, 5)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
P = wl.pool
marks = []
orig_finish, orig_submit = graphs.finish, graphs.submit

def submit(*a, **k):
    t0 = time.perf_counter(); p = orig_submit(*a, **k); marks.append(("submit", t0, time.perf_counter())); return p

def finish(p, run_post, clone=True):
    t0 = time.perf_counter()
    p.ready.synchronize()
    t1 = time.perf_counter()
    def rp(prep, norms):
        ta = time.perf_counter(); out = run_post(prep, norms); marks.append(("plan", ta, time.perf_counter())); return out
    out = orig_finish(p, rp, clone)
    marks.append(("finish", t0, t1, time.perf_counter()))
    return out
graphs.submit, graphs.finish = submit, finish
for t in range(50):
    wl.step(wl.Xd[t % P])
torch.cuda.synchronize()
gc.collect(); gc.freeze(); gc.disable()
rows = []
for t in range(N):
    flush.zero_(); torch.cuda.synchronize()
    del marks[:]
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    h0 = time.perf_counter()
    a.record(); rep = wl.step(wl.Xd[t % P]); b.record()
    h1 = time.perf_counter()
    b.synchronize()
    h2 = time.perf_counter()
    ev = a.elapsed_time(b)
    if ev > 2.0:
        d = {m[0]: m for m in marks}
        s, f, pl = d.get("submit"), d.get("finish"), d.get("plan")
        print(f"step {t}: event {ev:.2f} ms; host: call {1e3*(h1-h0):.2f} ms, final sync {1e3*(h2-h1):.2f}; "
              f"submit {1e3*(s[2]-s[1]):.2f} (starts +{1e3*(s[1]-h0):.2f}); wait norms {1e3*(f[2]-f[1]):.2f}; "
              f"plan {1e3*(pl[2]-pl[1]):.2f}; rest of finish {1e3*(f[3]-f[2]-(pl[2]-pl[1])):.2f}; after finish {1e3*(h1-f[3]):.2f}", flush=True)
    rows.append(ev)
r = np.array(rows)
print(f"{N} steps: median {np.median(r):.3f} ms, p99 {np.percentile(r, 99):.3f}, max {r.max():.2f}; steps > 2 ms: {(r > 2).sum()}, "
      f"mean {r.mean():.3f} ms")
