import time, sys, os, json
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "."))
import numpy as np, torch
import paper_2312_17396_b200 as mp
torch.cuda.set_device(0)
def synth(n, t, seed):
    G = np.random.default_rng(seed).standard_normal((n, n)); return G * (t / np.abs(G).sum(0).max())
rng = np.random.default_rng(1000)
A = torch.from_numpy(np.stack([synth(1024, t, i) for i, t in enumerate(10.0 ** rng.uniform(-2, 3, 16))])).cuda()
ctx = mp.PrecisionCtx(31)
X1 = torch.from_numpy(synth(32, 0.5, 0)).cuda()
import gc
mode = sys.argv[1] if len(sys.argv) > 1 else ""
if mode == "freeze":
    gc.collect(); gc.freeze()
elif mode == "off":
    gc.disable()
print("gc mode", mode, "tracked objects", len(gc.get_objects()))
for name, fn in (("cfg3", lambda: mp.expm_ss(A, ctx, timing=True)), ("cfg1", lambda: mp.ps_mixed_exp(X1, 16, mp.PrecisionCtx(15), timing=True))):
    for i in range(12):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        rep = fn()
        torch.cuda.synchronize(); t1 = time.perf_counter()
        r0 = rep[0] if hasattr(rep, "__getitem__") and not hasattr(rep, "plan") else rep
        sec = rep.seconds if hasattr(rep, "seconds") else None
        print(name, i, f"{(t1-t0)*1e3:.2f} ms", {k: round(v*1e3, 2) for k, v in (sec or {}).items()}, flush=True)
