"""Dev tool: cProfile of one steady-state evaluation (host-side overhead)."""
import cProfile, os, pstats, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2312_17396_b200 as mp
torch.cuda.set_device(0)
def synth(n, t, seed):
    G = np.random.default_rng(seed).standard_normal((n, n)); return G * (t / np.abs(G).sum(0).max())
cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
if cfg == "cfg3":
    rng = np.random.default_rng(1000)
    A = torch.from_numpy(np.stack([synth(1024, t, i) for i, t in enumerate(10.0 ** rng.uniform(-2, 3, 16))])).cuda()
    fn = lambda: mp.expm_ss(A, mp.PrecisionCtx(31), timing=False)
else:
    X = torch.from_numpy(np.stack([synth(256, 1.0, i) for i in range(64)])).cuda()
    fn = lambda: mp.ps_mixed_exp(X, 30, mp.PrecisionCtx(31), timing=False)
for _ in range(3):
    fn()
torch.cuda.synchronize()
t0 = time.perf_counter(); fn(); torch.cuda.synchronize(); print("step", (time.perf_counter() - t0) * 1e3, "ms")
pr = cProfile.Profile()
pr.enable(); fn(); torch.cuda.synchronize(); pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(25)
