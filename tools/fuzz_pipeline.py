"""Dev tool: random host-stream configurations (chunk sizes, streams, ahead / window modes, heterogeneous
norms so that plan structures change between chunks: speculation hits and misses, dd re-assembly) against
one direct device-resident call, bitwise."""
import sys, os, time
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import paper_2312_17396_b200 as mp
from paper_2312_17396_b200 import pipeline as pl, graphs
from _util import synth

N = int(sys.argv[1]) if len(sys.argv) > 1 else 60
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 0)
bad = 0
t0 = time.time()
for it in range(N):
    d = int(rng.choice([15, 31, 31]))
    n = int(rng.choice([8, 24, 40, 64, 96]))
    B = int(rng.integers(3, 25))
    m = int(rng.choice([9, 16, 18, 24, 30]))
    general = bool(rng.integers(2))
    lo, hi = sorted(rng.uniform(-4, 0.9, size=2))
    norms = 10.0 ** rng.uniform(lo, hi, size=B)
    X = np.stack([synth(n, float(norms[b]), int(rng.integers(1 << 30))) for b in range(B)])
    ctx = mp.PrecisionCtx(d)
    W = {15: 1, 31: 2}[d]
    k = int(rng.integers(1, min(B, 6) + 1))
    cuts = sorted(rng.choice(np.arange(1, B), size=k - 1, replace=False).tolist()) if k > 1 else []
    sizes = [b - a for a, b in zip([0] + cuts, cuts + [B])]
    streams = int(rng.integers(1, 3))
    ahead = bool(rng.integers(2)) if streams == 1 else True
    window = None if (not ahead or rng.integers(2)) else int(rng.integers(1, k + 1))
    tag = f"#{it} d={d} n={n} B={B} m={m} {'cos' if general else 'exp'} sizes={sizes} streams={streams} ahead={ahead} window={window}"
    try:
        series = mp.taylor_cos_coeffs(m)
        direct = (mp.ps_mixed_general(X, series, ctx) if general else mp.ps_mixed_exp(X, m, ctx)).result.data.clone()
        Xh = torch.from_numpy(X).pin_memory()
        out = torch.empty((W, B, n, n), dtype=torch.float64).pin_memory()
        sub = pl.mixed_general(series, ctx, timing=False) if general else pl.mixed_exp(m, ctx, timing=False)
        for rep_i in range(2):      # second pass: every graph replays, speculation from the previous chunk
            out.zero_()
            reps = pl.evaluate_host(sub, Xh, out, sizes, streams=streams, ahead=ahead, window=window)
            torch.cuda.synchronize()
            if not torch.equal(out, direct.cpu()):
                bad += 1
                print("MISMATCH", tag, "pass", rep_i, float((out - direct.cpu()).abs().max()), flush=True)
                break
    except Exception as e:
        bad += 1
        print("EXC", tag, type(e).__name__, str(e)[:200], flush=True)
print(f"{N} configurations, {bad} failures, {time.time() - t0:.0f} s; speculation {graphs.speculation_stats()}")
