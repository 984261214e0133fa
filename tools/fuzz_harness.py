"""Dev tool: the accuracy callers (harness.compare: mixed and fixed evaluations against reference_eval at
2x the digits) on random batches -- the reference's acceptance criterion C6 (acceptance.py:167-206):
eps_mixed <= max(10 r n u, 10 eps_fixed) for every case -- and with_bound reports (a bound or
BoundInvalidError, nothing else)."""
import sys, os, time
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import paper_2312_17396_b200 as mp
from paper_2312_17396_b200 import harness
from _util import synth

N = int(sys.argv[1]) if len(sys.argv) > 1 else 60
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 0)
bad = 0
within = total = 0
t0 = time.time()
for it in range(N):
    d = int(rng.choice([15, 31]))
    n = int(rng.integers(2, 60))
    B = int(rng.integers(1, 5))
    m = int(rng.integers(2, 36))
    kind = str(rng.choice(["exp", "cos"]))
    norms = 10.0 ** rng.uniform(-3, 0.7, size=B)
    X = np.stack([synth(n, float(norms[b]), int(rng.integers(1 << 30))) for b in range(B)])
    ctx = mp.PrecisionCtx(d)
    tag = f"#{it} {kind} d={d} n={n} B={B} m={m} lognorms={np.round(np.log10(norms), 1)}"
    try:
        series = mp.taylor_exp_coeffs(m) if kind == "exp" else mp.taylor_cos_coeffs(m)
        recs = harness.compare(X, series, ctx, m=m if kind == "exp" else None)
        for b, rec in enumerate(recs):
            total += 1
            gate = 10 * max(rec["rnu"], 10.0 ** -d)
            within += rec["eps_mixed"] <= gate
            if not rec["eps_mixed"] <= max(gate, 10 * rec["eps_fixed"]):
                bad += 1
                print("C6", tag, b, rec["eps_mixed"], rec["eps_fixed"], rec["rnu"], flush=True)
        try:
            rb = mp.ps_mixed_exp(X, m, ctx, with_bound=True) if kind == "exp" else mp.ps_mixed_general(X, series, ctx, with_bound=True)
            for r_ in rb:
                if r_.bound is not None and not float(r_.bound) >= 0:
                    bad += 1
                    print("BOUND", tag, r_.bound, flush=True)
        except mp.BoundInvalidError:
            pass
    except Exception as e:
        bad += 1
        print("EXC", tag, type(e).__name__, str(e)[:200], flush=True)
print(f"{N} batches ({total} matrices): {bad} failures; eps_mixed <= 10 r n u in {100.0 * within / max(total, 1):.1f} % "
      f"(reference criterion: >= 95 %), {time.time() - t0:.0f} s")
