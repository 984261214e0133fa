"""Dev tool: random BATCHES with heterogeneous norms (different plans inside one call) against the CPU
oracle (test infrastructure), member by member; every tenth batch is also checked for batch invariance
(member alone == member in the batch, bitwise)."""
import sys, os, time
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import oracle
import paper_2312_17396_b200 as mp
from _util import synth

N = int(sys.argv[1]) if len(sys.argv) > 1 else 150
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 0)
bad = 0
t0 = time.time()
for it in range(N):
    d = int(rng.choice([15, 31, 31, 63]))
    n = int(rng.integers(2, 48 if d < 63 else 24))
    B = int(rng.integers(2, 6))
    kind = str(rng.choice(["exp", "cos", "fixed"]))
    m = int(rng.integers(2, 36))
    norms = 10.0 ** rng.uniform(-4, 1.0, size=B)
    Xs = np.stack([synth(n, float(norms[b]), int(rng.integers(1 << 30))) for b in range(B)])
    ctx = mp.PrecisionCtx(d)
    tag = f"#{it} {kind} B={B} n={n} m={m} d={d} norms={np.round(np.log10(norms), 1)}"
    try:
        series = mp.taylor_cos_coeffs(m) if kind == "cos" else mp.taylor_exp_coeffs(m)
        if kind == "exp":
            reps = mp.ps_mixed_exp(Xs, m, ctx)
        elif kind == "cos":
            reps = mp.ps_mixed_general(Xs, series, ctx)
        else:
            reps = mp.ps_fixed(Xs, series, ctx)
        for b in range(B):
            ref = oracle.ps_eval(Xs[b], series.coeffs, d, mode="fixed" if kind == "fixed" else "mixed")
            p = reps[b].plan
            if kind != "fixed" and p.r > 0 and not getattr(p, "explicit_powers", False):
                if tuple(p.level_digits) != tuple(ref.digits) or p.nu != ref.nu:
                    bad += 1
                    print("SCHEDULE", tag, b, p.level_digits, ref.digits, flush=True)
                    continue
            diff, refn = ref.compare(reps.result.data[:, b].double().cpu().numpy())
            pabs = float(sum(abs(c) * float(norms[b]) ** k for k, c in enumerate(series.coeffs)))
            tol = 10 * max(p.r, 1) * n * 10.0 ** -d
            if not diff <= tol * max(refn, pabs):
                bad += 1
                print("VALUE", tag, b, diff / refn, tol, flush=True)
        if it % 10 == 0:
            b = int(rng.integers(B))
            solo = (mp.ps_mixed_exp(Xs[b], m, ctx) if kind == "exp" else
                    mp.ps_mixed_general(Xs[b], series, ctx) if kind == "cos" else mp.ps_fixed(Xs[b], series, ctx))
            if not torch.equal(solo.result.data[:, 0], reps.result.data[:, b]):
                bad += 1
                print("INVARIANCE", tag, b, flush=True)
    except Exception as e:
        bad += 1
        print("EXC", tag, type(e).__name__, str(e)[:150], flush=True)
print(f"{N} batches, {bad} failures, {time.time() - t0:.0f} s")
