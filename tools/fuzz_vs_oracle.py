"""Dev tool: random small evaluations (size, degree, digits, norm, evaluator) against the CPU oracle
(test infrastructure): schedule exactly equal, values within 10 r n 10^-d."""
import sys, os, time
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import oracle
import paper_2312_17396_b200 as mp
from _util import synth

N = int(sys.argv[1]) if len(sys.argv) > 1 else 200
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 0)
NMIN = int(sys.argv[3]) if len(sys.argv) > 3 else 1          # sizes: n in [NMIN, NMAX) (qd: half of NMAX)
NMAX = int(sys.argv[4]) if len(sys.argv) > 4 else 72
bad = 0
t0 = time.time()
for it in range(N):
    d = int(rng.choice([15, 31, 63, 15, 31]))
    n = int(rng.integers(NMIN, NMAX if d < 63 else max(NMIN + 1, NMAX // 2)))
    kind = str(rng.choice(["exp", "exp", "cos", "fixed", "pade"]))
    m = int(rng.integers(1, 41)) if kind != "pade" else int(rng.integers(2, 20))
    norm = float(10.0 ** rng.uniform(-4, 1.3))
    X = synth(n, norm, int(rng.integers(1 << 30)))
    ctx = mp.PrecisionCtx(d)
    tag = f"#{it} {kind} n={n} m={m} d={d} norm={norm:.3g}"
    try:
        if kind == "exp":
            series = mp.taylor_exp_coeffs(m)
            reps = [mp.ps_mixed_exp(X, m, ctx)]
            refs = [oracle.ps_eval(X, series.coeffs, d)]
        elif kind == "cos":
            series = mp.taylor_cos_coeffs(max(m, 1))
            reps = [mp.ps_mixed_general(X, series, ctx)]
            refs = [oracle.ps_eval(X, series.coeffs, d)]
        elif kind == "fixed":
            series = mp.taylor_exp_coeffs(m)
            reps = [mp.ps_fixed(X, series, ctx)]
            refs = [oracle.ps_eval(X, series.coeffs, d, mode="fixed")]
        else:
            pc, qc = mp.pade_exp_coeffs(m, m)
            reps = list(mp.ps_mixed_pade(X, m, ctx))
            refs = [oracle.ps_eval(X, pc.coeffs, d), oracle.ps_eval(X, qc.coeffs, d)]
        coeffs_of = ([pc.coeffs, qc.coeffs] if kind == "pade" else [series.coeffs])
        seen = []
        for rep, ref in zip(reps, refs):
            p = rep.plan
            if kind != "fixed" and p.r > 0 and not getattr(p, "explicit_powers", False):
                if tuple(p.level_digits) != tuple(ref.digits) or p.nu != ref.nu:
                    bad += 1
                    print("SCHEDULE", tag, p.level_digits, ref.digits, p.nu, ref.nu, flush=True)
                    continue
            diff, refn = ref.compare(rep.result.data[:, 0].double().cpu().numpy())
            tol = 10 * max(p.r, 1) * n * 10.0 ** -d
            # the gate is relative to |p|(||X||) = sum |b_k| ||X||^k, what Thm 2.1 bounds the error by
            # (for a cancelling p(X) -- tiny matrices at ||X|| ~ 10 -- it exceeds ||p(X)||)
            cs = coeffs_of[len(seen)]
            pabs = float(sum(abs(c) * norm ** k for k, c in enumerate(cs)))
            seen.append(1)
            if not diff <= tol * max(refn, pabs):
                bad += 1
                print("VALUE", tag, diff / refn, tol, flush=True)
    except Exception as e:
        bad += 1
        print("EXC", tag, type(e).__name__, str(e)[:150], flush=True)
print(f"{N} cases, {bad} failures, {time.time() - t0:.0f} s")
