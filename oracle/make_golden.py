"""TEST INFRASTRUCTURE: generate tests/golden/*.json from the UNMODIFIED
reference (/root/reference/pkg/src/mpps) run under oracle/gmpy2_shim.

    python oracle/make_golden.py [--quick]

Only runs in the build container (needs /root/reference)."""
import json
import math
import os
import random
import sys
import time
from fractions import Fraction

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
sys.path.insert(0, os.path.join(HERE, "gmpy2_shim"))
sys.path.insert(0, "/root/reference/pkg/src")
sys.dont_write_bytecode = True

import numpy as np  # noqa: E402
import gmpy2  # noqa: E402  (the shim)
from mpps import engine, precision, coefficients, harness  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden")


def words(x):
    """Exact fp64 word expansion of an mpfr (greedy nearest)."""
    f = x._fraction() if hasattr(x, "_fraction") else Fraction(x)
    out = []
    for _ in range(4):
        w = float(f)
        out.append(w)
        f -= Fraction(w)
    assert f == 0
    return out


def mat_words(A):
    return [[words(e.real) for e in row] for row in A.rows]


def synth(n, target, seed, cos=False):
    G = np.random.default_rng(seed).standard_normal((n, n))
    if cos:
        G = G / np.sqrt(n)
    return G * (target / np.abs(G).sum(axis=0).max())


def planner_cases(count, seed=2024):
    rng = random.Random(seed)
    cases = []
    for _ in range(count):
        r = rng.randint(1, 10)
        d = rng.choice([15, 16, 31, 32, 63, 64])
        delta = rng.choice([10.0, 10.0, 2.0])
        y = 10 ** rng.uniform(-3, 1.5)
        b = 10 ** rng.uniform(-2, 3)
        nb = []
        for i in range(r + 1):
            nb.append(b if rng.random() > 0.05 else 0.0)
            b *= 10 ** rng.uniform(-12, 0.3)
        if rng.random() < 0.03:
            y = 0.0
        ctx = precision.PrecisionCtx(d)
        plan = engine.plan_precisions(nb, y, ctx, delta, s=rng.randint(1, 9))
        cases.append({"norm_bs": nb, "norm_y": y, "d": d, "delta": delta, "s": plan.s,
                      "plan": plan.to_dict()})
    return cases


def eval_case(name, X, series, d, kind, m=None, fix_params=True):
    ctx = precision.PrecisionCtx(d)
    M = precision.MPMatrix(X.tolist(), ctx)
    t = time.time()
    if kind == "mixed_exp":
        rep = engine.ps_mixed_exp(M, m, ctx, fix_params=fix_params)
    elif kind == "mixed_general":
        rep = engine.ps_mixed_general(M, series, ctx)
    elif kind == "fixed":
        rep = engine.ps_fixed(M, series, ctx)
    else:
        raise ValueError(kind)
    print(f"  {name}: {time.time() - t:.1f}s plan {rep.plan.level_digits}", flush=True)
    j = json.loads(rep.to_json())
    j.pop("timing_buckets", None)
    return {"name": name, "kind": kind, "d": d, "m": m if m is not None else series.degree,
            "coeffs": [f"{c.numerator}/{c.denominator}" for c in series.coeffs],
            "fix_params": fix_params, "X": X.tolist(), "report": j,
            "result_words": mat_words(rep.result)}


def main(quick=False):
    os.makedirs(OUT, exist_ok=True)
    print("planner cases", flush=True)
    with open(os.path.join(OUT, "planner_reference.json"), "w") as f:
        json.dump({"source": "mpps.engine.plan_precisions (reference, under the gmpy2 shim)",
                   "cases": planner_cases(60 if quick else 400)}, f)
    print("evaluations", flush=True)
    ev = []
    te = coefficients.taylor_exp_coeffs
    pn, pd = coefficients.pade_exp_coeffs(13, 13)
    qn, qd = coefficients.pade_exp_coeffs(26, 26)
    ev.append(eval_case("cfg1_n8", synth(8, 0.5, 0), te(16), 15, "mixed_exp", m=16))
    ev.append(eval_case("cfg1_n8_seed3", synth(8, 0.5, 3), te(16), 15, "mixed_exp", m=16))
    ev.append(eval_case("cfg2_n6", synth(6, 1.0, 0), te(30), 31, "mixed_exp", m=30))
    ev.append(eval_case("cfg2_n6_fixed", synth(6, 1.0, 0), te(30), 31, "fixed"))
    ev.append(eval_case("cfg3_m42_n5", synth(5, 7 / math.e, 1), te(42), 31, "mixed_exp", m=42))
    ev.append(eval_case("pade13_num_n6", synth(6, 2.0, 0), pn, 15, "mixed_general"))
    ev.append(eval_case("pade13_den_n6", synth(6, 2.0, 0), pd, 15, "mixed_general"))
    ev.append(eval_case("pade26_num_n5", synth(5, 2.0, 0), qn, 63, "mixed_general"))
    ev.append(eval_case("pade26_den_n5", synth(5, 2.0, 0), qd, 63, "mixed_general"))
    # cosine: the reference forms Z = X X at the working precision first
    ctx31 = precision.PrecisionCtx(31)
    Xc = synth(6, 1.0, 0, cos=True)
    Zm = precision.mat_mul(precision.MPMatrix(Xc.tolist(), ctx31), precision.MPMatrix(Xc.tolist(), ctx31), ctx31)
    cz = {"name": "cos24_n6", "Xc": Xc.tolist(), "Z_words": mat_words(Zm)}
    repc = engine.ps_mixed_general(Zm, coefficients.taylor_cos_coeffs(24), ctx31)
    jc = json.loads(repc.to_json())
    jc.pop("timing_buckets", None)
    cz.update({"kind": "cos", "d": 31, "m": 24, "report": jc, "result_words": mat_words(repc.result),
               "coeffs": [f"{c.numerator}/{c.denominator}" for c in coefficients.taylor_cos_coeffs(24).coeffs]})
    ev.append(cz)
    ev.append(eval_case("growth_n4", synth(4, 0.02, 5), te(9), 24, "mixed_exp", m=9, fix_params=False))
    ev.append(eval_case("explicit_m1_n3", synth(3, 0.25, 7), te(1), 16, "mixed_exp", m=1, fix_params=False))
    with open(os.path.join(OUT, "evaluations_reference.json"), "w") as f:
        json.dump({"source": "mpps.engine evaluators (reference, under the gmpy2 shim)", "cases": ev}, f)
    if not quick:
        print("table 1 (plan_only on cauchy(100))", flush=True)
        rows = []
        for d, m in ((32, 42), (64, 64)):
            cfg = harness.ExperimentConfig(matrix="cauchy", n=100, family="taylor_exp", m=m, digits=d)
            t = time.time()
            X, series = harness.build_argument(cfg)
            plan = engine.plan_only(X, series, cfg.ctx)
            rows.append({"d": d, "m": m, "plan": plan.to_dict()})
            print(f"  d={d}: {plan.level_digits} {time.time() - t:.0f}s", flush=True)
        with open(os.path.join(OUT, "table1_reference.json"), "w") as f:
            json.dump({"source": "mpps.engine.plan_only on gallery cauchy(100)", "rows": rows}, f)


if __name__ == "__main__":
    main(quick="--quick" in sys.argv)
