"""TEST INFRASTRUCTURE: tests/golden/bounds_reference.json -- the
reference's Theorem 2.1 forward-error bound of evaluations run with
``with_bound=True`` (engine.py:283-292 -> bounds.py:101-113), from the
UNMODIFIED reference under oracle/gmpy2_shim, plus its own bound
containment check (acceptance.py:225-260, criterion C7a) outcome.

    python oracle/make_golden_bounds.py

Only runs in the build container (needs /root/reference)."""
import json
import math
import os
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
sys.path.insert(0, os.path.join(HERE, "gmpy2_shim"))
sys.path.insert(0, "/root/reference/pkg/src")
sys.dont_write_bytecode = True

import numpy as np  # noqa: E402
import gmpy2  # noqa: E402,F401  (the shim)
from mpps import engine, precision, coefficients, bounds  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden")


def synth(n, target, seed, cos=False):
    G = np.random.default_rng(seed).standard_normal((n, n))
    if cos:
        G = G / np.sqrt(n)
    return G * (target / np.abs(G).sum(axis=0).max())


def case(name, X, d, kind, m=None, series=None):
    ctx = precision.PrecisionCtx(d)
    M = precision.MPMatrix(X.tolist(), ctx)
    t = time.time()
    out = {"name": name, "kind": kind, "d": d, "m": m if m is not None else series.degree,
           "coeffs": [f"{c.numerator}/{c.denominator}" for c in (series or coefficients.taylor_exp_coeffs(m)).coeffs],
           "X": X.tolist()}
    try:
        if kind == "mixed_exp":
            rep = engine.ps_mixed_exp(M, m, ctx, with_bound=True)
        elif kind == "mixed_general":
            rep = engine.ps_mixed_general(M, series, ctx, with_bound=True)
        else:
            rep = engine.ps_fixed(M, series, ctx, with_bound=True)
    except bounds.BoundInvalidError as e:     # bounds.py:23-36 (k u >= 1)
        print(f"  {name}: BoundInvalidError {e}", flush=True)
        out.update({"bound": None, "error": "BoundInvalidError", "message": str(e)})
        return out
    j = json.loads(rep.to_json())
    print(f"  {name}: bound {j['bound']} plan {rep.plan.level_digits} ({time.time() - t:.1f}s)", flush=True)
    out.update({"bound": j["bound"], "plan": j["plan"]})
    return out


def main():
    te = coefficients.taylor_exp_coeffs
    pn, _ = coefficients.pade_exp_coeffs(13, 13)
    qn, _ = coefficients.pade_exp_coeffs(26, 26)
    cases = [
        case("cfg1_n8", synth(8, 0.5, 0), 15, "mixed_exp", m=16),
        case("cfg1_n8_seed5", synth(8, 0.5, 5), 15, "mixed_exp", m=16),
        case("cfg2_n6", synth(6, 1.0, 0), 31, "mixed_exp", m=30),
        case("cfg2_n6_big", synth(6, 4.0, 2), 31, "mixed_exp", m=30),
        case("cfg2_n6_fixed", synth(6, 1.0, 0), 31, "fixed", series=te(30)),
        case("pade13_num_n6", synth(6, 2.0, 0), 15, "mixed_general", series=pn),
        case("cfg3_m42_n5", synth(5, 7 / math.e, 1), 31, "mixed_exp", m=42),
        case("pade26_num_n5", synth(5, 2.0, 0), 63, "mixed_general", series=qn),
        case("cfg2_n7_norm3", synth(7, 3.0, 4), 31, "mixed_exp", m=30),
    ]
    with open(os.path.join(OUT, "bounds_reference.json"), "w") as f:
        json.dump({"source": "mpps.engine evaluators with_bound=True (reference, under the gmpy2 shim)",
                   "cases": cases}, f)


if __name__ == "__main__":
    main()
