"""TEST INFRASTRUCTURE: complex golden cases (tests/golden/complex_reference.json)
from the UNMODIFIED reference (its native element type is mpc,
precision.py:78-105) run under oracle/gmpy2_shim.

    python oracle/make_golden_complex.py

Only runs in the build container (needs /root/reference)."""
import json
import os
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
import make_golden as mg  # noqa: E402  (shim + reference on sys.path)
import numpy as np  # noqa: E402
from mpps import coefficients, engine, gallery, precision  # noqa: E402


def cwords(A):
    """[[re words, im words] per entry] of an MPMatrix."""
    return [[[mg.words(e.real), mg.words(e.imag)] for e in row] for row in A.rows]


def csynth(n, target, seed):
    rng = np.random.default_rng(seed)
    Z = rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))
    return Z * (target / np.abs(Z).sum(axis=0).max())


def case(name, Z, series, d, kind, m=None, M=None):
    ctx = precision.PrecisionCtx(d)
    if M is None:
        M = precision.MPMatrix([[complex(v) for v in row] for row in Z], ctx)
    t = time.time()
    if kind == "mixed_exp":
        rep = engine.ps_mixed_exp(M, m, ctx)
    elif kind == "mixed_general":
        rep = engine.ps_mixed_general(M, series, ctx)
    else:
        rep = engine.ps_fixed(M, series, ctx)
    print(f"  {name}: {time.time() - t:.1f}s plan {rep.plan.level_digits}", flush=True)
    j = json.loads(rep.to_json())
    j.pop("timing_buckets", None)
    return {"name": name, "kind": kind, "d": d, "m": m if m is not None else series.degree,
            "coeffs": [f"{c.numerator}/{c.denominator}" for c in series.coeffs],
            "X": cwords(M), "report": j, "result": cwords(rep.result)}


def main():
    te = coefficients.taylor_exp_coeffs
    pn, pd = coefficients.pade_exp_coeffs(13, 13)
    ev = []
    ctx31 = precision.PrecisionCtx(31)
    smoke = precision.round_to(gallery.gen_smoke(6, ctx31), ctx31)
    ev.append(case("smoke6_exp30_d31", None, te(30), 31, "mixed_exp", m=30, M=smoke))
    ev.append(case("rand5_exp30_d31", csynth(5, 1.0, 0), te(30), 31, "mixed_exp", m=30))
    ev.append(case("rand6_exp16_d15", csynth(6, 0.5, 1), te(16), 15, "mixed_exp", m=16))
    ev.append(case("rand5_pade13num_d15", csynth(5, 2.0, 2), pn, 15, "mixed_general"))
    ev.append(case("rand5_pade13den_d15", csynth(5, 2.0, 2), pd, 15, "mixed_general"))
    ev.append(case("rand4_exp30_fixed_d31", csynth(4, 1.0, 3), te(30), 31, "fixed"))
    out = os.path.join(mg.OUT, "complex_reference.json")
    with open(out, "w") as f:
        json.dump({"source": "mpps.engine evaluators on complex MPMatrix inputs (reference, under the gmpy2 shim)",
                   "cases": ev}, f)
    print("wrote", out)


if __name__ == "__main__":
    main()
