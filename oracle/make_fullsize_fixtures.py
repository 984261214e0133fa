"""TEST INFRASTRUCTURE: full-size (BASELINE-size) parity fixtures for the
configs whose n^3 MPFR evaluations cannot finish on a CPU (cfg3 n=1024 x16,
cfg4 n=2048, cfg5 n=8192) -- SURVEY.md 8(c) Tier C.

    python oracle/make_fullsize_fixtures.py [--only cfg3,cfg4,cfg5]

Writes
  tests/golden/fullsize_plans.json  per matrix/polynomial: the precision
      schedule the UNMODIFIED reference planner (engine.plan_precisions +
      snap_to_lattice, run here under oracle/gmpy2_shim) chooses from block
      norms computed in float64 (numpy BLAS), the norms, and the distance of
      every e_i from the nearest integer and from the delta threshold (the
      float64 norms' ~1e-13 relative error moves e_i by < 1e-12, so margins
      >= 1e-9 make the digits exact); cfg3's squaring count l comes from the
      reference's bounds.extra_squarings;
  tests/golden/fullsize_cols.npz    ground-truth columns p(X) e_j (cosine:
      p(X^2) e_j) at twice the working digits (the reference_eval rule,
      harness.py:105-109), by matrix-vector Horner in the C MPFR oracle
      (oracle.poly_columns), as exact 4-word planes.

Inputs are regenerated from their seeds by the tests (SURVEY 8d generator).
Only runs in the build container (needs /root/reference)."""
import argparse
import json
import math
import os
import sys
import time
from fractions import Fraction

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(HERE, "gmpy2_shim"))
sys.path.insert(0, "/root/reference/pkg/src")
sys.dont_write_bytecode = True

import numpy as np  # noqa: E402
import gmpy2  # noqa: E402,F401  (the shim)
from mpps import engine, precision, coefficients, bounds  # noqa: E402
import oracle  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden")
LATTICE = (7, 15, 31, 63)


def synth(n, target, seed, cos=False):
    G = np.random.default_rng(seed).standard_normal((n, n))
    if cos:
        G = G / np.sqrt(n)
    return G * (target / np.abs(G).sum(axis=0).max())


def one_norm(A):
    return float(np.abs(A).sum(axis=0).max())


def columns_for(n, key):
    return sorted(int(c) for c in np.random.default_rng(77 + key).choice(n, 2, replace=False))


def plan_record(X, coeffs, d, delta=10.0):
    """Reference planner on float64 block norms of X (engine.py:118-215)."""
    m = len(coeffs) - 1
    s = math.ceil(math.sqrt(m))
    r = m // s
    full = m // s
    n = X.shape[0]
    pw = [np.eye(n), X]
    for _ in range(2, s + 1):
        pw.append(pw[-1] @ X)            # X^k = X^{k-1} X (engine.py:151-153)
    b = [float(Fraction(c)) for c in coeffs]
    nb = []
    for i in range(r + 1):
        hi = s - 1 if i < full else m - s * full
        B = b[s * i] * np.eye(n)
        for j in range(1, hi + 1):
            B = B + b[s * i + j] * pw[j]
        nb.append(one_norm(B))
    ny = one_norm(pw[s])
    ctx = precision.PrecisionCtx(d)
    plan = engine.plan_precisions(nb, ny, ctx, delta, s=s)
    snapped = engine.snap_to_lattice(plan, [x for x in LATTICE if x <= d]).level_digits
    # margins of the digit rule in float64 (the rule itself ran in the reference)
    e = [d - math.log10(nb[0]) + math.log10(nb[i]) + i * math.log10(ny) + 1e-9
         for i in range(1, r + 1) if nb[i] > 0]
    lim = d - math.log10(delta)
    margin_int = min((abs(x - round(x)) for x in e if 1 <= x <= d), default=1.0)
    margin_delta = min((abs(x - lim) for x in e), default=1.0)
    return {"s": s, "r": r, "m": m, "d": d, "digits": list(plan.level_digits), "nu": plan.nu,
            "snapped": list(snapped), "norm_bs": nb, "norm_y": ny, "e": e,
            "margin_integer": margin_int, "margin_delta": margin_delta}


def truth_cols(X, coeffs, d, cols, squares=False):
    return oracle.poly_columns(X, coeffs, oracle.bits_of(2 * d), cols, squares=squares)


def cfg3(out, arrays):
    n, B, d, m = 1024, 16, 31, 42
    rng = np.random.default_rng(1000)
    targets = 10.0 ** rng.uniform(-2, 3, size=B)
    coeffs = coefficients.taylor_exp_coeffs(m).coeffs
    plans = []
    for b in range(B):
        A = synth(n, targets[b], b)
        ell = bounds.extra_squarings(one_norm(A), math.ceil(math.sqrt(m)))
        X = A * 2.0 ** -ell
        rec = plan_record(X, coeffs, d)
        rec.update({"seed": b, "target": float(targets[b]), "squarings": ell, "cols": columns_for(n, b)})
        t = time.time()
        arrays[f"cfg3_{b}"] = truth_cols(X, coeffs, d, rec["cols"])
        print(f"cfg3[{b}] l={ell} digits={rec['digits']} snapped={rec['snapped']} "
              f"margins {rec['margin_integer']:.2e}/{rec['margin_delta']:.2e} cols {time.time() - t:.1f}s", flush=True)
        plans.append(rec)
    out["cfg3"] = {"units": B, "n": n, "plans": plans,
                   "note": "seeds 0..15, ||A||_1 = 10^U(-2,3) from default_rng(1000); X = 2^-l A"}


def cfg4(out, arrays):
    n, d = 2048, 63
    X = synth(n, 2.0, 0)
    plans = []
    for k, dd in ((26, 63), (13, 15)):
        num, den = coefficients.pade_exp_coeffs(k, k)
        for which, series in (("num", num), ("den", den)):
            rec = plan_record(X, series.coeffs, dd)
            rec.update({"seed": 0, "pade": k, "which": which, "cols": columns_for(n, 100 + k),
                        "shared_powers_with_previous": which == "den"})
            t = time.time()
            arrays[f"cfg4_{k}_{which}"] = truth_cols(X, series.coeffs, dd, rec["cols"])
            print(f"cfg4 [{k}/{k}] {which} d={dd} digits={rec['digits']} snapped={rec['snapped']} "
                  f"margins {rec['margin_integer']:.2e}/{rec['margin_delta']:.2e} cols {time.time() - t:.1f}s",
                  flush=True)
            plans.append(rec)
    out["cfg4"] = {"units": 1, "n": n, "plans": [p for p in plans if p["pade"] == 26],
                   "fp64_pade13": [p for p in plans if p["pade"] == 13],
                   "note": "seed 0, ||X||_1 = 2; bench cfg4 = [26/26] at qd (plans); [13/13] at fp64 tested too"}


def cfg5(out, arrays):
    n, d, m = 8192, 31, 24
    X = synth(n, 1.0, 0, cos=True)
    t = time.time()
    Z = X @ X                                   # harness.py:100-101 (float64 here: norms only)
    rec = plan_record(Z, coefficients.taylor_cos_coeffs(m).coeffs, d)
    rec.update({"seed": 0, "argument_gemms": 1, "cols": columns_for(n, 5)})
    print(f"cfg5 digits={rec['digits']} snapped={rec['snapped']} margins "
          f"{rec['margin_integer']:.2e}/{rec['margin_delta']:.2e} ({time.time() - t:.1f}s)", flush=True)
    t = time.time()
    arrays["cfg5"] = truth_cols(X, coefficients.taylor_cos_coeffs(m).coeffs, d, rec["cols"], squares=True)
    print(f"cfg5 cols {time.time() - t:.1f}s", flush=True)
    out["cfg5"] = {"units": 1, "n": n, "plans": [rec],
                   "note": "seed 0, X ~ N(0,1)/sqrt(n) rescaled to ||X||_1 = 1; Z = X X"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", default="cfg3,cfg4,cfg5")
    args = ap.parse_args()
    oracle.build()
    pj = os.path.join(OUT, "fullsize_plans.json")
    pn = os.path.join(OUT, "fullsize_cols.npz")
    out = json.load(open(pj)) if os.path.exists(pj) else {}
    arrays = dict(np.load(pn)) if os.path.exists(pn) else {}
    for name in args.only.split(","):
        {"cfg3": cfg3, "cfg4": cfg4, "cfg5": cfg5}[name](out, arrays)
        json.dump(out, open(pj, "w"), indent=1)
        np.savez_compressed(pn, **arrays)


if __name__ == "__main__":
    main()
