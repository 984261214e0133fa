"""Pinning the oracle and the host planner to the reference itself.

tests/golden/*.json were produced by running the UNMODIFIED reference
(pkg/src/mpps) in the build container under the ctypes gmpy2 stand-in
(oracle/make_golden.py; the shim reproduces the reference's own test-suite
outcome, tests/golden/reference_suite_under_shim.txt).  Here, on CPU:

* the product planner (planner.plan_precisions) reproduces every reference
  plan record exactly -- digits, nu, and the 7-digit strings of roundoffs,
  taus and norms (engine.py:71-84);
* the C MPFR oracle, run at the reference's raw (unsnapped) digits,
  reproduces the reference's evaluation results BIT FOR BIT, and its
  norms/plans equal the reference's.
"""
import json
import math
import os
from fractions import Fraction

import numpy as np
import pytest

from paper_2312_17396_b200 import PrecisionCtx, plan_precisions
from paper_2312_17396_b200.bigfloat import fmt7

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load(name):
    path = os.path.join(GOLD, name)
    if not os.path.exists(path):
        pytest.skip(f"{name} not generated")
    with open(path) as f:
        return json.load(f)


def coeffs_of(case):
    out = []
    for c in case["coeffs"]:
        n, _, d = c.partition("/")
        out.append(Fraction(int(n), int(d)))
    return out


def test_planner_matches_reference_records():
    g = load("planner_reference.json")
    assert len(g["cases"]) >= 50
    for c in g["cases"]:
        p = plan_precisions(c["norm_bs"], c["norm_y"], PrecisionCtx(c["d"]), c["delta"], s=c["s"])
        assert p.to_dict() == c["plan"], c


def test_planner_oracle_matches_reference_records(oracle_lib):
    g = load("planner_reference.json")
    for c in g["cases"]:
        n2 = np.array([[x, 0.0] for x in c["norm_bs"]] + [[c["norm_y"], 0.0]])
        dig, nu, nil, _ = oracle_lib.plan_digits(n2, c["d"], c["delta"])
        assert list(dig) == c["plan"]["digits"] and nu == c["plan"]["nu"]
        assert nil == c["plan"]["nilpotent"]


def _oracle_eval_raw(oracle_lib, case):
    d = case["d"]
    coeffs = coeffs_of(case)
    m = len(coeffs) - 1
    s = math.ceil(math.sqrt(m))
    if case["kind"] == "cos":
        Z = np.array(case["Z_words"]).transpose(2, 0, 1)
        Xw = Z
    else:
        Xw = np.array(case["X"])[None]
    ps = oracle_lib.OraclePS(Xw.shape[-1])
    wb = oracle_lib.bits_of(d)
    n2 = ps.prepare(Xw, coeffs, s, wb)
    if case["kind"] == "fixed":
        digits, nu = (d,) * (m // s), m // s + 1
    else:
        digits, nu, nil, _ = oracle_lib.plan_digits(n2, d)
    ps.horner([wb] + [oracle_lib.bits_of(x) for x in digits])
    return ps, n2, digits, nu


def test_oracle_reproduces_reference_bitwise(oracle_lib):
    g = load("evaluations_reference.json")
    checked = 0
    for case in g["cases"]:
        if case["kind"] not in ("mixed_exp", "mixed_general", "fixed", "cos") or not case.get("fix_params", True):
            continue
        if case["kind"] == "mixed_exp" and case["m"] == 1:
            continue
        ps, n2, digits, nu = _oracle_eval_raw(oracle_lib, case)
        plan = case["report"]["plan"]
        assert list(digits) == plan["digits"] and nu == plan["nu"], case["name"]
        r = len(digits)
        got_norms = [fmt7(Fraction(a) + Fraction(b)) for a, b in n2]
        assert got_norms[:r + 1] == plan["norm_bs"] and got_norms[r + 1] == plan["norm_y"], case["name"]
        want = np.array(case["result_words"]).transpose(2, 0, 1)
        got = ps.result_words(4)
        assert np.array_equal(got, want), case["name"]
        checked += 1
    assert checked >= 9


def test_table1_reference_schedules_vs_planner(oracle_lib):
    """Table 1 rows (d=32 m=42, d=64 m=64, cauchy(100)): the reference's
    plan_only schedules, reproduced from oracle norms at 16 digits by the
    product planner."""
    g = load("table1_reference.json")
    n = 100
    from paper_2312_17396_b200.bigfloat import rn
    Xw = np.zeros((2, n, n))
    for i in range(n):
        for j in range(n):
            v = rn(rn(Fraction(1, i + j + 2), 133), 54)  # GEN_CTX 40 digits, then 16
            Xw[0, i, j] = float(v)
            Xw[1, i, j] = float(v - Fraction(float(v)))
    from paper_2312_17396_b200 import taylor_exp_coeffs
    for row in g["rows"]:
        d, m = row["d"], row["m"]
        s = math.ceil(math.sqrt(m))
        ps = oracle_lib.OraclePS(n)
        n2 = ps.prepare(Xw, taylor_exp_coeffs(m).coeffs, s, 54)
        fr = [Fraction(a) + Fraction(b) for a, b in n2]
        r = m // s
        p = plan_precisions(fr[:r + 1], fr[r + 1], PrecisionCtx(d), s=s)
        assert p.to_dict() == row["plan"]


def test_tier_c_columns_pinned_to_full_oracle(oracle_lib):
    """The Tier-C ground truth (oracle.poly_columns: matrix-vector Horner at
    2x digits) equals the full 2x-digit reference_eval (harness.py:105-109,
    fixed PS in MPFR) column by column, for exp and for the cosine's
    p(X^2); power_columns equals mat_mul products."""
    from _util import synth
    from paper_2312_17396_b200 import taylor_exp_coeffs, taylor_cos_coeffs
    n, d = 20, 31
    cols = [0, 7, 19]
    X = synth(n, 1.0, 3)
    co = taylor_exp_coeffs(30).coeffs
    ref = oracle_lib.reference_eval_words(X, co, d)
    pc = oracle_lib.poly_columns(X, co, oracle_lib.bits_of(2 * d), cols)
    nrm = np.abs(ref[0]).sum(0).max()
    assert (oracle_lib.column_diff(pc, ref[:, :, cols].transpose(0, 2, 1)) <= 1e-58 * nrm).all()
    Xc = synth(n, 1.0, 4, cos=True)
    cc = taylor_cos_coeffs(24).coeffs
    Z = oracle_lib.matmul(Xc, Xc, 2 * oracle_lib.bits_of(2 * d))
    ref = oracle_lib.reference_eval_words(Z, cc, d)
    pc = oracle_lib.poly_columns(Xc, cc, oracle_lib.bits_of(2 * d), cols, squares=True)
    assert (oracle_lib.column_diff(pc, ref[:, :, cols].transpose(0, 2, 1)) <= 1e-58).all()
    P = np.stack([X, X * 2.0 ** -60])
    P3 = oracle_lib.matmul(oracle_lib.matmul(P, P, 400), P, 400)
    pw = oracle_lib.power_columns(P, 3, 400, cols)
    assert (oracle_lib.column_diff(pw, P3[:, :, cols].transpose(0, 2, 1)) <= 1e-60).all()   # 4 output words ~ 212 bits


def test_fullsize_fixtures_consistent():
    """tests/golden/fullsize_*: one record (and truth columns) per cfg3 matrix,
    per cfg4 polynomial and for cfg5; snapped formats follow the digits."""
    import json
    import os
    here = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
    fx = json.load(open(os.path.join(here, "fullsize_plans.json")))
    cols = np.load(os.path.join(here, "fullsize_cols.npz"))
    assert len(fx["cfg3"]["plans"]) == 16 and len(fx["cfg4"]["plans"]) == 2 and len(fx["cfg5"]["plans"]) == 1
    lat = (7, 15, 31, 63)
    recs = fx["cfg3"]["plans"] + fx["cfg4"]["plans"] + fx["cfg4"]["fp64_pade13"] + fx["cfg5"]["plans"]
    for rec in recs:
        assert rec["snapped"] == [min(x for x in lat if x >= dd) for dd in rec["digits"]]
        assert rec["margin_integer"] > 1e-9 and rec["margin_delta"] > 1e-9
    for b in range(16):
        assert cols[f"cfg3_{b}"].shape == (4, 2, 1024)
    assert cols["cfg5"].shape == (4, 2, 8192)
