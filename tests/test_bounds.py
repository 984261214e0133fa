"""Theorem 2.1 bound parity (bounds.py:101-113 via engine.py:283-292): the
product's thm21_bound on plans the product planner builds from the oracle's
block norms (bit-identical to the reference's, test_oracle_golden.py)
reproduces the reference's ``with_bound=True`` report field string for
string, and raises BoundInvalidError exactly where the reference does
(bounds.py:23-36).  Goldens: oracle/make_golden_bounds.py (the unmodified
reference under the gmpy2 shim)."""
import json
import math
import os
from fractions import Fraction

import numpy as np
import pytest

from paper_2312_17396_b200 import PrecisionCtx, plan_precisions
from paper_2312_17396_b200.bigfloat import fmt7
from paper_2312_17396_b200.bounds import BoundInvalidError
from paper_2312_17396_b200.engine import _bound_for
from paper_2312_17396_b200.planner import fixed_plan

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "bounds_reference.json")


def cases():
    return json.load(open(GOLD))["cases"]


def _plan_from_oracle(oracle_lib, case):
    X = np.array(case["X"])
    coeffs = [Fraction(c) for c in case["coeffs"]]
    d = case["d"]
    m = len(coeffs) - 1
    s = math.ceil(math.sqrt(m))
    ps = oracle_lib.OraclePS(X.shape[0])
    n2 = ps.prepare(X, coeffs, s, oracle_lib.bits_of(d))
    fr = [Fraction(a) + Fraction(b) for a, b in n2]
    r = m // s
    ctx = PrecisionCtx(d)
    if case["kind"] == "fixed":
        return fixed_plan(fr[:r + 1], fr[r + 1], ctx, s), X.shape[0]
    return plan_precisions(fr[:r + 1], fr[r + 1], ctx, 10.0, s=s), X.shape[0]


@pytest.mark.parametrize("case", cases(), ids=lambda c: c["name"])
def test_thm21_bound_matches_reference(oracle_lib, case):
    plan, n = _plan_from_oracle(oracle_lib, case)
    if case["bound"] is None:
        with pytest.raises(BoundInvalidError) as ei:
            _bound_for(plan, n)
        want = float(case["message"].split(" = ")[1].split(" >=")[0])
        got = float(str(ei.value).split(" = ")[1].split(" >=")[0])
        assert abs(got - want) <= 1e-12 * want
    else:
        assert plan.to_dict() == case["plan"]
        assert fmt7(_bound_for(plan, n)) == case["bound"]


def test_bound_goldens_cover_both_outcomes():
    cs = cases()
    assert sum(c["bound"] is None for c in cs) >= 3 and sum(c["bound"] is not None for c in cs) >= 4
