"""Coefficient series (coefficients.py restated) against the reference's
known answers: Pade [13/13] numerator golden values (acceptance.py:49-60),
Taylor/cos identities (test_coefficients.py:13-68)."""
from fractions import Fraction
from math import factorial

import numpy as np
import pytest

from paper_2312_17396_b200 import (PrecisionCtx, eval_coeff, pade_exp_coeffs, series_from_json,
                                   series_to_json, taylor_cos_coeffs, taylor_exp_coeffs)
from paper_2312_17396_b200.coefficients import coeff_words, split_words
from paper_2312_17396_b200.bigfloat import rn

PADE_GOLDEN = (Fraction(1, 2), Fraction(3, 25), Fraction(11, 600), Fraction(11, 5520),
               Fraction(3, 18400), Fraction(1, 96600), Fraction(1, 1932000))


def test_pade_13_golden():
    num, den = pade_exp_coeffs(13, 13)
    assert num.coeffs[0] == 1 and num.coeffs[1:8] == PADE_GOLDEN
    assert all(q == (-1) ** j * p for j, (p, q) in enumerate(zip(num.coeffs, den.coeffs)))


def test_pade_1_1_and_norm():
    p, q = pade_exp_coeffs(1, 1)
    assert p.coeffs == (1, Fraction(1, 2)) and q.coeffs == (1, Fraction(-1, 2))
    with pytest.raises(ValueError):
        pade_exp_coeffs(-1, 2)


def test_taylor_and_cos():
    assert taylor_exp_coeffs(4).coeffs == (1, 1, Fraction(1, 2), Fraction(1, 6), Fraction(1, 24))
    c = taylor_exp_coeffs(12).coeffs
    assert all(c[i] / c[i - 1] == Fraction(1, i) for i in range(1, 13))
    assert taylor_cos_coeffs(2).coeffs == (1, Fraction(-1, 2), Fraction(1, 24))
    k = taylor_cos_coeffs(8).coeffs
    assert all(abs(k[j] / k[j - 1]) == Fraction(1, 2 * j * (2 * j - 1)) for j in range(1, 9))
    with pytest.raises(ValueError):
        taylor_exp_coeffs(-1)


def test_eval_coeff_correct_rounding():
    assert eval_coeff(Fraction(1, 2), PrecisionCtx(8)) == 0.5
    v = eval_coeff(Fraction(1, 3), PrecisionCtx(31))
    assert v.prec == 103 and abs(v.value - Fraction(1, 3)) <= Fraction(1, 3) / 2 ** 103


def test_json_roundtrip():
    s = pade_exp_coeffs(6, 6)[1]
    t = series_from_json(series_to_json(s))
    assert t == s


@pytest.mark.parametrize("d", [7, 15, 31, 63])
def test_coefficient_words_exact(d):
    ctx = PrecisionCtx(d)
    series = taylor_exp_coeffs(42)
    w = coeff_words(series, ctx)
    for k, c in enumerate(series.coeffs):
        assert sum(Fraction(x) for x in w[k]) == rn(c, ctx.binary_precision)
        # non-overlapping, decreasing words
        nz = [abs(x) for x in w[k] if x != 0]
        assert all(a > b for a, b in zip(nz, nz[1:]))
