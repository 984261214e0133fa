"""Exact MPFR emulation used by the host planner (bigfloat.py)."""
import math
import random
from fractions import Fraction

from paper_2312_17396_b200.bigfloat import (MPF, exp10_rn, fmt7, fmt_sci, log10_rn, rn)


def test_rn53_matches_python_float_rounding():
    rng = random.Random(1)
    for _ in range(20000):
        q = Fraction(rng.randrange(1, 10 ** 30), rng.randrange(1, 10 ** 30)) * rng.choice([1, -1])
        assert rn(q, 53) == Fraction(float(q))


def test_rn_ties_to_even():
    # 1 + 2^-53 is a tie at 53 bits -> rounds to 1 (even); 1 + 3*2^-53 -> up
    assert rn(Fraction(1) + Fraction(1, 2 ** 53), 53) == 1
    assert rn(Fraction(1) + Fraction(3, 2 ** 53), 53) == 1 + Fraction(4, 2 ** 53)
    assert rn(Fraction(5), 2) == 4 and rn(Fraction(7), 2) == 8 and rn(Fraction(6), 2) == 6


def test_rn_idempotent_and_exact():
    for p in (24, 50, 53, 103, 107, 210):
        v = rn(Fraction(1, 3), p)
        assert rn(v, p) == v
        assert abs(v - Fraction(1, 3)) <= Fraction(1, 3) * Fraction(1, 2 ** p)


def test_log10_exact_powers_and_accuracy():
    assert log10_rn(Fraction(1000), 107) == 3
    assert log10_rn(Fraction(1), 107) == 0
    v = log10_rn(Fraction(2), 107)
    assert abs(float(v) - math.log10(2)) < 1e-16


def test_exp10_roundoffs():
    assert exp10_rn(-1, 107) == rn(Fraction(1, 10), 107)
    assert float(exp10_rn(-15, 64)) == 1e-15


def test_fmt_sci_matches_reference_format():
    # precision.py:256-269 format: d.dddddde<exp>
    assert fmt7(0.5) == "5.000000e-1"
    assert fmt7(1e-27) == "1.000000e-27"
    assert fmt7(123456789.0) == "1.234568e8"
    assert fmt7(-2.5e-3) == "-2.500000e-3"
    assert fmt_sci(Fraction(0), 7) == "0.0e0"
    assert fmt7(MPF.inf()) == "inf"
    # rounding to 7 significant digits, ties-to-even on the exact value
    assert fmt7(9.9999995) in ("9.999999e0", "1.000000e1")


def test_mpf_ordering():
    a, b = MPF(1), MPF(2)
    assert a < b and b > a and a <= 1 and a == 1.0 and MPF.inf() > b
