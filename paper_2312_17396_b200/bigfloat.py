"""Exact emulation of the reference's MPFR scalar arithmetic on the host.

The reference planner and bounds run a handful of scalar operations per
evaluation through gmpy2 contexts of fixed bit precision: 64-bit norms
(engine.py:170-171), the 107-bit ``BOUND_CTX`` (precision.py:75) for
log10/add/mul/div, the 54-bit ``NORM_CTX`` (precision.py:72) for the growth
test, and Python ``float()`` conversions (engine.py:196).  Every one of those
is a correctly rounded round-to-nearest-even operation, so it can be
reproduced bit for bit with exact rational arithmetic followed by one
explicit rounding:

* ``rn(q, p)`` rounds an exact ``Fraction`` to ``p`` significant bits
  (ties to even, unbounded exponent -- MPFR's default exponent range is
  never reached by these values);
* transcendental functions (log10, ln, exp) are evaluated with the
  ``decimal`` module, whose ``ln``/``log10``/``exp`` are correctly rounded,
  at 100 significant digits, then rounded once to ``p`` bits.  The double
  rounding can only differ from MPFR when the exact value lies within
  1e-100 (relative) of a ``p``-bit midpoint, i.e. never in practice; the
  planner tests pin the result against the C MPFR oracle on 10^5 inputs.

No gmpy2/MPFR is needed by this module (the product's host planner).
"""

from __future__ import annotations

import decimal
import math
from fractions import Fraction
from typing import Union

Number = Union[int, float, Fraction, "MPF"]

_DEC = decimal.Context(prec=100, rounding=decimal.ROUND_HALF_EVEN,
                       Emax=999999, Emin=-999999)


def _floor_log2(a: Fraction) -> int:
    """floor(log2(a)) for a > 0, exactly."""
    n, d = a.numerator, a.denominator
    e = n.bit_length() - d.bit_length()
    if e >= 0:
        return e if n >= (d << e) else e - 1
    return e if (n << -e) >= d else e - 1


def rn(q: Fraction, p: int) -> Fraction:
    """Round q to p significant bits, nearest, ties to even."""
    if q == 0:
        return Fraction(0)
    sign = -1 if q < 0 else 1
    a = -q if q < 0 else q
    E = _floor_log2(a)
    sh = p - 1 - E
    n, d = a.numerator, a.denominator
    if sh >= 0:
        num, den = n << sh, d
    else:
        num, den = n, d << (-sh)
    m, rem = divmod(num, den)
    twice = 2 * rem
    if twice > den or (twice == den and (m & 1)):
        m += 1
    if sh >= 0:
        return Fraction(sign * m, 1 << sh)
    return Fraction(sign * m * (1 << (-sh)))


def to_fraction(x) -> Fraction:
    if isinstance(x, MPF):
        if x.special is not None:
            raise ValueError(f"non-finite value {x.special}")
        return x.value
    if isinstance(x, Fraction):
        return x
    if isinstance(x, int):
        return Fraction(x)
    if isinstance(x, float):
        if not math.isfinite(x):
            raise ValueError("non-finite float")
        return Fraction(x)
    # mpfr-like objects from the reference (gmpy2 or a shim): go through
    # their exact rational value when available.
    if hasattr(x, "as_integer_ratio"):
        n, d = x.as_integer_ratio()
        return Fraction(n, d)
    return Fraction(x)


def _dec_of(q: Fraction) -> decimal.Decimal:
    return _DEC.divide(decimal.Decimal(q.numerator), decimal.Decimal(q.denominator))


def _frac_of_dec(x: decimal.Decimal) -> Fraction:
    return Fraction(x)


def log10_rn(q: Fraction, p: int) -> Fraction:
    """RN_p(log10(q)), q > 0."""
    if q <= 0:
        raise ValueError("log10 of a non-positive value")
    # exact powers of ten (only non-negative ones are dyadic)
    if q.denominator == 1:
        n = q.numerator
        k = len(str(n)) - 1
        if 10 ** k == n:
            return Fraction(k)
    return rn(_frac_of_dec(_DEC.log10(_dec_of(q))), p)


def ln_rn(q: Fraction, p: int) -> Fraction:
    if q <= 0:
        raise ValueError("log of a non-positive value")
    if q == 1:
        return Fraction(0)
    return rn(_frac_of_dec(_DEC.ln(_dec_of(q))), p)


def exp_rn(q: Fraction, p: int) -> Fraction:
    if q == 0:
        return Fraction(1)
    return rn(_frac_of_dec(_DEC.exp(_dec_of(q))), p)


def log2_rn(q: Fraction, p: int) -> Fraction:
    if q <= 0:
        raise ValueError("log2 of a non-positive value")
    n, d = q.numerator, q.denominator
    if n & (n - 1) == 0 and d & (d - 1) == 0:  # exact power of two
        return Fraction(n.bit_length() - d.bit_length())
    return rn(_frac_of_dec(_DEC.divide(_DEC.ln(_dec_of(q)), _DEC.ln(decimal.Decimal(2)))), p)


def exp10_rn(k: int, p: int) -> Fraction:
    return rn(Fraction(10) ** k, p)


def decimal_digits(v: Fraction, n: int):
    """mpfr_get_str(base 10, n digits, RNDN) of a nonzero v: returns
    (digit string with sign, exponent) such that v ~ 0.DIGITS * 10^exp."""
    sign = "-" if v < 0 else ""
    a = -v if v < 0 else v
    # e10 with 10^(e10-1) <= a < 10^e10
    e10 = int((a.numerator.bit_length() - a.denominator.bit_length()) * 0.30102999566398120) + 1
    while a >= Fraction(10) ** e10:
        e10 += 1
    while a < Fraction(10) ** (e10 - 1):
        e10 -= 1
    scaled = a * Fraction(10) ** (n - e10)
    m, rem = divmod(scaled.numerator, scaled.denominator)
    twice = 2 * rem
    if twice > scaled.denominator or (twice == scaled.denominator and (m & 1)):
        m += 1
    if m == 10 ** n:
        m //= 10
        e10 += 1
    return sign + str(m), e10


class MPF:
    """An exactly known binary floating-point value with a nominal precision.

    Stands in for the ``gmpy2.mpfr`` values the reference stores in its plan
    and report records (engine.py:32-108): the plan's roundoffs, taus and
    norms.  Supports float(), ordering against numbers, and exact rational
    access (``as_integer_ratio``)."""

    __slots__ = ("value", "prec", "special")

    def __init__(self, value=0, prec: int = 53, special: str = None):
        self.prec = prec
        self.special = special
        self.value = Fraction(0) if special else to_fraction(value)

    @classmethod
    def inf(cls, prec: int = 53) -> "MPF":
        return cls(0, prec, special="inf")

    @classmethod
    def rounded(cls, value, prec: int) -> "MPF":
        return cls(rn(to_fraction(value), prec), prec)

    def is_inf(self) -> bool:
        return self.special == "inf"

    def __float__(self) -> float:
        if self.special == "inf":
            return math.inf
        return float(self.value)

    def as_integer_ratio(self):
        if self.special:
            raise OverflowError("cannot convert infinity to integer ratio")
        return self.value.numerator, self.value.denominator

    def _cmp_key(self, other):
        if isinstance(other, MPF):
            return other
        if isinstance(other, float) and math.isinf(other):
            return MPF.inf() if other > 0 else None
        return MPF(other)

    def __eq__(self, other):
        try:
            o = self._cmp_key(other)
        except (TypeError, ValueError):
            return NotImplemented
        if o is None:
            return False
        return self.special == o.special and self.value == o.value

    def __hash__(self):
        return hash((self.special, self.value))

    def __lt__(self, other):
        o = self._cmp_key(other)
        if self.special == "inf":
            return False
        if o is None or o.special == "inf":
            return o is not None
        return self.value < o.value

    def __le__(self, other):
        return self == other or self < other

    def __gt__(self, other):
        o = self._cmp_key(other)
        if self.special == "inf":
            return o is None or o.special != "inf"
        if o is None:
            return True
        if o.special == "inf":
            return False
        return self.value > o.value

    def __ge__(self, other):
        return self == other or self > other

    def __bool__(self):
        return self.special is not None or self.value != 0

    def __repr__(self):
        return f"MPF({fmt_sci(self, 17)!r}, prec={self.prec})"


def fmt_sci(x, sig_digits: int) -> str:
    """precision.py:256-269 restated: scientific notation with sig_digits
    correctly rounded significant digits."""
    if isinstance(x, MPF) and x.special == "inf":
        return "inf"
    v = to_fraction(x)
    if v == 0:
        return "0.0e0"
    ds, exp = decimal_digits(v, sig_digits)
    sign = ""
    if ds.startswith("-"):
        sign, ds = "-", ds[1:]
    return f"{sign}{ds[0]}.{ds[1:]}e{exp - 1}"


def fmt7(x) -> str:
    """engine.py:28-29 ``_fmt``: 7 significant digits of mpfr(x, 64)."""
    if isinstance(x, MPF) and x.special == "inf":
        return "inf"
    if isinstance(x, float) and math.isinf(x):
        return "inf" if x > 0 else "-inf"
    return fmt_sci(rn(to_fraction(x), 64), 7)
