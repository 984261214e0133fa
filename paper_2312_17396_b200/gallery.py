"""Deterministic test-matrix generators (gallery.py:1-107 restated).

Every generator returns the reference's entries exactly: each entry is the
value the reference's ``as_mpc(..., ctx)`` / ``mpc(..., precision=p)``
produces at p = ceil(d log2 10) bits, kept as exact ``Fraction`` pairs
(re, im).  ``generate`` places them on the device in the smallest hardware
format holding p bits (fp64 / dd / qd, as ``matio`` does for decimal
input); ``generate_fp64`` gives the nearest fp64 array, enough for the
planner-only callers (``plan_only`` forms its powers at 16 digits,
engine.py:485-504) at any working precision, including d > 63.

* cauchy(n): A(i,j) = 1/(i+j), 1-based (gallery.py:21-28)
* ward: the 3x3 stiff integer matrix (31-34)
* nonnormal2: [[-0.1, 1e6], [0, -0.1]] from the fp64 literals (37-39)
* lotkin(n): Hilbert with its first row replaced by ones (42-50)
* triu_rand(n, scale, seed): strictly upper triangular
  scale * N(0,1) from ``numpy.random.default_rng(seed)`` (53-63)
* smoke(n): roots of unity on the diagonal, ones on the superdiagonal, a one
  in the (n,1) corner; cos/sin of RN_p(RN_p(2 pi_p i) / n) (66-83)
"""

from __future__ import annotations

from fractions import Fraction
from typing import List, Tuple

import numpy as np

from .bigfloat import rn
from .precision import PrecisionCtx

#: gallery.py:18 -- default generation context (40 digits).
GEN_CTX = PrecisionCtx(40)

Entry = Tuple[Fraction, Fraction]
Values = List[List[Entry]]


def _re(x, p: int) -> Entry:
    return rn(Fraction(x), p), Fraction(0)


def _check_n(n: int):
    if n < 1:
        raise ValueError("n must be >= 1")


def gen_cauchy(n: int, ctx: PrecisionCtx = GEN_CTX) -> Values:
    _check_n(n)
    p = ctx.binary_precision
    return [[_re(Fraction(1, i + j), p) for j in range(1, n + 1)] for i in range(1, n + 1)]


def gen_ward(ctx: PrecisionCtx = GEN_CTX) -> Values:
    p = ctx.binary_precision
    data = [[-131, 19, 18], [-390, 56, 54], [-387, 57, 52]]
    return [[_re(v, p) for v in row] for row in data]


def gen_nonnormal2(ctx: PrecisionCtx = GEN_CTX) -> Values:
    p = ctx.binary_precision
    return [[_re(-0.1, p), _re(10 ** 6, p)], [_re(0, p), _re(-0.1, p)]]


def gen_lotkin(n: int, ctx: PrecisionCtx = GEN_CTX) -> Values:
    _check_n(n)
    p = ctx.binary_precision
    rows = [[_re(1, p)] * n]
    for i in range(2, n + 1):
        rows.append([_re(Fraction(1, i + j - 1), p) for j in range(1, n + 1)])
    return rows[:n]


def gen_triu_rand(n: int, scale: float = 100.0, seed: int = 0, ctx: PrecisionCtx = GEN_CTX) -> Values:
    _check_n(n)
    p = ctx.binary_precision
    g = np.random.default_rng(seed).standard_normal((n, n))
    # scale * g[i][j] is a Python float product (fp64), then rounded to p bits
    return [[_re(float(scale) * float(g[i][j]), p) if j > i else _re(0, p) for j in range(n)]
            for i in range(n)]


def _cos_sin(i: int, n: int, p: int) -> Entry:
    """cos/sin of ang = RN_p(RN_p(RN_p(2 pi) * i) / n) at p bits, each op
    rounded to nearest as the reference's gmpy2 context does."""
    import mpmath
    with mpmath.workprec(p):
        two_pi = mpmath.mpf(2) * +mpmath.pi         # 2 * RN_p(pi), exact doubling
        ang = (two_pi * i) / n
        return _mpf_frac(mpmath.cos(ang)), _mpf_frac(mpmath.sin(ang))


def _mpf_frac(x) -> Fraction:
    sign, man, exp, _ = x._mpf_
    man = -int(man) if sign else int(man)
    return Fraction(man * (1 << exp)) if exp >= 0 else Fraction(man, 1 << (-exp))


def gen_smoke(n: int, ctx: PrecisionCtx = GEN_CTX) -> Values:
    _check_n(n)
    p = ctx.binary_precision
    rows = [[_re(0, p) for _ in range(n)] for _ in range(n)]
    for i in range(n):
        rows[i][i] = _cos_sin(i, n, p)
        if i + 1 < n:
            rows[i][i + 1] = _re(1, p)
    rows[n - 1][0] = _re(1, p)
    return rows


GENERATORS = {
    "cauchy": gen_cauchy,
    "lotkin": gen_lotkin,
    "smoke": gen_smoke,
    "ward": gen_ward,
    "nonnormal2": gen_nonnormal2,
    "triu_rand": gen_triu_rand,
}


def generate_values(name: str, n: int = 0, seed: int = 0, scale: float = 100.0,
                    ctx: PrecisionCtx = GEN_CTX) -> Values:
    """gallery.py:96-107 dispatch, exact entries."""
    if name == "ward":
        return gen_ward(ctx)
    if name == "nonnormal2":
        return gen_nonnormal2(ctx)
    if name == "triu_rand":
        return gen_triu_rand(n, scale, seed, ctx)
    if name in GENERATORS:
        return GENERATORS[name](n, ctx)
    raise KeyError(f"unknown generator {name!r}")


def scale_values(values: Values, ell: int) -> Values:
    """scale_pow2 (precision.py:220-224): exact multiplication by 2^-ell."""
    f = Fraction(1, 1 << ell) if ell >= 0 else Fraction(1 << (-ell))
    return [[(re * f, im * f) for (re, im) in row] for row in values]


def round_values(values: Values, ctx: PrecisionCtx) -> Values:
    """round_to (precision.py:153-157) of exact entries."""
    p = ctx.binary_precision
    return [[(rn(re, p), rn(im, p)) for (re, im) in row] for row in values]


def to_device(values: Values, ctx: PrecisionCtx, device=None):
    """Exact entries (<= p bits of ctx) -> MatBatch / ComplexMatBatch of batch 1
    in the storage format of ctx (d <= 63)."""
    from .matio import _build
    return _build(values, ctx.decimal_digits, device)


def to_fp64(values: Values) -> np.ndarray:
    """Nearest fp64 (complex128 when any imaginary part is nonzero)."""
    re = np.array([[float(e[0]) for e in row] for row in values], dtype=np.float64)
    if any(e[1] != 0 for row in values for e in row):
        im = np.array([[float(e[1]) for e in row] for row in values], dtype=np.float64)
        return re + 1j * im
    return re


def generate(name: str, n: int = 0, seed: int = 0, scale: float = 100.0,
             ctx: PrecisionCtx = GEN_CTX, device=None):
    """The generated matrix on the device at ctx's storage format."""
    return to_device(generate_values(name, n, seed, scale, ctx), ctx, device)
