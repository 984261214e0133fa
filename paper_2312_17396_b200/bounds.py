"""Host-side scalar bounds and decay diagnostics used by the planner and the
evaluation reports, restated from pkg/src/mpps/bounds.py with every
BOUND_CTX (107-bit) operation emulated exactly (see bigfloat.py).

Only the pieces the hot path consumes are here: ``tau_sequence`` (recorded
in every plan, engine.py:172), ``gamma``/``thm21_bound`` (the optional
``with_bound`` report field, engine.py:283-292) and ``extra_squarings``
(the scaling count of the config-3 scaling-and-squaring driver,
bounds.py:216-227).
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from fractions import Fraction
from typing import List, Optional, Sequence, Tuple

from .bigfloat import MPF, exp_rn, log2_rn, rn, to_fraction

_P = 107  # BOUND_CTX binary precision (precision.py:75 -> ceil(32*log2 10))


class BoundInvalidError(ArithmeticError):
    """k*u >= 1: the gamma constant is vacuous (bounds.py:23-24)."""


def _f(x) -> Fraction:
    if isinstance(x, MPF) and x.is_inf():
        raise ValueError("infinite operand")
    return rn(to_fraction(x), _P)


def _mpf(v: Fraction) -> MPF:
    return MPF(v, _P)


def gamma(k, u) -> MPF:
    """gamma_k = k u / (1 - k u) (bounds.py:31-36)."""
    ku = rn(_f(k) * _f(u), _P)
    if ku >= 1:
        raise BoundInvalidError(f"k*u = {float(ku)} >= 1")
    return _mpf(rn(ku / rn(1 - ku, _P), _P))


@dataclass(frozen=True)
class BoundInputs:
    """bounds.py:39-60: precisions/norm_bs over levels nu-1..r, base first."""
    n: int
    precisions: Tuple
    norm_y: object
    norm_bs: Tuple
    s: int = 0
    r: int = 0
    nu: int = 1
    sigma: Optional[object] = None

    def __post_init__(self):
        if len(self.precisions) != len(self.norm_bs):
            raise ValueError("precisions and norm_bs must align")
        for a, b in zip(self.precisions, self.precisions[1:]):
            if _f(b) < _f(a):
                raise ValueError("precisions must ascend outward")


def f_constants_closed(precisions: Sequence, n: int) -> List[MPF]:
    """bounds.py:63-80 (closed form of the accumulated multipliers)."""
    us = [_f(u) for u in precisions]
    L = len(us) - 1
    fs = [Fraction(2)]
    base = us[0]
    for j in range(1, L + 1):
        lead = n if j == L else n + 2
        acc = rn(_f(lead) * rn(us[j] / base, _P), _P)
        for t in range(1, j):
            acc = rn(acc + rn(_f(n + 1) * rn(us[t] / base, _P), _P), _P)
        fs.append(rn(acc + 1, _P))
    return [_mpf(v) for v in fs]


def thm21_bound(inp: BoundInputs) -> MPF:
    """bounds.py:101-113: sum_i gamma_{f_i}(u_base) ||Y||^i ||B_i||."""
    fs = f_constants_closed(inp.precisions, inp.n)
    u_base = inp.precisions[0]
    y = _f(inp.norm_y)
    total = Fraction(0)
    ypow = Fraction(1)
    for fi, nb in zip(fs, inp.norm_bs):
        g = to_fraction(gamma(fi, u_base))
        term = rn(g * rn(ypow * _f(nb), _P), _P)
        total = rn(total + term, _P)
        ypow = rn(ypow * y, _P)
    return _mpf(total)


def tau_sequence(norm_bs: Sequence, norm_y) -> List[MPF]:
    """bounds.py:151-162: tau_i = ||B_i|| ||Y|| / ||B_{i-1}|| (inf if the
    denominator is zero)."""
    y = _f(norm_y)
    out = []
    for prev, cur in zip(norm_bs, norm_bs[1:]):
        pv = _f(prev)
        if pv == 0:
            out.append(MPF.inf(_P))
        else:
            out.append(_mpf(rn(rn(_f(cur) * y, _P) / pv, _P)))
    return out


def extra_squarings(normX, s: int) -> int:
    """bounds.py:216-227: max(0, ceil(log2(e ||X|| / s)))."""
    if s < 1:
        raise ValueError("s must be >= 1")
    x = _f(normX)
    if x <= 0:
        raise ValueError("normX must be > 0")
    e1 = exp_rn(Fraction(1), _P)
    arg = rn(rn(e1 * x, _P) / _f(s), _P)
    if arg <= 1:
        return 0
    return int(math.ceil(log2_rn(arg, _P)))


def alpha_m(X, m: int):
    """bounds.py:193-213: the degree-selection norm surrogate
    max(||X^d||^(1/d), ||X^(d+1)||^(1/(d+1))) at d = floor((1+sqrt(4m+5))/2)
    (adjusted so d(d-1) <= m+1 < d(d+1)).  The powers are formed on the
    device at fp64 (the reference forms them at the 16-digit NORM_CTX; this
    is a magnitude diagnostic).  ``X``: a device MatBatch of batch 1.
    Returns (alpha as float, d)."""
    if m < 1:
        raise ValueError("m must be >= 1")
    from . import ops
    from .precision import NORM_CTX
    d_star = int((1 + math.isqrt(4 * m + 5)) // 2)
    while (d_star + 1) * d_star <= m + 1:
        d_star += 1
    while d_star * (d_star - 1) > m + 1:
        d_star -= 1
    X = ops.round_to(X, NORM_CTX)
    P = X
    for _ in range(d_star - 1):
        P = ops.mat_mul(P, X, NORM_CTX)
    nd = float(ops.one_norm(P)[0])
    P = ops.mat_mul(P, X, NORM_CTX)
    nd1 = float(ops.one_norm(P)[0])
    return max(nd ** (1.0 / d_star), nd1 ** (1.0 / (d_star + 1))), d_star
