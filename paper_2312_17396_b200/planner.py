"""Precision planner, lattice snapping and the digit-weighted cost model.

Bit-exact host restatement of engine.py:32-84 (``EvaluationPlan``),
engine.py:157-215 (``plan_precisions``), engine.py:218-240
(``snap_to_lattice``) and engine.py:255-262 (``cost_ratio``).  Every MPFR
operation of the reference is reproduced with exact rationals plus one
correct rounding at the same precision (bigfloat.py), so for the same input
norms the digits, the switch index nu, the roundoffs and the tau sequence
are identical to the reference's.

The device-facing addition is ``level_formats``: the lattice format that
executes each Horner level (digits -> fp32/fp64/dd/qd).
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field
from fractions import Fraction
from typing import Dict, Sequence, Tuple

from .bigfloat import MPF, exp10_rn, fmt7, log10_rn, rn, to_fraction
from .bounds import tau_sequence
from .precision import LATTICE, PrecisionCtx, format_for_digits

_P = 107                       # BOUND_CTX bits (engine.py:25 _G)
_ONE_E_MINUS_9 = rn(Fraction(1, 10 ** 9), 53)   # mpfr("1e-9") at 53 bits


_ROUNDOFF = {}


def _roundoff(k: int) -> MPF:
    v = _ROUNDOFF.get(k)
    if v is None:
        v = _ROUNDOFF[k] = MPF(exp10_rn(-k, _P), _P)
    return v


@dataclass(frozen=True)
class EvaluationPlan:
    """engine.py:32-84.  Level digits/roundoffs are indexed 1..r (stored
    0-based); levels below nu run at the working precision."""
    s: int
    r: int
    nu: int
    d_working: int
    level_digits: Tuple[int, ...]
    level_roundoffs: Tuple[MPF, ...]
    tau_seq: Tuple[MPF, ...]
    norm_bs: Tuple[MPF, ...]
    norm_y: MPF
    delta: float = 10.0
    fix_params: bool = True
    degenerate_levels: Tuple[int, ...] = ()
    nilpotent: bool = False
    explicit_powers: bool = False

    def __post_init__(self):
        if not (1 <= self.s):
            raise ValueError("s must be >= 1")
        if not (1 <= self.nu <= self.r + 1):
            raise ValueError("nu out of range")
        if len(self.level_digits) != self.r:
            raise ValueError("need r level digits")
        for a, b in zip(self.level_digits, self.level_digits[1:]):
            if a < b:
                raise ValueError("digit schedule must be non-increasing")

    def level_ctx(self, i: int) -> PrecisionCtx:
        if i == 0:
            return PrecisionCtx(self.d_working)
        return PrecisionCtx(self.level_digits[i - 1])

    @property
    def level_formats(self) -> Tuple[int, ...]:
        """Lattice format of levels 0..r (level 0 = working precision)."""
        return (format_for_digits(self.d_working),) + tuple(
            format_for_digits(d) for d in self.level_digits)

    def to_dict(self) -> dict:
        return {
            "s": self.s, "r": self.r, "nu": self.nu,
            "working_digits": self.d_working,
            "digits": list(self.level_digits),
            "roundoffs": [fmt7(u) for u in self.level_roundoffs],
            "tau": [fmt7(t) for t in self.tau_seq],
            "norm_bs": [fmt7(b) for b in self.norm_bs],
            "norm_y": fmt7(self.norm_y),
            "delta": self.delta, "fix_params": self.fix_params,
            "degenerate_levels": list(self.degenerate_levels),
            "nilpotent": self.nilpotent,
            "explicit_powers": self.explicit_powers,
        }


def _n64(x) -> MPF:
    """mpfr(x, 64)."""
    if isinstance(x, MPF) and x.is_inf():
        return x
    return MPF(rn(to_fraction(x), 64), 64)


def plan_precisions(norm_bs: Sequence, norm_y, ctx: PrecisionCtx,
                    delta: float = 10.0, *, s: int, apply_switch: bool = True,
                    fix_params: bool = True) -> EvaluationPlan:
    """engine.py:157-215: e_i = d - log10||B0|| + log10||B_i|| + i log10||Y||
    at 107 bits, +1e-9, float(); d_i = clamp(floor(e_i), 1, d); nu = first
    level with e_i <= d - log10(delta); levels < nu at d; running max."""
    d = ctx.decimal_digits
    r = len(norm_bs) - 1
    nb = tuple(_n64(b) for b in norm_bs)
    ny = _n64(norm_y)
    taus = tuple(tau_sequence(nb, ny))
    degenerate = tuple(i for i, b in enumerate(nb) if b == 0)

    if ny == 0:
        return EvaluationPlan(
            s=s, r=r, nu=1, d_working=d, level_digits=(1,) * r,
            level_roundoffs=(_roundoff(1),) * r, tau_seq=taus, norm_bs=nb,
            norm_y=ny, delta=delta, fix_params=fix_params,
            degenerate_levels=degenerate, nilpotent=True)

    b0 = nb[0].value
    log_b0 = log10_rn(b0, _P) if b0 > 0 else Fraction(0)
    log_y = log10_rn(ny.value, _P)
    digits, qualifies = [], []
    lim = d - math.log10(delta)
    for i in range(1, r + 1):
        bi = nb[i].value
        if bi == 0 or b0 == 0:
            digits.append(1)
            qualifies.append(True)
            continue
        e = rn(rn(Fraction(d) - log_b0, _P) +
               rn(log10_rn(bi, _P) + rn(Fraction(i) * log_y, _P), _P), _P)
        e = float(rn(e + _ONE_E_MINUS_9, _P))
        digits.append(max(1, min(d, math.floor(e))))
        qualifies.append(e <= lim)

    nu = r + 1
    for i in range(1, r + 1):
        if qualifies[i - 1]:
            nu = i
            break
    if apply_switch:
        for i in range(1, nu):
            digits[i - 1] = d
    for i in range(r - 2, -1, -1):
        digits[i] = max(digits[i], digits[i + 1])
    return EvaluationPlan(
        s=s, r=r, nu=nu, d_working=d, level_digits=tuple(digits),
        level_roundoffs=tuple(_roundoff(k) for k in digits), tau_seq=taus,
        norm_bs=nb, norm_y=ny, delta=delta, fix_params=fix_params,
        degenerate_levels=degenerate)


# ----------------------------------------------------- batched fast path
_CERT_MARGIN = 1e-8


def plan_digits_batch(norm_bs, norm_y, d: int, delta: float = 10.0, apply_switch: bool = True):
    """Digits / nu / nilpotent flags of ``plan_precisions`` for a whole batch.

    Vectorised float64 evaluation of e_i, certified: the digit rule only
    consumes floor(e_i) and the test e_i <= d - log10(delta), and the float64
    evaluation is within ~1e-11 of the 107-bit value, so every row whose e_i
    all lie farther than 1e-8 from an integer and from the threshold gets the
    exact reference digits.  Uncertain rows (and any non-finite input) are
    recomputed with the exact scalar ``plan_precisions``.

    norm_bs: (B, r+1) float64, norm_y: (B,) float64 (the exact norm values).
    Returns (digits (B, r) int64, nu (B,) int64, nilpotent (B,) bool)."""
    import numpy as np
    nb = np.asarray(norm_bs, dtype=np.float64)
    ny = np.asarray(norm_y, dtype=np.float64)
    B, r1 = nb.shape
    if B <= 4:
        return _plan_rows_small(nb, ny, d, delta, apply_switch)
    r = r1 - 1
    digits = np.ones((B, r), dtype=np.int64)
    nu = np.full(B, r + 1, dtype=np.int64)
    nil = ny == 0
    lim = d - math.log10(delta)
    with np.errstate(divide="ignore", invalid="ignore"):
        lb0 = np.where(nb[:, 0] > 0, np.log10(np.where(nb[:, 0] > 0, nb[:, 0], 1.0)), 0.0)
        ly = np.log10(np.where(ny > 0, ny, 1.0))
        li = np.log10(np.where(nb[:, 1:] > 0, nb[:, 1:], 1.0))
        i = np.arange(1, r + 1, dtype=np.float64)
        e = (d - lb0)[:, None] + (li + i[None, :] * ly[:, None]) + 1e-9
    zero = (nb[:, 1:] == 0) | (nb[:, :1] == 0)
    qual = np.where(zero, True, e <= lim)
    dig = np.where(zero, 1, np.clip(np.floor(e), 1, d)).astype(np.int64)
    risky = ~zero & ((np.abs(e - np.round(e)) < _CERT_MARGIN) | (np.abs(e - lim) < _CERT_MARGIN))
    bad = ~np.isfinite(nb).all(axis=1) | ~np.isfinite(ny) | risky.any(axis=1)
    anyq = qual.any(axis=1)
    first = np.where(anyq, qual.argmax(axis=1) + 1, r + 1)
    if apply_switch:
        cols = np.arange(1, r + 1)[None, :]
        dig = np.where(cols < first[:, None], d, dig)
    # running max from the outermost level inward (engine.py:209-210)
    dig = np.maximum.accumulate(dig[:, ::-1], axis=1)[:, ::-1]
    digits[:] = dig
    nu[:] = first
    digits[nil] = 1
    nu[nil] = 1
    for b in np.nonzero(bad & ~nil)[0]:
        p = plan_precisions(nb[b], ny[b], PrecisionCtx(d), delta, s=1, apply_switch=apply_switch)
        digits[b] = p.level_digits
        nu[b] = p.nu
        nil[b] = p.nilpotent
    return digits, nu, nil


def _plan_rows_small(nb, ny, d: int, delta: float, apply_switch: bool):
    """plan_digits_batch for a few rows in scalar Python (numpy's per-call
    overhead dominates a one-matrix evaluation): the same certified float64
    rule -- digits exact away from integers and the delta threshold, the
    exact plan_precisions otherwise -- so the result is identical."""
    import numpy as np
    B, r1 = nb.shape
    r = r1 - 1
    lim = d - math.log10(delta)
    digits = np.ones((B, r), dtype=np.int64)
    nu = np.full(B, r + 1, dtype=np.int64)
    nil = np.zeros(B, dtype=bool)
    for b in range(B):
        row = [float(x) for x in nb[b]]
        y = float(ny[b])
        if y == 0:
            nil[b], nu[b] = True, 1
            continue
        risky = not (all(math.isfinite(x) for x in row) and math.isfinite(y))
        dig, qual = [], []
        if not risky:
            lb0 = math.log10(row[0]) if row[0] > 0 else 0.0
            ly = math.log10(y)
            for i in range(1, r + 1):
                if row[i] == 0 or row[0] == 0:
                    dig.append(1)
                    qual.append(True)
                    continue
                e = (d - lb0) + (math.log10(row[i]) + i * ly) + 1e-9
                if abs(e - round(e)) < _CERT_MARGIN or abs(e - lim) < _CERT_MARGIN:
                    risky = True
                    break
                dig.append(min(max(math.floor(e), 1), d))
                qual.append(e <= lim)
        if risky:
            p = plan_precisions(nb[b], ny[b], PrecisionCtx(d), delta, s=1, apply_switch=apply_switch)
            digits[b], nu[b], nil[b] = p.level_digits, p.nu, p.nilpotent
            continue
        first = next((i + 1 for i, q in enumerate(qual) if q), r + 1)
        if apply_switch:
            for i in range(first - 1):
                dig[i] = d
        for i in range(r - 2, -1, -1):
            if dig[i + 1] > dig[i]:
                dig[i] = dig[i + 1]
        digits[b] = dig
        nu[b] = first
    return digits, nu, nil


_FMT_OF_DIGITS = {}


def formats_of_digits(digits):
    """Lattice format of each digit count (cached)."""
    out = []
    for x in digits:
        f = _FMT_OF_DIGITS.get(x)
        if f is None:
            f = _FMT_OF_DIGITS[x] = format_for_digits(int(x))
        out.append(f)
    return tuple(out)


def fixed_plan(norm_bs: Sequence, norm_y, ctx: PrecisionCtx, s: int) -> EvaluationPlan:
    """The all-working plan ps_fixed builds (engine.py:336-340)."""
    d = ctx.decimal_digits
    r = len(norm_bs) - 1
    nb = tuple(_n64(b) for b in norm_bs)
    ny = _n64(norm_y)
    return EvaluationPlan(
        s=s, r=r, nu=r + 1, d_working=d, level_digits=(d,) * r,
        level_roundoffs=(ctx.unit_roundoff,) * r,
        tau_seq=tuple(tau_sequence(nb, ny)), norm_bs=nb, norm_y=ny)


def snap_to_lattice(plan: EvaluationPlan, lattice: Sequence[int]) -> EvaluationPlan:
    """engine.py:218-240: each level to the smallest lattice member >= it."""
    lat = sorted(set(int(x) for x in lattice))
    if not lat:
        raise ValueError("empty lattice")
    if plan.d_working not in lat:
        raise ValueError("lattice must contain the working digits")
    snapped = []
    for di in plan.level_digits:
        up = [x for x in lat if x >= di]
        if not up:
            raise ValueError(f"no lattice member >= {di}")
        snapped.append(up[0])
    return EvaluationPlan(
        s=plan.s, r=plan.r, nu=plan.nu, d_working=plan.d_working,
        level_digits=tuple(snapped),
        level_roundoffs=tuple(_roundoff(k) for k in snapped),
        tau_seq=plan.tau_seq, norm_bs=plan.norm_bs, norm_y=plan.norm_y,
        delta=plan.delta, fix_params=plan.fix_params,
        degenerate_levels=plan.degenerate_levels, nilpotent=plan.nilpotent,
        explicit_powers=plan.explicit_powers)


def hardware_lattice(d_working: int) -> Tuple[int, ...]:
    """The B200 lattice restricted to [1, d_working] (SURVEY 8c recipe)."""
    return tuple(x for x in LATTICE if x <= d_working)


def cost_ratio(plan: EvaluationPlan) -> Tuple[float, float]:
    """engine.py:255-262: ((s-1) d + sum d_i) / ((s+r-1) d) and 1 - that."""
    s, r, d = plan.s, plan.r, plan.d_working
    if s + r - 1 <= 0:
        return 1.0, 0.0
    cr = Fraction((s - 1) * d + sum(plan.level_digits), (s + r - 1) * d)
    return float(cr), float(1 - cr)


def matmul_counts(plan: EvaluationPlan) -> Dict[int, int]:
    """engine.py:384-386: {d: s-1} plus one per Horner level digit."""
    counts: Dict[int, int] = {plan.d_working: plan.s - 1}
    for di in plan.level_digits:
        counts[di] = counts.get(di, 0) + 1
    return counts


def default_block_size(m: int) -> int:
    """engine.py:111-112."""
    return math.ceil(math.sqrt(m))
