"""Self-verification suite behind ``mpps verify`` (acceptance.py:1-407
restated for the device build).

Each criterion keeps the reference's name, inputs and pass rule where the
device lattice can execute them; evaluations that need more than quad-double
(the reference's 32/64-digit accuracy runs need a 64/128-digit ground truth)
run at the lattice digits 15 and 31, whose 2x-digit ground truth (dd / qd)
the device holds.

    pade_coefficient_golden        acceptance.py:49-63    (host, exact)
    cost_ratio_formula             acceptance.py:82-116   (host, exact)
    planner_schedule_reproduction  acceptance.py:119-145  (device plan_only)
    nonnormal_diagnostics          acceptance.py:148-164  (device alpha_m)
    accuracy_suite                 acceptance.py:167-209  (device, d in {15, 31})
    degenerate_equivalence         acceptance.py:332-362  (device, d in {15, 31})

Not restated: ward_block_norms (a 64-digit evaluation; it fails by design in
the reference too, README.md:96-101), bound_containment and f_recurrence
(MPFR arithmetic at 40-96 random digit counts, no device formats).
"""

from __future__ import annotations

from dataclasses import dataclass
from fractions import Fraction
from typing import Callable, List, Tuple

import numpy as np

from .coefficients import CoefficientSeries, pade_exp_coeffs
from .planner import EvaluationPlan, cost_ratio, _roundoff
from .bigfloat import MPF
from .precision import PrecisionCtx


@dataclass
class CriterionResult:
    name: str
    passed: bool
    detail: str

    def line(self) -> str:
        return f"[{'PASS' if self.passed else 'FAIL'}] {self.name}: {self.detail}"


_PADE_GOLDEN = (Fraction(1, 2), Fraction(3, 25), Fraction(11, 600), Fraction(11, 5520), Fraction(3, 18400),
                Fraction(1, 96600), Fraction(1, 1932000))


def check_pade_golden() -> CriterionResult:
    num, _ = pade_exp_coeffs(13, 13)
    got = tuple(num.coeffs[1:8])
    ok = got == _PADE_GOLDEN and num.coeffs[0] == 1
    return CriterionResult("pade_coefficient_golden", ok, f"numerator j=1..7 = {[str(c) for c in got]}")


#: acceptance.py:84-89 -- the paper's published Table-1 rows.
_TABLE1 = (
    (32, 42, 7, 6, (30, 25, 18, 11, 3, 1), 0.271),
    (64, 64, 8, 8, (61, 55, 47, 38, 28, 18, 7, 1), 0.268),
    (128, 100, 10, 10, (124, 115, 104, 92, 78, 64, 49, 34, 18, 1), 0.247),
    (256, 182, 14, 13, (248, 234, 217, 197, 176, 154, 131, 107, 82, 57, 31, 4, 1), 0.254),
)


def _plan_from_schedule(s, r, d, schedule) -> EvaluationPlan:
    return EvaluationPlan(s=s, r=r, nu=1, d_working=d, level_digits=tuple(schedule),
                          level_roundoffs=tuple(_roundoff(k) for k in schedule), tau_seq=(),
                          norm_bs=(MPF(1, 64),) * (r + 1), norm_y=MPF(1, 64))


def check_cost_ratio() -> CriterionResult:
    worst, details = 0.0, []
    for d, m, s, r, schedule, want in _TABLE1:
        _, sav = cost_ratio(_plan_from_schedule(s, r, d, schedule))
        worst = max(worst, abs(sav - want))
        details.append(f"d={d}: {100 * sav:.1f}% vs {100 * want:.1f}%")
    return CriterionResult("cost_ratio_formula", worst <= 0.001 + 1e-12,
                           "; ".join(details) + f" (max dev {100 * worst:.2f} pts)")


def check_planner_table1() -> CriterionResult:
    from .cli import run_table1
    rows = run_table1("cauchy", 100, 0, 100.0, 0, "taylor_exp", 42, [d for d, *_ in _TABLE1],
                      [m for _, m, *_ in _TABLE1])
    problems = []
    for row, (d, m, s, r, schedule, want) in zip(rows, _TABLE1):
        if (row["s"], row["r"]) != (s, r):
            problems.append(f"d={d}: (s,r)=({row['s']},{row['r']})")
            continue
        dev = max(abs(a - b) for a, b in zip(row["schedule"], schedule))
        if dev > 2:
            problems.append(f"d={d}: schedule off by {dev}")
        if any(a < b for a, b in zip(row["schedule"], row["schedule"][1:])):
            problems.append(f"d={d}: schedule not monotone")
        if row["schedule"][-1] > 2:
            problems.append(f"d={d}: final level {row['schedule'][-1]} > 2")
        if abs(row["savings"] - want) > 0.03:
            problems.append(f"d={d}: savings {row['savings']:.3f}")
    return CriterionResult("planner_schedule_reproduction", not problems,
                           "; ".join(problems) if problems else
                           "all four schedules within +-2 digits, savings within 3 points")


def check_nonnormal_diagnostics() -> CriterionResult:
    from . import gallery, ops
    from .bounds import alpha_m, extra_squarings
    ctx = gallery.GEN_CTX
    X = gallery.to_device(gallery.scale_values(gallery.gen_nonnormal2(ctx), 1), PrecisionCtx(15))
    a, d_star = alpha_m(X, 42)
    nx = float(ops.one_norm(X)[0])
    norm_ok = nx == 500000.05 and round(nx, -4) == 5e5
    ell0 = extra_squarings(nx, 7)
    ok = d_star == 7 and 0.61 <= a <= 0.71 and norm_ok and ell0 == 18
    return CriterionResult("nonnormal_diagnostics", ok,
                           f"d*={d_star} (want 7), alpha_m={a:.4f} (want [0.61,0.71]), ||X||_1={nx} "
                           f"(5e5 at 2 sig figs), extra_squarings={ell0} (want 18)")


_FAMS = [("taylor_exp", 20), ("pade_exp_num", 13), ("pade_exp_den", 13), ("taylor_cos", 8)]


def _accuracy_configs() -> List[Tuple[str, int, int, str, int, int]]:
    """acceptance.py:167-188 with the 32/64-digit runs at 15/31 digits."""
    cfgs = []
    gens = ("cauchy", "lotkin", "smoke", "triu_rand")
    for gi, gen in enumerate(gens):
        for ni, n in enumerate((8, 20)):
            for fi in range(3):
                fam, m = _FAMS[(gi + ni + fi) % 4]
                cfgs.append((gen, n, gi * 7 + ni, fam, m, 15 if fi % 2 == 0 else 31))
    for gi, gen in enumerate(gens):
        fam, m = _FAMS[gi]
        cfgs.append((gen, 50, gi, fam, m, 15))
    for gi, gen in enumerate(gens):
        fam, m = _FAMS[(gi + 1) % 4]
        cfgs.append((gen, 8, gi + 100, fam, m, 31))
    return cfgs


def check_accuracy_suite() -> CriterionResult:
    from .cli import build_argument
    from .harness import compare
    cfgs = _accuracy_configs()
    n_soft, hard_fail = 0, []
    for gen, n, seed, fam, m, d in cfgs:
        ctx = PrecisionCtx(d)
        X, series = build_argument(gen, n, seed, 1.0, 0, fam, m, ctx)
        rec = compare(X, series, ctx, m=m if fam == "taylor_exp" else None)[0]
        if rec["eps_mixed"] <= 10.0 * rec["rnu"]:
            n_soft += 1
        if rec["eps_mixed"] > max(10.0 * rec["rnu"], 10.0 * rec["eps_fixed"]):
            hard_fail.append(f"{gen}(n={n},seed={seed},{fam},d={d})")
    frac = n_soft / len(cfgs)
    return CriterionResult("accuracy_suite", frac >= 0.95 and not hard_fail,
                           f"{len(cfgs)} runs, eps_v <= 10*r*n*u in {100 * frac:.0f}%, "
                           f"hard failures: {hard_fail or 'none'}")


def check_degenerate_equivalence() -> CriterionResult:
    """acceptance.py:332-362: a flat series clamps the plan to the working
    precision everywhere, and the mixed result must equal the fixed one
    bit for bit (the reference's d = 20 / 32 runs at 15 / 31 digits)."""
    from . import gallery
    from .engine import ps_fixed, ps_mixed_general
    flat = lambda m: CoefficientSeries(tuple(Fraction(1) for _ in range(m + 1)))  # noqa: E731
    configs = [(g, n, m, 15) for g in ("cauchy", "lotkin", "smoke") for n in (3, 4, 5) for m in (5, 9)]
    configs = configs[:18] + [("smoke", 6, 12, 31), ("cauchy", 6, 7, 31)]
    mismatches, not_clamped = [], []
    for gen, n, m, d in configs:
        ctx = PrecisionCtx(d)
        X = gallery.to_device(gallery.round_values(gallery.generate_values(gen, n), ctx), ctx)
        mixed = ps_mixed_general(X, flat(m), ctx)
        fixed = ps_fixed(X, flat(m), ctx)
        p = mixed.plan
        if p.nu != p.r + 1 or any(k != d for k in p.level_digits):
            not_clamped.append(f"{gen}(n={n},m={m})")
            continue
        a = _words(mixed.result)
        b = _words(fixed.result)
        if a.shape != b.shape or not np.array_equal(a, b):
            mismatches.append(f"{gen}(n={n},m={m})")
    ok = not mismatches and not not_clamped
    return CriterionResult("degenerate_equivalence", ok,
                           f"{len(configs)} clamped configs, bitwise mismatches: {mismatches or 'none'}"
                           + (f"; not clamped: {not_clamped}" if not_clamped else ""))


def _words(M) -> np.ndarray:
    emb = getattr(M, "emb", M)
    return emb.words_numpy()


ALL_CRITERIA: Tuple[Callable[[], CriterionResult], ...] = (
    check_pade_golden,
    check_cost_ratio,
    check_planner_table1,
    check_nonnormal_diagnostics,
    check_accuracy_suite,
    check_degenerate_equivalence,
)


def run_all(verbose: bool = True) -> List[CriterionResult]:
    """acceptance.py:400-407."""
    results = []
    for fn in ALL_CRITERIA:
        res = fn()
        results.append(res)
        if verbose:
            print(res.line())
    return results


__all__ = ["CriterionResult", "ALL_CRITERIA", "run_all"]
