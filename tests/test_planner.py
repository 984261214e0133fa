"""Host planner (planner.py) vs the C MPFR restatement of engine.py:157-215
(oracle/mpfr_oracle.c orc_plan), plus the reference's own planner tests
(test_engine.py:93-147, 290-326) and cost-ratio goldens."""
import math
import random
from fractions import Fraction

import numpy as np
import pytest

from paper_2312_17396_b200 import (EvaluationPlan, PrecisionCtx, cost_ratio, plan_precisions,
                                   snap_to_lattice, tau_sequence, taylor_exp_coeffs)
from paper_2312_17396_b200.bigfloat import MPF, rn
from paper_2312_17396_b200.planner import fixed_plan


def _norms2_to_frac(n2):
    return [Fraction(a) + Fraction(b) for a, b in n2]


def _random_norms(rng, r):
    """Decaying block norms like the PS blocks of a Taylor series, with
    54-bit values (as one_norm produces) written as (hi, lo) pairs."""
    out = []
    y = 10 ** rng.uniform(-3, 2)
    b = 10 ** rng.uniform(-2, 4)
    for i in range(r + 1):
        v = rn(Fraction(b), 54)
        if rng.random() < 0.3:
            v = rn(Fraction(b) * (1 + Fraction(rng.randrange(1 << 20), 1 << 53)), 54)
        hi = float(v)
        out.append((hi, float(v - Fraction(hi))))
        b = b * 10 ** rng.uniform(-12, 0.5)
    yv = rn(Fraction(y), 54)
    out.append((float(yv), float(yv - Fraction(float(yv)))))
    return np.array(out)


@pytest.mark.parametrize("seed", range(4))
def test_planner_matches_mpfr_oracle_random(oracle_lib, seed):
    rng = random.Random(seed)
    count = 5000
    for _ in range(count):
        r = rng.randint(1, 13)
        d = rng.choice([15, 16, 31, 32, 63, 64, 128])
        delta = rng.choice([10.0, 10.0, 2.0, 100.0])
        n2 = _random_norms(rng, r)
        fr = _norms2_to_frac(n2)
        p = plan_precisions(fr[:r + 1], fr[r + 1], PrecisionCtx(d), delta, s=3)
        dig, nu, nil, _ = oracle_lib.plan_digits(n2, d, delta)
        assert p.level_digits == dig and p.nu == nu and p.nilpotent == nil, (fr, d, delta)


def test_planner_integer_and_zero_edges(oracle_lib):
    cases = [
        [1.0, 1.0, 1.0, 1.0], [10.0, 1.0, 0.1, 0.01], [100.0, 0.0, 1e-5, 3.0],
        [0.0, 1.0, 1.0, 1.0], [1000.0, 1e-300, 1e-310, 0.5], [2.0 ** 30, 2.0 ** -60, 2.0 ** -90, 2.0 ** -3],
    ]
    for c in cases:
        n2 = np.array([[x, 0.0] for x in c])
        r = len(c) - 2
        for d in (15, 31, 63):
            p = plan_precisions(c[:r + 1], c[r + 1], PrecisionCtx(d), s=2)
            dig, nu, nil, _ = oracle_lib.plan_digits(n2, d)
            assert (p.level_digits, p.nu) == (dig, nu), c


def test_flat_is_fixed():
    plan = plan_precisions([1.0, 1.0, 1.0], 1.0, PrecisionCtx(24), 10.0, s=2)
    assert plan.nu == plan.r + 1 and plan.level_digits == (24, 24)


def test_monotone_and_bounded():
    plan = plan_precisions([10.0, 1e-3, 1e-9, 1e-20], 0.5, PrecisionCtx(32), 10.0, s=2)
    ds = plan.level_digits
    assert all(a >= b for a, b in zip(ds, ds[1:]))
    assert all(1 <= x <= 32 for x in ds)
    assert all(ds[i - 1] == 32 for i in range(1, plan.nu))


def test_nilpotent_flag():
    plan = plan_precisions([5.0, 3.0, 1.0], 0.0, PrecisionCtx(16), 10.0, s=2)
    assert plan.nilpotent and plan.nu == 1 and plan.level_digits == (1, 1)
    assert [float(u) for u in plan.level_roundoffs] == [0.1, 0.1]


def test_tau_sequence_exact():
    t = tau_sequence([MPF(4), MPF(2), MPF(0), MPF(1)], MPF(3))
    assert float(t[0]) == 1.5 and float(t[1]) == 0.0 and t[2].is_inf()


def _plan(s, r, d, digits):
    return EvaluationPlan(s=s, r=r, nu=1, d_working=d, level_digits=tuple(digits),
                          level_roundoffs=tuple(PrecisionCtx(k).unit_roundoff for k in digits),
                          tau_seq=(), norm_bs=(MPF(1),) * (r + 1), norm_y=MPF(1))


def test_snap_to_lattice_cases():
    assert snap_to_lattice(_plan(2, 3, 16, [12, 5, 1]), [16]).level_digits == (16, 16, 16)
    assert snap_to_lattice(_plan(2, 1, 16, [5]), [3, 8, 16]).level_digits == (8,)
    assert snap_to_lattice(_plan(2, 1, 16, [16]), [3, 8, 16]).level_digits == (16,)
    with pytest.raises(ValueError):
        snap_to_lattice(_plan(2, 1, 16, [5]), [3, 8])
    # the B200 lattice
    assert snap_to_lattice(_plan(6, 5, 31, [22, 10, 1, 1, 1]), [7, 15, 31]).level_digits == (31, 15, 7, 7, 7)


def test_cost_ratio_table1_goldens():
    cr, sav = cost_ratio(_plan(8, 8, 64, (61, 55, 47, 38, 28, 18, 7, 1)))
    assert abs(cr - 703 / 960) < 1e-12 and abs(sav - 0.268) < 0.001
    rows = [(32, 7, 6, (30, 25, 18, 11, 3, 1), 0.271),
            (128, 10, 10, (124, 115, 104, 92, 78, 64, 49, 34, 18, 1), 0.247),
            (256, 14, 13, (248, 234, 217, 197, 176, 154, 131, 107, 82, 57, 31, 4, 1), 0.254)]
    for d, s, r, sched, want in rows:
        assert abs(cost_ratio(_plan(s, r, d, sched))[1] - want) <= 0.001
    assert cost_ratio(_plan(3, 4, 16, (16,) * 4)) == (1.0, 0.0)


def test_plan_validation():
    with pytest.raises(ValueError):
        EvaluationPlan(s=2, r=2, nu=1, d_working=16, level_digits=(5, 9), level_roundoffs=(),
                       tau_seq=(), norm_bs=(), norm_y=MPF(1))
    with pytest.raises(ValueError):
        EvaluationPlan(s=2, r=1, nu=5, d_working=16, level_digits=(16,), level_roundoffs=(),
                       tau_seq=(), norm_bs=(), norm_y=MPF(1))


def test_table1_schedules_via_oracle_norms(oracle_lib):
    """acceptance.py:119-142 (C4): cauchy(100) plan_only schedules within
    +-2 digits of Table 1 (rows 1-2).  Norms from the oracle at the
    reference's 16-digit NORM_CTX; digits from the product planner."""
    n = 100
    A = np.array([[1.0 / (i + j) for j in range(1, n + 1)] for i in range(1, n + 1)])
    # the reference builds cauchy at GEN_CTX (40 digits) then rounds to 16
    from paper_2312_17396_b200.bigfloat import rn as _rn
    Xw = np.zeros((2, n, n))
    for i in range(n):
        for j in range(n):
            v = _rn(Fraction(1, i + j + 2), 54)
            Xw[0, i, j] = float(v)
            Xw[1, i, j] = float(v - Fraction(float(v)))
    for d, m, want in ((32, 42, (30, 25, 18, 11, 3, 1)), (64, 64, (61, 55, 47, 38, 28, 18, 7, 1))):
        s = math.ceil(math.sqrt(m))
        ps = oracle_lib.OraclePS(n)
        n2 = ps.prepare(Xw, taylor_exp_coeffs(m).coeffs, s, 54)
        fr = _norms2_to_frac(n2)
        r = m // s
        plan = plan_precisions(fr[:r + 1], fr[r + 1], PrecisionCtx(d), s=s)
        assert plan.r == len(want)
        assert all(abs(a - b) <= 2 for a, b in zip(plan.level_digits, want)), plan.level_digits
        assert plan.level_digits[-1] <= 2


def test_batched_planner_certified_equals_exact():
    """plan_digits_batch (vectorised, certified, used on the execution path)
    equals the exact plan_precisions row by row, including rows placed on
    integer boundaries that force the exact fallback."""
    from paper_2312_17396_b200.planner import plan_digits_batch
    rng = random.Random(7)
    for d in (15, 31, 63):
        rows = []
        for _ in range(300):
            r = 5
            n2 = _random_norms(rng, r)
            rows.append([Fraction(a) + Fraction(b) for a, b in n2])
        # boundary rows: ||B_i|| ||Y||^i / ||B_0|| = 10^-k exactly-ish
        rows.append([1.0, 1e-5, 1e-10, 1e-15, 1e-20, 1e-25, 1.0])
        rows.append([1.0, 0.0, 1e-10, 0.0, 1e-20, 1e-25, 0.5])
        rows.append([1.0, 1e-5, 1e-10, 1e-15, 1e-20, 1e-25, 0.0])
        nb = np.array([[float(x) for x in row[:-1]] for row in rows])
        ny = np.array([float(row[-1]) for row in rows])
        dig, nu, nil = plan_digits_batch(nb, ny, d)
        for b in range(len(rows)):
            p = plan_precisions(nb[b], ny[b], PrecisionCtx(d), s=2)
            assert tuple(dig[b]) == p.level_digits and nu[b] == p.nu and nil[b] == p.nilpotent


def test_level_planes_from_planned_digits():
    """gemm_engine.planes_for_digits: the smallest compiled 8-bit plane count
    with 6 + 8 (S-1) >= ceil(d log2 10) + 4 bits, capped at the format's
    plane count; 7-bit digits keep the format's count."""
    import math
    from paper_2312_17396_b200 import gemm_engine as ge

    class H:
        def slices_for(self, fmt, db):
            return {8: {7: 4, 15: 8, 31: 14, 63: 28}, 7: {7: 4, 15: 8, 31: 16, 63: 31}}[db][fmt]

    h = H()
    assert [ge.planes_for_digits(h, 31, d, 8) for d in (22, 31, 16)] == [10, 14, 8]
    assert [ge.planes_for_digits(h, 15, d, 8) for d in (10, 15, 8)] == [5, 8, 5]
    assert [ge.planes_for_digits(h, 7, d, 8) for d in (1, 3, 4, 7)] == [2, 2, 3, 4]
    assert ge.planes_for_digits(h, 31, 22, 7) == 16
    for fmt, dmax in ((7, 7), (15, 15), (31, 31)):
        for d in range(1, dmax + 1):
            S = ge.planes_for_digits(h, fmt, d, 8)
            assert 6 + 8 * (S - 1) >= min(math.ceil(d * math.log2(10)) + 4, 6 + 8 * (h.slices_for(fmt, 8) - 1))


def test_execution_planner_vs_mpfr_oracle_1e5(oracle_lib):
    """SURVEY 8c / VERDICT r1: >= 10^5 random norm vectors through the
    planner the evaluators execute (plan_digits_batch: certified float64 +
    exact fallback) against the C MPFR restatement of engine.py:184-215.
    The norms are float64 values (what the device norms are); 2% of the rows
    are pushed onto digit boundaries (e_i within 1e-12 of an integer) so the
    exact fallback is exercised too."""
    from paper_2312_17396_b200.planner import plan_digits_batch
    rng = np.random.default_rng(11)
    total = 0
    for r in (1, 3, 4, 5, 6, 8, 13):
        for d in (15, 31, 63):
            B = 100_000 // 21 + 1
            y = 10 ** rng.uniform(-3, 2, B)
            b0 = 10 ** rng.uniform(-2, 4, B)
            steps = 10 ** rng.uniform(-12, 0.5, (B, r))
            nb = np.concatenate([b0[:, None], b0[:, None] * np.cumprod(steps, axis=1)], axis=1)
            nb[rng.random((B, r + 1)) < 0.02] = 0.0
            edge = rng.random(B) < 0.02          # ||B_1|| so that e_1 lands on an integer
            k = rng.integers(1, d, B)
            nb[edge, 1] = nb[edge, 0] * 10.0 ** (k[edge] - d - 1e-9) / y[edge]
            y[rng.random(B) < 0.005] = 0.0
            dig, nu, nil = plan_digits_batch(nb, y, d)
            for i in range(B):
                n2 = np.zeros((r + 2, 2))
                n2[:r + 1, 0] = nb[i]
                n2[r + 1, 0] = y[i]
                od, onu, onil, _ = oracle_lib.plan_digits(n2, d)
                assert tuple(dig[i]) == od and nu[i] == onu and bool(nil[i]) == onil, (nb[i], y[i], d)
            total += B
    assert total >= 100_000


def test_small_batch_planner_rows_vs_mpfr_oracle(oracle_lib):
    """plan_digits_batch's scalar path for batches of <= 4 rows (one-matrix
    evaluations) against the C MPFR digit rule, boundary rows included."""
    from paper_2312_17396_b200.planner import plan_digits_batch
    rng = np.random.default_rng(12)
    for r in (1, 4, 6):
        for d in (15, 31, 63):
            for _ in range(400):
                B = int(rng.integers(1, 5))
                y = 10 ** rng.uniform(-3, 2, B)
                b0 = 10 ** rng.uniform(-2, 4, B)
                nb = np.concatenate([b0[:, None], b0[:, None] * np.cumprod(10 ** rng.uniform(-12, 0.5, (B, r)), axis=1)],
                                    axis=1)
                if rng.random() < 0.2:
                    k = int(rng.integers(1, d))
                    nb[0, 1] = nb[0, 0] * 10.0 ** (k - d - 1e-9) / y[0]
                if rng.random() < 0.05:
                    y[0] = 0.0
                if rng.random() < 0.05:
                    nb[-1, -1] = 0.0
                dig, nu, nil = plan_digits_batch(nb, y, d)
                for i in range(B):
                    n2 = np.zeros((r + 2, 2))
                    n2[:r + 1, 0] = nb[i]
                    n2[r + 1, 0] = y[i]
                    od, onu, onil, _ = oracle_lib.plan_digits(n2, d)
                    assert tuple(dig[i]) == od and nu[i] == onu and bool(nil[i]) == onil
