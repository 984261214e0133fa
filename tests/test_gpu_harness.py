"""Accuracy callers (harness.py:105-155 restated on the device): the 2x-digit
truth, relative errors and the mixed-vs-fixed comparison, checked with the
reference's own acceptance criterion eps_mixed <= max(10 r n u, 10 eps_fixed)
(acceptance.py:191-206, test_harness.py:112-122)."""
import numpy as np
import pytest

from _util import synth

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("d,m,n,target", [(15, 16, 32, 0.5), (31, 30, 48, 1.0)])
def test_compare_mixed_fixed_truth(cuda, d, m, n, target):
    import paper_2312_17396_b200 as mp
    from paper_2312_17396_b200 import harness
    ctx = mp.PrecisionCtx(d)
    X = np.stack([synth(n, target, s) for s in range(3)])
    recs = harness.compare(X, mp.taylor_exp_coeffs(m), ctx, m=m)
    assert len(recs) == 3
    u = 10.0 ** (-d)
    for rec in recs:
        r = rec["plan"]["r"]
        assert rec["eps_fixed"] <= 10 * r * n * u
        assert rec["eps_mixed"] <= max(10 * r * n * u, 10 * rec["eps_fixed"])
        assert 0 < rec["savings"] < 1


def test_relative_error_basics(cuda):
    import paper_2312_17396_b200 as mp
    from paper_2312_17396_b200 import harness
    ctx = mp.PrecisionCtx(31)
    X = synth(24, 1.0, 9)
    series = mp.taylor_exp_coeffs(30)
    truth = harness.reference_eval(X, series, ctx)
    assert truth.fmt == mp.DD
    assert harness.relative_error(truth, truth)[0] == 0.0
    mixed = mp.ps_mixed_exp(X, 30, ctx)
    eps = harness.relative_error(mixed, truth)[0]
    assert 0.0 <= eps <= 10 * mixed.plan.r * 24 * 1e-31
    with pytest.raises(mp.UnsupportedPrecisionError):
        harness.reference_eval(X, series, mp.PrecisionCtx(63))


def test_compare_complex(cuda):
    import paper_2312_17396_b200 as mp
    from paper_2312_17396_b200 import harness
    rng = np.random.default_rng(5)
    Z = rng.standard_normal((16, 16)) + 1j * rng.standard_normal((16, 16))
    Z /= np.abs(Z).sum(axis=0).max()
    ctx = mp.PrecisionCtx(31)
    rec = harness.compare(Z, mp.taylor_exp_coeffs(30), ctx, m=30)[0]
    r = rec["plan"]["r"]
    assert rec["eps_mixed"] <= max(10 * r * 16 * 1e-31, 10 * rec["eps_fixed"])


# ---------------------------------------------------------------- oracle pins
def _bound_cases():
    import json
    import os
    p = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "bounds_reference.json")
    return json.load(open(p))["cases"]


@pytest.mark.parametrize("case", _bound_cases(), ids=lambda c: c["name"])
def test_with_bound_report_matches_reference(cuda, case):
    """with_bound=True on the device path (engine.py:283-292): the report's
    bound equals the reference's to its 7 printed digits' rounding (device
    norms are fp64 column sums, not the reference's 54-bit MPFR ones), and
    BoundInvalidError is raised where the reference raises it."""
    from fractions import Fraction
    import paper_2312_17396_b200 as mp
    from paper_2312_17396_b200.bounds import BoundInvalidError
    X = np.array(case["X"])
    ctx = mp.PrecisionCtx(case["d"])
    series = mp.CoefficientSeries(tuple(Fraction(c) for c in case["coeffs"]))

    def run():
        if case["kind"] == "mixed_exp":
            return mp.ps_mixed_exp(X, case["m"], ctx, with_bound=True)
        if case["kind"] == "mixed_general":
            return mp.ps_mixed_general(X, series, ctx, with_bound=True)
        return mp.ps_fixed(X, series, ctx, with_bound=True)
    if case["bound"] is None:
        with pytest.raises(BoundInvalidError):
            run()
        return
    import json
    rep = run()
    got = json.loads(rep.to_json())
    assert list(rep.plan.level_digits) == case["plan"]["digits"]
    assert abs(float(got["bound"]) - float(case["bound"])) <= 2e-6 * float(case["bound"])


@pytest.mark.parametrize("d,m,n", [(15, 16, 20), (31, 30, 20)])
def test_reference_eval_and_errors_vs_oracle(cuda, oracle_lib, d, m, n):
    """harness.py:105-121: the device 2x-digit truth (fixed PS at 2d digits,
    on qd / dd) against the oracle's fixed PS at 2d digits in MPFR; the
    device relative_error against the exact one of the same words; and the
    hard acceptance criterion eps_gpu <= max(10 r n u, 10 eps_oracle)
    (acceptance.py:199) with eps_oracle from the oracle's own mixed run."""
    from fractions import Fraction
    import paper_2312_17396_b200 as mp
    from paper_2312_17396_b200 import harness
    X = synth(n, 1.0, 40 + d)
    series = mp.taylor_exp_coeffs(m)
    coeffs = series.coeffs
    ctx = mp.PrecisionCtx(d)
    wide = oracle_lib.ps_eval(X, coeffs, 2 * d, mode="fixed")       # reference_eval's values
    r = wide.ps.r
    # device ps_fixed at 2d digits (the unrounded truth) vs the oracle's
    fx = mp.ps_fixed(X, series, mp.PrecisionCtx(2 * d))
    diff, refn = wide.compare(fx.result.data[:, 0].double().cpu().numpy())
    assert diff <= 10 * r * n * 10.0 ** (-2 * d) * refn, diff / refn
    # reference_eval = that truth rounded back to the working format
    T = harness.reference_eval(X, series, ctx)
    tw = T.data[:, 0].double().cpu().numpy()
    diff, refn = wide.compare(tw)
    assert diff <= (2.0 ** -52 if d == 15 else 2.0 ** -104) * refn
    # relative_error vs the exact quotient of the same words
    mixed = mp.ps_mixed_exp(X, m, ctx)
    eps = float(harness.relative_error(mixed, T)[0])
    mw = mixed.result.data[:, 0].double().cpu().numpy()
    dmat = [[abs(sum(Fraction(float(x)) for x in mw[:, i, j]) - sum(Fraction(float(x)) for x in tw[:, i, j]))
             for j in range(n)] for i in range(n)]
    tmat = [[abs(sum(Fraction(float(x)) for x in tw[:, i, j])) for j in range(n)] for i in range(n)]
    exact = float(max(sum(dmat[i][j] for i in range(n)) for j in range(n)) /
                  max(sum(tmat[i][j] for i in range(n)) for j in range(n)))
    assert abs(eps - exact) <= 1e-10 * exact + 1e-300, (eps, exact)
    # acceptance.py:199 with the oracle's epsilon
    om = oracle_lib.ps_eval(X, coeffs, d)
    d_gpu, tn = wide.compare(mw)
    d_orc, _ = wide.compare(om.ps.result_words(4))
    eps_gpu, eps_orc = d_gpu / tn, d_orc / tn
    rp = mixed.plan.r
    assert eps_gpu <= max(10 * rp * n * 10.0 ** -d, 10 * eps_orc), (eps_gpu, eps_orc)


def test_c7a_bound_containment_device(cuda):
    """acceptance.py:225-260 (C7a, part a) on the device: horner_mixed with
    random ladders over random blocks/Y exact at the coarsest level's
    precision stays within the Theorem 2.1 bound (bounds.py:101-113) of the
    exact (rational) Horner value."""
    import random
    from fractions import Fraction
    import paper_2312_17396_b200 as mp
    from paper_2312_17396_b200 import ops
    from paper_2312_17396_b200.bigfloat import MPF, to_fraction
    from paper_2312_17396_b200.bounds import BoundInputs, thm21_bound
    from paper_2312_17396_b200.planner import EvaluationPlan
    rng = random.Random(20240517)
    nprng = np.random.default_rng(7)
    checked = 0
    for trial in range(40):
        n = rng.randint(2, 8)
        r = rng.randint(1, 4)
        d = rng.choice([15, 31])
        ladder = sorted([rng.randint(2, d) for _ in range(r)], reverse=True)
        # exact inputs at fp32 (every level format holds them exactly)
        Y = (nprng.standard_normal((n, n)) * 0.5 / n).astype(np.float32).astype(np.float64)
        Bs = [(nprng.standard_normal((n, n)) * 2.0 ** -(3 * i)).astype(np.float32).astype(np.float64)
              for i in range(r + 1)]
        fY = [[Fraction(float(v)) for v in row] for row in Y]
        fB = [[[Fraction(float(v)) for v in row] for row in B] for B in Bs]

        def norm1(M):
            return max(sum(abs(M[i][j]) for i in range(n)) for j in range(n))
        plan = EvaluationPlan(s=2, r=r, nu=1, d_working=d, level_digits=tuple(ladder),
                              level_roundoffs=tuple(mp.PrecisionCtx(k).unit_roundoff for k in ladder),
                              tau_seq=(), norm_bs=tuple(MPF(norm1(B), 64) for B in fB),
                              norm_y=MPF(norm1(fY), 64))
        wf = 31 if d == 31 else 15
        got = mp.horner_mixed([ops.from_numpy(B, wf) for B in Bs], ops.from_numpy(Y, wf), plan)
        gw = got.data[:, 0].double().cpu().numpy()
        # exact Horner (the wide oracle of acceptance.py, here exact rationals)
        phi = fB[r]
        for j in range(r, 0, -1):
            phi = [[fB[j - 1][i][k] + sum(fY[i][t] * phi[t][k] for t in range(n)) for k in range(n)]
                   for i in range(n)]
        err = norm1([[sum(Fraction(float(x)) for x in gw[:, i, k]) - phi[i][k] for k in range(n)]
                     for i in range(n)])
        inp = BoundInputs(n=n, precisions=(mp.PrecisionCtx(d).unit_roundoff,) +
                          tuple(mp.PrecisionCtx(k).unit_roundoff for k in ladder),
                          norm_y=plan.norm_y, norm_bs=plan.norm_bs, s=2, r=r, nu=1)
        try:
            bound = to_fraction(thm21_bound(inp))
        except mp.BoundInvalidError:
            continue
        assert err <= bound, (trial, float(err), float(bound))
        checked += 1
    assert checked >= 20


def test_store_host_moves_planner_norms_without_the_copy_engine(cuda):
    """mpps_store_host / Handle.host_array: a kernel's stores into pinned
    memory deliver the exact values, also while a large device-to-host copy
    occupies the copy engine on another stream (the situation of the host
    stream, where a memcpy of the norms would wait for that copy)."""
    import time
    import torch
    from paper_2312_17396_b200 import _lib
    h = _lib.handle_for()
    src = torch.randn(64, 7, dtype=torch.float64, device="cuda")
    got = h.host_array(src)
    assert got.shape == (64, 7) and np.array_equal(got, src.cpu().numpy())
    pin = torch.empty(src.numel(), dtype=torch.float64).pin_memory()
    h.store_host(src.reshape(-1).contiguous(), pin)
    torch.cuda.synchronize()
    assert np.array_equal(pin.numpy().reshape(64, 7), src.cpu().numpy())
    with pytest.raises(ValueError):
        h.store_host(src, torch.empty(src.numel(), dtype=torch.float64))      # not pinned
    # behind a 512 MiB download on another stream the kernel path returns long before the copy ends
    big = torch.empty(64 << 20, dtype=torch.float64, device="cuda")
    big_h = torch.empty(64 << 20, dtype=torch.float64).pin_memory()
    side = torch.cuda.Stream()
    torch.cuda.synchronize()
    with torch.cuda.stream(side):
        big_h.copy_(big, non_blocking=True)
        done = torch.cuda.Event()
        done.record(side)
    t0 = time.perf_counter()
    got = h.host_array(src)
    t_kernel = time.perf_counter() - t0
    finished_early = not done.query()
    done.synchronize()
    assert np.array_equal(got, src.cpu().numpy())
    assert finished_early, f"host_array took {t_kernel * 1e3:.2f} ms: it waited for the download"
