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
