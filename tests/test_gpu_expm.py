"""Config 3: scaling-and-squaring exp (m = 42, s = 7, l = extra_squarings)
vs the oracle (C MPFR: the same scaled PS at the snapped digits, then l
squarings at 103 bits), with the squaring-phase error growth accounted for.
The full-size (16 x n=1024) checks are in test_gpu_fullsize.py."""
import math

import numpy as np
import pytest

from _util import synth

pytestmark = pytest.mark.gpu


def test_cfg3_small_vs_oracle(cuda, oracle_lib):
    import paper_2312_17396_b200 as m
    from paper_2312_17396_b200.bounds import extra_squarings
    n, d = 24, 31
    norms = [0.05, 1.0, 7.5, 40.0]
    A = np.stack([synth(n, v, 100 + i) for i, v in enumerate(norms)])
    rep = m.expm_ss(A, m.PrecisionCtx(d))
    coeffs = m.taylor_exp_coeffs(42).coeffs
    for b, v in enumerate(norms):
        ell = extra_squarings(np.abs(A[b]).sum(0).max(), 7)
        assert rep[b].diagnostics["squarings"] == ell
        X = A[b] * 2.0 ** -ell
        ref = oracle_lib.ps_eval(X, coeffs, d)
        assert rep[b].plan.level_digits == ref.digits
        P = ref.ps.result_words(4)
        growth = 1.0
        for _ in range(ell):
            P2 = oracle_lib.matmul(P, P, oracle_lib.bits_of(d))
            n1 = np.abs(P.sum(0)).sum(0).max()
            n2 = np.abs(P2.sum(0)).sum(0).max()
            growth *= 2.0 * n1 * n1 / n2
            P = P2
        got = rep.result.data[:, b].cpu().numpy()
        diff = np.abs((got[0] - P[0]) + (got[1] - P[1] - P[2] - P[3])).sum(0).max()
        refn = np.abs(P.sum(0)).sum(0).max()
        assert diff <= 10 * 6 * n * 1e-31 * max(growth, 1.0) * refn, (b, diff / refn, growth)
