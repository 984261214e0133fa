"""Parity at the BASELINE sizes, through the same public calls
the bench times.

  cfg2  64 x n=256, seeds 0..63: every matrix against the full C MPFR oracle
        (oracle.ps_eval: blocks/norms at the working digits, the reference's
        digit rule, snap, Horner at the snapped digits' bits) -- schedule
        exactly equal, values within 10 r n 10^-31 (acceptance.py:197,
        harness.py:139-155).
  cfg3  16 x n=1024 scaling-and-squaring: l and the PS-stage schedule equal
        the reference's extra_squarings / plan_precisions (fixture, float64
        norms, margins recorded); the PS stage p_42(2^-l A) against Tier-C
        truth columns at 2x digits; every squaring GEMM against its own
        matrix-vector truth, and the squaring chain bitwise equal to
        expm_ss's result.
  cfg4  Pade [26/26] at qd and [13/13] at fp64, n=2048: schedules and Tier-C
        columns.
  cfg5  cosine deg 24 in Z = X^2, n=8192: schedule and Tier-C columns, on the
        single-GPU path and on the SUMMA path (1x1 grid) the multi-GPU bench
        uses.
Tier C (fixtures from oracle/make_fullsize_fixtures.py): exact columns
p(X) e_j at twice the working digits by matrix-vector Horner in MPFR; the
gate per column is ||(P_gpu - P_true) e_j||_1 <= 10 r n 10^-d ||P_gpu||_1,
implied by (weaker than) the normwise gate."""
import json
import os

import numpy as np
import pytest

from _util import synth, tol

pytestmark = pytest.mark.gpu

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@pytest.fixture(scope="module")
def fx():
    return json.load(open(os.path.join(GOLD, "fullsize_plans.json")))


@pytest.fixture(scope="module")
def cols_fx():
    return dict(np.load(os.path.join(GOLD, "fullsize_cols.npz")))


def mp():
    import paper_2312_17396_b200 as m
    return m


def _gpu_cols(res, b, cols):
    """(W, ncols, n) words of columns `cols` of batch member b."""
    import torch
    idx = torch.tensor(cols, device=res.data.device)
    return res.data[:, b].index_select(2, idx).double().cpu().numpy().transpose(0, 2, 1)


def _norm1(res, b):
    from paper_2312_17396_b200 import ops
    from paper_2312_17396_b200.precision import MatBatch
    return float(ops.one_norm(MatBatch(res.data[:, b:b + 1], res.fmt))[0])


def _check_schedule(plan, rec, formats=None):
    assert list(plan.level_digits) == rec["digits"], (plan.level_digits, rec["digits"])
    assert plan.nu == rec["nu"]
    # float64 fixture norms: the digits are exact only away from integer / delta boundaries
    assert rec["margin_integer"] > 1e-9 and rec["margin_delta"] > 1e-9
    if formats is not None:
        assert list(formats) == rec["snapped"], (formats, rec["snapped"])


def _check_cols(oracle_lib, res, b, rec, truth, r, n, d):
    got = _gpu_cols(res, b, rec["cols"])
    diff = oracle_lib.column_diff(got, truth)
    nrm = _norm1(res, b)
    assert (diff <= tol(r, n, d) * nrm).all(), (diff / nrm, tol(r, n, d))
    return float((diff / nrm).max())


def test_cfg2_full_batch_vs_oracle(cuda, oracle_lib):
    """All 64 matrices of the benched cfg2 batch against the full oracle."""
    m = mp()
    n, d, B = 256, 31, 64
    X = np.stack([synth(n, 1.0, s) for s in range(B)])
    rep = m.ps_mixed_exp(X, 30, m.PrecisionCtx(d))
    coeffs = m.taylor_exp_coeffs(30).coeffs
    words = rep.result.data.double().cpu().numpy()
    worst = 0.0
    for b in range(B):
        ref = oracle_lib.ps_eval(X[b], coeffs, d)
        p = rep[b].plan
        assert p.level_digits == ref.digits and p.nu == ref.nu, (b, p.level_digits, ref.digits)
        assert tuple(rep[b].diagnostics["snapped_digits"]) == tuple(ref.snapped)
        diff, refn = ref.compare(words[:, b])
        assert diff <= tol(p.r, n, d) * refn, (b, diff / refn)
        worst = max(worst, diff / refn)
    print(f"cfg2 64/64 schedules equal; worst ||G-R||/||R|| = {worst:.3e} (gate {tol(5, n, d):.1e})")


def test_cfg3_full_ps_stage_and_squarings(cuda, oracle_lib, fx, cols_fx):
    import torch
    from paper_2312_17396_b200 import ops
    from paper_2312_17396_b200.precision import MatBatch, FORMAT_NAME
    m = mp()
    spec = fx["cfg3"]
    n, B, d = spec["n"], spec["units"], 31
    recs = spec["plans"]
    A = np.stack([synth(n, rec["target"], rec["seed"]) for rec in recs])
    ctx = m.PrecisionCtx(d)
    rep, P = m.expm_ss(A, ctx, return_stage=True)
    worst = 0.0
    for b, rec in enumerate(recs):
        assert rep[b].diagnostics["squarings"] == rec["squarings"], b
        plan = rep[b].plan
        fm = [int(x) for x in rep[b].diagnostics["snapped_digits"]]
        _check_schedule(plan, rec, fm)
        worst = max(worst, _check_cols(oracle_lib, P, b, rec, cols_fx[f"cfg3_{b}"], plan.r, n, d))
    # squaring phase: every dd squaring of every matrix against its
    # matrix-vector truth (two products at 2x digits), and the chain equal
    # bit for bit to expm_ss's result
    bits2 = oracle_lib.bits_of(2 * d)
    for b, rec in enumerate(recs):
        Q = MatBatch(P.data[:, b:b + 1].clone(), P.fmt)
        cols = rec["cols"]
        for _ in range(rec["squarings"]):
            Q2 = ops.mat_mul(Q, Q, ctx)
            qw = Q.data[:, 0].double().cpu().numpy()
            truth = oracle_lib.power_columns(qw, 2, bits2, cols)
            got = _gpu_cols(Q2, 0, cols)
            diff = oracle_lib.column_diff(got, truth)
            aq = np.abs(qw[0])
            scale = np.abs(aq @ aq[:, cols]).sum(axis=0)        # || |Q| |Q| e_j ||_1
            assert (diff <= 10 * n * 10.0 ** -d * scale).all(), (b, diff / scale)
            Q = Q2
        assert torch.equal(Q.data[:, 0], rep.result.data[:, b]), b
    print(f"cfg3 16/16 schedules and l equal; worst PS-stage column error {worst:.3e} (gate {tol(6, n, d):.1e})")


@pytest.mark.parametrize("k,d", [(26, 63), (13, 15)])
def test_cfg4_full_pade(cuda, oracle_lib, fx, cols_fx, k, d):
    m = mp()
    spec = fx["cfg4"]
    recs = spec["plans"] if k == 26 else spec["fp64_pade13"]
    n = spec["n"]
    X = synth(n, 2.0, 0)
    num, den = m.ps_mixed_pade(X, k, m.PrecisionCtx(d))
    for rep, rec in zip((num, den), recs):
        assert rec["which"] == ("num" if rep is num else "den")
        fm = [int(x) for x in rep.diagnostics["snapped_digits"]]
        _check_schedule(rep.plan, rec, fm)
        e = _check_cols(oracle_lib, rep.result, 0, rec, cols_fx[f"cfg4_{k}_{rec['which']}"], rep.plan.r, n, d)
        print(f"cfg4 [{k}/{k}] {rec['which']} column error {e:.3e} (gate {tol(rep.plan.r, n, d):.1e})")


def test_cfg5_full_cosine(cuda, oracle_lib, fx, cols_fx):
    m = mp()
    rec = fx["cfg5"]["plans"][0]
    n, d = fx["cfg5"]["n"], 31
    ctx = m.PrecisionCtx(d)
    X = synth(n, 1.0, rec["seed"], cos=True)
    Z = m.cos_argument(X, ctx)
    rep = m.ps_mixed_general(Z, m.taylor_cos_coeffs(24), ctx)
    fm = [int(x) for x in rep.diagnostics["snapped_digits"]]
    _check_schedule(rep.plan, rec, fm)
    e = _check_cols(oracle_lib, rep.result, 0, rec, cols_fx["cfg5"], rep.plan.r, n, d)
    print(f"cfg5 single-GPU column error {e:.3e} (gate {tol(rep.plan.r, n, d):.1e})")


def test_cfg5_full_cosine_summa_path(cuda, oracle_lib, fx, cols_fx):
    """The 2-D block SUMMA driver (bench at N > 1) on a 1x1 grid: the same
    schedule and the same Tier-C columns."""
    import torch
    from paper_2312_17396_b200 import summa
    from paper_2312_17396_b200.precision import MatBatch
    m = mp()
    rec = fx["cfg5"]["plans"][0]
    n, d = fx["cfg5"]["n"], 31
    ctx = m.PrecisionCtx(d)
    X = synth(n, 1.0, rec["seed"], cos=True)
    grid = summa.ProcessGrid.single()
    blk = MatBatch(torch.from_numpy(X).cuda().reshape(1, 1, n, n), 15)
    ops = summa.DeviceOps()
    Zb = summa.cos_argument_dist(blk, ctx, grid, ops)
    res = summa.ps_mixed_dist(Zb, m.taylor_cos_coeffs(24), ctx, grid, ops)
    plan = res.plan(ctx)
    assert list(plan.level_digits) == rec["digits"] and plan.nu == rec["nu"]
    e = _check_cols(oracle_lib, res.block, 0, rec, cols_fx["cfg5"], plan.r, n, d)
    print(f"cfg5 SUMMA 1x1 column error {e:.3e}")


# ------------------------------------------------- worst-case accumulators
def _const_poly_exact(x, n, coeffs):
    """X = x J (n x n, every entry x): X^k = n^(k-1) x^k J exactly, so
    p(X) = b_0 I + (sum_{k>=1} b_k n^(k-1) x^k) J.  Returns (diagonal, off-diagonal)."""
    from fractions import Fraction
    xf = Fraction(x)
    off = sum(Fraction(c) * n ** (k - 1) * xf ** k for k, c in enumerate(coeffs) if k >= 1)
    return Fraction(coeffs[0]) + off, off


def _check_const(res, diag, off, n, d, r):
    from fractions import Fraction
    import torch
    data = res.data.double()[:, 0]
    worst = Fraction(0)
    for (i, j) in ((0, 0), (0, 1), (n - 1, n - 1), (n - 1, 0), (n // 2, n // 3), (n // 2, n // 2)):
        v = sum(Fraction(float(data[w][i, j])) for w in range(data.shape[0]))
        worst = max(worst, abs(v - (diag if i == j else off)))
    # every row and column has the same digits: the off-diagonal entries agree to the bit
    hi = data[0].clone()
    hi.fill_diagonal_(float(data[0][0, 1]))
    assert (hi.max() - hi.min()).item() == 0.0
    normp = abs(diag) + (n - 1) * abs(off)
    assert float(worst * n / normp) <= tol(r, n, d), (float(worst * n / normp), tol(r, n, d))


@pytest.mark.parametrize("n,a", [(256, 0.99), (1024, 0.7123456789012345), (8192, 0.99999999999), (8192, 0.501)])
def test_constant_matrices_fill_the_int32_accumulators(cuda, n, a):
    """Size-independent property with an exact answer at the BASELINE sizes: for X = x J all
    products of a digit-plane pair have one sign, so every int32 diagonal accumulator of the
    tensor-core GEMMs reaches K d_i d_j (random matrices never come near: their sums grow like
    sqrt(K)).  exp (Taylor m = 30: cfg2 / cfg3 kernels) and the cosine in Z = X X (cfg5 path) at
    dd against the exact rational value."""
    import torch
    import paper_2312_17396_b200 as mp
    ctx = mp.PrecisionCtx(31)
    x = a / n
    X = torch.full((n, n), x, dtype=torch.float64, device="cuda")
    rep = mp.ps_mixed_exp(X, 30, ctx)
    diag, off = _const_poly_exact(x, n, mp.taylor_exp_coeffs(30).coeffs)
    _check_const(rep.result, diag, off, n, 31, rep.plan.r)
    del rep
    from fractions import Fraction
    Z = mp.cos_argument(X, ctx)
    rep = mp.ps_mixed_general(Z, mp.taylor_cos_coeffs(24), ctx)
    z = n * Fraction(x) ** 2          # Z = X X = n x^2 J exactly (Z itself is rounded to dd: within the gate)
    diag, off = _const_poly_exact(z, n, mp.taylor_cos_coeffs(24).coeffs)
    _check_const(rep.result, diag, off, n, 31, rep.plan.r)


def test_constant_matrix_qd_pade(cuda):
    """The same worst case on the qd kernels (cfg4 shape: Pade [26/26], n = 2048, ||X||_1 = 2)."""
    import torch
    import paper_2312_17396_b200 as mp
    n = 2048
    x = 1.9999 / n
    X = torch.full((n, n), x, dtype=torch.float64, device="cuda")
    num, den = mp.ps_mixed_pade(X, 26, mp.PrecisionCtx(63))
    pc, qc = mp.pade_exp_coeffs(26, 26)
    for rep, cs in ((num, pc), (den, qc)):
        diag, off = _const_poly_exact(x, n, cs.coeffs)
        _check_const(rep.result, diag, off, n, 63, rep.plan.r)
