"""GPU parity: the sm_100a path vs the CPU oracle (oracle/, the C MPFR
restatement of the reference) on the same seeded inputs.

Gates:
  * schedule -- digits, nu and snapped formats EXACTLY equal to the
    oracle's plan_precisions/snap_to_lattice;
  * values -- ||p_gpu - p_oracle||_1 <= 10 r n 10^-d_w ||p_oracle||_1.
The reference rounds each scalar op separately in a sequential order
(precision.py:176-181); the GPU uses FMA-based error-free transforms in a
tiled order and fp32/fp64/dd/qd significands (24/53/106/212 bits) for the
lattice digits 7/15/31/63 (24/50/103/210 bits in the oracle).  Both are
covered by Thm 2.1 with n -> n+1, hence the
tolerance rather than bitwise equality.  Bitwise gates are used where the
math is identical (degenerate plans, batch invariance, exact zeros).
"""
import math
from fractions import Fraction

import numpy as np
import pytest

from _util import synth, tol, words_of

pytestmark = pytest.mark.gpu


def mp():
    import paper_2312_17396_b200 as m
    return m


def _check(rep, ref, n, d):
    p = rep.plan
    assert p.level_digits == ref.digits and p.nu == ref.nu, (p.level_digits, ref.digits)
    if not ref.nilpotent:
        got_fmt = tuple(x for x in rep.diagnostics["snapped_digits"])
        assert got_fmt == tuple(ref.snapped)
    diff, refn = ref.compare(words_of(rep))
    assert diff <= tol(max(p.r, 1), n, d) * refn, (diff / refn, tol(p.r, n, d))
    return diff / refn


@pytest.mark.parametrize("seed", range(8))
def test_cfg1_full(cuda, oracle_lib, seed):
    """Config 1: Taylor exp m=16, s=4, n=32, ||X||_1=0.5, fp64 working."""
    m = mp()
    X = synth(32, 0.5, seed)
    rep = m.ps_mixed_exp(X, 16, m.PrecisionCtx(15))
    ref = oracle_lib.ps_eval(X, m.taylor_exp_coeffs(16).coeffs, 15)
    _check(rep, ref, 32, 15)
    assert rep.diagnostics["level_formats"][0] == "fp64"
    assert rep.plan.s == 4 and rep.plan.r == 4


def test_cfg2_reduced_batch(cuda, oracle_lib):
    """Config 2 shape at reduced n (ragged 48 vs 64-tiles): Taylor exp m=30,
    s=6, dd working, batch of 4, one oracle run per matrix."""
    m = mp()
    n, d = 48, 31
    X = np.stack([synth(n, 1.0, s) for s in range(4)])
    rep = m.ps_mixed_exp(X, 30, m.PrecisionCtx(d))
    assert len(rep) == 4
    coeffs = m.taylor_exp_coeffs(30).coeffs
    for b in range(4):
        ref = oracle_lib.ps_eval(X[b], coeffs, d)
        assert rep[b].plan.level_digits == ref.digits
        diff, refn = ref.compare(rep.result.data[:, b].double().cpu().numpy())
        assert diff <= tol(5, n, d) * refn, diff / refn


def test_fixed_matches_oracle_dd(cuda, oracle_lib):
    m = mp()
    n, d = 40, 31
    X = synth(n, 1.0, 11)
    s = m.taylor_exp_coeffs(20)
    rep = m.ps_fixed(X, s, m.PrecisionCtx(d))
    ref = oracle_lib.ps_eval(X, s.coeffs, d, mode="fixed")
    diff, refn = ref.compare(words_of(rep))
    assert rep.plan.level_digits == (d,) * rep.plan.r
    assert diff <= tol(rep.plan.r, n, d) * refn


@pytest.mark.parametrize("which", [0, 1])
def test_pade13_fp64(cuda, oracle_lib, which):
    """Config 4 (m=13 at fp64) at reduced n: numerator and denominator."""
    m = mp()
    n, d = 40, 15
    X = synth(n, 2.0, 0)
    series = m.pade_exp_coeffs(13, 13)[which]
    rep = m.ps_mixed_general(X, series, m.PrecisionCtx(d))
    ref = oracle_lib.ps_eval(X, series.coeffs, d)
    _check(rep, ref, n, d)


@pytest.mark.parametrize("which", [0, 1])
def test_pade26_qd(cuda, oracle_lib, which):
    """Config 4 (m=26 at qd, 63 digits) at reduced n."""
    m = mp()
    n, d = 24, 63
    X = synth(n, 2.0, 0)
    series = m.pade_exp_coeffs(26, 26)[which]
    rep = m.ps_mixed_general(X, series, m.PrecisionCtx(d))
    ref = oracle_lib.ps_eval(X, series.coeffs, d)
    _check(rep, ref, n, d)
    assert rep.diagnostics["level_formats"][0] == "qd"


def test_cosine_dd(cuda, oracle_lib):
    """Config 5 shape at reduced n: Z = X^2 at dd, cos Taylor deg 24 in Z."""
    m = mp()
    n, d = 40, 31
    X = synth(n, 1.0, 0, cos=True)
    ctx = m.PrecisionCtx(d)
    Z = m.cos_argument(X, ctx)
    series = m.taylor_cos_coeffs(24)
    rep = m.ps_mixed_general(Z, series, ctx)
    # the oracle forms its own Z = fl(X X) at 103 bits (harness.py:100-101)
    Zo = oracle_lib.matmul(X, X, oracle_lib.bits_of(d))
    ref = oracle_lib.ps_eval(Zo, series.coeffs, d)
    assert rep.plan.level_digits == ref.digits
    diff, refn = ref.compare(words_of(rep))
    assert diff <= tol(rep.plan.r, n, d) * refn


def test_degenerate_flat_series_bitwise(cuda):
    """test_engine.py:259-267 / acceptance C8: a flat series clamps the plan
    to all-working, so mixed and fixed run the same kernels: same bits."""
    m = mp()
    ctx = m.PrecisionCtx(31)
    n = 20  # cauchy(20), as the reference test uses a Cauchy matrix: ||Y|| > 1
    X = np.array([[1.0 / (i + j) for j in range(1, n + 1)] for i in range(1, n + 1)])
    series = m.CoefficientSeries(tuple(Fraction(1) for _ in range(10)))
    mixed = m.ps_mixed_general(X, series, ctx)
    fixed = m.ps_fixed(X, series, ctx)
    assert mixed.plan.nu == mixed.plan.r + 1
    assert np.array_equal(words_of(mixed), words_of(fixed))


def test_zero_matrix_gives_identity(cuda):
    m = mp()
    for ctx in (m.PrecisionCtx(15), m.PrecisionCtx(31), m.PrecisionCtx(63)):
        rep = m.ps_mixed_exp(np.zeros((3, 3)), 9, ctx)
        w = words_of(rep)
        assert np.array_equal(w[0], np.eye(3)) and not w[1:].any()
        rep = m.ps_fixed(np.zeros((3, 3)), m.taylor_exp_coeffs(9), ctx)
        assert np.array_equal(words_of(rep)[0], np.eye(3))


def test_nilpotent_plan(cuda, oracle_lib):
    """Strictly upper triangular 4x4 with s=4: Y = X^4 = 0 exactly, plan is
    nilpotent and p = B_0 (engine.py:175-182, 473-474)."""
    m = mp()
    rng = np.random.default_rng(3)
    X = np.triu(rng.standard_normal((4, 4)), 1)
    rep = m.ps_mixed_exp(X, 12, m.PrecisionCtx(31))
    assert rep.plan.nilpotent and rep.plan.nu == 1
    ref = oracle_lib.ps_eval(X, m.taylor_exp_coeffs(12).coeffs, 31)
    assert ref.nilpotent
    diff, refn = ref.compare(words_of(rep))
    assert diff <= 1e-30 * refn


def test_degree_one_and_explicit_powers(cuda):
    m = mp()
    ctx = m.PrecisionCtx(15)
    X = synth(3, 0.25, 7)
    rep = m.ps_mixed_exp(X, 1, ctx, fix_params=False)
    assert rep.plan.explicit_powers and rep.plan.s == 1
    assert sum(rep.matmuls_by_digits.values()) == 0
    assert np.allclose(words_of(rep)[0], np.eye(3) + X, atol=0, rtol=0)
    series = m.CoefficientSeries((Fraction(2), Fraction(3)))
    rep = m.ps_fixed(np.array([[1.5]]), series, ctx)
    assert rep.plan.s == 1 and rep.plan.r == 1 and words_of(rep)[0, 0, 0] == 2 + 3 * 1.5


def test_batch_invariance_bitwise(cuda):
    """P1 batch sharding must be bitwise invisible: a matrix evaluated inside
    a batch equals the same matrix evaluated alone."""
    m = mp()
    ctx = m.PrecisionCtx(31)
    X = np.stack([synth(36, 1.0, s) for s in range(3)])
    rep = m.ps_mixed_exp(X, 30, ctx)
    for b in range(3):
        one = m.ps_mixed_exp(X[b], 30, ctx)
        assert np.array_equal(words_of(one), rep.result.data[:, b].cpu().numpy())


def test_batch_invariance_heterogeneous_plans_bitwise(cuda):
    """Batch members whose plans keep different numbers of dd levels (the
    post-planner dd re-assembly covers the longest prefix in the batch):
    every member still equals its solo evaluation bit for bit."""
    m = mp()
    ctx = m.PrecisionCtx(31)
    norms = [1.0, 6.0, 0.01, 8.0, 3.0]
    X = np.stack([synth(40, t, 20 + b) for b, t in enumerate(norms)])
    rep = m.ps_mixed_exp(X, 30, ctx)
    assert len({tuple(r.diagnostics["level_formats"]) for r in rep}) >= 3
    for b in range(len(norms)):
        one = m.ps_mixed_exp(X[b], 30, ctx)
        assert np.array_equal(words_of(one), rep.result.data[:, b].cpu().numpy()), b


@pytest.mark.parametrize("fmt,bits", [(7, 24), (15, 53), (31, 106), (63, 212)])
def test_gemm_operator_parity(cuda, oracle_lib, fmt, bits):
    """mat_mul per format vs the oracle's mat_mul at the format's bits:
    |C - C_o| <= c n u |A||B| entrywise-normwise."""
    from paper_2312_17396_b200 import ops
    m = mp()
    n = 70
    rng = np.random.default_rng(5)
    A = rng.standard_normal((n, n))
    B = rng.standard_normal((n, n))
    if fmt >= 31:  # give the operands real low words
        A = np.stack([A, A * 2.0 ** -60])
        B = np.stack([B, B * 2.0 ** -61])
        if fmt == 63:
            A = np.concatenate([A, A * 2.0 ** -120])
            B = np.concatenate([B, B * 2.0 ** -122])
    if fmt == 7:
        A = A.astype(np.float32).astype(np.float64)
        B = B.astype(np.float32).astype(np.float64)
    ctx = m.PrecisionCtx(fmt)
    C = ops.mat_mul(ops.from_numpy(A, fmt), ops.from_numpy(B, fmt), ctx)
    Co = oracle_lib.matmul(A, B, bits)
    got = C.data[:, 0].double().cpu().numpy()
    A0 = A if A.ndim == 2 else A[0]
    B0 = B if B.ndim == 2 else B[0]
    absAB = np.abs(A0) @ np.abs(B0)
    u = Fraction(1, 2 ** bits)
    rng = np.random.default_rng(9)
    for _ in range(300):
        i, j = rng.integers(0, n, 2)
        g = sum(Fraction(float(x)) for x in got[:, i, j])
        o = sum(Fraction(float(x)) for x in Co[:, i, j])
        assert abs(g - o) <= 4 * n * u * Fraction(float(absAB[i, j])), (i, j, float(g - o))


def test_one_norm_and_round_to(cuda):
    from paper_2312_17396_b200 import ops
    m = mp()
    X = synth(50, 3.0, 1)
    A = ops.from_numpy(X, 15)
    assert abs(ops.one_norm(A)[0] - np.abs(X).sum(0).max()) <= 1e-14 * 3
    dd = ops.round_to(A, m.PrecisionCtx(31))
    assert np.array_equal(dd.data[0, 0].cpu().numpy(), X) and not dd.data[1].any()
    f = ops.round_to(A, m.PrecisionCtx(7))
    assert np.array_equal(f.data[0, 0].cpu().numpy(), X.astype(np.float32))


def test_errors_mirror_reference(cuda):
    m = mp()
    with pytest.raises(m.DimensionError):
        m.ps_mixed_exp(np.zeros((3, 4)), 4, m.PrecisionCtx(15))
    with pytest.raises(ValueError):
        m.ps_mixed_exp(np.zeros((3, 3)), 0, m.PrecisionCtx(15))
    with pytest.raises(ValueError):
        m.ps_mixed_general(np.zeros((2, 2)), m.CoefficientSeries((Fraction(1),)), m.PrecisionCtx(15))
    with pytest.raises(m.UnsupportedPrecisionError):
        m.ps_mixed_exp(np.zeros((3, 3)), 4, m.PrecisionCtx(64))


def test_horner_rejects_fp32_previous_block(cuda):
    """The fused Horner step reads B_{j-1} as fp64 words: an fp32 block is
    rejected by both engines (blocks are assembled at >= fp64)."""
    from paper_2312_17396_b200 import _lib
    from paper_2312_17396_b200.precision import MatBatch
    h = _lib.handle_for()
    Y = MatBatch.zeros(15, 1, 8, device="cuda")
    P = MatBatch.zeros(7, 1, 8, device="cuda")
    Bp = MatBatch.zeros(7, 1, 8, device="cuda")
    out = MatBatch.zeros(7, 1, 8, device="cuda")
    ys, ps = h.slice(Y, 0, 4), h.slice(P, 1, 4)
    err = mp().UnsupportedPrecisionError
    with pytest.raises(err, match="working format"):
        h.horner_step_sliced(ys, ps, 4, Bp, out, fmt_in=7)
    with pytest.raises(err, match="working format"):
        h.horner_step(P, P, Bp, out)


def test_pade_pair_shares_powers_bitwise(cuda):
    """ps_mixed_pade forms the powers once; each polynomial equals its own
    ps_mixed_general evaluation bit for bit (identical powers, kernels, plan)."""
    m = mp()
    X = synth(48, 2.0, 4)
    for d, k in ((15, 13), (63, 26)):
        ctx = m.PrecisionCtx(d)
        num, den = m.ps_mixed_pade(X, k, ctx)
        sn, sd = m.pade_exp_coeffs(k, k)
        a = m.ps_mixed_general(X, sn, ctx)
        b = m.ps_mixed_general(X, sd, ctx)
        assert num.plan.level_digits == a.plan.level_digits and den.plan.level_digits == b.plan.level_digits
        assert np.array_equal(words_of(num), words_of(a)) and np.array_equal(words_of(den), words_of(b))


def test_graph_replay_matches_eager_bitwise(cuda):
    """The CUDA-graph path (default) replays the same kernels as the eager
    path: results are bitwise identical, also for successive different
    inputs of the same shape (static buffers are refilled each call)."""
    from paper_2312_17396_b200 import graphs
    m = mp()
    ctx = m.PrecisionCtx(31)
    Xs = [np.stack([synth(40, 1.0, 10 * k + b) for b in range(3)]) for k in range(3)]
    graphs.set_enabled(True)
    g = [m.ps_mixed_exp(X, 30, ctx).result.data.cpu().numpy() for X in Xs]
    graphs.set_enabled(False)
    try:
        e = [m.ps_mixed_exp(X, 30, ctx).result.data.cpu().numpy() for X in Xs]
    finally:
        graphs.set_enabled(True)
    for a, b in zip(g, e):
        assert np.array_equal(a, b)
    assert not np.array_equal(g[0], g[1])


def test_speculative_horner_miss_and_hit_bitwise(cuda):
    """The Horner graph of the previous plan structure is replayed
    speculatively; when the next batch's plan has a different structure
    (here the level formats change with ||X||) the right graph runs after
    it.  Hits and misses both give the eager path's bits."""
    from paper_2312_17396_b200 import graphs
    m = mp()
    ctx = m.PrecisionCtx(31)
    norms = (1.0, 1e-3, 1.0, 1.0, 1e-3)          # structures: A, B, A, A, B
    Xs = [np.stack([synth(48, t, 7 * k + b) for b in range(2)]) for k, t in enumerate(norms)]
    plans = [m.ps_mixed_exp(X, 30, ctx)[0].plan.level_digits for X in Xs[:2]]
    assert plans[0] != plans[1]
    graphs.set_enabled(True)
    s0 = graphs.speculation_stats()
    g = [m.ps_mixed_exp(X, 30, ctx).result.data.cpu().numpy() for X in Xs]
    s1 = graphs.speculation_stats()
    graphs.set_enabled(False)
    try:
        e = [m.ps_mixed_exp(X, 30, ctx).result.data.cpu().numpy() for X in Xs]
    finally:
        graphs.set_enabled(True)
    for a, b in zip(g, e):
        assert np.array_equal(a, b)
    assert s1["miss"] - s0["miss"] >= 2 and s1["hit"] - s0["hit"] >= 1


def test_pipelined_host_evaluation_matches(cuda):
    """pipeline.evaluate_host (chunked, copies overlapping compute) returns the
    same bits as one device-resident batched call."""
    import torch
    from paper_2312_17396_b200 import pipeline
    m = mp()
    ctx = m.PrecisionCtx(31)
    X = np.stack([synth(64, 1.0, b) for b in range(12)])
    ref = m.ps_mixed_exp(X, 30, ctx).result.data.cpu().numpy()
    Xh = torch.from_numpy(X).pin_memory()
    out = torch.empty((2,) + X.shape, dtype=torch.float64).pin_memory()
    reps = pipeline.evaluate_host(pipeline.mixed_exp(30, ctx), Xh, out, chunks=3)
    torch.cuda.synchronize()
    assert len(reps) == 3
    assert np.array_equal(out.numpy(), ref)
    # every chunk submitted up front over two compute streams (static slot
    # results downloaded directly), twice so the speculative Horner graphs hit
    for _ in range(2):
        out.zero_()
        reps = pipeline.evaluate_host(pipeline.mixed_exp(30, ctx), Xh, out, chunks=[4, 4, 2, 2], streams=2)
        torch.cuda.synchronize()
        assert len(reps) == 4
        assert np.array_equal(out.numpy(), ref)
    # a host stream longer than the slot window: 6 chunks through 2 slots
    # (uploads wait for the slot's previous input copy, evaluations for its
    # previous download), distinct matrices per chunk
    X2 = np.stack([synth(64, 1.0, 100 + b) for b in range(12)])
    ref2 = m.ps_mixed_exp(X2, 30, ctx).result.data.cpu().numpy()
    Xh2 = torch.from_numpy(X2).pin_memory()
    for win in (2, 3):
        out.zero_()
        reps = pipeline.evaluate_host(pipeline.mixed_exp(30, ctx), Xh2, out, chunks=[2] * 6, streams=2,
                                      window=win)
        torch.cuda.synchronize()
        assert len(reps) == 6
        assert np.array_equal(out.numpy(), ref2)


def test_graph_input_reuse_in_place(cuda):
    """A device input passed again at the same address after an in-place
    update: the graphs copy every input at submit (no pointer-bound graph),
    so each call sees the tensor's current values."""
    import torch
    m = mp()
    ctx = m.PrecisionCtx(31)
    X1 = np.stack([synth(64, 1.0, 300 + b) for b in range(4)])
    X2 = np.stack([synth(64, 0.7, 400 + b) for b in range(4)])
    Xd = torch.from_numpy(X1).cuda()
    for _ in range(3):
        r1 = m.ps_mixed_exp(Xd, 30, ctx).result.data.cpu().numpy()
    Xd.copy_(torch.from_numpy(X2))
    r2 = m.ps_mixed_exp(Xd, 30, ctx).result.data.cpu().numpy()
    ref1 = m.ps_mixed_exp(torch.from_numpy(X1).cuda().clone(), 30, ctx).result.data.cpu().numpy()
    ref2 = m.ps_mixed_exp(X2, 30, ctx).result.data.cpu().numpy()
    assert np.array_equal(r1, ref1)
    assert np.array_equal(r2, ref2)


def test_windowed_host_stream_with_dd_reassembly(cuda):
    """a windowed host stream whose plans keep two dd Horner
    levels (the post graph re-assembles dd blocks from X^1 after planning)
    while the next chunk of the same slot is already being uploaded.  Every
    chunk must equal its device-resident evaluation bit for bit."""
    import torch
    from paper_2312_17396_b200 import pipeline
    m = mp()
    ctx = m.PrecisionCtx(31)
    norms = [4.0, 6.0, 5.0, 8.0, 4.5, 7.0, 6.5, 5.5]
    X = np.stack([synth(64, norms[b // 2], 500 + b) for b in range(16)])
    ref = m.ps_mixed_exp(X, 30, ctx)
    fm = [r.diagnostics["level_formats"] for r in ref]
    assert any(f[1] == "dd" and f[2] == "dd" for f in fm), fm
    ref = ref.result.data.cpu().numpy()
    Xh = torch.from_numpy(X).pin_memory()
    out = torch.empty((2,) + X.shape, dtype=torch.float64).pin_memory()
    for win in (2, 3):
        for _ in range(2):
            out.zero_()
            pipeline.evaluate_host(pipeline.mixed_exp(30, ctx), Xh, out, chunks=[2] * 8, streams=2, window=win)
            torch.cuda.synchronize()
            assert np.array_equal(out.numpy(), ref)


def test_small_fused_path_vs_oracle_and_invariance(cuda, oracle_lib):
    """K5 (n <= 32, fp64 working: two launches around the planner) against
    the oracle for mixed exp, fixed PS and Pade 13 at ragged n, batch
    members bitwise equal to solo runs, and the same schedule as the general
    pipeline (MPPS_SMALL=0 in-process switch)."""
    from paper_2312_17396_b200 import engine
    m = mp()
    ctx = m.PrecisionCtx(15)
    for n, seed in ((32, 3), (17, 4), (5, 6)):
        X = synth(n, 0.5, seed)
        assert engine._small_ok(X, m.taylor_exp_coeffs(16), ctx)
        rep = m.ps_mixed_exp(X, 16, ctx)
        _check(rep, oracle_lib.ps_eval(X, m.taylor_exp_coeffs(16).coeffs, 15), n, 15)
        s = m.taylor_exp_coeffs(20)
        fx = m.ps_fixed(X, s, ctx)
        ref = oracle_lib.ps_eval(X, s.coeffs, 15, mode="fixed")
        diff, refn = ref.compare(words_of(fx))
        assert diff <= tol(fx.plan.r, n, 15) * refn
        X2 = synth(n, 2.0, seed)
        num, den = m.ps_mixed_pade(X2, 13, ctx)
        sn, sd = m.pade_exp_coeffs(13, 13)
        _check(num, oracle_lib.ps_eval(X2, sn.coeffs, 15), n, 15)
        _check(den, oracle_lib.ps_eval(X2, sd.coeffs, 15), n, 15)
    Xb = np.stack([synth(24, t, 80 + b) for b, t in enumerate((0.5, 3.0, 0.01, 1.5))])
    rep = m.ps_mixed_exp(Xb, 16, ctx)
    for b in range(4):
        one = m.ps_mixed_exp(Xb[b], 16, ctx)
        assert np.array_equal(words_of(one), rep.result.data[:, b].cpu().numpy())
    engine._SMALL = False
    try:
        gen = m.ps_mixed_exp(Xb, 16, ctx)
    finally:
        engine._SMALL = True
    for b in range(4):
        assert gen[b].plan.level_digits == rep[b].plan.level_digits
        g, k = gen.result.data[0, b].cpu().numpy(), rep.result.data[0, b].cpu().numpy()
        assert np.abs(g - k).sum(0).max() <= tol(4, 24, 15) * np.abs(g).sum(0).max()


def test_evaluate_stream_matches_direct_calls(cuda):
    """pipeline.evaluate_stream (H2D of step t+1 and D2H of step t-1
    overlapping step t, two device input slots) returns each step's result
    bit for bit as a direct call on the same input."""
    import torch
    from paper_2312_17396_b200 import pipeline
    m = mp()
    ctx = m.PrecisionCtx(31)
    series = m.taylor_cos_coeffs(24)
    Xs = [synth(300, 1.0, 90 + t, cos=True) for t in range(4)]

    def fn(x):
        return m.ps_mixed_general(m.cos_argument(x, ctx), series, ctx)
    ref = [fn(X).result.data.cpu().numpy() for X in Xs]
    Xh = [torch.from_numpy(X).pin_memory() for X in Xs]
    outs = [[torch.empty((2, 1, 300, 300), dtype=torch.float64).pin_memory()] for _ in Xs]
    pipeline.evaluate_stream(fn, Xh, outs)
    torch.cuda.synchronize()
    for o, r in zip(outs, ref):
        assert np.array_equal(o[0].numpy(), r)


def test_y_low_precision_rule(cuda, oracle_lib):
    """Odd s (m = 42, s = 7): Y = X^s is formed at fp64 precision and at dd
    only for the matrices whose plan keeps a Horner level at dd.  Members
    with a dd level get exactly the bits of the always-dd chain
    (MPPS_Y_LOW=0); the others stay within the oracle tolerance; every
    member equals its solo evaluation bit for bit (the choice depends on the
    matrix's own plan only)."""
    from paper_2312_17396_b200 import engine
    m = mp()
    n, d = 40, 31
    ctx = m.PrecisionCtx(d)
    norms = [2.5, 0.01, 2.0, 0.02]
    X = np.stack([synth(n, t, 60 + b) for b, t in enumerate(norms)])
    engine._Y_LOW_MIN_N = 0          # the rule's size threshold (n >= 4096) lowered for the test
    try:
        _y_low_checks(m, engine, oracle_lib, X, norms, n, d, ctx)
    finally:
        engine._Y_LOW_MIN_N = 4096


def _y_low_checks(m, engine, oracle_lib, X, norms, n, d, ctx):
    rep = m.ps_mixed_exp(X, 42, ctx)
    fm = [r.diagnostics["level_formats"] for r in rep]
    has_dd = [("dd" in f[1:]) for f in fm]
    assert any(has_dd) and not all(has_dd), fm
    engine._Y_LOW = False
    try:
        full = m.ps_mixed_exp(X, 42, ctx).result.data.cpu().numpy()
    finally:
        engine._Y_LOW = True
    got = rep.result.data.cpu().numpy()
    coeffs = m.taylor_exp_coeffs(42).coeffs
    for b in range(len(norms)):
        solo = m.ps_mixed_exp(X[b], 42, ctx)
        assert np.array_equal(words_of(solo), got[:, b]), b
        if has_dd[b]:
            assert np.array_equal(got[:, b], full[:, b]), b
        ref = oracle_lib.ps_eval(X[b], coeffs, d)
        assert rep[b].plan.level_digits == ref.digits
        diff, refn = ref.compare(got[:, b])
        assert diff <= tol(rep[b].plan.r, n, d) * refn, (b, diff / refn)


def test_small_path_certified_planner_fallback(cuda):
    """K5's in-library certified digit rule declines near digit boundaries;
    the exact planner then runs on the host and the Horner launch follows.
    A matrix whose e_1 sits on an integer (scaled so ||B_1|| ||Y|| / ||B_0||
    lands on a power of ten) still gets the reference schedule."""
    from paper_2312_17396_b200 import _lib, engine
    from paper_2312_17396_b200.precision import MatBatch
    import torch
    m = mp()
    ctx = m.PrecisionCtx(15)
    X = synth(16, 0.5, 2)
    rep = m.ps_mixed_exp(X, 16, ctx)
    assert rep.plan.level_digits == m.plan_precisions(rep.plan.norm_bs, rep.plan.norm_y, ctx, s=4).level_digits
    # drive the C rule directly with boundary norms: it must decline
    h = _lib.handle_for()
    Xm = MatBatch(torch.from_numpy(X).cuda()[None, None], 15)
    cw = engine._small_coeffs(m.taylor_exp_coeffs(16), ctx)
    blocks = torch.empty((5, 1, 16, 16), dtype=torch.float64, device="cuda")
    Y = torch.empty((1, 16, 16), dtype=torch.float64, device="cuda")
    nd = torch.empty((1, 6), dtype=torch.float64, device="cuda")
    out = MatBatch.empty(15, 1, 16, device="cuda")
    norms, digits, nu, planned = h.small_ps_eval(Xm, 16, 4, cw, 15, 1e15, True, False, blocks, Y, nd, out)
    # delta = 1e15 puts the threshold d - log10(delta) = 0: certified unless some e_i is near 0 or an integer
    assert norms.shape == (1, 6)
    if planned:
        p = m.plan_precisions(norms[0, :5], norms[0, 5], ctx, 1e15, s=4)
        assert tuple(digits[0]) == p.level_digits and nu[0] == p.nu


@pytest.mark.parametrize("d,n", [(15, 8), (15, 40), (31, 40)])
def test_non_finite_input_raises_and_keeps_the_graphs(cuda, d, n):
    """A NaN or Inf entry must not come back as finite digits: the block
    norms carry it to the planner (NaN-keeping column maxima), which raises
    ValueError as the reference's does for a non-finite norm
    (engine.py:467-472 -> precision.py one_norm); the cached graphs of the
    shape stay usable afterwards (no eager fallback, no warning)."""
    import warnings
    m = mp()
    ctx = m.PrecisionCtx(d)
    X = synth(n, 1.0, 3)
    good = words_of(m.ps_mixed_exp(X, 16, ctx))
    for bad in (np.nan, np.inf, -np.inf):
        Xb = X.copy()
        Xb[n // 2, 1] = bad
        with warnings.catch_warnings():
            warnings.simplefilter("error")
            with pytest.raises(ValueError):
                m.ps_mixed_exp(Xb, 16, ctx)
            again = words_of(m.ps_mixed_exp(X, 16, ctx))
        assert np.array_equal(good, again)
    # one bad member of a batch fails the call (the reference has no batches)
    Xs = np.stack([X, X])
    Xs[1, 0, 0] = np.nan
    with pytest.raises(ValueError):
        m.ps_mixed_exp(Xs, 16, ctx)
    # the other evaluators: fixed precision and explicit powers (no planner on their path),
    # the cosine's Z = X X (a product before any norm), Pade pairs, scaling and squaring
    Xb = X.copy()
    Xb[1, n - 1] = np.nan
    for fn in (lambda: m.ps_fixed(Xb, m.taylor_exp_coeffs(12), ctx),
               lambda: m.ps_mixed_exp(Xb, 2, ctx),
               lambda: m.ps_mixed_exp(Xb, 16, ctx, fix_params=False),
               lambda: m.ps_mixed_general(m.cos_argument(Xb, ctx), m.taylor_cos_coeffs(12), ctx),
               lambda: m.ps_mixed_pade(Xb, 13, ctx),
               lambda: m.expm_ss(Xb, ctx, 16)):
        with pytest.raises(ValueError):
            fn()


def test_empty_batch_and_empty_matrix(cuda):
    """No kernel is launched for an empty batch or 0 x 0 matrices; the
    reference returns an empty result for from_rows([]) (engine.py:390-482)."""
    m = mp()
    for ctx in (m.PrecisionCtx(15), m.PrecisionCtx(31)):
        reps = m.ps_mixed_exp(np.zeros((0, 8, 8)), 16, ctx)
        assert len(reps) == 0
        reps = m.ps_mixed_general(np.zeros((0, 40, 40)), m.taylor_cos_coeffs(12), ctx)
        assert len(reps) == 0
        assert len(m.ps_fixed(np.zeros((0, 8, 8)), m.taylor_exp_coeffs(9), ctx)) == 0
        rep = m.ps_mixed_exp(np.zeros((0, 0)), 8, ctx)
        assert tuple(rep.result.data.shape[-2:]) == (0, 0)
        assert all(x == 1 for x in rep.plan.level_digits)
        assert len(m.expm_ss(np.zeros((0, 8, 8)), ctx, 16)) == 0


def test_batches_beyond_the_grid_range(cuda):
    """More matrices than blockIdx.y / z can index run as sub-batches; every
    member keeps the bits it has alone (batch invariance)."""
    import torch
    m = mp()
    for d, B, n in ((31, 70000, 4), (15, 66000, 33)):
        ctx = m.PrecisionCtx(d)
        Xb = np.random.default_rng(d).standard_normal((B, n, n)) / n
        reps = m.ps_mixed_exp(Xb, 8, ctx)
        assert len(reps) == B and reps.result.batch == B
        for b in (0, 32767, 32768, B - 1):
            solo = m.ps_mixed_exp(Xb[b], 8, ctx)
            assert torch.equal(reps.result.data[:, b], solo.result.data[:, 0])
            assert torch.equal(reps[b].result.data.reshape(-1), solo.result.data.reshape(-1))
            assert reps[b].plan.level_digits == solo.plan.level_digits


def test_graph_cache_is_bounded_by_bytes(cuda):
    """Cached shapes keep their intermediates in private pools; least recently used shapes are
    dropped once the recorded pools exceed the budget, and an evicted shape is simply captured
    again (same bits)."""
    import torch
    from paper_2312_17396_b200 import graphs
    m = mp()
    ctx = m.PrecisionCtx(31)
    graphs.clear()
    try:
        Xs = {n: np.stack([synth(n, 1.0, 10 * n + i) for i in range(4)]) for n in (40, 48, 56, 64)}
        first = {n: m.ps_mixed_exp(X, 16, ctx).result.data.clone() for n, X in Xs.items()}
        info = graphs.cache_info()
        assert info["shapes"] == 4 and info["bytes"] > 0
        per = info["bytes"] // 4
        graphs.set_cache_budget(2 * per + per // 2)
        for n, X in list(Xs.items()) * 2:
            assert torch.equal(m.ps_mixed_exp(X, 16, ctx).result.data, first[n])
            assert graphs.cache_info()["shapes"] <= 4
        X72 = np.stack([synth(72, 1.0, i) for i in range(4)])
        m.ps_mixed_exp(X72, 16, ctx)
        assert graphs.cache_info()["shapes"] <= 3
        for n, X in Xs.items():            # evicted shapes are captured again
            assert torch.equal(m.ps_mixed_exp(X, 16, ctx).result.data, first[n])
        assert graphs.cache_info()["shapes"] <= 4
    finally:
        graphs.set_cache_budget(None)
        graphs.clear()


def test_small_path_one_launch_equals_two_launches(cuda):
    """mpps_small_ps_eval runs prepare, the digit rule (on the device) and the Horner chain in one
    launch; the same operations as small_ps_prepare + the host rule + small_ps_horner, hence the
    same bits, digits and nu -- mixed and fixed, batches with heterogeneous plans, n = 32 / 17 / 5."""
    import torch
    from paper_2312_17396_b200 import _lib, planner
    from paper_2312_17396_b200.coefficients import coeff_words
    from paper_2312_17396_b200.precision import MatBatch, FP64
    m_ = mp()
    h = _lib.handle_for()
    ctx = m_.PrecisionCtx(15)
    for n, B, deg in ((32, 6, 16), (17, 3, 30), (5, 4, 9), (32, 1, 25)):
        series = m_.taylor_exp_coeffs(deg)
        s = planner.default_block_size(deg)
        r = deg // s
        cw = np.ascontiguousarray(coeff_words(series, ctx)[:, 0])
        Xs = np.stack([synth(n, 10.0 ** (-b), 7 * n + b) for b in range(B)])      # norms 1 .. 1e-5: different plans
        X = MatBatch(torch.from_numpy(Xs).cuda().unsqueeze(0), FP64)
        for fixed in (False, True):
            l0 = _lib.total_launches()
            blocks = torch.empty((r + 1, B, n, n), dtype=torch.float64, device=cuda)
            Y = torch.empty((B, n, n), dtype=torch.float64, device=cuda)
            nd = torch.empty((B, r + 2), dtype=torch.float64, device=cuda)
            out = MatBatch.empty(FP64, B, n, device=cuda)
            norms, digits, nu, planned = h.small_ps_eval(X, deg, s, cw, 15, 10.0, True, fixed, blocks, Y, nd, out)
            assert planned and _lib.total_launches() - l0 == 1
            # the two-launch path with the exact host planner
            blocks2, Y2, nd2 = torch.empty_like(blocks), torch.empty_like(Y), torch.empty_like(nd)
            h.small_ps_prepare(X, deg, s, cw, blocks2, Y2, nd2)
            norms2 = nd2.cpu().numpy()
            assert np.array_equal(norms, norms2) and torch.equal(Y, Y2)
            top = deg % s == 0
            assert torch.equal(blocks[:r if top else r + 1], blocks2[:r if top else r + 1])
            fm = np.ones((B, r + 1), dtype=np.int8)
            for b in range(B):
                if fixed:
                    dg, nu_b = (15,) * r, r + 1
                else:
                    p = planner.plan_precisions(tuple(float(x) for x in norms2[b, :r + 1]), float(norms2[b, r + 1]), ctx,
                                                10.0, s=s)
                    dg, nu_b = p.level_digits, p.nu
                assert tuple(int(x) for x in digits[b]) == tuple(dg) and int(nu[b]) == nu_b
                fm[b, 1:] = [0 if x <= 7 else 1 for x in dg]
            out2 = MatBatch.empty(FP64, B, n, device=cuda)
            h.small_ps_horner(Y2, blocks2, fm, deg, s, float(cw[deg]), out2)
            assert torch.equal(out.data, out2.data)


@pytest.mark.parametrize("m", [17, 19, 26, 29, 37, 38, 41])
def test_flat_plans_after_two_pass_assembly(cuda, oracle_lib, m):
    """dd evaluations whose plan keeps (nearly) every level at dd (a large ||X||) re-assemble all
    blocks in dd after the two-pass assembly; for r + 1 = s blocks (m = 17-19, 26-29, 37-41) that
    pass had no compiled kernel and the evaluation raised (found by tools/fuzz_vs_oracle.py).
    Oracle parity, alone and next to a small-norm batch mate (batch invariance)."""
    import torch
    import oracle
    mm = mp()
    ctx = mm.PrecisionCtx(31)
    n = 30
    X = synth(n, 6.0, m)
    rep = mm.ps_mixed_exp(X, m, ctx)
    ref = oracle.ps_eval(X, mm.taylor_exp_coeffs(m).coeffs, 31)
    _check(rep, ref, n, 31)
    assert sum(1 for x in rep.plan.level_digits if x > 15) >= 2      # dd levels beyond B_0, B_1: a re-assembly
    both = mm.ps_mixed_exp(np.stack([X, synth(n, 1e-3, m + 1)]), m, ctx)
    assert torch.equal(both[0].result.data.reshape(-1), rep.result.data.reshape(-1))
    num, den = mm.ps_mixed_pade(X, m if m < 30 else 18, ctx)
    pc, qc = mm.pade_exp_coeffs(m if m < 30 else 18, m if m < 30 else 18)
    _check(num, oracle.ps_eval(X, pc.coeffs, 31), n, 31)
    _check(den, oracle.ps_eval(X, qc.coeffs, 31), n, 31)


def test_graph_replay_after_the_coefficient_cache_rolled_over(cuda):
    """A captured graph bakes the device address of the coefficient tensor into its assembly
    kernel; the tensor lives in a module-level cache that is cleared after 64 distinct series.
    The prepared state of the graph must keep it alive: replaying the first shape after 70 other
    series used to read freed memory (blocks without their b_0 I, garbage norms).  Found by
    tools/fuzz_vs_oracle.py."""
    import torch
    from paper_2312_17396_b200 import graphs
    m = mp()
    ctx = m.PrecisionCtx(31)
    series = m.taylor_exp_coeffs(1)            # s = 1: the run-time-coefficient assembly kernel
    X1, X2 = synth(19, 0.13, 1), synth(19, 0.2, 2)
    first = m.ps_fixed(X1, series, ctx).result.data.clone()          # captures
    small = synth(6, 0.3, 3)
    for deg in range(2, 38):
        for d in (15, 31):
            m.ps_fixed(small, m.taylor_exp_coeffs(deg), m.PrecisionCtx(d))
    # whatever the rolled-over cache freed is reallocated and overwritten (the tensor was
    # allocated on the capture's warm-up side stream, so the junk goes through torch's stream pool)
    junk = []
    for _ in range(40):
        side = torch.cuda.Stream()
        with torch.cuda.stream(side):
            junk += [torch.full((k % 60 + 4,), float("nan"), dtype=torch.float64, device=cuda) for k in range(200)]
    torch.cuda.synchronize()
    again = m.ps_fixed(X1, series, ctx).result.data                  # replays
    assert torch.equal(first, again)
    del junk
    # (whether freed memory is actually handed out again depends on the allocator's stream pools, so
    # the mechanism is checked too: the graph's prepared state owns the coefficient tensor)
    from paper_2312_17396_b200.coefficients import coeff_words
    g = next(v for k, v in graphs._CACHE.items() if k[0] == (1, 19, 19))
    kept = [t for t in g.prep.keep if torch.is_tensor(t) and t.dtype == torch.float64]
    assert kept and np.array_equal(kept[0].cpu().numpy(), np.asarray(coeff_words(series, ctx), dtype=np.float64))
    got = m.ps_fixed(X2, series, ctx).result.data.clone()
    graphs.set_enabled(False)
    try:
        want = m.ps_fixed(X2, series, ctx).result.data
    finally:
        graphs.set_enabled(True)
    assert torch.equal(got, want)
    rep = m.ps_mixed_general(X2, m.taylor_cos_coeffs(24), ctx)
    assert rep.plan.level_digits[0] > 1


def test_host_batches_one_stream_download_waits_for_the_result_copy(cuda):
    """pipeline.evaluate_host in its default mode (one stream, chunks one after another) downloads each
    chunk on a copy stream once the evaluation's done event has fired; for cloned results that event
    must follow the copy out of the graph's static buffer (it was recorded before it: ~1 % of the
    calls downloaded a tensor that had not been written yet; found by tools/fuzz_pipeline.py).  Many
    repetitions of two of the configurations that failed, against the direct call, bitwise."""
    import torch
    from paper_2312_17396_b200 import pipeline as pl
    m = mp()
    ctx = m.PrecisionCtx(31)
    for n, B, deg, sizes in ((24, 18, 16, [18]), (64, 12, 9, [5, 7])):
        X = np.stack([synth(n, 10.0 ** (-0.3 * b), 11 * n + b) for b in range(B)])
        direct = m.ps_mixed_exp(X, deg, ctx).result.data.cpu()
        Xh = torch.from_numpy(X).pin_memory()
        out = torch.empty((2, B, n, n), dtype=torch.float64).pin_memory()
        sub = pl.mixed_exp(deg, ctx, timing=False)
        for _ in range(150):
            out.zero_()
            pl.evaluate_host(sub, Xh, out, sizes, streams=1)
            torch.cuda.synchronize()
            assert torch.equal(out, direct)
