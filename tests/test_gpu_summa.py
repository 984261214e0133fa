"""SUMMA driver on the GPU over NCCL (one rank, 1x1 grid -- the box has one
GPU; the multi-rank plumbing is covered by tests/test_summa_gloo.py).  The
distributed pipeline keeps the reference's association (X^k = X^{k-1} X,
Y phi), format plane counts and an all-dd block assembly, while the
single-GPU engine pairs powers, runs phi Y with per-level planes and
assembles fp32/fp64-level blocks in fp64: same schedule, values within the
c n u tolerance of each other and of the oracle."""
import os
import socket

import numpy as np
import pytest

from _util import synth, tol

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def nccl1(cuda):
    import torch.distributed as dist
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1)
    yield
    dist.destroy_process_group()


def test_summa_1x1_matches_single_gpu(nccl1):
    import torch
    import paper_2312_17396_b200 as m
    from paper_2312_17396_b200 import summa
    from paper_2312_17396_b200.precision import MatBatch
    n = 96
    ctx = m.PrecisionCtx(31)
    X = synth(n, 1.0, 0, cos=True)
    grid = summa.ProcessGrid(1, 1)
    blk = MatBatch(torch.from_numpy(X).cuda()[None, None], m.FP64)
    Z = summa.cos_argument_dist(blk, ctx, grid, summa.DeviceOps())
    res = summa.ps_mixed_dist(Z, m.taylor_cos_coeffs(24), ctx, grid)
    ref = m.ps_mixed_general(m.cos_argument(X, ctx), m.taylor_cos_coeffs(24), ctx)
    assert res.digits == ref.plan.level_digits and res.nu == ref.plan.nu
    a = res.block.data.cpu().numpy()
    b = ref.result.data.cpu().numpy()
    va, vb = a[0, 0] + a[1, 0], b[0, 0] + b[1, 0]
    d = np.abs((a[0, 0] - b[0, 0]) + (a[1, 0] - b[1, 0])).sum(axis=0).max()
    assert d <= tol(ref.plan.r, n, 31) * np.abs(vb).sum(axis=0).max()
    pa, pb = res.plan(ctx).to_dict(), ref.plan.to_dict()
    for k in ("s", "r", "nu", "working_digits", "digits", "roundoffs", "nilpotent"):
        assert pa[k] == pb[k], k


def test_summa_1x1_vs_oracle(nccl1, oracle_lib):
    import torch
    import paper_2312_17396_b200 as m
    from paper_2312_17396_b200 import summa
    from paper_2312_17396_b200.precision import MatBatch
    n, d = 64, 31
    X = synth(n, 1.0, 2)
    grid = summa.ProcessGrid(1, 1)
    res = summa.ps_mixed_dist(MatBatch(torch.from_numpy(X).cuda()[None, None], m.FP64),
                              m.taylor_exp_coeffs(30), m.PrecisionCtx(d), grid)
    ref = oracle_lib.ps_eval(X, m.taylor_exp_coeffs(30).coeffs, d)
    assert res.digits == ref.digits
    diff, refn = ref.compare(res.block.data[:, 0].cpu().numpy())
    assert diff <= tol(res.r, n, d) * refn


def test_summa_chunked_overlap_is_bitwise_invisible(cuda):
    """The chunked (overlapped) power and Horner chains give exactly the
    unchunked result: row chunks of a left operand and column chunks of a
    right operand (ragged last chunk, strided views into the block) are
    split and multiplied independently of the rest."""
    import torch
    import paper_2312_17396_b200 as m
    from paper_2312_17396_b200 import summa
    from paper_2312_17396_b200.precision import MatBatch
    n = 640
    ctx = m.PrecisionCtx(31)
    grid = summa.ProcessGrid.single()
    for family, X in (("exp", synth(n, 1.0, 5)), ("cos", synth(n, 1.0, 6, cos=True))):
        blk = MatBatch(torch.from_numpy(X).cuda()[None, None], m.FP64)
        ops = summa.DeviceOps()
        if family == "cos":
            blk = summa.cos_argument_dist(blk, ctx, grid, ops)
            series = m.taylor_cos_coeffs(24)
        else:
            series = m.taylor_exp_coeffs(30)
        a = summa.ps_mixed_dist(blk, series, ctx, grid, ops, chunks=1)
        b = summa.ps_mixed_dist(blk, series, ctx, grid, ops, chunks=3)
        assert a.digits == b.digits
        assert torch.equal(a.block.data, b.block.data), family


@pytest.mark.parametrize("db,fmt", [(8, 31), (7, 31), (8, 15)])
def test_plane_panel_equals_split_of_the_panel(cuda, db, fmt):
    """SUMMA panels move as digit planes: a block split with the panel's
    scales (mpps_slice_ex: mode 1 scales of each block, max over the blocks,
    mode 2 split) and concatenated along K gives exactly the planes and
    scales of the split of the whole panel -- row panels (side 0, blocks
    along columns) and column panels (side 1, blocks along rows)."""
    import torch
    from paper_2312_17396_b200 import _lib
    from paper_2312_17396_b200.precision import MatBatch
    h = _lib.handle_for()
    rng = np.random.default_rng(12)
    rows, K, parts = 200, 384, 3            # blocks of K/parts = 128
    W = 2 if fmt == 31 else 1
    A = rng.standard_normal((W, 1, rows, K)) * np.logspace(0, -9, K)[None, None, None, :]
    if W == 2:
        A[1] *= 2.0 ** -57
    S = h.slices_for(fmt, db)
    for side in (0, 1):
        src = A if side == 0 else A.transpose(0, 1, 3, 2).copy()
        M = MatBatch(torch.from_numpy(src).cuda(), fmt)
        whole = h.slice(M, side, S, None, db)
        kb = K // parts
        blocks = []
        for p in range(parts):
            sub = src[..., :, p * kb:(p + 1) * kb] if side == 0 else src[..., p * kb:(p + 1) * kb, :]
            B = MatBatch(torch.from_numpy(np.ascontiguousarray(sub)).cuda(), fmt)
            sl = _lib.Slices(S, 1, rows, kb, "cuda", db)
            h.slice_ex(B, side, sl, 1)
            blocks.append((B, sl))
        ex = torch.stack([sl.exps for _, sl in blocks]).amax(dim=0)
        for B, sl in blocks:
            sl.exps.copy_(ex)
            h.slice_ex(B, side, sl, 2)
        digits = torch.cat([sl.digits for _, sl in blocks], dim=3)
        assert torch.equal(ex[:, :rows], whole.exps[:, :rows]), side
        assert torch.equal(digits[:, :, :rows], whole.digits[:, :, :rows]), side
