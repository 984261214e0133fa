"""SUMMA driver host logic on CPU with gloo and the float64 test double
(world sizes 2, 4 and 8: grids 1x2, 2x1, 2x2, 2x4): block layout, the
chunked asynchronous panel gathers (row chunks in the power chain, column
chunks in the Horner chain), the norm reduction (column sums over the
process column, max over the grid), the plan broadcast and the Horner chain
must reproduce the 1x1 evaluation."""
import os
import socket
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

HERE = os.path.dirname(os.path.abspath(__file__))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _synth(n, target, seed):
    G = np.random.default_rng(seed).standard_normal((n, n))
    return G * (target / np.abs(G).sum(axis=0).max())


def _run(rank, world, port, pr, pc, n, family, out_q, chunks):
    sys.path.insert(0, HERE)
    sys.path.insert(0, os.path.dirname(HERE))
    from _cpu_ops import CpuOps
    import paper_2312_17396_b200 as m
    from paper_2312_17396_b200 import summa
    from paper_2312_17396_b200.precision import MatBatch
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        grid = summa.ProcessGrid(pr, pc)
        ctx = m.PrecisionCtx(31)
        X = _synth(n, 1.0, 0)
        r0, mr, c0, nc = grid.block(n)
        blk = MatBatch(torch.from_numpy(X[r0:r0 + mr, c0:c0 + nc].copy())[None, None], m.FP64)
        ops = CpuOps()
        if family == "cos":
            Z = summa.cos_argument_dist(blk, ctx, grid, ops)
            res = summa.ps_mixed_dist(Z, m.taylor_cos_coeffs(24), ctx, grid, ops, chunks=chunks, chunk_align=2)
        else:
            res = summa.ps_mixed_dist(blk, m.taylor_exp_coeffs(30), ctx, grid, ops, chunks=chunks, chunk_align=2)
        full = grid.gather_full(res.block, n)
        if rank == 0:
            out_q.put((res.digits, res.nu, res.norms.tolist(), full[0].tolist()))
    finally:
        dist.destroy_process_group()


def _eval(world, pr, pc, n, family, chunks=1):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_run, args=(r, world, port, pr, pc, n, family, q, chunks)) for r in range(world)]
    for p in procs:
        p.start()
    out = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return out


@pytest.mark.parametrize("family", ["exp", "cos"])
@pytest.mark.parametrize("grid,chunks", [((1, 2), 1), ((2, 1), 3), ((2, 2), 2), ((2, 4), 3)])
def test_summa_matches_single_rank(family, grid, chunks):
    n = 16
    d1, nu1, norms1, full1 = _eval(1, 1, 1, n, family)
    d2, nu2, norms2, full2 = _eval(grid[0] * grid[1], grid[0], grid[1], n, family, chunks)
    assert d1 == d2 and nu1 == nu2
    np.testing.assert_allclose(norms2, norms1, rtol=1e-13)
    np.testing.assert_allclose(np.array(full2), np.array(full1), rtol=1e-12, atol=1e-14)
    if family == "exp":
        import scipy.linalg as sl
        np.testing.assert_allclose(np.array(full1), sl.expm(_synth(n, 1.0, 0)), rtol=0, atol=1e-12)


def test_chunk_bounds():
    from paper_2312_17396_b200.summa import chunk_bounds
    assert chunk_bounds(4096, 4) == [(0, 1024), (1024, 2048), (2048, 3072), (3072, 4096)]
    assert chunk_bounds(1000, 4) == [(0, 256), (256, 512), (512, 768), (768, 1000)]
    assert chunk_bounds(100, 4) == [(0, 100)]
    assert chunk_bounds(8, 3, 2) == [(0, 4), (4, 8)]
    assert chunk_bounds(4096, 1) == [(0, 4096)]


def test_grid_shapes():
    from paper_2312_17396_b200.summa import ProcessGrid
    assert [ProcessGrid.for_world(w) for w in (1, 2, 4, 8)] == [(1, 1), (1, 2), (2, 2), (2, 4)]
