"""2-D block SUMMA driver: one large matrix polynomial over a pr x pc grid of
GPUs, NCCL collectives through torch.distributed.

Every rank owns block (I, J) of X, of each power X^k, of every coefficient
block B_i and of every Horner iterate: rows [I n/pr, (I+1) n/pr), columns
[J n/pc, (J+1) n/pc).  A product C = A B is formed block-locally as
C_IJ = A_I: B_:J from two gathered panels:

  * power chain X^k = X^{k-1} X (engine.py:151-153): the column panel X_:J is
    gathered ONCE per evaluation (all-gather along the process column), the
    row panel of X^{k-1} each step (all-gather along the process row);
  * Horner Y phi_j (engine.py:249-251): the row panel Y_I: is gathered once
    (at the working planes; each level uses a prefix), the column panel of
    phi_j each level -- at the level format's planes;
  * panels move as digit planes: each rank reduces the row (column) scales
    of its block over the process row (column), splits only its own block
    with them and all-gathers the planes -- exactly the split of the whole
    panel, without splitting it pc (pr) times over, and S bytes per entry
    instead of the dd words' 16;
  * block assembly, the Horner add and all format conversions are local;
  * overlap: every product is issued in row chunks (power chain) or column
    chunks (Horner) and each finished chunk's panel all-gather is started
    at once (async collective on NCCL's stream), so the gather of chunk t
    runs while chunk t+1 is computed, and the next product's chunk t waits
    only for its own gathered rows/columns.  Rows of a left operand and
    columns of a right operand are split independently (per-row / per-column
    digit scales), so chunking changes no bit of the result;
  * planner norms: local column abs-sums (mpps_assemble_blocks_dist) ->
    all-reduce(sum) along the process column -> column max -> all-reduce(max)
    over the grid; every rank then runs the same deterministic planner and
    rank 0's digits are broadcast so the schedule is identical everywhere.

The arithmetic is the same C-ABI kernels as the single-GPU path (rectangular
GEMM blocks with the fused Horner epilogue).  The ``ops`` object isolates the
device calls so the collective plumbing is testable on CPU with gloo
(tests/test_summa_gloo.py).
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from typing import Dict, List, Optional, Tuple

import numpy as np

from .coefficients import CoefficientSeries, coeff_words
from .planner import default_block_size, formats_of_digits, plan_digits_batch, plan_precisions
from .precision import FP32, FP64, MatBatch, PrecisionCtx


def _torch():
    import torch
    return torch


def _dist():
    import torch.distributed as dist
    return dist


class ProcessGrid:
    """pr x pc process grid over the default process group (row-major ranks)
    with one communicator per process row and per process column."""

    def __init__(self, pr: int, pc: int):
        dist = _dist()
        world = dist.get_world_size()
        if pr * pc != world:
            raise ValueError(f"grid {pr}x{pc} != world size {world}")
        self.pr, self.pc = pr, pc
        self.rank = dist.get_rank()
        self.I, self.J = divmod(self.rank, pc)
        # every rank must create every group, in the same order
        rows = [dist.new_group([i * pc + j for j in range(pc)]) if pc > 1 else None for i in range(pr)]
        cols = [dist.new_group([i * pc + j for i in range(pr)]) if pr > 1 else None for j in range(pc)]
        self.row_group = rows[self.I]
        self.col_group = cols[self.J]

    @classmethod
    def single(cls) -> "ProcessGrid":
        """A 1x1 grid without a process group (one GPU, no collectives)."""
        g = cls.__new__(cls)
        g.pr = g.pc = 1
        g.rank = g.I = g.J = 0
        g.row_group = g.col_group = None
        return g

    @staticmethod
    def for_world(world: int) -> Tuple[int, int]:
        """1x1, 1x2, 2x2, 2x4, ... (pr <= pc, pr a power-of-two split)."""
        pr = 1
        while (pr * 2) * (pr * 2) <= world and world % (pr * 2) == 0:
            pr *= 2
        return pr, world // pr

    def block(self, n: int):
        if n % self.pr or n % self.pc:
            raise ValueError(f"n={n} must be divisible by the grid {self.pr}x{self.pc}")
        mr, nc = n // self.pr, n // self.pc
        return self.I * mr, mr, self.J * nc, nc

    # --- panels ------------------------------------------------------
    def row_panel(self, A: MatBatch) -> MatBatch:
        """A_I: = [A_I0 ... A_I(pc-1)] (all-gather along the process row)."""
        if self.pc == 1:
            return A
        torch, dist = _torch(), _dist()
        parts = [torch.empty_like(A.data) for _ in range(self.pc)]
        dist.all_gather(parts, A.data.contiguous(), group=self.row_group)
        return MatBatch(torch.cat(parts, dim=3), A.fmt)

    def col_panel(self, A: MatBatch) -> MatBatch:
        """A_:J = [A_0J; ...; A_(pr-1)J] (all-gather along the process column)."""
        if self.pr == 1:
            return A
        torch, dist = _torch(), _dist()
        parts = [torch.empty_like(A.data) for _ in range(self.pr)]
        dist.all_gather(parts, A.data.contiguous(), group=self.col_group)
        return MatBatch(torch.cat(parts, dim=2), A.fmt)

    # --- chunked, asynchronous panels (compute/communication overlap) ---
    def row_panel_start(self, A: MatBatch):
        """Start the all-gather of A's rows along the process row; the
        returned handle's panel_finish() gives [A_I0 ... A_I(pc-1)]."""
        if self.pc == 1:
            return _Done(A)
        torch, dist = _torch(), _dist()
        src = A.data.contiguous()
        parts = [torch.empty_like(src) for _ in range(self.pc)]
        work = dist.all_gather(parts, src, group=self.row_group, async_op=True)
        return _Pending(work, parts, 3, A.fmt)

    def col_panel_start(self, A: MatBatch):
        """Start the all-gather of A's columns along the process column."""
        if self.pr == 1:
            return _Done(A)
        torch, dist = _torch(), _dist()
        src = A.data.contiguous()
        parts = [torch.empty_like(src) for _ in range(self.pr)]
        work = dist.all_gather(parts, src, group=self.col_group, async_op=True)
        return _Pending(work, parts, 2, A.fmt)

    def sum_over_column(self, t):
        if self.pr > 1:
            _dist().all_reduce(t, op=_dist().ReduceOp.SUM, group=self.col_group)
        return t

    def max_over_grid(self, t):
        if self.pr * self.pc > 1:
            _dist().all_reduce(t, op=_dist().ReduceOp.MAX)
        return t

    def broadcast(self, t):
        if self.pr * self.pc > 1:
            _dist().broadcast(t, src=0)
        return t

    def gather_full(self, A: MatBatch, n: int) -> Optional[np.ndarray]:
        """Assemble the global (words, n, n) matrix on every rank (checking
        and tests only; not on the timed path)."""
        torch, dist = _torch(), _dist()
        if self.pr * self.pc == 1:
            return A.data[:, 0].double().cpu().numpy()
        parts = [torch.empty_like(A.data) for _ in range(self.pr * self.pc)]
        dist.all_gather(parts, A.data.contiguous())
        rows = []
        for i in range(self.pr):
            rows.append(torch.cat(parts[i * self.pc:(i + 1) * self.pc], dim=3))
        return torch.cat(rows, dim=2)[:, 0].double().cpu().numpy()


class _Done:
    __slots__ = ("A",)

    def __init__(self, A):
        self.A = A

    def panel_finish(self) -> MatBatch:
        return self.A


class _Pending:
    """An in-flight panel all-gather; panel_finish() makes the caller's
    stream wait for it (no host block on NCCL) and concatenates the parts."""
    __slots__ = ("work", "parts", "dim", "fmt")

    def __init__(self, work, parts, dim, fmt):
        self.work, self.parts, self.dim, self.fmt = work, parts, dim, fmt

    def panel_finish(self) -> MatBatch:
        self.work.wait()
        return MatBatch(_torch().cat(self.parts, dim=self.dim), self.fmt)


def chunk_bounds(extent: int, chunks: int, align: int = 128) -> List[Tuple[int, int]]:
    """[lo, hi) pieces of ``extent`` for chunked products: at most
    ``chunks`` pieces, interior boundaries on multiples of ``align`` (the
    tensor-core row tile) where the extent allows."""
    chunks = max(1, int(chunks))
    if chunks == 1 or extent <= align:
        return [(0, extent)]
    step = -(-extent // chunks)
    step = -(-step // align) * align
    out, lo = [], 0
    while lo < extent:
        hi = min(extent, lo + step)
        out.append((lo, hi))
        lo = hi
    return out


def rows_of(A: MatBatch, lo: int, hi: int) -> MatBatch:
    return MatBatch(A.data[:, :, lo:hi, :], A.fmt)


def cols_of(A: MatBatch, lo: int, hi: int) -> MatBatch:
    return MatBatch(A.data[:, :, :, lo:hi], A.fmt)


DEFAULT_CHUNKS = 4


class _PlanePending:
    """An in-flight digit-plane panel (DeviceOps.panel_start); finish()
    makes the caller's stream wait for the gather and returns the operand."""
    __slots__ = ("work", "parts", "sl", "rows", "k", "db", "fmt", "side")

    def __init__(self, work, parts, sl, rows, k, db, fmt, side):
        self.work, self.parts, self.sl, self.rows, self.k = work, parts, sl, rows, k
        self.db, self.fmt, self.side = db, fmt, side

    def finish(self):
        from . import _lib
        from . import gemm_engine as ge
        if self.work is not None:
            self.work.wait()
        sl = _lib.Slices.__new__(_lib.Slices)
        sl.digits = self.parts[0] if len(self.parts) == 1 else _torch().cat(self.parts, dim=3)
        sl.exps = self.sl.exps
        sl.S, sl.rows, sl.k, sl.db = self.sl.S, self.rows, self.k, self.db
        return ge.Operand(None, sl, self.fmt, self.side)


class DeviceOps:
    """The C-ABI kernels, for SummaPS (one matrix per call, batch = 1)."""

    def __init__(self, handle=None):
        from . import _lib
        self.h = handle or _lib.handle_for()
        torch = _torch()
        self.device = torch.device("cuda", torch.cuda.current_device())

    def empty(self, fmt, rows, cols):
        return MatBatch.empty(fmt, 1, rows, cols, device=self.device)

    def _e(self, e):
        if not e:
            return None
        return _torch().tensor([int(e)], dtype=_torch().int32, device=self.device)

    def convert(self, src, dst, exp=0):
        self.h.convert(src, dst, None, self._e(exp))

    def gemm(self, A, B, C):
        self.gemm_op(self.prepare(A, 0, C.fmt), self.prepare(B, 1, C.fmt), C)

    # prepared operands (tensor-core digit planes or SIMT matrices)
    def prepare(self, A, side, fmt, exp=0):
        from . import gemm_engine as ge
        # the digit width follows the evaluation's working format (set by
        # the drivers below), so every product's operands share it
        return ge.prepare(self.h, A, side, fmt, None, self._e(exp), wf=getattr(self, "wf", None))

    def gemm_op(self, L, R, C):
        from . import gemm_engine as ge
        ge.gemm(self.h, L, R, C)

    def panel_start(self, grid: "ProcessGrid", A: MatBatch, side: int, fmt: int, k_total: int):
        """Start the digit-plane panel of this rank's block A: side 0, the row
        panel A_I: (the blocks of the process row concatenated along K); side
        1, the column panel A_:J (along the process column).  Each rank
        splits only its own block, with the row / column scales reduced
        (max) over the panel first, so the gathered planes are exactly the
        split of the whole panel; the planes (S bytes per entry instead of
        the dd words' 16) are all-gathered asynchronously."""
        from . import _lib
        from . import gemm_engine as ge
        torch, dist = _torch(), _dist()
        h = self.h
        db = ge.digit_bits_for(h, k_total, getattr(self, "wf", None) or fmt)
        S = h.slices_for(fmt, db)
        rows, k = (A.rows, A.cols) if side == 0 else (A.cols, A.rows)
        parts_n, group = (grid.pc, grid.row_group) if side == 0 else (grid.pr, grid.col_group)
        sl = _lib.Slices(S, 1, rows, k, self.device, db)
        if parts_n == 1:
            h.slice_ex(A, side, sl, 0)
            return _PlanePending(None, [sl.digits], sl, rows, k, db, fmt, side)
        if k % 32:
            raise ValueError(f"SUMMA plane gathers need block extents divisible by 32 (got {k})")
        h.slice_ex(A, side, sl, 1)                                   # this block's scales
        dist.all_reduce(sl.exps, op=dist.ReduceOp.MAX, group=group)  # the panel's scales
        h.slice_ex(A, side, sl, 2)                                   # split with them
        parts = [torch.empty_like(sl.digits) for _ in range(parts_n)]
        work = dist.all_gather(parts, sl.digits, group=group, async_op=True)
        return _PlanePending(work, parts, sl, rows, k * parts_n, db, fmt, side)

    def concat_rows(self, ops_):
        """One row-split operand from row chunks (digit planes and scales)."""
        from . import _lib
        from . import gemm_engine as ge
        if len(ops_) == 1:
            return ops_[0]
        torch = _torch()
        s0 = ops_[0].slices
        sl = _lib.Slices.__new__(_lib.Slices)
        sl.digits = torch.cat([o.slices.digits for o in ops_], dim=2)
        sl.exps = torch.cat([o.slices.exps for o in ops_], dim=1)
        sl.S, sl.rows, sl.k, sl.db = s0.S, sl.digits.shape[2], s0.k, s0.db
        return ge.Operand(None, sl, ops_[0].fmt, 0)

    def horner_op(self, Y, phi, fmt_level, Bprev, out, ey=0, ei=0, eo=0):
        from . import gemm_engine as ge
        ge.horner(self.h, Y, phi, fmt_level, Bprev, out, None, self._e(ey), self._e(ei), self._e(eo))

    def coeffs(self, series, ctx):
        return _torch().tensor(coeff_words(series, ctx), dtype=_torch().float64, device=self.device)

    def assemble_dist(self, powers, m, coeffs, blocks, row0, col0):
        torch = _torch()
        r = len(blocks) - 1
        colsums = torch.empty((1, r + 2, powers[0].cols), dtype=torch.float64, device=self.device)
        self.h.assemble_blocks_dist(powers, m, coeffs, blocks, colsums, row0, col0)
        return colsums

    def colmax(self, colsums):
        torch = _torch()
        out = torch.empty((colsums.shape[0], colsums.shape[1]), dtype=torch.float64, device=self.device)
        self.h.colmax(colsums, colsums.shape[1], colsums.shape[2], colsums.shape[0], out)
        return out

    def horner_step(self, Y, phi, Bprev, out, ey=0, ei=0, eo=0):
        self.h.horner_step(Y, phi, Bprev, out, None, self._e(ey), self._e(ei), self._e(eo))

    def scalar_top(self, bm_words, fmt_top, Y, Bprev, out, eo=0):
        self.h.horner_scalar_top(bm_words, fmt_top, Y, Bprev, out, None, self._e(eo))


@dataclass
class DistResult:
    block: MatBatch            # this rank's block of p(X) at the working format
    digits: Tuple[int, ...]
    nu: int
    nilpotent: bool
    norms: np.ndarray          # (r+2,) global ||B_0..B_r||, ||Y||
    s: int
    r: int

    def plan(self, ctx: PrecisionCtx, delta: float = 10.0):
        """The full EvaluationPlan (exact planner on the global norms)."""
        return plan_precisions(tuple(float(x) for x in self.norms[:self.r + 1]), float(self.norms[self.r + 1]),
                               ctx, delta, s=self.s)


def _exp_for(v: float) -> int:
    return -int(round(math.log2(v))) if v > 0 and math.isfinite(v) else 0


def _working(ctx):
    f = ctx.fmt
    return FP64 if f == FP32 else f


def cos_argument_dist(Xblk: MatBatch, ctx: PrecisionCtx, grid: ProcessGrid, ops) -> MatBatch:
    """Z_IJ = X_I: X_:J at the working format (harness.py:100-101)."""
    wf = _working(ctx)
    ops.wf = wf
    Xw = Xblk
    if Xblk.fmt != wf:
        Xw = ops.empty(wf, Xblk.rows, Xblk.cols)
        ops.convert(Xblk, Xw)
    Z = ops.empty(wf, Xw.rows, Xw.cols)
    n = Xw.rows * grid.pr
    rp = ops.panel_start(grid, Xw, 0, wf, n)
    cp = ops.panel_start(grid, Xw, 1, wf, n)
    ops.gemm_op(rp.finish(), cp.finish(), Z)
    return Z


def ps_mixed_dist(Xblk: MatBatch, series: CoefficientSeries, ctx: PrecisionCtx, grid: ProcessGrid,
                  ops=None, delta: float = 10.0, fixed: bool = False, chunks: Optional[int] = None,
                  chunk_align: int = 128) -> DistResult:
    """ps_mixed_general (engine.py:348-387) -- or ps_fixed (304-345) with
    ``fixed`` -- of one n x n matrix distributed over ``grid``; Xblk is this
    rank's block (fp64 or working format).  ``chunks``: row / column pieces
    per product for communication overlap (default DEFAULT_CHUNKS on a
    multi-rank grid, 1 on 1x1); the result does not depend on it."""
    torch = _torch()
    ops = ops or DeviceOps()
    if chunks is None:
        chunks = 1 if grid.pr * grid.pc == 1 else DEFAULT_CHUNKS
    m = series.degree
    if m < 1:
        raise ValueError("series degree must be >= 1")
    d = ctx.decimal_digits
    wf = _working(ctx)
    ops.wf = wf
    s = default_block_size(m)
    r = m // s
    n = Xblk.rows * grid.pr
    row0, mr, col0, nc = grid.block(n)
    if (Xblk.rows, Xblk.cols) != (mr, nc):
        raise ValueError(f"block shape {(Xblk.rows, Xblk.cols)} != {(mr, nc)} for n={n}")
    # powers (engine.py:141-154): X^k = X^{k-1} X
    P1 = Xblk
    if Xblk.fmt != wf:
        P1 = ops.empty(wf, mr, nc)
        ops.convert(Xblk, P1)
    powers = [P1]
    rch = chunk_bounds(mr, chunks, chunk_align)
    # row-panel gathers of the newest power, one per row chunk, in flight
    # while the chunks after it are computed (and, for Y = X^s, while the
    # blocks are assembled and the norms reduced)
    pend = [ops.panel_start(grid, rows_of(P1, lo, hi), 0, wf, n) for lo, hi in rch]
    if s > 1:
        Xr = ops.panel_start(grid, P1, 1, wf, n).finish()      # gathered and split once
        for _ in range(1, s):
            C = ops.empty(wf, mr, nc)
            nxt = []
            for (lo, hi), pnd in zip(rch, pend):
                ops.gemm_op(pnd.finish(), Xr, rows_of(C, lo, hi))
                nxt.append(ops.panel_start(grid, rows_of(C, lo, hi), 0, wf, n))
            pend = nxt
            powers.append(C)
    blocks = [ops.empty(wf, mr, nc) for _ in range(r + 1)]
    coeffs = ops.coeffs(series, ctx)
    colsums = ops.assemble_dist(powers, m, coeffs, blocks, row0, col0)
    grid.sum_over_column(colsums)
    norms_t = grid.max_over_grid(ops.colmax(colsums))
    norms = norms_t.double().cpu().numpy()[0]
    # planner (identical inputs on all ranks; rank 0's digits broadcast)
    if fixed:
        digits = np.full(r, d, dtype=np.int64)
        nu, nil = r + 1, False
    else:
        dg, nv, nl = plan_digits_batch(norms[None, :r + 1], norms[None, r + 1], d, delta)
        digits, nu, nil = dg[0], int(nv[0]), bool(nl[0])
    pk = torch.tensor(list(digits) + [nu, int(nil)], dtype=torch.int64).to(norms_t.device)
    grid.broadcast(pk)
    pk = pk.cpu().numpy()
    digits, nu, nil = tuple(int(x) for x in pk[:r]), int(pk[r]), bool(pk[r + 1])
    if nil:
        return DistResult(blocks[0], digits, nu, True, norms, s, r)
    fm = (wf,) + formats_of_digits(digits)
    ex = [(_exp_for(float(norms[j])) if fm[j] == FP32 else 0) for j in range(r + 1)]
    ey = _exp_for(float(norms[r + 1]))
    # Horner (engine.py:243-252)
    Y = powers[s - 1]
    # Y's row panel: the row chunks gathered during the assembly / norm
    # reduction, at the working planes (each level uses a prefix)
    Yrow = ops.concat_rows([p.finish() for p in pend])
    yrow = {}
    for f in sorted(set(fm[1:])):
        yrow[f] = (ops.prepare(Yrow.mat, 0, f, ey if f == FP32 else 0) if getattr(ops, "host_double", False)
                   else Yrow)
    if m % s == 0:
        out = ops.empty(fm[r - 1], mr, nc)
        ops.scalar_top(coeff_words(series, ctx)[m], fm[r], Y, blocks[r - 1], out, ex[r - 1])
        phi, j0 = out, r - 1
    else:
        phi = ops.empty(fm[r], mr, nc)
        ops.convert(blocks[r], phi, ex[r])
        j0 = r
    # Horner levels in column chunks: chunk t of level j-1 needs only the
    # gathered column chunk t of phi_j; its own gather starts as soon as it
    # is written
    cch = chunk_bounds(nc, chunks, chunk_align)
    pend = [ops.panel_start(grid, cols_of(phi, lo, hi), 1, fm[j0], n) for lo, hi in cch] if j0 > 0 else []
    for j in range(j0, 0, -1):
        out = ops.empty(fm[j - 1], mr, nc)
        nxt = []
        for (lo, hi), pnd in zip(cch, pend):
            ops.horner_op(yrow[fm[j]], pnd.finish(), fm[j],
                          cols_of(blocks[j - 1], lo, hi), cols_of(out, lo, hi),
                          ey if fm[j] == FP32 else 0, ex[j], ex[j - 1])
            if j > 1:
                nxt.append(ops.panel_start(grid, cols_of(out, lo, hi), 1, fm[j - 1], n))
        pend = nxt
        phi = out
    return DistResult(phi, digits, nu, False, norms, s, r)
