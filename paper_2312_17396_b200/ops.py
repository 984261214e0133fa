"""The reference's per-op precision-context layer (precision.py:153-249) on
device batches: each call is one kernel of libmpps_b200.so.

    round_to(A, ctx)            precision.py:153-157   mpps_convert
    mat_mul(A, B, ctx)          precision.py:160-184   mpps_gemm
    mat_axpy(alpha, A, B, ctx)  precision.py:187-197   mpps_axpy
    one_norm(A)                 precision.py:235-249   mpps_one_norm

``ctx`` selects the lattice format (PrecisionCtx.fmt); operands are
converted (exactly widened, or rounded) to it first.
"""

from __future__ import annotations

from fractions import Fraction

import numpy as np

from . import _lib
from .bigfloat import rn
from .coefficients import split_words
from .precision import FP32, DimensionError, MatBatch, PrecisionCtx


def _torch():
    import torch
    return torch


def from_numpy(words, fmt: int, device=None) -> MatBatch:
    """Host words -> MatBatch (exact).  (n, n): one fp64 matrix;
    (w, n, n): the w word planes of one matrix; (w, B, n, n): a batch."""
    torch = _torch()
    a = np.asarray(words, dtype=np.float64)
    if a.ndim == 2:
        a = a[None, None]
    elif a.ndim == 3:
        a = a[:, None]
    from .precision import FORMAT_WORDS
    w = FORMAT_WORDS[fmt]
    if a.shape[0] < w:
        a = np.concatenate([a, np.zeros((w - a.shape[0],) + a.shape[1:])], axis=0)
    elif a.shape[0] > w:
        raise DimensionError(f"{a.shape[0]} words do not fit format {fmt}")
    dt = torch.float32 if fmt == FP32 else torch.float64
    dev = device or torch.device("cuda", torch.cuda.current_device())
    return MatBatch(torch.from_numpy(np.ascontiguousarray(a)).to(dev).to(dt), fmt)


def round_to(A: MatBatch, ctx: PrecisionCtx) -> MatBatch:
    out = MatBatch.empty(ctx.fmt, A.batch, A.rows, A.cols, device=A.device)
    _lib.handle_for().convert(A, out)
    return out


def _at(A: MatBatch, fmt: int) -> MatBatch:
    if A.fmt == fmt:
        return A
    out = MatBatch.empty(fmt, A.batch, A.rows, A.cols, device=A.device)
    _lib.handle_for().convert(A, out)
    return out


def mat_mul(A: MatBatch, B: MatBatch, ctx: PrecisionCtx) -> MatBatch:
    if A.cols != B.rows or A.batch != B.batch:
        raise DimensionError(f"mat_mul: {A.shape} x {B.shape}")
    f = ctx.fmt
    C = MatBatch.empty(f, A.batch, A.rows, B.cols, device=A.device)
    from . import gemm_engine as ge
    h = _lib.handle_for()
    ge.gemm(h, ge.prepare(h, _at(A, f), 0, f), ge.prepare(h, _at(B, f), 1, f), C)
    return C


def mat_axpy(alpha, A: MatBatch, B: MatBatch, ctx: PrecisionCtx) -> MatBatch:
    if A.shape != B.shape or A.batch != B.batch:
        raise DimensionError(f"mat_axpy: {A.shape} vs {B.shape}")
    f = ctx.fmt
    C = MatBatch.empty(f, A.batch, A.rows, A.cols, device=A.device)
    words = split_words(rn(Fraction(alpha), ctx.binary_precision))
    _lib.handle_for().axpy(words, _at(A, f), _at(B, f), C)
    return C


def one_norm(A: MatBatch) -> np.ndarray:
    """Max column abs-sum of every batch member (fp64 sums of the leading
    word, deterministic order)."""
    torch = _torch()
    out = torch.empty(A.batch, dtype=torch.float64, device=A.device)
    _lib.handle_for().one_norm(A, out)
    return out.cpu().numpy()
