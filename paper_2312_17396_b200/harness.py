"""Accuracy callers of the hot path (harness.py:105-155 restated on the
device): the 2x-digit ground truth, the normwise relative error and the
mixed-vs-fixed-vs-truth comparison record.  The experiment front end around
them (gallery generators, ExperimentConfig, table/CSV runners) is out of
scope.

* ``reference_eval(X, series, ctx)`` -- harness.py:105-109: fixed-precision
  PS at twice the working digits, rounded back to the working format.  On
  the hardware lattice that is fixed PS in dd for d <= 15 and in qd for
  d <= 31; beyond that the 2x context exceeds quad-double and
  ``UnsupportedPrecisionError`` is raised.
* ``relative_error(approx, truth)`` -- harness.py:112-121: ||A - T||_1 /
  ||T||_1 with the difference formed in qd (exact for operands of <= 2
  words with overlapping exponent ranges, otherwise within 2^-210), the
  norms in fp64 as ``one_norm`` (NORM_CTX).  Per batch member.
* ``compare(X, series, ctx, m=None)`` -- harness.py:139-155 (run_compare):
  mixed and fixed evaluations against ``reference_eval``; returns the
  ComparisonRecord fields per batch member.
"""

from __future__ import annotations

from typing import Dict, List, Optional

import numpy as np

from . import _lib
from .complexmat import ComplexMatBatch, complex_input
from .precision import FP64, QD, MatBatch, PrecisionCtx, UnsupportedPrecisionError


def _torch():
    import torch
    return torch


def _matrix(x):
    """report / batch report / MatBatch / ComplexMatBatch -> (MatBatch, n_complex or None)."""
    if hasattr(x, "result") and not isinstance(x, (MatBatch, ComplexMatBatch)):
        x = x.result
    if isinstance(x, ComplexMatBatch):
        return x.emb, x.n
    if isinstance(x, MatBatch):
        return x, None
    raise TypeError(f"expected a device matrix or report, got {type(x).__name__}")


def _to_format(h, A: MatBatch, fmt: int) -> MatBatch:
    if A.fmt == fmt:
        return A
    out = MatBatch.empty(fmt, A.batch, A.rows, A.cols, device=A.device)
    h.convert(A, out)
    return out


def reference_eval(X, series, ctx: PrecisionCtx):
    """harness.py:105-109."""
    from .engine import _working_format, ps_fixed
    wide = PrecisionCtx(2 * ctx.decimal_digits)
    if wide.decimal_digits > 63:
        raise UnsupportedPrecisionError(
            f"reference_eval needs {wide.decimal_digits} digits (2x {ctx.decimal_digits}); quad-double holds 63")
    rep = ps_fixed(X, series, wide, timing=False)
    res, nc = _matrix(rep)
    out = _to_format(_lib.handle_for(), res, _working_format(ctx))
    return ComplexMatBatch(out, nc) if nc is not None else out


def _norms(h, A: MatBatch, nc: Optional[int]):
    torch = _torch()
    out = torch.empty(A.batch, dtype=torch.float64, device=A.device)
    if nc is not None:
        h.one_norm_complex(A, nc, out, 1)
    else:
        h.one_norm(A, out)
    return out


def relative_error(approx, truth) -> np.ndarray:
    """harness.py:112-121, per batch member (float64 array)."""
    h = _lib.handle_for()
    A, na = _matrix(approx)
    T, nt = _matrix(truth)
    if A.shape != T.shape or na != nt:
        raise ValueError("approx and truth must have the same shape")
    Aq, Tq = _to_format(h, A, QD), _to_format(h, T, QD)
    D = MatBatch.empty(QD, A.batch, A.rows, A.cols, device=A.device)
    h.axpy((-1.0, 0.0, 0.0, 0.0), Tq, Aq, D)           # RN_qd(A - T)
    dn = _norms(h, _to_format(h, D, FP64), na).cpu().numpy()
    tn = _norms(h, _to_format(h, T, FP64), na).cpu().numpy()
    return np.where(tn == 0, dn, dn / np.where(tn == 0, 1.0, tn))


def compare(X, series, ctx: PrecisionCtx, m: Optional[int] = None, delta: float = 10.0,
            fix_params: bool = True) -> List[Dict[str, object]]:
    """harness.py:139-155 (run_compare) for a batch: ``m`` given -> the
    Taylor exp evaluator (ps_mixed_exp), else ps_mixed_general(series)."""
    from .engine import ps_fixed, ps_mixed_exp, ps_mixed_general
    if m is not None:
        mixed = ps_mixed_exp(X, m, ctx, fix_params, delta, timing=False)
    else:
        mixed = ps_mixed_general(X, series, ctx, delta, timing=False)
    fixed = ps_fixed(X, series, ctx, timing=False)
    ref = reference_eval(X, series, ctx)
    eps_m = relative_error(mixed, ref)
    eps_f = relative_error(fixed, ref)
    reps = list(mixed) if isinstance(mixed, list) else [mixed]
    cx = complex_input(X)
    n = cx[1] if cx is not None else (X.rows if isinstance(X, MatBatch) else np.shape(X)[-1])
    out = []
    for b, rep in enumerate(reps):
        p = rep.plan
        out.append({"eps_mixed": float(eps_m[b]), "eps_fixed": float(eps_f[b]),
                    "rnu": float(p.r * n) * 10.0 ** (-ctx.decimal_digits), "savings": rep.savings,
                    "plan": p.to_dict()})
    return out
