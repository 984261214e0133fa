"""Scaling-and-squaring exp driven by the mixed-precision PS Taylor
evaluation (config 3).

The reference stops at the polynomial: degree/scaling selection and the
squaring phase are out of its scope and only the
``extra_squarings`` diagnostic exists (bounds.py:216-227).  The build rule,
as documented in SURVEY 8(d):

  * degree m = 42, s = ceil(sqrt(42)) = 7, r = 6 (Table 1's degree at 32
    digits); at ||X||_1 <= s/e the truncation term
    ||X||^43/43! e^||X|| ~ 1e-34 < 1e-31 (dd);
  * l = extra_squarings(||A||_1, s) = max(0, ceil(log2(e ||A||_1 / s)))
    (bounds.py:216-227, exact 107-bit emulation), so ||2^-l A||_1 <= s/e
    (Eq. 3.1);
  * X = 2^-l A exactly (scale_pow2, precision.py:220-224);
  * P = p_42(X) by ps_mixed_exp (per-matrix plans, heterogeneous within the
    batch), then l squarings P <- P P at the working format (dd GEMMs),
    batched over the matrices that still need one.
"""

from __future__ import annotations

from typing import List, Optional

import numpy as np

from . import _lib
from . import gemm_engine as ge
from .bounds import extra_squarings
from .engine import BatchReport, _input, ps_mixed_exp
from .planner import default_block_size
from .precision import FP64, MatBatch, PrecisionCtx, to_device_async

DEFAULT_M = 42


def _torch():
    import torch
    return torch


def scaling_of(norms: np.ndarray, m: int = DEFAULT_M) -> List[int]:
    s = default_block_size(m)
    return [extra_squarings(float(v), s) if v > 0 else 0 for v in norms]


def expm_ss(A, ctx: PrecisionCtx, m: int = DEFAULT_M, delta: float = 10.0, timing: bool = True,
            return_stage: bool = False):
    """exp(A) for an (n, n) or (B, n, n) batch.  Returns a BatchReport (or a
    single report) whose ``diagnostics['squarings']`` holds l per matrix and
    whose ``result`` is exp(A) at the working format.  ``return_stage``
    returns (report, P) with P a copy of the PS stage p_m(2^-l A) before the
    squarings (full-size parity tests check the two phases separately)."""
    torch = _torch()
    h = _lib.handle_for()
    At, Aw, single = _input(A)
    if Aw is None:
        Aw = MatBatch(At.unsqueeze(0), FP64)
    B, n = Aw.batch, Aw.rows
    if B == 0 or n == 0:      # nothing to launch: the PS stage's empty report
        rep = ps_mixed_exp(Aw, m, ctx, delta=delta, timing=timing)
        return (rep, None) if return_stage else rep
    normsA = torch.empty(B, dtype=torch.float64, device=Aw.device)
    h.one_norm(Aw, normsA)
    na = h.host_array(normsA)
    if not np.isfinite(na).all():
        raise ValueError("non-finite float")
    ells = scaling_of(na, m)
    wf = ctx.fmt if ctx.fmt != 7 else FP64
    # X = 2^-l A, exact (the widening to the working format is exact too)
    X = MatBatch.empty(wf, B, n, device=Aw.device)
    exps = to_device_async([-e for e in ells], torch.int32, Aw.device)
    h.convert(Aw, X, None, exps)
    rep = ps_mixed_exp(X, m, ctx, delta=delta, timing=timing)
    from .engine import EvaluationReport
    reps = [rep] if isinstance(rep, EvaluationReport) else list(rep)
    P = rep.result
    stage = MatBatch(P.data.clone(), P.fmt) if return_stage else None
    Q = MatBatch.empty(P.fmt, P.batch, n, device=P.device)
    sels = {}
    for t in range(1, max(ells) + 1 if ells else 1):
        members = tuple(b for b in range(B) if ells[b] >= t)
        if members not in sels:
            sels[members] = to_device_async(members, torch.int32, P.device)
    for t in range(1, max(ells) + 1 if ells else 1):
        members = tuple(b for b in range(B) if ells[b] >= t)
        sel = sels[members]
        ge.gemm(h, ge.prepare(h, P, 0, P.fmt, sel), ge.prepare(h, P, 1, P.fmt, sel), Q, sel)  # Q = P P
        h.convert(Q, P, sel)          # copy back (same format: exact)
    for b, r_ in enumerate(reps):
        r_._diag_extra = dict(r_._diag_extra or {}, squarings=int(ells[b]), degree=m,
                              norm_A=float(normsA[b]))
    return (rep, stage) if return_stage else rep
