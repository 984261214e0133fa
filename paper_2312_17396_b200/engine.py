"""Paterson-Stockmeyer evaluators on B200: the drop-in for engine.py.

Same entry points, signatures, defaults, plan/report records and errors as
pkg/src/mpps/engine.py:

    ps_fixed(X, series, ctx, with_bound=False)                 engine.py:304-345
    ps_mixed_general(X, series, ctx, delta=10., with_bound=False)  348-387
    ps_mixed_exp(X, m, ctx, fix_params=True, delta=10., with_bound=False) 390-482
    plan_only(X, series, ctx, delta=10., fix_params=True)          485-504

``X`` is an (n, n) array (numpy / torch, host or device, or a reference
``MPMatrix`` with real entries) or an (B, n, n) batch; a batch returns a
``BatchReport`` whose entries are per-matrix ``EvaluationReport`` records
(every matrix gets its own plan, exactly as if evaluated alone).

Device pipeline per batch (one host sync, for the planner's norms):

  1. convert X (fp64) -> working format (exact widening)           K4
  2. X^2..X^s by GEMMs at the working format                        K1
  3. one fused pass: B_0..B_r in index order + column abs-sums       K1b
  4. norms -> host; bit-exact planner per matrix (planner.py)
  5. matrix Horner, grouped by each matrix's level formats:
     top level K3 (B_r = b_m I) or convert B_r; then r GEMMs whose
     epilogue adds B_{j-1} and rounds into the level-(j-1) format     K2

All arithmetic runs in the sm_100a kernels of libmpps_b200.so; this module
only plans, allocates (torch caching allocator) and launches.
"""

from __future__ import annotations

import json
import math
import time
from dataclasses import dataclass, field
from fractions import Fraction
from typing import Dict, List, Optional, Sequence, Tuple

import numpy as np

from . import _lib
from . import complexmat
from . import gemm_engine as ge
from .bigfloat import MPF, exp_rn, fmt7, ln_rn, rn, to_fraction
from .bounds import BoundInputs, thm21_bound, tau_sequence
from .coefficients import (CoefficientSeries, coeff_words, eval_coeff,
                           split_words, taylor_exp_coeffs)
from .planner import (EvaluationPlan, cost_ratio, default_block_size,
                      fixed_plan, formats_of_digits, hardware_lattice,
                      matmul_counts, plan_digits_batch, plan_precisions,
                      snap_to_lattice)
from .precision import (DD, FORMAT_NAME, FP32, FP64, NORM_CTX, QD,
                        DimensionError, MatBatch, PrecisionCtx, as_fp64_batch,
                        to_device_async)

BUCKETS = ("power_formation", "norm_estimation", "mixed_horner", "coefficient_assembly")

import os as _os
#: two-pass block assembly for the mixed evaluators (MPPS_LOWP_ASSEMBLY=0: one dd pass)
_LOWP = _os.environ.get("MPPS_LOWP_ASSEMBLY", "1") != "0"
#: two powers per power-chain GEMM (MPPS_PAIRED_POWERS=0: X^{k+1} = X^k X one by one)
_PAIRED = _os.environ.get("MPPS_PAIRED_POWERS", "1") != "0"
#: K5 fused small-matrix evaluation (n <= 32, fp64 working; MPPS_SMALL=0: general pipeline)
_SMALL = _os.environ.get("MPPS_SMALL", "1") != "0"
#: mixed evaluators with an odd s >= 5 form Y = X^s at fp64 precision and at dd only for the
#: matrices whose plan keeps a Horner level at dd (MPPS_Y_LOW=0: Y always at dd)
_Y_LOW = _os.environ.get("MPPS_Y_LOW", "1") != "0"
_Y_LOW_MIN_N = 4096


def _torch():
    import torch
    return torch


class EvaluationReport:
    """engine.py:87-108.  ``result`` is a device ``MatBatch`` of batch 1.

    Batched evaluations build the per-matrix plan lazily: execution uses the
    certified batched digit rule (planner.plan_digits_batch), and the full
    ``EvaluationPlan`` (taus, roundoffs, norms) is produced by the exact
    ``plan_precisions`` on first access and checked against the executed
    digits."""

    def __init__(self, result: Optional[MatBatch], plan: Optional[EvaluationPlan] = None,
                 matmuls_by_digits: Optional[Dict[int, int]] = None, cost_ratio: Optional[float] = None,
                 savings: Optional[float] = None, timing_buckets: Optional[Dict[str, float]] = None,
                 bound: Optional[MPF] = None, diagnostics: Optional[Dict[str, object]] = None,
                 *, plan_fn=None, counts_mode: str = "mixed", executed=None, batch_view=None):
        self._result = result
        self._batch_view = batch_view   # (batch MatBatch, index) -> lazy view
        self._plan = plan
        self._plan_fn = plan_fn
        self._counts = matmuls_by_digits
        self._cr = None if cost_ratio is None else (cost_ratio, savings)
        self.timing_buckets = timing_buckets if timing_buckets is not None else {k: 0.0 for k in BUCKETS}
        self.bound = bound
        self._diag_extra = diagnostics or {}
        self._counts_mode = counts_mode
        self._executed = executed

    _cplx_n = None      # n of a complex evaluation (result is a ComplexMatBatch)

    @property
    def result(self) -> MatBatch:
        if self._result is None:
            bm, i = self._batch_view
            self._result = bm.select(i)
        if self._cplx_n is not None and not isinstance(self._result, complexmat.ComplexMatBatch):
            self._result = complexmat.ComplexMatBatch(self._result, self._cplx_n)
        return self._result

    @property
    def plan(self) -> EvaluationPlan:
        if self._plan is None:
            p = self._plan_fn()
            if self._executed is not None:
                digits, nu = self._executed
                if tuple(p.level_digits) != tuple(digits) or p.nu != nu:
                    raise RuntimeError(f"executed schedule {digits}/{nu} != exact plan "
                                       f"{p.level_digits}/{p.nu}")
            self._plan = p
        return self._plan

    @property
    def matmuls_by_digits(self) -> Dict[int, int]:
        if self._counts is None:
            p = self.plan
            d = p.d_working
            if self._counts_mode == "fixed":
                self._counts = {d: p.s - 1 + p.r} if p.r else {}
            elif self._counts_mode == "explicit" or p.nilpotent:
                self._counts = {d: p.s - 1}
            else:
                self._counts = matmul_counts(p)
        return self._counts

    @property
    def cost_ratio(self) -> float:
        if self._cr is None:
            self._cr = cost_ratio(self.plan)
        return self._cr[0]

    @property
    def savings(self) -> float:
        if self._cr is None:
            self._cr = cost_ratio(self.plan)
        return self._cr[1]

    @property
    def diagnostics(self) -> Dict[str, object]:
        p = self.plan
        lat = hardware_lattice(p.d_working)
        diag = {"level_formats": [FORMAT_NAME[f] for f in p.level_formats],
                "snapped_digits": list(snap_to_lattice(p, lat).level_digits) if p.d_working in lat else None}
        diag.update(self._diag_extra)
        return diag

    def to_json(self) -> str:
        return json.dumps({
            "plan": self.plan.to_dict(),
            "matmuls_by_digits": {str(k): v for k, v in self.matmuls_by_digits.items()},
            "cost_ratio": self.cost_ratio,
            "savings": self.savings,
            "timing_buckets": self.timing_buckets,
            "bound": None if self.bound is None else fmt7(self.bound),
            "diagnostics": self.diagnostics,
        })

    def result_numpy(self) -> np.ndarray:
        return self.result.to_numpy()[0]

    def __repr__(self):
        return f"EvaluationReport({self.result!r})"


class BatchReport(list):
    """A list of per-matrix ``EvaluationReport`` plus the batched result."""

    def __init__(self, reports, result: MatBatch, seconds: Dict[str, float]):
        super().__init__(reports)
        self.result = result
        self.seconds = seconds


# kernels index the batch with blockIdx.y / blockIdx.z (<= 65535)
_MAX_BATCH = 32768


def _chunked(fn):
    """Batches beyond the grid's y / z range run as consecutive sub-batches
    (a matrix gets the same bits in any batch); one BatchReport comes back."""
    import functools

    @functools.wraps(fn)
    def wrapper(X, *args, **kw):
        if isinstance(X, MatBatch):
            B = X.batch
        else:
            shp = getattr(X, "shape", None)
            B = shp[0] if shp is not None and len(shp) == 3 else 0
        if B <= _MAX_BATCH:
            return fn(X, *args, **kw)
        reps, parts, sec = [], [], {}
        for lo in range(0, B, _MAX_BATCH):
            hi = min(B, lo + _MAX_BATCH)
            part = MatBatch(X.data[:, lo:hi], X.fmt) if isinstance(X, MatBatch) else X[lo:hi]
            out = fn(part, *args, **kw)
            reps.extend(out)
            parts.append(out.result.data)
            for k, v in (out.seconds or {}).items():
                sec[k] = sec.get(k, 0.0) + v
        return BatchReport(reps, MatBatch(_torch().cat(parts, dim=1), out.result.fmt), sec)
    return wrapper


# ---------------------------------------------------------------- timing
class _Buckets:
    """CUDA-event timing of the reference's four buckets (engine.py:268-280);
    read once at the end, reported as fractions like the reference."""

    def __init__(self, enabled: bool):
        self.enabled = enabled
        self.marks: List[Tuple[str, object, object]] = []
        self._open = None

    def start(self, name: str):
        if not self.enabled:
            return
        torch = _torch()
        ev = torch.cuda.Event(enable_timing=True)
        ev.record()
        self._open = (name, ev)

    def stop(self):
        if not self.enabled or self._open is None:
            return
        torch = _torch()
        ev = torch.cuda.Event(enable_timing=True)
        ev.record()
        self.marks.append((self._open[0], self._open[1], ev))
        self._open = None

    def seconds(self) -> Dict[str, float]:
        out: Dict[str, float] = {}
        if not self.enabled:
            return out
        _torch().cuda.synchronize()
        for name, a, b in self.marks:
            out[name] = out.get(name, 0.0) + a.elapsed_time(b) * 1e-3
        return out


def _fractions(sec: Dict[str, float]) -> Dict[str, float]:
    total = sum(sec.values())
    if total <= 0:
        return {k: 0.0 for k in BUCKETS}
    return {k: sec.get(k, 0.0) / total for k in BUCKETS}


# ------------------------------------------------------------- internals
def _working_format(ctx: PrecisionCtx) -> int:
    f = ctx.fmt
    # fp32 working contexts (d <= 7) run at fp64: the block assembly and the
    # planner norms need at least fp64; u_hw <= 10^-d still holds.
    return FP64 if f == FP32 else f


def _exp_for(norm: float) -> int:
    """Exponent e with 2^e * norm ~ 1 (exact power-of-two level scaling)."""
    if not (norm > 0) or not math.isfinite(norm):
        return 0
    return -int(round(math.log2(norm)))


def _exps_for(norms: np.ndarray) -> np.ndarray:
    """Vectorised _exp_for."""
    v = np.asarray(norms, dtype=np.float64)
    ok = np.isfinite(v) & (v > 0)
    with np.errstate(divide="ignore", invalid="ignore"):
        e = -np.round(np.log2(np.where(ok, v, 1.0)))
    return np.where(ok, e, 0).astype(np.int32)


class _Workspace:
    """Per-format ping-pong buffers for the Horner chain."""

    def __init__(self, batch: int, n: int, device):
        self.batch, self.n, self.device = batch, n, device
        self.bufs: Dict[int, List[MatBatch]] = {}
        self.turn: Dict[int, int] = {}

    def next(self, fmt: int) -> MatBatch:
        if fmt not in self.bufs:
            self.bufs[fmt] = [MatBatch.empty(fmt, self.batch, self.n, device=self.device) for _ in range(2)]
            self.turn[fmt] = 0
        t = self.turn[fmt]
        self.turn[fmt] = 1 - t
        return self.bufs[fmt][t]


_COEFF_DEV: Dict[tuple, object] = {}


@dataclass
class _Prepared:
    """Device state after power formation and block assembly."""
    wf: int
    s: int
    r: int
    m: int
    powers: List[MatBatch]
    blocks: List[MatBatch]
    norms: np.ndarray          # (B, r+2) float64: ||B_0..B_r||, ||Y||
    coeffs: np.ndarray         # (m+1, 4) words at the working precision
    norms_dev: object = None   # the same norms on the device (level scalings)
    lowp: bool = False         # blocks are fp64 (two-pass assembly): dd ones are made per plan in _horner
    y_low: bool = False        # Y = X^s is at fp64 precision: groups with a dd level get a dd Y in _horner
    # device tensors from module-level caches (coefficients, member selections) that this state's
    # kernels read: a captured graph bakes their addresses into its kernel nodes and outlives the
    # caches' clear() -- without this reference a replay after the cache rolled over read freed
    # memory (wrong blocks and norms; found by tools/fuzz_vs_oracle.py after > 64 distinct series)
    keep: list = field(default_factory=list)


def _form_powers(h, Xt, wf: int, s: int, timer: _Buckets, x_is_working: Optional[MatBatch] = None,
                 x_fp64_ok: bool = False, y_low: bool = False):
    """X, X^2..X^s at the working format (engine.py:141-154 power chain).
    ``x_fp64_ok``: an fp64 input X under a dd chain on the tensor cores
    stays fp64 (its digit split and the block assembly read it directly:
    widening it to dd is exact and changes no value)."""
    dev = Xt.device if Xt is not None else x_is_working.device
    B = Xt.shape[0] if Xt is not None else x_is_working.batch
    n = Xt.shape[1] if Xt is not None else x_is_working.rows
    timer.start("power_formation")
    powers = [MatBatch.empty(wf, B, n, device=dev) for _ in range(s)]
    if x_is_working is not None:
        if x_is_working.fmt == wf:
            powers[0] = x_is_working
        else:
            h.convert(x_is_working, powers[0])
    elif x_fp64_ok and wf == DD and s >= 4 and _PAIRED and ge.uses_tc(wf):
        powers[0] = MatBatch(Xt.unsqueeze(0), FP64)
    else:
        h.convert(MatBatch(Xt.unsqueeze(0), FP64), powers[0])
    if s > 1 and _PAIRED and ge.uses_tc(wf) and s >= 4:
        powers = _paired_powers(h, powers[0], wf, s, y_low)
    elif s > 1:
        Xr = ge.prepare(h, powers[0], 1, wf)          # X: right operand of every step
        for k in range(1, s):       # X^{k+1} = X^k X   (engine.py:151-153)
            ge.gemm(h, ge.prepare(h, powers[k - 1], 0, wf), Xr, powers[k])
    timer.stop()
    return powers


def _y_low_ok(wf: int, s: int, lowp: bool, n: int) -> bool:
    """Y = X^s at fp64 precision first (see _paired_powers): mixed evaluators
    on the dd tensor-core chain whose last power is a single GEMM (odd s),
    for n >= 4096, where the 8-plane product runs on the 128-byte-box kernel
    at ~0.36 of the dd product's time (at n = 1024 it takes ~0.52 of it, so
    cfg3, whose plans mostly keep a dd level and then recompute Y at dd, was
    2.5 % slower with it)."""
    return (_Y_LOW and lowp and wf == DD and s >= 5 and s % 2 == 1 and _PAIRED and n >= _Y_LOW_MIN_N
            and complexmat.scope() is None)


def _paired_powers(h, X: MatBatch, wf: int, s: int, y_low: bool = False) -> List[MatBatch]:
    """X, X^2..X^s with two powers per tensor-core GEMM: the right operand
    is the column split of [X | X^2] (one slice buffer, 2n columns), so
    [X^{k+1} | X^{k+2}] = X^k [X | X^2] is one product of N = 2n.  s = 6:
    3 GEMMs and 3 row splits instead of 5 and 5 (powers are the same
    working-precision products, associated differently than the
    reference's X^{k+1} = X^k X; engine.py:151-153)."""
    B, n, dev = X.batch, X.rows, X.device
    db = ge.digit_bits_for(h, n, wf)
    S = h.slices_for(wf, db)
    SP = _lib.Slices(S, B, 2 * n, n, dev, db)
    h.slice_into(X, SP, 0)
    X2 = MatBatch.empty(wf, B, n, device=dev)
    h.gemm_sliced(h.slice(X, 0, S, None, db), SP, S, X2)        # X^2 = X X (first n slice rows)
    h.slice_into(X2, SP, n)
    out = [X, X2]
    A = X2
    while len(out) < s:
        if s - len(out) >= 2:
            Q = MatBatch.empty(wf, B, n, 2 * n, device=dev)
            h.gemm_sliced(h.slice(A, 0, S, None, db), SP, S, Q)  # [A X | A X^2]
            lo, hi = MatBatch(Q.data[..., :n], wf), MatBatch(Q.data[..., n:], wf)
            out += [lo, hi]
            A = hi
        elif y_low:
            # Y = X^s, the last (single) product, at fp64 precision: it enters
            # only the Horner products, which use a level's digit planes of it,
            # and ||Y||.  Plans that keep a level at dd get Y at dd in _horner
            # (the same product as below, so their bits are unchanged).
            S64 = h.slices_for(FP64, db)
            C = MatBatch.empty(FP64, B, n, device=dev)
            h.gemm_sliced(h.slice(A, 0, S64, None, db), SP, S64, C)
            out.append(C)
        else:
            C = MatBatch.empty(wf, B, n, device=dev)
            h.gemm_sliced(h.slice(A, 0, S, None, db), SP, S, C)
            out.append(C)
    return out


def _lowp_blocks(h, wf: int, s: int, m: int) -> int:
    """Number of blocks the fp64 pass of the two-pass assembly makes (0: not
    applicable): dd working format, real inputs, a compiled shape."""
    if wf != DD or complexmat.scope() is not None or s < 2 or not _LOWP:
        return 0
    r = m // s
    nlo = r if m % s == 0 else r + 1
    return nlo if nlo >= 2 and h.assemble_hc_n_supported(-1, s, m, nlo) else 0


def _assemble(h, powers: List[MatBatch], series: CoefficientSeries, ctx: PrecisionCtx, wf: int, s: int,
              timer: _Buckets, sync: bool = True, lowp: bool = False) -> _Prepared:
    """assemble_block for every block + one_norm (engine.py:127-138,
    467-468), then the one host sync for the planner's norms.

    ``lowp`` (mixed evaluators, dd working format): B_0 and B_1 in dd, the
    other blocks in fp64 from the powers' high words (they serve the planner's
    norms -- the reference plans from 16-digit norms -- and the B_{j-1} of
    fp32 / fp64 Horner levels, to ~2^-53 |b| |X^j|).  If a plan keeps more
    levels at dd, _horner assembles those blocks in dd (post-planner, per
    plan structure).  cfg2: 60 % less FP64 work and 15 % fewer bytes."""
    torch = _torch()
    dev = powers[0].device
    B, n = powers[0].batch, powers[0].rows
    m = series.degree
    r = m // s
    cw = coeff_words(series, ctx)
    key = (series.token, ctx.binary_precision, str(dev))
    coeffs = _COEFF_DEV.get(key)
    if coeffs is None:
        coeffs = to_device_async(cw, torch.float64, dev)
        if len(_COEFF_DEV) > 64:
            _COEFF_DEV.clear()
        _COEFF_DEV[key] = coeffs
    timer.start("coefficient_assembly")
    norms = torch.empty((B, r + 2), dtype=torch.float64, device=dev)
    nlo = _lowp_blocks(h, wf, s, m) if lowp else 0
    if nlo:
        blocks = [MatBatch.empty(DD if k < 2 else FP64, B, n, device=dev) for k in range(nlo)]
        lo_norms = torch.empty((B, nlo + 1), dtype=torch.float64, device=dev)
        h.assemble_blocks_hc_n(powers, m, cw, blocks, lo_norms)
        norms[:, :nlo] = lo_norms[:, :nlo]
        norms[:, r + 1] = lo_norms[:, nlo]
        if nlo == r:    # B_r = b_m I (not assembled): ||B_r|| = |hi(b_m)| as the one-pass kernel reports
            norms[:, r] = abs(float(cw[m][0]))
            blocks.append(MatBatch.empty(wf, 1, 1, device=dev))
        timer.stop()
        if not sync:
            return _Prepared(wf, s, r, m, powers, blocks, None, cw, norms, lowp=True, keep=[coeffs])
        timer.start("norm_estimation")
        norms_h = h.host_array(norms)
        timer.stop()
        return _Prepared(wf, s, r, m, powers, blocks, norms_h, cw, norms, lowp=True, keep=[coeffs])
    hc = h.assemble_hc_supported(wf, s, m)
    # B_r = b_m I when m mod s == 0: the K3 Horner step uses b_m itself, so
    # the constant-coefficient kernel does not store it (norm still reported)
    skip_top = hc and m % s == 0
    blocks = [MatBatch.empty(wf, B, n, device=dev) if not (skip_top and k == r) else MatBatch.empty(wf, 1, 1, device=dev)
              for k in range(r + 1)]
    if hc:
        h.assemble_blocks_hc(powers, m, cw, blocks, norms, skip_top)
    else:
        h.assemble_blocks(powers, m, coeffs, blocks, norms)
    nc = complexmat.scope()
    if nc is not None:
        # complex inputs run on their real embeddings; the planner needs the
        # complex one_norm (sum of |z|), not the embedding's abs-sums (the
        # unstored B_r = b_m I has the same norm either way)
        for k in range(r + 1 - (1 if skip_top else 0)):
            h.one_norm_complex(blocks[k], nc, norms[:, k], r + 2)
        h.one_norm_complex(powers[s - 1], nc, norms[:, r + 1], r + 2)
    timer.stop()
    if not sync:
        return _Prepared(wf, s, r, m, powers, blocks, None, cw, norms, keep=[coeffs])
    timer.start("norm_estimation")
    norms_h = h.host_array(norms)   # the one host sync of the pipeline (no copy engine: _lib.host_array)
    timer.stop()
    return _Prepared(wf, s, r, m, powers, blocks, norms_h, cw, norms, keep=[coeffs])


def _prepare(h, Xt, series: CoefficientSeries, ctx: PrecisionCtx, wf: int, s: int,
             timer: _Buckets, x_is_working: Optional[MatBatch] = None, sync: bool = True,
             lowp: bool = False) -> _Prepared:
    """eval_b0_and_power + assemble_block + one_norm (engine.py:141-154,
    127-138, 467-468) for the whole batch."""
    m = series.degree
    # fp64 X may stay unwidened when the assembly runs the constant-coefficient
    # kernels (both the mixed and the all-dd ones read an fp64 X^1)
    x64 = (wf == DD and complexmat.scope() is None and h.assemble_hc_supported(wf, s, m)
           and (not lowp or _lowp_blocks(h, wf, s, m) > 0))
    n = Xt.shape[-1] if Xt is not None else x_is_working.rows
    y_low = _y_low_ok(wf, s, lowp, n)
    powers = _form_powers(h, Xt, wf, s, timer, x_is_working, x_fp64_ok=x64, y_low=y_low)
    prep = _assemble(h, powers, series, ctx, wf, s, timer, sync, lowp)
    prep.y_low = y_low and powers[s - 1].fmt != wf
    return prep


def _dd_blocks(h, prep: _Prepared, structure) -> List[MatBatch]:
    """The blocks of a two-pass assembly for this plan structure: B_k in dd
    for B_0 and every level k the plan keeps at dd (formats are
    non-increasing, so a prefix), fp64 for the rest."""
    r, s, m, wf = prep.r, prep.s, prep.m, prep.wf
    group_list, _ = structure
    nd = 1
    for (fm, _st), _ in group_list:
        k = 1
        while k <= r and fm[k] == DD:
            k += 1
        nd = max(nd, k)
    if m % s == 0:
        nd = min(nd, r)          # B_r = b_m I is never assembled
    if nd <= len(prep.blocks) and prep.blocks[nd - 1].fmt != DD:
        B, n, dev = prep.powers[0].batch, prep.powers[0].rows, prep.powers[0].device
        if h.assemble_hc_n_supported(DD, s, m, nd):
            dd = [MatBatch.empty(DD, B, n, device=dev) for _ in range(nd)]
            h.assemble_blocks_hc_n(prep.powers, m, prep.coeffs, dd)
        else:                    # (nearly) flat plan: the one-pass dd assembly
            skip_top = m % s == 0
            dd = [MatBatch.empty(DD, B, n, device=dev) if not (skip_top and k == r)
                  else MatBatch.empty(DD, 1, 1, device=dev) for k in range(r + 1)]
            scratch = _torch().empty((B, r + 2), dtype=_torch().float64, device=dev)
            h.assemble_blocks_hc(prep.powers, m, prep.coeffs, dd, scratch, skip_top)
        return dd[:nd] + list(prep.blocks[nd:])
    return list(prep.blocks)


def _structure(prep: _Prepared, digits: np.ndarray, nil: np.ndarray):
    """Batch members grouped by (level formats, level digit planes), plus the
    nilpotent ones.  The planes of every level's tensor-core GEMM follow the
    member's own planned digits (gemm_engine.planes_for_digits), so a matrix
    gets the same bits alone or inside any batch (batch invariance)."""
    groups: Dict[Tuple, List[int]] = {}
    nil_idx = []
    tc = prep.wf in (FP64, DD) and ge.uses_tc(prep.wf)
    h = _lib.handle_for() if tc else None
    db = ge.digit_bits_for(h, prep.powers[0].rows, prep.wf) if tc else None
    memo = {}
    nil_l = np.asarray(nil, dtype=bool).tolist()
    for b, dg in enumerate(map(tuple, np.asarray(digits).tolist())):
        if nil_l[b]:
            nil_idx.append(b)
            continue
        key = memo.get(dg)
        if key is None:
            fm = (prep.wf,) + formats_of_digits(dg)
            st = tuple(ge.planes_for_digits(h, fm[j], dg[j - 1], db) for j in range(1, prep.r + 1)) if tc else ()
            key = memo[dg] = (fm, st)
        groups.setdefault(key, []).append(b)
    return tuple((key, tuple(mem)) for key, mem in groups.items()), tuple(nil_idx)


_SEL_CACHE: Dict[tuple, object] = {}


def _selection_of(members, dev):
    """Device index tensor of a member list (cached: created outside graph
    captures on first use, reused by the replays)."""
    key = (tuple(members), str(dev))
    t = _SEL_CACHE.get(key)
    if t is None:
        if len(_SEL_CACHE) > 256:
            _SEL_CACHE.clear()
        t = _SEL_CACHE[key] = to_device_async(list(members), _torch().int32, dev)
    return t


def _selections(structure, dev):
    """Device index tensors of a structure (created eagerly, outside any
    graph capture)."""
    torch = _torch()
    groups, nil_idx = structure
    whole = len(groups) == 1 and not nil_idx
    sels = {key: (None if whole else to_device_async(mem, torch.int32, dev)) for key, mem in groups}
    sels["nil"] = to_device_async(nil_idx, torch.int64, dev) if nil_idx else None
    return sels


def _horner(h, prep: _Prepared, digits: np.ndarray, nil: np.ndarray, timer: _Buckets,
            structure=None, sels=None, commute: bool = True) -> MatBatch:
    """horner_mixed (engine.py:243-252) for every matrix of the batch,
    grouped by level-format tuple (one launch per level per group).
    ``commute``: Y and the blocks are polynomials in one X (every evaluator),
    so the tensor-core levels may run phi_j Y; the public horner_mixed on
    arbitrary blocks passes False and gets Y phi_j as the reference computes."""
    torch = _torch()
    wf, s, r, m = prep.wf, prep.s, prep.r, prep.m
    Y = prep.powers[s - 1]
    B, n, dev = Y.batch, Y.rows, Y.device
    result = MatBatch.empty(wf, B, n, device=dev)
    timer.start("mixed_horner")
    if structure is None:
        structure = _structure(prep, digits, nil)
    # two-pass assembly: dd blocks exist for the longest dd prefix of any
    # group; each group takes B_k in dd only where its own level k is dd
    # (fp64 block otherwise), so a matrix gets the same bits in any batch
    dd_blocks = _dd_blocks(h, prep, structure) if prep.lowp else prep.blocks
    if sels is None:
        sels = _selections(structure, dev)
    group_list, nil_idx = structure
    groups = {fm: list(mem) for fm, mem in group_list}
    Y_dd = None
    if prep.y_low and any(DD in key[0][1:] for key, _ in group_list):
        # groups with a dd level need Y at dd: the chain's last product again
        # at the working planes (X^s = X^(s-1) X), for those members only
        dd_mem = sorted(b for key, mem in group_list if DD in key[0][1:] for b in mem)
        sel_dd = None if len(dd_mem) == B else _selection_of(dd_mem, dev)
        if sel_dd is not None:
            prep.keep.append(sel_dd)
        Y_dd = MatBatch.empty(DD, B, n, device=dev)
        ge.gemm(h, ge.prepare(h, prep.powers[s - 2], 0, wf, sel_dd, wf=wf),
                ge.prepare(h, prep.powers[0], 1, wf, sel_dd, wf=wf), Y_dd, sel_dd)
    if nil_idx:
        # p = B_0 (engine.py:378-379, 473-474)
        ii = sels["nil"]
        result.data[:, ii] = dd_blocks[0].data[:, ii]
    ws = _Workspace(B, n, dev)
    scalar_top = (m % s == 0)
    bm_words = prep.coeffs[m]
    for key, members in groups.items():
        fm, st = key
        sel = sels[key]
        blocks = [dd_blocks[k] if fm[k] == DD else prep.blocks[k] for k in range(r + 1)]
        Y = Y_dd if (Y_dd is not None and DD in fm[1:]) else prep.powers[s - 1]
        exps = exp_y = None
        if FP32 in fm:
            # exact power-of-two level scalings, computed on the device from
            # the device copy of the norms (no host round trip on the
            # critical path): e = -round(log2 ||B_j||) for fp32 levels
            if prep.norms_dev is not None:
                mask = sum(1 << j for j in range(1, r + 1) if fm[j] == FP32)
                exps = torch.empty((r + 2, B), dtype=torch.int32, device=dev)
                exp_y = torch.empty((B,), dtype=torch.int32, device=dev)
                h.level_exps(prep.norms_dev, r, mask, exps, exp_y)
            else:
                e = np.zeros((r + 1, B), dtype=np.int32)
                ey = np.zeros(B, dtype=np.int32)
                idx = np.asarray(members)
                for j in range(1, r + 1):
                    if fm[j] == FP32:
                        e[j, idx] = _exps_for(prep.norms[idx, j])
                ey[idx] = _exps_for(prep.norms[idx, r + 1])
                exps = to_device_async(e, torch.int32, dev)
                exp_y = to_device_async(ey, torch.int32, dev)

        def ex(j):
            return None if (exps is None or fm[j] != FP32) else exps[j]

        # Y as the left operand of every level: one split at the finest
        # tensor-core level format (coarser levels use a prefix of its digit
        # planes); fp32 levels get a scaled fp32 copy (FFMA GEMM)
        ys: Dict[int, ge.Operand] = {}
        tc_fmts = [f for f in set(fm[1:]) if ge.uses_tc(f)] if commute else []
        if tc_fmts:
            # tensor cores: the level products run as phi_j Y (Y and phi_j
            # commute: both are polynomials in X), so each phi_j is split by
            # rows (one pass, no column-exponent pre-pass) and Y by columns
            # once, at the finest level's planes
            ytc = ge.prepare(h, Y, 1, max(tc_fmts), sel, nslices=max(st) if st else None, wf=wf)
            for f in tc_fmts:
                ys[f] = ytc
        for f in sorted(set(fm[1:])):
            if f not in ys:
                ys[f] = ge.prepare(h, Y, 0, f, sel, exp_y if f == FP32 else None, wf=wf)
        if scalar_top:
            out = result if r - 1 == 0 else ws.next(fm[r - 1])
            h.horner_scalar_top(bm_words, fm[r], Y, blocks[r - 1], out, sel, ex(r - 1))
            phi, j0 = out, r - 1
        else:
            phi = ws.next(fm[r])
            h.convert(blocks[r], phi, sel, ex(r))
            j0 = r
        for j in range(j0, 0, -1):
            out = result if j - 1 == 0 else ws.next(fm[j - 1])
            ns = st[j - 1] if st else None       # this level's digit planes
            if ge.uses_tc(fm[j]) and commute:
                # phi_j (rows) x Y (columns): left operand first
                ge.horner(h, ge.prepare(h, phi, 0, fm[j], sel, nslices=ns, wf=wf), ys[fm[j]], fm[j], blocks[j - 1], out,
                          sel, None, ex(j), ex(j - 1), nslices=ns)
            else:
                ge.horner(h, ys[fm[j]], ge.prepare(h, phi, 1, fm[j], sel, wf=wf), fm[j], blocks[j - 1], out, sel,
                          exp_y if fm[j] == FP32 else None, ex(j), ex(j - 1))
            phi = out
    timer.stop()
    return result


def _input(X, device=None):
    """(torch fp64 (B,n,n) on device or None, working MatBatch or None, single)."""
    if isinstance(X, MatBatch):
        return None, X, X.batch == 1
    Xt, single = as_fp64_batch(X, device)
    return Xt, None, single


def _bound_for(plan: EvaluationPlan, n: int) -> MPF:
    """engine.py:283-292."""
    u = PrecisionCtx(plan.d_working).unit_roundoff
    nu = plan.nu
    precisions = [u] + [plan.level_roundoffs[i - 1] for i in range(nu, plan.r + 1)]
    inp = BoundInputs(n=n, precisions=tuple(precisions), norm_y=plan.norm_y,
                      norm_bs=tuple(plan.norm_bs[nu - 1:]), s=plan.s, r=plan.r, nu=nu)
    return thm21_bound(inp)


def _check_square(Xt, Xw):
    if Xt is not None:
        return Xt.shape[0], Xt.shape[1]
    if Xw.rows != Xw.cols:
        raise DimensionError("X must be square")
    return Xw.batch, Xw.rows


def _require_finite_norms(norms) -> None:
    """The evaluators without a planner on their path (fixed precision,
    explicit powers) reject a non-finite input the way the planner of the
    mixed ones does (one_norm of a block with a NaN / Inf entry, engine.py:
    467-472): the digit splits carry non-finite entries into the block
    norms, never into finite digits."""
    if not np.isfinite(np.asarray(norms, dtype=np.float64)).all():
        raise ValueError("non-finite float")


def _degenerate_shape(Xt, Xw, single, series, ctx, kind, delta=10.0, apply_switch=True, fix_params=True):
    """An empty batch or 0 x 0 matrices: nothing to launch.  The reference
    returns an empty result whose plan comes from zero norms
    (engine.py:390-482 on ``from_rows([])``); a batch of none returns an
    empty BatchReport.  None for every other shape."""
    B, n = _check_square(Xt, Xw)
    if B > 0 and n > 0:
        return None
    dev = Xt.device if Xt is not None else Xw.device
    if dev.type != "cuda":
        dev = "cuda"
    res = MatBatch.empty(_working_format(ctx), B, n, device=dev)
    m = series.degree
    s = default_block_size(m) if m >= 1 else 1
    r = m // s
    zeros = np.zeros(r + 2)
    if kind == "fixed":
        fns = [(lambda: fixed_plan(tuple([0.0] * (r + 1)), 0.0, ctx, s)) for _ in range(B)]
    else:
        fns = [_plan_fn(zeros, r, ctx, delta, s, apply_switch, fix_params) for _ in range(B)]
    return _reports(res, fns, None, kind, {}, False, single and B > 0)


def _reports(result: MatBatch, plan_fns, executed, counts_mode, sec, with_bound, single, extra=None):
    frac = _fractions(sec)
    n = result.rows
    reps = []
    for b, fn in enumerate(plan_fns):
        rep = EvaluationReport(result if single else None, plan_fn=fn, batch_view=(result, b),
                               counts_mode=counts_mode, timing_buckets=frac, diagnostics=extra,
                               executed=None if executed is None else executed[b])
        if with_bound:
            p = rep.plan
            if not p.nilpotent and p.r > 0 and counts_mode != "explicit":
                rep.bound = _bound_for(p, n)
        reps.append(rep)
    if single:
        return reps[0]
    return BatchReport(reps, result, sec)


def _plan_fn_list(row, r, ctx, delta, s, apply_switch, fix_params):
    """_plan_fn for a row of python floats."""
    nb, ny = tuple(row[:r + 1]), row[r + 1]
    return lambda: plan_precisions(nb, ny, ctx, delta, s=s, apply_switch=apply_switch, fix_params=fix_params)


def _plan_fn(norms_row, r, ctx, delta, s, apply_switch, fix_params):
    nb = tuple(float(x) for x in norms_row[:r + 1])
    ny = float(norms_row[r + 1])
    return lambda: plan_precisions(nb, ny, ctx, delta, s=s, apply_switch=apply_switch,
                                   fix_params=fix_params)


# ------------------------------------------------- K5: small matrices
_SMALL_OK: Dict[tuple, bool] = {}


def _small_ok(X, series: CoefficientSeries, ctx: PrecisionCtx) -> bool:
    """Whether the two-kernel small-matrix path (csrc/small_ps.cuh) runs
    this evaluation: fp64 working format, real n <= 32, s < m, coefficients
    well inside the fp64 range (the kernels keep fp32 levels as 24-bit
    roundings in fp64, whose exponent range must hold every level)."""
    if not _SMALL or complexmat.scope() is not None or _working_format(ctx) != FP64:
        return False
    shp = X.data.shape[2:] if isinstance(X, MatBatch) else getattr(X, "shape", None)
    key = (series.token, ctx.binary_precision, tuple(shp) if shp is not None else None,
           X.fmt if isinstance(X, MatBatch) else None)
    ok = _SMALL_OK.get(key)
    if ok is None:
        ok = _SMALL_OK[key] = _small_ok_uncached(X, series, ctx)
    return ok


def _small_ok_uncached(X, series: CoefficientSeries, ctx: PrecisionCtx) -> bool:
    if isinstance(X, MatBatch):
        if X.fmt != FP64 or X.rows != X.cols:
            return False
        n = X.rows
    else:
        shp = getattr(X, "shape", None)
        if shp is None or len(shp) not in (2, 3) or shp[-1] != shp[-2]:
            return False
        n = shp[-1]
    m = series.degree
    if not _lib.handle_for().small_ps_supported(n, m, FP64):
        return False
    c = np.abs(coeff_words(series, ctx)[:, 0])
    nz = c[c != 0]
    return bool(nz.size == 0 or (nz.min() > 2.0 ** -900 and nz.max() < 2.0 ** 900))


def _small_eval(X, series: CoefficientSeries, ctx: PrecisionCtx, kind: str, delta: float, apply_switch: bool,
                fix_params: bool, with_bound: bool, timing: bool):
    """K5: powers, blocks and norms in one launch, the planner's
    digit rule in certified float64 inside the library (mpps_small_ps_eval:
    no Python between the two launches), the mixed Horner chain in a second
    launch -- engine.py:141-154, 127-138, 157-215, 243-252.  When the
    certified rule declines (an e_i within 1e-8 of a digit boundary) the
    exact planner runs here and the Horner launch follows.  kind: "mixed" or
    "fixed"."""
    torch = _torch()
    Xt, Xw, single = _input(X)
    B, n = _check_square(Xt, Xw)
    Xm = Xw if Xw is not None else MatBatch(Xt.unsqueeze(0), FP64)
    h = _lib.handle_for()
    m = series.degree
    s = default_block_size(m)
    r = m // s
    d = ctx.decimal_digits
    cw = _small_coeffs(series, ctx)
    dev = Xm.device
    timer = _Buckets(timing)
    blocks = torch.empty((r + 1, B, n, n), dtype=torch.float64, device=dev)
    Y = torch.empty((B, n, n), dtype=torch.float64, device=dev)
    norms_d = torch.empty((B, r + 2), dtype=torch.float64, device=dev)
    result = MatBatch.empty(FP64, B, n, device=dev)
    timer.start("power_formation")
    norms, digits, nu, planned = h.small_ps_eval(Xm, m, s, cw, d, delta, apply_switch, kind == "fixed", blocks, Y,
                                                 norms_d, result)
    timer.stop()
    if not planned:
        digits, nu, _ = plan_digits_batch(norms[:, :r + 1], norms[:, r + 1], d, delta, apply_switch)
        fm = np.ones((B, r + 1), dtype=np.int8)
        for b, dg in enumerate(np.asarray(digits).tolist()):
            fm[b, 1:] = [0 if f == FP32 else 1 for f in formats_of_digits(dg)]
        timer.start("mixed_horner")
        h.small_ps_horner(Y, blocks, fm, m, s, float(cw[m]), result)
        timer.stop()
    if kind == "fixed":
        _require_finite_norms(norms)
        fns = [(lambda nb=tuple(float(x) for x in norms[b, :r + 1]), ny=float(norms[b, r + 1]):
                fixed_plan(nb, ny, ctx, s)) for b in range(B)]
        return _reports(result, fns, None, "fixed", timer.seconds(), with_bound, single)
    fns = [_plan_fn(norms[b], r, ctx, delta, s, apply_switch, fix_params) for b in range(B)]
    dl, nl = np.asarray(digits).tolist(), np.asarray(nu).tolist()
    executed = [(tuple(dl[b]), int(nl[b])) for b in range(B)]
    return _reports(result, fns, executed, "mixed", timer.seconds(), with_bound, single)


_SMALL_COEFFS: Dict[tuple, np.ndarray] = {}


def _small_coeffs(series: CoefficientSeries, ctx: PrecisionCtx) -> np.ndarray:
    key = (series.token, ctx.binary_precision)
    c = _SMALL_COEFFS.get(key)
    if c is None:
        if len(_SMALL_COEFFS) > 64:
            _SMALL_COEFFS.clear()
        c = _SMALL_COEFFS[key] = np.ascontiguousarray(coeff_words(series, ctx)[:, 0])   # fp64: one word each
    return c


# ------------------------------------------------------------ evaluators
def _graph_stages(Xt, series: CoefficientSeries, ctx: PrecisionCtx, wf: int, s: int, kind: str, delta: float,
                  apply_switch: bool):
    """(key, build_pre, run_post) of the graphed batched pipeline."""
    d = ctx.decimal_digits
    key = (tuple(Xt.shape), str(Xt.device if Xt.is_cuda else "host"), series.token, d, wf, s, kind, delta,
           apply_switch, ge.engine(), complexmat.scope(), _y_low_ok(wf, s, kind == "mixed", Xt.shape[-1]))

    def build_pre(xstatic, capture):
        return _prepare(_lib.handle_for(), xstatic, series, ctx, wf, s, _Buckets(False), None, sync=False,
                        lowp=(kind == "mixed"))

    def run_post(prep, norms):
        r = prep.r
        if kind == "fixed":
            _require_finite_norms(norms)
            digits = np.full((norms.shape[0], r), d, dtype=np.int64)
            nu = np.full(norms.shape[0], r + 1, dtype=np.int64)
            nil = np.zeros(norms.shape[0], dtype=bool)
        else:
            digits, nu, nil = plan_digits_batch(norms[:, :r + 1], norms[:, r + 1], d, delta, apply_switch)
        structure = _structure(prep, digits, nil)
        sels = _selections(structure, prep.norms_dev.device)

        def post_fn(p):
            return _horner(_lib.handle_for(), p, digits, nil, _Buckets(False), structure, sels)
        return structure, post_fn, (digits, nu, nil)
    return key, build_pre, run_post


def _graphed(Xt, series: CoefficientSeries, ctx: PrecisionCtx, wf: int, s: int, kind: str, delta: float,
             apply_switch: bool, timer: _Buckets):
    """The batched pipeline through cached CUDA graphs (graphs.py); returns
    (prep, digits, nu, nil, result) or None (eager path)."""
    from . import graphs
    if Xt is None or not graphs.enabled():
        return None
    key, build_pre, run_post = _graph_stages(Xt, series, ctx, wf, s, kind, delta, apply_switch)
    out = graphs.run(key, Xt, build_pre, run_post, timer)
    if out is None:
        return None
    prep, norms, result, info = out
    digits, nu, nil = info
    return prep, digits, nu, nil, result


class PendingEvaluation:
    """A batched mixed-precision evaluation whose device work before the
    planner is already enqueued (see submit_mixed_exp).  ``finish()`` waits
    for this evaluation's block norms only, plans, enqueues the Horner chain
    and returns the report exactly as the one-shot evaluator would."""

    def __init__(self, finish, pending=None):
        self._finish = finish
        self._report = None
        self._pending = pending     # graphs.Pending of a graphed evaluation

    @property
    def done_event(self):
        """CUDA event after which the result is final (graphed evaluations
        after finish(); None otherwise)."""
        return self._pending.done if self._pending is not None else None

    def finish(self):
        if self._report is None:
            self._report = self._finish()
            self._finish = None
        return self._report


def submit_mixed_general(X, series: CoefficientSeries, ctx: PrecisionCtx, delta: float = 10.0,
                         with_bound: bool = False, timing: bool = True, slot: int = 0,
                         static_result: bool = False) -> PendingEvaluation:
    """Two-phase ps_mixed_general: enqueue everything up to the block norms
    now, plan and run the Horner phase at ``finish()``.  Submitting batch c+1
    (another ``slot``) before finishing batch c keeps the GPU busy while the
    host plans; results are bit-identical to ps_mixed_general.
    ``static_result``: the report's result is the slot's graph buffer (no
    device copy; valid until the slot is submitted again)."""
    return _submit(X, series, ctx, delta, True, with_bound, timing, slot,
                   lambda: ps_mixed_general(X, series, ctx, delta, with_bound, timing), static_result)


def submit_mixed_exp(X, m: int, ctx: PrecisionCtx, delta: float = 10.0, with_bound: bool = False,
                     timing: bool = True, slot: int = 0, static_result: bool = False) -> PendingEvaluation:
    """Two-phase ps_mixed_exp (fix_params=True; see submit_mixed_general)."""
    if m < 1:
        raise ValueError("m must be >= 1")
    series = taylor_exp_coeffs(m)
    if default_block_size(m) == m:
        rep = ps_mixed_exp(X, m, ctx, True, delta, with_bound, timing)
        return PendingEvaluation(lambda: rep)
    return _submit(X, series, ctx, delta, True, with_bound, timing, slot,
                   lambda: ps_mixed_exp(X, m, ctx, True, delta, with_bound, timing), static_result)


def _submit(X, series, ctx, delta, fix_params, with_bound, timing, slot, eager, static_result=False):
    from . import graphs
    Xt, Xw, single = _input(X)
    B, n = _check_square(Xt, Xw)
    if series.degree < 1:
        raise ValueError("series degree must be >= 1")
    if B == 0 or n == 0 or Xt is None or not graphs.enabled() or _small_ok(Xt, series, ctx):
        rep = eager()
        return PendingEvaluation(lambda: rep)
    timer = _Buckets(timing)
    wf = _working_format(ctx)
    s = default_block_size(series.degree)
    key, build_pre, run_post = _graph_stages(Xt, series, ctx, wf, s, "mixed", delta, True)
    pend = graphs.submit(key, Xt, build_pre, timer, slot)
    if pend is None:
        rep = eager()
        return PendingEvaluation(lambda: rep)

    def fin():
        try:
            prep, norms, result, (digits, nu, nil) = graphs.finish(pend, run_post, clone=not static_result)
        except graphs.PlanError as pe:
            raise pe.orig
        return _graphed_reports((prep, digits, nu, nil, result), ctx, delta, True, fix_params, with_bound,
                                single, timer)
    return PendingEvaluation(fin, pend)


@complexmat.complex_aware
@_chunked
def ps_fixed(X, series: CoefficientSeries, ctx: PrecisionCtx, with_bound: bool = False,
             timing: bool = True):
    """Fixed-precision PS with s = ceil(sqrt(m)) (engine.py:304-345)."""
    Xt, Xw, single = _input(X)
    B, n = _check_square(Xt, Xw)
    if B == 0 or n == 0:
        return _degenerate_shape(Xt, Xw, single, series, ctx, "fixed")
    h = _lib.handle_for()
    timer = _Buckets(timing)
    d = ctx.decimal_digits
    m = series.degree
    wf = _working_format(ctx)
    torch = _torch()
    if m == 0:
        dev = Xt.device if Xt is not None else Xw.device
        res = MatBatch.zeros(wf, B, n, device=dev)
        w = split_words(rn(Fraction(series.coeffs[0]), ctx.binary_precision))
        idx = torch.arange(n, device=dev)
        for k in range(res.words):
            res.data[k][:, idx, idx] = w[k]
        c0 = abs(rn(Fraction(series.coeffs[0]), ctx.binary_precision))
        plan = EvaluationPlan(s=1, r=0, nu=1, d_working=d, level_digits=(), level_roundoffs=(),
                              tau_seq=(), norm_bs=(MPF(rn(c0, 54), 54),), norm_y=MPF(0, 64))
        return _reports(res, [lambda: plan] * B, None, "fixed", {}, False, single)
    s = default_block_size(m)
    if _small_ok(X, series, ctx):
        return _small_eval(X, series, ctx, "fixed", 10.0, True, True, with_bound, timing)
    g = _graphed(Xt, series, ctx, wf, s, "fixed", 10.0, True, timer) if Xw is None else None
    if g is not None:
        prep, digits, _, _, result = g
        r = prep.r
    else:
        prep = _prepare(h, Xt, series, ctx, wf, s, timer, Xw)
        _require_finite_norms(prep.norms)
        r = prep.r
        digits = np.full((B, r), d, dtype=np.int64)
        result = _horner(h, prep, digits, np.zeros(B, dtype=bool), timer)
    fns = []
    for b in range(B):
        nb = tuple(float(x) for x in prep.norms[b, :r + 1])
        ny = float(prep.norms[b, r + 1])
        fns.append((lambda nb=nb, ny=ny: fixed_plan(nb, ny, ctx, s)))
    return _reports(result, fns, None, "fixed", timer.seconds(), with_bound, single)


@complexmat.complex_aware
@_chunked
def ps_mixed_general(X, series: CoefficientSeries, ctx: PrecisionCtx, delta: float = 10.0,
                     with_bound: bool = False, timing: bool = True):
    """Mixed-precision PS for decaying coefficients (engine.py:348-387)."""
    Xt, Xw, single = _input(X)
    B, n = _check_square(Xt, Xw)
    m = series.degree
    if m < 1:
        raise ValueError("series degree must be >= 1")
    if B == 0 or n == 0:
        return _degenerate_shape(Xt, Xw, single, series, ctx, "mixed", delta)
    if _small_ok(X, series, ctx):
        return _small_eval(X, series, ctx, "mixed", delta, True, True, with_bound, timing)
    h = _lib.handle_for()
    timer = _Buckets(timing)
    wf = _working_format(ctx)
    s = default_block_size(m)
    g = _graphed(Xt, series, ctx, wf, s, "mixed", delta, True, timer) if Xw is None else None
    if g is not None:
        return _graphed_reports(g, ctx, delta, True, True, with_bound, single, timer)
    prep = _prepare(h, Xt, series, ctx, wf, s, timer, Xw, lowp=True)
    return _mixed_tail(h, prep, ctx, delta, True, True, with_bound, single, timer)


def _mixed_tail(h, prep, ctx, delta, apply_switch, fix_params, with_bound, single, timer):
    """Planner + Horner + reports of the mixed evaluators (engine.py:376-387,
    471-482)."""
    d = ctx.decimal_digits
    r, s = prep.r, prep.s
    timer.start("norm_estimation")
    digits, nu, nil = plan_digits_batch(prep.norms[:, :r + 1], prep.norms[:, r + 1], d, delta, apply_switch)
    timer.stop()
    result = _horner(h, prep, digits, nil, timer)
    B = prep.norms.shape[0]
    # built after the Horner launches so the GPU is not kept waiting
    fns = [_plan_fn(prep.norms[b], r, ctx, delta, s, apply_switch, fix_params) for b in range(B)]
    executed = [(tuple(int(x) for x in digits[b]), int(nu[b])) for b in range(B)]
    return _reports(result, fns, executed, "mixed", timer.seconds(), with_bound, single)


@complexmat.complex_aware
@_chunked
def ps_mixed_exp(X, m: int, ctx: PrecisionCtx, fix_params: bool = True, delta: float = 10.0,
                 with_bound: bool = False, timing: bool = True):
    """Mixed-precision PS for the order-m Taylor approximant of exp
    (engine.py:390-482), including the growth branch (fix_params=False and
    ||X||_1 <= s/e) and the explicit-powers degenerate case s == m."""
    Xt, Xw, single = _input(X)
    B, n = _check_square(Xt, Xw)
    if m < 1:
        raise ValueError("m must be >= 1")
    series = taylor_exp_coeffs(m)
    s = default_block_size(m)
    if B == 0 or n == 0:
        return _degenerate_shape(Xt, Xw, single, series, ctx, "mixed", delta, True, fix_params)
    if not fix_params:
        # growth decisions are per matrix (host loop over norms), so the
        # batch is split; the common fixed-s case stays batched.
        norm_x = _one_norms(Xt, Xw)
        grow = [float(v) <= s / math.e for v in norm_x]
        if any(grow):
            reps = []
            for b in range(B):
                xb = Xt[b:b + 1] if Xt is not None else None
                wb = Xw.select(b) if Xw is not None else None
                reps.append(_ps_mixed_exp_one(xb, wb, m, ctx, fix_params, delta, with_bound, timing,
                                              grow[b], float(norm_x[b])))
            if single:
                return reps[0]
            res = MatBatch(_torch().cat([r_.result.data for r_ in reps], dim=1), reps[0].result.fmt)
            return BatchReport(reps, res, {})
    if s == m:
        return _explicit_powers(Xt, Xw, m, ctx, s, series, delta, True, fix_params, single, timing)
    if _small_ok(X, series, ctx):
        return _small_eval(X, series, ctx, "mixed", delta, True, fix_params, with_bound, timing)
    h = _lib.handle_for()
    timer = _Buckets(timing)
    wf = _working_format(ctx)
    g = _graphed(Xt, series, ctx, wf, s, "mixed", delta, True, timer) if Xw is None else None
    if g is not None:
        return _graphed_reports(g, ctx, delta, True, fix_params, with_bound, single, timer)
    prep = _prepare(h, Xt, series, ctx, wf, s, timer, Xw, lowp=True)
    return _mixed_tail(h, prep, ctx, delta, True, fix_params, with_bound, single, timer)


def _graphed_reports(g, ctx, delta, apply_switch, fix_params, with_bound, single, timer):
    prep, digits, nu, nil, result = g
    r, s = prep.r, prep.s
    # one tolist() per array instead of per-element conversions: this runs
    # on the host between the Horner graph launch and the caller's next
    # step (64 reports at cfg2)
    rows = prep.norms.tolist()
    fns = [_plan_fn_list(row, r, ctx, delta, s, apply_switch, fix_params) for row in rows]
    executed = [(tuple(dg), n) for dg, n in zip(digits.tolist(), nu.tolist())]
    return _reports(result, fns, executed, "mixed", timer.seconds(), with_bound, single)


def _one_norms(Xt, Xw) -> np.ndarray:
    torch = _torch()
    h = _lib.handle_for()
    A = Xw if Xw is not None else MatBatch(Xt.unsqueeze(0), FP64)
    out = torch.empty(A.batch, dtype=torch.float64, device=A.device)
    nc = complexmat.scope()
    if nc is not None:
        h.one_norm_complex(A, nc, out, 1)
    else:
        h.one_norm(A, out)
    return out.cpu().numpy()


def _explicit_powers(Xt, Xw, m, ctx, s, series, delta, apply_switch, fix_params, single, timing):
    """engine.py:439-459: p = B_0 + b_m Y with no Horner phase."""
    h = _lib.handle_for()
    timer = _Buckets(timing)
    wf = _working_format(ctx)
    # blocks of the s == m layout: r = 1, B_0 = sum_{j<s} b_j X^j, B_1 = b_m I
    prep = _prepare(h, Xt, series, ctx, wf, s, timer, Xw)
    _require_finite_norms(prep.norms)
    Y = prep.powers[s - 1]
    res = MatBatch.empty(wf, Y.batch, Y.rows, device=Y.device)
    timer.start("coefficient_assembly")
    h.axpy(prep.coeffs[m], Y, prep.blocks[0], res)
    timer.stop()
    bm_norm = MPF(abs(rn(Fraction(series.coeffs[m]), NORM_CTX.binary_precision)), 54)

    def fn(b):
        nb0, ny = float(prep.norms[b, 0]), float(prep.norms[b, prep.r + 1])

        def make():
            p = plan_precisions((nb0, bm_norm), ny, ctx, delta, s=s, apply_switch=apply_switch,
                                fix_params=fix_params)
            return EvaluationPlan(
                s=p.s, r=p.r, nu=p.nu, d_working=p.d_working, level_digits=p.level_digits,
                level_roundoffs=p.level_roundoffs, tau_seq=p.tau_seq, norm_bs=p.norm_bs,
                norm_y=p.norm_y, delta=delta, fix_params=fix_params,
                degenerate_levels=p.degenerate_levels, nilpotent=p.nilpotent, explicit_powers=True)
        return make
    return _reports(res, [fn(b) for b in range(Y.batch)], None, "explicit", timer.seconds(), False, single)


def _ps_mixed_exp_one(Xt, Xw, m, ctx, fix_params, delta, with_bound, timing, grow, norm_x):
    """Single-matrix ps_mixed_exp with the growth branch (engine.py:417-437):
    s grows while ||X^s|| > ||B_0|| ||X||^s (54-bit NORM_CTX arithmetic)."""
    series = taylor_exp_coeffs(m)
    s = default_block_size(m)
    if not grow:
        if s == m:
            return _explicit_powers(Xt, Xw, m, ctx, s, series, delta, True, fix_params, True, timing)
        h = _lib.handle_for()
        timer = _Buckets(timing)
        prep = _prepare(h, Xt, series, ctx, _working_format(ctx), s, timer, Xw, lowp=True)
        return _mixed_tail(h, prep, ctx, delta, True, fix_params, with_bound, True, timer)
    p54 = NORM_CTX.binary_precision
    nx = rn(Fraction(norm_x), p54)
    while s < m:
        h = _lib.handle_for()
        prep = _prepare(h, Xt, series, ctx, _working_format(ctx), s, _Buckets(False), Xw)
        nb0, ny = Fraction(float(prep.norms[0, 0])), Fraction(float(prep.norms[0, prep.r + 1]))
        xs = exp_rn(rn(Fraction(s) * ln_rn(nx, p54), p54), p54) if nx > 0 else Fraction(0)
        if ny <= rn(nb0 * xs, p54):
            break
        s += 1
    if s == m:
        return _explicit_powers(Xt, Xw, m, ctx, s, series, delta, False, fix_params, True, timing)
    h = _lib.handle_for()
    timer = _Buckets(timing)
    prep = _prepare(h, Xt, series, ctx, _working_format(ctx), s, timer, Xw, lowp=True)
    return _mixed_tail(h, prep, ctx, delta, False, fix_params, with_bound, True, timer)


@complexmat.complex_aware
def ps_mixed_pade(X, k: int, ctx: PrecisionCtx, delta: float = 10.0, with_bound: bool = False,
                  timing: bool = True):
    """Numerator and denominator of the diagonal [k/k] Pade approximant of
    exp, each by ps_mixed_general (engine.py:348-387) with its own plan
    (config 4), sharing one power chain: both series have degree k, so both
    use s = ceil(sqrt(k)) and the reference forms identical powers X^2..X^s
    for the two calls -- forming them once is exact.  Returns (num, den)."""
    from .coefficients import pade_exp_coeffs
    Xt, Xw, single = _input(X)
    B, n = _check_square(Xt, Xw)
    if k < 1:
        raise ValueError("series degree must be >= 1")
    num, den = pade_exp_coeffs(k, k)
    if _small_ok(X, num, ctx):      # K5: two launches per polynomial, nothing to share
        return (ps_mixed_general(X, num, ctx, delta, with_bound, timing),
                ps_mixed_general(X, den, ctx, delta, with_bound, timing))
    h = _lib.handle_for()
    timer = _Buckets(timing)
    wf = _working_format(ctx)
    s = default_block_size(k)
    powers = _form_powers(h, Xt, wf, s, timer, Xw)
    out = []
    for series in (num, den):
        prep = _assemble(h, powers, series, ctx, wf, s, timer, lowp=True)
        out.append(_mixed_tail(h, prep, ctx, delta, True, True, with_bound, single, timer))
    return tuple(out)


@complexmat.complex_aware
def plan_only(X, series: CoefficientSeries, ctx: PrecisionCtx, delta: float = 10.0,
              fix_params: bool = True):
    """Planner only (engine.py:485-504).  The reference forms powers and
    blocks at the 16-digit NORM_CTX; the B200 build forms them in fp64 (the
    nearest lattice format; the planner consumes orders of magnitude)."""
    m = series.degree
    if m < 1:
        raise ValueError("series degree must be >= 1")
    Xt, Xw, single = _input(X)
    B, n = _check_square(Xt, Xw)
    s = default_block_size(m)
    h = _lib.handle_for()
    scaled, sig = _fp64_range_series(series, s)
    prep = _prepare(h, Xt, scaled, NORM_CTX, FP64, s, _Buckets(False), Xw)
    r = prep.r
    if sig is None:
        nbs = [prep.norms[b, :r + 1] for b in range(B)]
    else:   # undo the exact per-block 2^sigma_i scalings on the norms
        nbs = [[Fraction(float(prep.norms[b, i])) * Fraction(2) ** -sig[i] for i in range(r + 1)]
               for b in range(B)]
    plans = [plan_precisions(nbs[b], prep.norms[b, r + 1], ctx, delta, s=s,
                             apply_switch=True, fix_params=fix_params) for b in range(B)]
    return plans[0] if single else plans


def _fp64_range_series(series: CoefficientSeries, s: int):
    """(series, None) when every RN_54 coefficient is comfortably inside the
    fp64 exponent range; otherwise (scaled series, sigma) with block i's
    coefficients multiplied by 2^sigma_i so that its largest |b_k| is in
    [1, 2).  The reference's MPFR exponents are unbounded (e.g. 1/182! for
    Table 1's d = 256 row is below the fp64 range); power-of-two scaling
    commutes exactly with RN_54 and with the block assembly, so
    ||B_i|| = 2^-sigma_i ||B'_i|| exactly (barring fp64 range limits of the
    scaled blocks themselves)."""
    nz = [abs(Fraction(c)) for c in series.coeffs if c != 0]
    if not nz or (min(nz) > Fraction(2) ** -900 and max(nz) < Fraction(2) ** 900):
        return series, None
    m = series.degree
    r = m // s
    sig = []
    for i in range(r + 1):
        hi = m if i == r else s * i + s - 1
        blk = [abs(Fraction(c)) for c in series.coeffs[s * i:hi + 1] if c != 0]
        if not blk:
            sig.append(0)
            continue
        big = max(blk)
        sig.append(-(big.numerator.bit_length() - big.denominator.bit_length()))
    coeffs = tuple(Fraction(c) * Fraction(2) ** sig[min(k // s, r)] for k, c in enumerate(series.coeffs))
    return CoefficientSeries(coeffs, series.family, series.variable_note), sig


@complexmat.complex_aware
def cos_argument(X, ctx: PrecisionCtx) -> MatBatch:
    """harness.py:100-101: the cosine polynomial variable Z = fl(X X) at the
    working precision (formed on device, returned as a working-format batch
    ready for ps_mixed_general)."""
    Xt, Xw, _ = _input(X)
    wf = _working_format(ctx)
    h = _lib.handle_for()
    if Xw is None:
        Xw = MatBatch(Xt.unsqueeze(0), FP64)
    Xk = Xw
    if Xw.fmt != wf:
        Xk = MatBatch.empty(wf, Xw.batch, Xw.rows, device=Xw.device)
        h.convert(Xw, Xk)
    Z = MatBatch.empty(wf, Xk.batch, Xk.rows, device=Xk.device)
    ge.gemm(h, ge.prepare(h, Xk, 0, wf), ge.prepare(h, Xk, 1, wf), Z)
    return Z


def horner_mixed(Bs: Sequence[MatBatch], Y: MatBatch, plan: EvaluationPlan) -> MatBatch:
    """engine.py:243-252 on device blocks: phi = B_r; phi = RN_{j-1}(B_{j-1}
    + RN_j(Y phi)), j = r..1.  Bs and Y at the working format."""
    if len(Bs) != plan.r + 1:
        raise ValueError("need r+1 coefficient blocks")
    if plan.r == 0:
        return Bs[0]
    h = _lib.handle_for()
    norms = np.array([[float(b) for b in plan.norm_bs] + [float(plan.norm_y)]] * Y.batch)
    m = plan.r * plan.s + 1       # m mod s != 0: B_r is a general block here
    prep = _Prepared(Y.fmt, plan.s, plan.r, m, [Y] * plan.s, list(Bs), norms, np.zeros((m + 1, 4)))
    digits = np.array([plan.level_digits] * Y.batch, dtype=np.int64)
    return _horner(h, prep, digits, np.zeros(Y.batch, dtype=bool), _Buckets(False), commute=False)
