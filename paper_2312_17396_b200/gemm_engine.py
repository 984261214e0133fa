"""The GEMMs of the PS pipeline: every product (power chain, Horner levels,
squarings, SUMMA blocks, the operator-level mat_mul) runs on the INT8
tensor cores (tcgen05.mma kind::i8) on exact digit-plane splittings of the
operands (csrc/ozaki.cuh): fp32 (4 planes), fp64 (8), dd (14 / 16), qd
(28 / 31).  The operand that stays fixed across a chain (X in the power
chain, Y in the Horner chain) is split once per evaluation.  (Round 1 also
kept a SIMT DFMA engine behind MPPS_GEMM=simt; it was retired in round 2.)

Digit width: products with inner dimension K <= 4800 split into 8-bit
digits -- dd in 14 planes (110 bits) instead of 16 7-bit ones (111 bits):
105 plane pairs instead of 136 and 12.5 % fewer plane bytes (GEMM -7..-9 %
at n = 256..2048); qd in 28 instead of 31 (GEMM -18 % at n = 2048).  fp32 /
fp64 / dd operands are split into 8-bit digits by exact fixed-point integer
arithmetic (carry-free bytes, as cheap as the 7-bit FP64 split); qd keeps a
floating-point split with a bottom-up carry pass.  Above K = 4800 the int32
diagonal accumulators of qd's 28 planes could overflow, so larger K keeps
7-bit digits.  Both operands of a product share K, hence the width.
``MPPS_DIGITS=7`` forces 7-bit digits everywhere.
"""

from __future__ import annotations

import os

from .precision import FP32, MatBatch

_DIGITS = os.environ.get("MPPS_DIGITS", "auto")
_MIN_K_8BIT = 0


def set_digit_bits(db) -> None:
    """Digit width policy of the tensor-core splits: 7, 8 or "auto"."""
    global _DIGITS
    if db not in (7, 8, "7", "8", "auto"):
        raise ValueError("digit bits must be 7, 8 or 'auto'")
    _DIGITS = str(db)


def digit_bits_for(h, K: int, fmt: int = 63) -> int:
    """Digit width of the products of an evaluation at working format
    ``fmt`` with inner dimension K: 8-bit while fmt's full plane count keeps
    the int32 diagonal accumulators exact at K (dd up to K = 10070, qd up to
    4851; mpps_oz_max_k), 7-bit above.  Every split of one evaluation must
    pass the same (K, fmt) -- the working format, also for the coarser
    levels' operands -- so both operands of every product share the width.
    The default fmt (qd) is the conservative bound for any format."""
    if _DIGITS == "7" or K > h.max_k(fmt, 8):
        return 7
    if _DIGITS == "8":
        return 8
    return 8 if K >= _MIN_K_8BIT else 7


def engine() -> str:
    return "tc"


def uses_tc(fmt: int) -> bool:
    return True


class Operand:
    """A GEMM operand prepared for one side: its digit planes (``slices``)
    plus the source matrix; ``fmt`` is the format it was prepared at.  The
    host test double of the SUMMA driver (tests/_cpu_ops.py) builds
    Operands without planes."""

    __slots__ = ("mat", "slices", "fmt", "side")

    def __init__(self, mat, slices, fmt, side):
        self.mat, self.slices, self.fmt, self.side = mat, slices, fmt, side


#: plane counts with an 8-bit-digit kernel set (csrc: 2, 3, 5, 6, 10, 12
#: exist for the Horner chain's column operand only)
_PLANES_8 = (2, 3, 4, 5, 6, 8, 10, 12, 14)
_PER_LEVEL = os.environ.get("MPPS_LEVEL_PLANES", "1") != "0"


def planes_for_digits(h, fmt: int, digits: int, db: int) -> int:
    """Digit planes for a Horner level planned at ``digits`` decimal digits
    (engine.py:184-215) stored in ``fmt``: the level's GEMM needs the
    reference's p = ceil(d log2 10) bits (its mat_mul runs at ctx_j,
    engine.py:249-251), not the full storage format.  8-bit planes carry
    6 + 8 (S-1) bits; S is the smallest compiled count with >= p + 4 bits,
    capped at the format's own count (the snapped-lattice kernels)."""
    full = h.slices_for(fmt, db)
    if db != 8 or not _PER_LEVEL or fmt not in (7, 15, 31):
        return full
    import math
    p = math.ceil(digits * math.log2(10))
    for S in _PLANES_8:
        if 6 + 8 * (S - 1) >= p + 4:
            return min(S, full)
    return full


def prepare(h, A: MatBatch, side: int, fmt: int, sel=None, exp=None, nslices=None, wf=None) -> Operand:
    """Prepare A as the left (side 0) or right (side 1) operand of GEMMs at
    ``fmt``: its digit planes at the finest format any later use needs (the
    caller passes it as ``fmt``); a coarser level uses a prefix of the
    planes.  The planes carry their own per-row/column power-of-two scales,
    so no extra level scaling applies (``exp`` is accepted and ignored).
    ``wf``: the evaluation's working format, which fixes the digit width
    (digit_bits_for); default ``fmt``."""
    K = A.cols if side == 0 else A.rows
    db = digit_bits_for(h, K, wf if wf is not None else fmt)
    return Operand(A, h.slice(A, side, nslices or h.slices_for(fmt, db), sel, db), fmt, side)


def gemm(h, L: Operand, R: Operand, C: MatBatch, sel=None) -> None:
    """C = L R at C's format on the tensor cores."""
    h.gemm_sliced(L.slices, R.slices, h.slices_for(C.fmt, L.slices.db), C, sel)


def horner(h, Y: Operand, phi: Operand, fmt_level: int, Bprev, out, sel=None, exp_y=None, exp_in=None,
           exp_out=None, nslices=None) -> None:
    """out = RN_out(2^eo (Bprev + 2^-ei RN_level(Y phi))): the Y planes are
    unscaled (exp_y does not apply); phi keeps its level scaling 2^exp_in,
    undone in the epilogue."""
    h.horner_step_sliced(Y.slices, phi.slices, nslices or h.slices_for(fmt_level, Y.slices.db), Bprev, out, sel,
                         None, exp_in, exp_out, fmt_in=fmt_level)
