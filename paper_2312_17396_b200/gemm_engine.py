"""GEMM engine selection for the PS pipeline.

Two sm_100a implementations of every multiword GEMM exist in
libmpps_b200.so:

* ``tc``   -- INT8 tensor cores (tcgen05.mma kind::i8) on exact digit-plane
  splittings of the operands (csrc/ozaki.cuh): fp64 (8 planes), dd (16),
  qd (31).  The operand that stays fixed across a chain (X in the power
  chain, Y in the Horner chain) is split once per evaluation.
* ``simt`` -- FP64-pipe error-free-transform GEMMs and FFMA fp32 GEMMs
  (csrc/gemm.cuh).

fp32 levels use 4 digit planes (27 bits >= 24) on the tensor cores.

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

The default is ``tc``; ``MPPS_GEMM=simt`` (environment) or
``set_engine("simt")`` selects the SIMT kernels (A/B evidence, tests).
"""

from __future__ import annotations

import os

from .precision import FP32, MatBatch

_ENGINE = os.environ.get("MPPS_GEMM", "tc").lower()
_DIGITS = os.environ.get("MPPS_DIGITS", "auto")
_MIN_K_8BIT = 0


def set_digit_bits(db) -> None:
    """Digit width policy of the tensor-core splits: 7, 8 or "auto"."""
    global _DIGITS
    if db not in (7, 8, "7", "8", "auto"):
        raise ValueError("digit bits must be 7, 8 or 'auto'")
    _DIGITS = str(db)


def digit_bits_for(h, K: int) -> int:
    """Digit width of a product with inner dimension K."""
    if _DIGITS == "7" or K > h.max_k_8bit():
        return 7
    if _DIGITS == "8":
        return 8
    return 8 if K >= _MIN_K_8BIT else 7


def set_engine(name: str) -> None:
    global _ENGINE
    if name not in ("tc", "simt"):
        raise ValueError("engine must be 'tc' or 'simt'")
    _ENGINE = name


def engine() -> str:
    return _ENGINE


def uses_tc(fmt: int) -> bool:
    return _ENGINE == "tc"


class Operand:
    """A GEMM operand prepared for one side: the MatBatch itself (SIMT) or
    its digit planes (tensor cores).  ``fmt`` is the format it was prepared
    at (for SIMT the data is converted to it)."""

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


def prepare(h, A: MatBatch, side: int, fmt: int, sel=None, exp=None, nslices=None) -> Operand:
    """Prepare A as the left (side 0) or right (side 1) operand of GEMMs at
    ``fmt``.  For the tensor-core engine the split uses the planes of the
    finest format any later use needs (the caller passes it as ``fmt``);
    a coarser level uses a prefix of the planes."""
    if uses_tc(fmt):
        # digit planes carry their own per-row/column power-of-two scales,
        # so no extra level scaling is applied (exp is ignored)
        K = A.cols if side == 0 else A.rows
        db = digit_bits_for(h, K)
        return Operand(A, h.slice(A, side, nslices or h.slices_for(fmt, db), sel, db), fmt, side)
    if A.fmt != fmt or exp is not None:
        B = MatBatch.empty(fmt, A.batch, A.rows, A.cols, device=A.device)
        h.convert(A, B, sel, exp)
        A = B
    return Operand(A, None, fmt, side)


def gemm(h, L: Operand, R: Operand, C: MatBatch, sel=None) -> None:
    """C = L R at C's format."""
    if L.slices is not None and R.slices is not None:
        h.gemm_sliced(L.slices, R.slices, h.slices_for(C.fmt, L.slices.db), C, sel)
    else:
        h.gemm(L.mat, R.mat, C, sel)


def horner(h, Y: Operand, phi: Operand, fmt_level: int, Bprev, out, sel=None, exp_y=None, exp_in=None,
           exp_out=None, nslices=None) -> None:
    """out = RN_out(2^eo (Bprev + 2^-(ey+ei) RN_level(Y phi)))."""
    if Y.slices is not None and phi.slices is not None:
        # the Y planes are unscaled (exp_y does not apply); phi keeps its
        # level scaling 2^exp_in, undone in the epilogue
        h.horner_step_sliced(Y.slices, phi.slices, nslices or h.slices_for(fmt_level, Y.slices.db), Bprev, out, sel,
                             None, exp_in, exp_out, fmt_in=fmt_level)
    else:
        h.horner_step(Y.mat, phi.mat, Bprev, out, sel, exp_y, exp_in, exp_out)
