"""Precision contexts, the B200 format lattice and device matrix batches.

Mirrors the reference's precision core (pkg/src/mpps/precision.py):
``PrecisionCtx`` (precision.py:29-57) with the same digit -> bit map,
``NORM_CTX``/``BOUND_CTX`` (72, 75) and ``DimensionError`` (25-26).

Where the reference rounds every scalar through an MPFR context of
``ceil(d*log2 10)`` bits, the B200 build executes each context on the
smallest hardware format whose significand is at least that wide
(SURVEY.md section 0, fact 2):

    digits <= 7  -> fp32 (24 bits)      digits <= 15 -> fp64 (53 bits)
    digits <= 31 -> dd   (106 bits)     digits <= 63 -> qd   (212 bits)

``MatBatch`` is the device container: a torch tensor of shape
(words, batch, rows, cols) holding the word planes of a batch of row-major
matrices (SoA), tagged with its lattice format.  It is the device analogue of
``MPMatrix`` (precision.py:89-126).
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from typing import Optional, Sequence

import numpy as np

from .bigfloat import MPF, exp10_rn

FP32, FP64, DD, QD = 7, 15, 31, 63
LATTICE = (FP32, FP64, DD, QD)
FORMAT_BITS = {FP32: 24, FP64: 53, DD: 106, QD: 212}
FORMAT_WORDS = {FP32: 1, FP64: 1, DD: 2, QD: 4}
FORMAT_NAME = {FP32: "fp32", FP64: "fp64", DD: "dd", QD: "qd"}


class DimensionError(ValueError):
    """Operand shapes are incompatible (precision.py:25-26)."""


class UnsupportedPrecisionError(ValueError):
    """A context wider than the widest B200 format (qd, 63 digits)."""


@dataclass(frozen=True)
class PrecisionCtx:
    """A working precision in decimal digits (precision.py:29-57).

    ``binary_precision`` = ceil(d * log2 10) as in the reference;
    ``unit_roundoff`` = 10^-d (an ``MPF`` at 64 bits, like the reference's
    ``_pow10``); ``fmt`` is the lattice format that executes it."""

    decimal_digits: int

    def __post_init__(self):
        if self.decimal_digits < 1:
            raise ValueError("decimal_digits must be >= 1")

    @property
    def binary_precision(self) -> int:
        return math.ceil(self.decimal_digits * math.log2(10))

    @property
    def unit_roundoff(self) -> MPF:
        return MPF(exp10_rn(-self.decimal_digits, 64), 64)

    @property
    def fmt(self) -> int:
        return format_for_digits(self.decimal_digits)

    def __repr__(self):
        return f"PrecisionCtx(d={self.decimal_digits})"


#: Norm context of the reference (16 digits, 54 bits; precision.py:72).
NORM_CTX = PrecisionCtx(16)
#: Bound-evaluation context (32 digits, 107 bits; precision.py:75).
BOUND_CTX = PrecisionCtx(32)


def format_for_digits(d: int) -> int:
    """Smallest lattice format whose significand holds ceil(d*log2 10) bits."""
    bits = math.ceil(d * math.log2(10))
    for f in LATTICE:
        if bits <= FORMAT_BITS[f]:
            return f
    raise UnsupportedPrecisionError(
        f"{d} digits ({bits} bits) exceed the widest B200 format (qd, 212 bits)")


def _torch():
    import torch
    return torch


class MatBatch:
    """A batch of real square-or-rectangular matrices on one CUDA device,
    stored as word planes of one lattice format.

    data: torch tensor (words, batch, rows, cols), float32 for fp32 and
    float64 otherwise, contiguous."""

    __slots__ = ("data", "fmt")

    def __init__(self, data, fmt: int):
        if fmt not in LATTICE:
            raise UnsupportedPrecisionError(f"unknown format {fmt}")
        torch = _torch()
        want = torch.float32 if fmt == FP32 else torch.float64
        if data.dim() != 4 or data.shape[0] != FORMAT_WORDS[fmt] or data.dtype != want:
            raise DimensionError(
                f"MatBatch({FORMAT_NAME[fmt]}) needs a ({FORMAT_WORDS[fmt]}, B, R, C) "
                f"{want} tensor, got {tuple(data.shape)} {data.dtype}")
        if data.stride(3) != 1 or data.stride(2) < data.shape[3]:
            data = data.contiguous()
        self.data = data
        self.fmt = fmt

    @classmethod
    def empty(cls, fmt: int, batch: int, rows: int, cols: Optional[int] = None,
              device=None) -> "MatBatch":
        torch = _torch()
        cols = rows if cols is None else cols
        dt = torch.float32 if fmt == FP32 else torch.float64
        return cls(torch.empty((FORMAT_WORDS[fmt], batch, rows, cols), dtype=dt,
                               device=device), fmt)

    @classmethod
    def zeros(cls, fmt: int, batch: int, rows: int, cols: Optional[int] = None,
              device=None) -> "MatBatch":
        m = cls.empty(fmt, batch, rows, cols, device)
        m.data.zero_()
        return m

    @property
    def batch(self) -> int:
        return self.data.shape[1]

    @property
    def rows(self) -> int:
        return self.data.shape[2]

    @property
    def cols(self) -> int:
        return self.data.shape[3]

    @property
    def shape(self):
        return (self.rows, self.cols)

    @property
    def words(self) -> int:
        return self.data.shape[0]

    @property
    def device(self):
        return self.data.device

    def select(self, idx: int) -> "MatBatch":
        """Batch member idx as a batch-1 view (no copy; the C-ABI takes the
        plane and batch strides explicitly)."""
        return MatBatch(self.data[:, idx:idx + 1], self.fmt)

    def words_numpy(self) -> np.ndarray:
        """(words, batch, rows, cols) float64 copy on the host."""
        return self.data.detach().to("cpu", torch_float64()).numpy()

    def to_numpy(self) -> np.ndarray:
        """Round-to-nearest fp64 value of every entry, (batch, rows, cols)."""
        w = self.data.detach().double()
        if self.words > 1:
            # words are non-overlapping and decreasing: the fp64 rounding of
            # the sum is the rounded sum of the leading two (exactness of the
            # tail is irrelevant at 2^-53)
            v = w[0] + w[1]
        else:
            v = w[0]
        return v.cpu().numpy()

    def __repr__(self):
        return (f"MatBatch({FORMAT_NAME[self.fmt]}, batch={self.batch}, "
                f"{self.rows}x{self.cols}, {self.device})")


def to_device_async(values, dtype, device):
    """Small host array -> device without stalling the stream: staged in
    (cached) pinned memory and copied with non_blocking=True, so the launch
    queue is not drained (a pageable torch.tensor(..., device=cuda) copy
    synchronises the stream)."""
    torch = _torch()
    a = np.asarray(values)
    if isinstance(a, np.ndarray) and not a.flags.writeable:
        a = a.copy()
    t = torch.as_tensor(a, dtype=dtype)
    if t.device.type != "cpu":
        return t.to(device)
    return t.pin_memory().to(device, non_blocking=True)


def torch_float64():
    return _torch().float64


def as_fp64_batch(X, device=None):
    """Accept an (n,n) / (B,n,n) numpy array or torch tensor (any device) or
    a MatBatch; return (torch float64 tensor (B,n,n) on the CUDA device,
    was_single)."""
    torch = _torch()
    if isinstance(X, MatBatch):
        raise TypeError("as_fp64_batch takes raw arrays")
    if isinstance(X, np.ndarray):
        t = torch.from_numpy(np.ascontiguousarray(X, dtype=np.float64))
    elif isinstance(X, torch.Tensor):
        t = X.to(torch.float64)
    elif hasattr(X, "rows") and hasattr(X, "n_rows"):
        t = torch.tensor(mpmatrix_to_float(X), dtype=torch.float64)
    else:
        t = torch.as_tensor(np.asarray(X, dtype=np.float64))
    single = t.dim() == 2
    if single:
        t = t.unsqueeze(0)
    if t.dim() != 3:
        raise DimensionError(f"expected (n,n) or (B,n,n), got {tuple(t.shape)}")
    if t.shape[1] != t.shape[2]:
        raise DimensionError("X must be square")
    dev = device if device is not None else (t.device if t.is_cuda else torch.device("cuda", torch.cuda.current_device()))
    if t.device != dev:
        if t.device.type == "cpu" and not t.is_pinned():
            t = t.pin_memory()
        t = t.to(dev, non_blocking=True)
    return t.contiguous(), single


def mpmatrix_to_float(A) -> np.ndarray:
    """Real fp64 values of a reference ``MPMatrix`` (complex entries with a
    zero imaginary part); matrices with imaginary parts are routed to the
    complex path (complexmat.py) by the entry points before reaching here."""
    out = np.empty((A.n_rows, A.n_cols))
    for i, row in enumerate(A.rows):
        for j, e in enumerate(row):
            im = getattr(e, "imag", 0)
            if float(im) != 0.0:
                raise NotImplementedError("complex matrices are not supported on the B200 path")
            out[i, j] = float(getattr(e, "real", e))
    return out
