"""Decimal matrix I/O with two guard digits (precision.py:252-341 restated):
JSON ``{"n_rows", "n_cols", "decimal_digits", "entries"}`` and CSV with a
``digits,d`` header row; every entry is ``fmt_sci(x, d + 2)`` (correctly
rounded scientific notation), complex entries as ``re{+|-}imj``, so binary
values round-trip exactly through text.

Reading rounds each decimal string to the reference's p = ceil(d log2 10)
bits (``mpfr(s, p)``, precision.py:296-307) and stores the result exactly in
the smallest hardware format that holds p bits (fp64 for d <= 15, dd for
d <= 31, qd for d <= 63), so a matrix read here carries exactly the values
the reference reads.  Writing prints the exact value of each entry (the sum
of its fp64 words).  Matrices are device ``MatBatch`` / ``ComplexMatBatch``
of batch 1 (or the ``result`` of a report); reading returns them on
``device`` (default: the current CUDA device when there is one, else CPU).
"""

from __future__ import annotations

import csv
import decimal
import io
import json
from fractions import Fraction
from typing import Optional

import numpy as np

from .bigfloat import fmt_sci, rn
from .coefficients import split_words
from .complexmat import ComplexMatBatch
from .precision import DD, FP32, FP64, QD, MatBatch, PrecisionCtx, UnsupportedPrecisionError

_DIGITS_OF_FMT = {FP32: 7, FP64: 15, DD: 31, QD: 63}
_WORDS = {FP64: 1, DD: 2, QD: 4}


def _torch():
    import torch
    return torch


def storage_format(d: int) -> int:
    """Smallest format holding the reference's p-bit values at d digits."""
    if d <= 15:
        return FP64
    if d <= 31:
        return DD
    if d <= 63:
        return QD
    raise UnsupportedPrecisionError(f"{d} digits exceed quad-double")


def _entry_values(words: np.ndarray):
    """(W, n, m) float64 words -> n x m exact Fractions."""
    W, n, m = words.shape
    out = []
    for i in range(n):
        row = []
        for j in range(m):
            row.append(sum((Fraction(float(words[w, i, j])) for w in range(W)), Fraction(0)))
        out.append(row)
    return out


def _fmt_real(x: Fraction, digits: int) -> str:
    return fmt_sci(x, digits + 2)


def _entry_to_str(re: Fraction, im: Fraction, digits: int) -> str:
    if im == 0:
        return _fmt_real(re, digits)
    im_s = _fmt_real(im, digits)
    sign = "" if im_s.startswith("-") else "+"
    return f"{_fmt_real(re, digits)}{sign}{im_s}j"


def _parse_real(s: str, p: int) -> Fraction:
    s = s.strip()
    low = s.lower()
    if low in ("nan", "inf", "+inf", "-inf"):
        raise ValueError(f"non-finite entry {s!r} cannot be stored in a hardware format")
    try:
        q = Fraction(decimal.Decimal(s))
    except decimal.InvalidOperation:
        raise ValueError(f"malformed entry: {s!r}") from None
    return rn(q, p)


def _entry_from_str(s: str, p: int):
    s = s.strip()
    if s.endswith("j"):
        body = s[:-1]
        # the sign separating real and imaginary parts (not a leading sign,
        # not an exponent sign), as precision.py:296-307
        for idx in range(len(body) - 1, 0, -1):
            ch = body[idx]
            if ch in "+-" and body[idx - 1] not in "eE":
                return _parse_real(body[:idx], p), _parse_real(body[idx:], p)
        raise ValueError(f"malformed complex entry: {s!r}")
    return _parse_real(s, p), Fraction(0)


def _parts(A):
    """(real words (W,n,m), imag words or None, default digits)."""
    if hasattr(A, "result") and not isinstance(A, (MatBatch, ComplexMatBatch)):
        A = A.result
    if isinstance(A, ComplexMatBatch):
        if A.batch != 1:
            raise ValueError("matrix I/O takes one matrix (batch 1)")
        return A.real.words_numpy()[:, 0], A.imag.words_numpy()[:, 0], _DIGITS_OF_FMT[A.fmt]
    if isinstance(A, MatBatch):
        if A.batch != 1:
            raise ValueError("matrix I/O takes one matrix (batch 1)")
        return A.words_numpy()[:, 0], None, _DIGITS_OF_FMT[A.fmt]
    arr = np.asarray(A)
    if np.iscomplexobj(arr):
        return arr.real[None].astype(np.float64), arr.imag[None].astype(np.float64), 15
    return arr[None].astype(np.float64), None, 15


def _strings(A, digits: Optional[int]):
    re_w, im_w, d0 = _parts(A)
    d = d0 if digits is None else int(digits)
    re = _entry_values(re_w)
    im = _entry_values(im_w) if im_w is not None else None
    n, m = re_w.shape[1], re_w.shape[2]
    rows = [[_entry_to_str(re[i][j], im[i][j] if im is not None else Fraction(0), d) for j in range(m)]
            for i in range(n)]
    return rows, d


def matrix_to_json(A, digits: Optional[int] = None) -> str:
    """precision.py:310-317.  ``digits``: the decimal digits the matrix was
    produced at (default: the lattice digits of its format)."""
    rows, d = _strings(A, digits)
    n = len(rows)
    m = len(rows[0]) if rows else 0
    return json.dumps({"n_rows": n, "n_cols": m, "decimal_digits": d,
                       "entries": [e for row in rows for e in row]})


def matrix_to_csv(A, digits: Optional[int] = None) -> str:
    """precision.py:330-337."""
    rows, d = _strings(A, digits)
    buf = io.StringIO()
    w = csv.writer(buf)
    w.writerow(["digits", d])
    for row in rows:
        w.writerow(row)
    return buf.getvalue()


def _build(values, d: int, device):
    """n x m (re, im) Fractions at p bits -> MatBatch / ComplexMatBatch."""
    torch = _torch()
    fmt = storage_format(d)
    W = _WORDS[fmt]
    n = len(values)
    m = len(values[0]) if n else 0
    cplx = any(im != 0 for row in values for (_, im) in row)
    if cplx and n != m:
        raise ValueError("complex matrices are held as square real embeddings")
    R = np.zeros((W, n, m))
    I = np.zeros((W, n, m)) if cplx else None
    for i in range(n):
        for j in range(m):
            re, im = values[i][j]
            R[:, i, j] = split_words(re, W)
            if cplx:
                I[:, i, j] = split_words(im, W)
    if device is None:
        device = torch.device("cuda", torch.cuda.current_device()) if torch.cuda.is_available() else "cpu"
    if not cplx:
        return MatBatch(torch.from_numpy(R[:, None]).to(device), fmt)
    E = np.zeros((W, 1, 2 * n, 2 * n))
    E[:, 0, :n, :n] = R
    E[:, 0, n:, n:] = R
    E[:, 0, n:, :n] = I
    E[:, 0, :n, n:] = -I
    return ComplexMatBatch(MatBatch(torch.from_numpy(E).to(device), fmt), n)


def values_from_json(text: str):
    """precision.py:320-327 on the host: (exact (re, im) entries at p bits, d)."""
    obj = json.loads(text)
    d = int(obj["decimal_digits"])
    p = PrecisionCtx(d).binary_precision
    nr, nc = int(obj["n_rows"]), int(obj["n_cols"])
    ent = obj["entries"]
    if len(ent) != nr * nc:
        raise ValueError("entry count mismatch")
    return [[_entry_from_str(ent[i * nc + j], p) for j in range(nc)] for i in range(nr)], d


def values_from_csv(text: str):
    """precision.py:340-346 on the host: (exact (re, im) entries at p bits, d)."""
    rows_in = [r for r in csv.reader(io.StringIO(text)) if r]
    if not rows_in or rows_in[0][0] != "digits":
        raise ValueError("missing digits header row")
    d = int(rows_in[0][1])
    p = PrecisionCtx(d).binary_precision
    values = [[_entry_from_str(s, p) for s in r] for r in rows_in[1:]]
    if any(len(r) != len(values[0]) for r in values):
        raise ValueError("ragged rows")
    return values, d


def matrix_from_json(text: str, device=None):
    """precision.py:320-327."""
    values, d = values_from_json(text)
    return _build(values, d, device)


def matrix_from_csv(text: str, device=None):
    """precision.py:340-346."""
    values, d = values_from_csv(text)
    return _build(values, d, device)
