"""TEST INFRASTRUCTURE ONLY: the CPU oracle of the mixed-precision
Paterson-Stockmeyer hot path.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its
``cpu_baseline`` and ``--impl reference`` legs) may import this package, and
only as the checker or the timed CPU baseline -- never as the product.

``libmpps_oracle.so`` (mpfr_oracle.c) restates the reference's MPFR
arithmetic op for op (pkg/src/mpps/precision.py:160-249, engine.py:118-252);
this module composes it into the "oracle at hardware precisions" of
SURVEY.md 8(c):

  1. eval_b0_and_power + assemble_block + one_norm at the working digits;
  2. plan_precisions (the C MPFR restatement of engine.py:184-215, with the
     tau/roundoff fields left to the product planner, which the tests check
     separately);
  3. snap_to_lattice(plan, {7,15,31,63} & [1, d_w])  (engine.py:218-240);
  4. horner_mixed at the snapped digits' bit counts (engine.py:243-252).

Parity pins: the oracle is checked against the reference itself (run in the
build container under a ctypes gmpy2 shim, oracle/gmpy2_shim) through the
committed fixtures in tests/golden/ and against the reference's own
known-answer tests (tests/test_oracle_golden.py).
"""

from __future__ import annotations

import ctypes
import math
import os
import subprocess
from fractions import Fraction
from typing import List, Optional, Sequence

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "_build", "libmpps_oracle.so")
LATTICE = (7, 15, 31, 63)


def bits_of(d: int) -> int:
    """precision.py:44-46."""
    return math.ceil(d * math.log2(10))


def build(force: bool = False) -> str:
    if force or not os.path.exists(LIB):
        subprocess.check_call(["make", "-s", "-C", HERE])
    return LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB):
            build()
        L = ctypes.CDLL(LIB)
        P = ctypes.POINTER
        dp = P(ctypes.c_double)
        L.orc_new.restype = ctypes.c_void_p
        L.orc_new.argtypes = [ctypes.c_int]
        L.orc_free.argtypes = [ctypes.c_void_p]
        L.orc_prepare.argtypes = [ctypes.c_void_p, dp, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                  ctypes.c_long, P(ctypes.c_char_p), P(ctypes.c_char_p), dp]
        L.orc_horner.argtypes = [ctypes.c_void_p, P(ctypes.c_long)]
        L.orc_result_words.argtypes = [ctypes.c_void_p, dp, ctypes.c_int]
        L.orc_matrix_words.argtypes = [ctypes.c_void_p, ctypes.c_int, dp]
        L.orc_compare.argtypes = [ctypes.c_void_p, dp, ctypes.c_int, dp, dp]
        L.orc_matmul.argtypes = [ctypes.c_int, dp, ctypes.c_int, dp, ctypes.c_int, ctypes.c_long, dp]
        L.orc_result_from_block.argtypes = [ctypes.c_void_p, ctypes.c_int]
        L.orc_poly_cols.argtypes = [ctypes.c_int, dp, ctypes.c_int, ctypes.c_int, P(ctypes.c_char_p),
                                    P(ctypes.c_char_p), ctypes.c_long, ctypes.c_int, P(ctypes.c_int), ctypes.c_int, dp]
        L.orc_matpow_cols.argtypes = [ctypes.c_int, dp, ctypes.c_int, ctypes.c_int, ctypes.c_long, P(ctypes.c_int),
                                      ctypes.c_int, dp]
        L.orc_plan.argtypes = [dp, dp, ctypes.c_int, ctypes.c_int, ctypes.c_double, ctypes.c_int,
                               P(ctypes.c_int), P(ctypes.c_int), dp]
        _lib = L
    return _lib


def _dp(a: np.ndarray):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def _words(A: np.ndarray) -> np.ndarray:
    """(w, n, n) or (n, n) float64 -> contiguous (w, n, n)."""
    A = np.asarray(A, dtype=np.float64)
    if A.ndim == 2:
        A = A[None]
    return np.ascontiguousarray(A)


def split2(v: Fraction):
    hi = float(v)
    return hi, float(v - Fraction(hi))


class OraclePS:
    """One matrix through the C restatement of the reference hot path."""

    def __init__(self, n: int):
        self.n = n
        self.h = lib().orc_new(n)
        self.r = None
        self.s = None

    def __del__(self):
        try:
            lib().orc_free(self.h)
        except Exception:
            pass

    def prepare(self, X_words: np.ndarray, coeffs: Sequence[Fraction], s: int, wbits: int) -> np.ndarray:
        """Powers, blocks (engine.py:127-154) and the 54-bit norms as an
        (r+2, 2) array of exact (hi, lo) word pairs."""
        Xw = _words(X_words)
        m = len(coeffs) - 1
        r = m // s
        nums = (ctypes.c_char_p * (m + 1))(*[str(Fraction(c).numerator).encode() for c in coeffs])
        dens = (ctypes.c_char_p * (m + 1))(*[str(Fraction(c).denominator).encode() for c in coeffs])
        norms = np.zeros((r + 2, 2))
        rc = lib().orc_prepare(self.h, _dp(Xw), Xw.shape[0], m, s, wbits, nums, dens, _dp(norms))
        if rc:
            raise ValueError("oracle prepare failed")
        self.r, self.s, self.m = r, s, m
        return norms

    def horner(self, level_bits: Sequence[int]):
        arr = (ctypes.c_long * len(level_bits))(*level_bits)
        if lib().orc_horner(self.h, arr):
            raise RuntimeError("oracle horner before prepare")

    def result_words(self, nw: int = 4) -> np.ndarray:
        out = np.zeros((nw, self.n, self.n))
        lib().orc_result_words(self.h, _dp(out), nw)
        return out

    def matrix_words(self, which: int) -> np.ndarray:
        out = np.zeros((4, self.n, self.n))
        if lib().orc_matrix_words(self.h, which, _dp(out)):
            raise IndexError(which)
        return out

    def compare(self, gpu_words: np.ndarray):
        """(||G - R||_1, ||R||_1) with the difference taken at 1024 bits."""
        g = _words(gpu_words)
        diff, refn = ctypes.c_double(), ctypes.c_double()
        lib().orc_compare(self.h, _dp(g), g.shape[0], ctypes.byref(diff), ctypes.byref(refn))
        return diff.value, refn.value


def plan_digits(norms2: np.ndarray, d: int, delta: float = 10.0, apply_switch: bool = True):
    """C MPFR restatement of the plan_precisions digit rule.
    norms2: (r+2, 2) exact word pairs (blocks then Y).  Returns
    (digits, nu, nilpotent, e_values)."""
    n2 = np.ascontiguousarray(norms2, dtype=np.float64)
    r = n2.shape[0] - 2
    digits = (ctypes.c_int * max(r, 1))()
    nu = ctypes.c_int()
    e = np.zeros(max(r, 1))
    rc = lib().orc_plan(_dp(n2[:r + 1].copy()), _dp(n2[r + 1].copy()), r, d, delta, int(apply_switch),
                        digits, ctypes.byref(nu), _dp(e))
    return tuple(digits[i] for i in range(r)), nu.value, rc == 1, e[:r]


def snap(digits: Sequence[int], d_w: int) -> tuple:
    lat = [x for x in LATTICE if x <= d_w]
    return tuple(min(x for x in lat if x >= di) for di in digits)


def matmul(A_words: np.ndarray, B_words: np.ndarray, bits: int) -> np.ndarray:
    """mat_mul (precision.py:160-184) at `bits`; returns (4, n, n) words."""
    A, B = _words(A_words), _words(B_words)
    n = A.shape[1]
    C = np.zeros((4, n, n))
    lib().orc_matmul(n, _dp(A), A.shape[0], _dp(B), B.shape[0], bits, _dp(C))
    return C


class OracleResult:
    def __init__(self, ps: OraclePS, norms2, digits, nu, nil, snapped, level_bits):
        self.ps, self.norms2, self.digits, self.nu = ps, norms2, digits, nu
        self.nilpotent, self.snapped, self.level_bits = nil, snapped, level_bits

    @property
    def norms(self) -> np.ndarray:
        return self.norms2[:, 0] + self.norms2[:, 1]

    def compare(self, gpu_words):
        return self.ps.compare(gpu_words)


def ps_eval(X_words, coeffs: Sequence[Fraction], d_w: int, *, mode: str = "mixed", delta: float = 10.0,
            snap_levels: bool = True, wbits: Optional[int] = None) -> OracleResult:
    """The oracle composition of SURVEY.md 8(c) for one matrix.
    mode = "mixed" (plan_precisions + snap) or "fixed" (all levels at d_w,
    ps_fixed engine.py:304-345)."""
    Xw = _words(X_words)
    n = Xw.shape[1]
    m = len(coeffs) - 1
    s = math.ceil(math.sqrt(m))
    wb = bits_of(d_w) if wbits is None else wbits
    ps = OraclePS(n)
    norms2 = ps.prepare(Xw, coeffs, s, wb)
    r = m // s
    if mode == "fixed":
        digits, nu, nil = (d_w,) * r, r + 1, False
    else:
        digits, nu, nil, _ = plan_digits(norms2, d_w, delta)
    if nil:
        # p = B_0 (engine.py:378-379, 473-474)
        lib().orc_result_from_block(ps.h, 0)
        return OracleResult(ps, norms2, digits, nu, True, tuple(digits), [wb] + [bits_of(1)] * r)
    snapped = snap(digits, d_w) if (snap_levels and mode != "fixed") else tuple(digits)
    level_bits = [wb] + [bits_of(x) for x in snapped]
    ps.horner(level_bits)
    return OracleResult(ps, norms2, digits, nu, False, snapped, level_bits)


def reference_eval_words(X_words, coeffs: Sequence[Fraction], d: int) -> np.ndarray:
    """harness.py:105-109: ps_fixed at 2d digits (returned unrounded, 4 words)."""
    res = ps_eval(X_words, coeffs, 2 * d, mode="fixed")
    return res.ps.result_words(4)


def _cols_arg(cols):
    cols = [int(c) for c in cols]
    return (ctypes.c_int * len(cols))(*cols), len(cols)


def poly_columns(X_words, coeffs: Sequence[Fraction], bits: int, cols, squares: bool = False) -> np.ndarray:
    """Tier C: columns ``cols`` of p(X) -- or of p(X^2) with
    ``squares`` (the cosine's Z = X X, harness.py:100-101) -- by
    matrix-vector Horner at ``bits`` (use 2x the working digits' bits, as
    reference_eval does, harness.py:105-109).  Returns (4, len(cols), n)
    exact word planes."""
    Xw = _words(X_words)
    n = Xw.shape[1]
    m = len(coeffs) - 1
    nums = (ctypes.c_char_p * (m + 1))(*[str(Fraction(c).numerator).encode() for c in coeffs])
    dens = (ctypes.c_char_p * (m + 1))(*[str(Fraction(c).denominator).encode() for c in coeffs])
    ca, nc = _cols_arg(cols)
    out = np.zeros((4, nc, n))
    if lib().orc_poly_cols(n, _dp(Xw), Xw.shape[0], m, nums, dens, bits, int(bool(squares)), ca, nc, _dp(out)):
        raise ValueError("bad column index")
    return out


def power_columns(P_words, count: int, bits: int, cols) -> np.ndarray:
    """Columns ``cols`` of P^count at ``bits`` (repeated matrix-vector
    products); (4, len(cols), n) word planes."""
    Pw = _words(P_words)
    n = Pw.shape[1]
    ca, nc = _cols_arg(cols)
    out = np.zeros((4, nc, n))
    if lib().orc_matpow_cols(n, _dp(Pw), Pw.shape[0], int(count), bits, ca, nc, _dp(out)):
        raise ValueError("bad column index")
    return out


def column_diff(gpu_cols: np.ndarray, ref_cols: np.ndarray) -> np.ndarray:
    """Per column ||g - r||_1, every entry's difference of word expansions
    formed exactly (rationals): gpu_cols (W, ncols, n), ref_cols (4, ncols, n)."""
    g = np.asarray(gpu_cols, dtype=np.float64)
    r = np.asarray(ref_cols, dtype=np.float64)
    out = np.zeros(g.shape[1])
    for c in range(g.shape[1]):
        tot = Fraction(0)
        for i in range(g.shape[2]):
            d = sum(Fraction(float(x)) for x in g[:, c, i]) - sum(Fraction(float(x)) for x in r[:, c, i])
            tot += abs(d)
        out[c] = float(tot)
    return out
