"""Complex matrices (the reference's native element type: every ``MPMatrix``
entry is a ``gmpy2.mpc``, precision.py:78-105).

A complex n x n matrix Z = A + iB runs through the real evaluators as its
real embedding

    E(Z) = [[A, -B],
            [B,  A]]        (2n x 2n),

which is an algebra homomorphism: E(Z1 Z2) = E(Z1) E(Z2), E(Z1 + Z2) =
E(Z1) + E(Z2), E(cI) = cI for real c -- so p(E(X)) = E(p(X)) for the real
coefficient series of exp / Pade / cos, and the power chain, block assembly
and Horner GEMMs of the embedding compute exactly the real sums of the
complex products (Re(z w) = ar br - ai bi, Im(z w) = ar bi + ai br, with
K = 2n terms per entry).  The reference rounds each mpc product component
once (MPC, correctly rounded); the B200 path rounds the K-term sums like
every other GEMM (Thm 2.1 with n -> 2n covers it).

What differs from the real path is the planner's input: ``one_norm`` of a
complex matrix sums |z_ij| = hypot(Re, Im) (precision.py:235-249 with
mpc_abs), not the absolute values of the embedding's entries.  While an
evaluation of a complex input runs, ``scope()`` holds n and the engine
replaces every block / power norm by ``mpps_one_norm_complex`` of the
embedding, so the schedule is planned on the reference's norms.

Cost: a complex GEMM as the embedding is 8 n^3 real multiply-adds against
4 n^3 for the four-real-product form; the embedding keeps every kernel and
the plan machinery unchanged (a dedicated complex GEMM is future work).
"""

from __future__ import annotations

import contextlib
import functools
import threading
from typing import Optional

import numpy as np

from .precision import DimensionError, MatBatch

_TLS = threading.local()


def scope() -> Optional[int]:
    """n of the complex evaluation running in this thread (None: real)."""
    return getattr(_TLS, "n", None)


@contextlib.contextmanager
def _complex_scope(n: int):
    prev = scope()
    _TLS.n = n
    try:
        yield
    finally:
        _TLS.n = prev


def _torch():
    import torch
    return torch


class ComplexMatBatch:
    """A batch of complex matrices held as real embeddings (words, B, 2n, 2n)
    at one format; ``real`` / ``imag`` are views of its left block column."""

    def __init__(self, emb: MatBatch, n: int):
        if emb.rows != 2 * n or emb.cols != 2 * n:
            raise DimensionError(f"embedding must be {2 * n}x{2 * n}, got {emb.rows}x{emb.cols}")
        self.emb = emb
        self.n = n

    @property
    def fmt(self) -> int:
        return self.emb.fmt

    @property
    def batch(self) -> int:
        return self.emb.batch

    @property
    def rows(self) -> int:
        return self.n

    @property
    def cols(self) -> int:
        return self.n

    @property
    def words(self) -> int:
        return self.emb.words

    @property
    def device(self):
        return self.emb.device

    @property
    def real(self) -> MatBatch:
        return MatBatch(self.emb.data[:, :, :self.n, :self.n], self.emb.fmt)

    @property
    def imag(self) -> MatBatch:
        return MatBatch(self.emb.data[:, :, self.n:, :self.n], self.emb.fmt)

    def select(self, idx: int) -> "ComplexMatBatch":
        return ComplexMatBatch(self.emb.select(idx), self.n)

    def words_numpy(self) -> np.ndarray:
        """(2, words, batch, n, n): real and imaginary word planes."""
        return np.stack([self.real.words_numpy(), self.imag.words_numpy()])

    def to_numpy(self) -> np.ndarray:
        """complex128 (batch, n, n), each part rounded to fp64."""
        return self.real.to_numpy() + 1j * self.imag.to_numpy()

    def __repr__(self):
        return f"ComplexMatBatch({self.emb!r} embedding, {self.n}x{self.n} complex)"


def _mp_complex(A) -> Optional[np.ndarray]:
    """complex128 values of a reference ``MPMatrix`` with a nonzero imaginary
    part somewhere (None for real matrices)."""
    vals = np.empty((A.n_rows, A.n_cols), dtype=np.complex128)
    cplx = False
    for i, row in enumerate(A.rows):
        for j, e in enumerate(row):
            re = float(getattr(e, "real", e))
            im = float(getattr(e, "imag", 0))
            cplx = cplx or im != 0.0
            vals[i, j] = complex(re, im)
    return vals if cplx else None


def complex_input(X):
    """None for real inputs; otherwise (embedding: torch fp64 (B,2n,2n) or a
    working-format MatBatch, n, single)."""
    torch = _torch()
    if isinstance(X, ComplexMatBatch):
        return X.emb, X.n, X.batch == 1
    if isinstance(X, MatBatch):
        return None
    if isinstance(X, np.ndarray):
        if not np.iscomplexobj(X):
            return None
        Z = torch.from_numpy(np.ascontiguousarray(X, dtype=np.complex128))
    elif isinstance(X, torch.Tensor):
        if not X.is_complex():
            return None
        Z = X.to(torch.complex128)
    elif hasattr(X, "rows") and hasattr(X, "n_rows"):
        v = _mp_complex(X)
        if v is None:
            return None
        Z = torch.from_numpy(v)
    else:
        return None
    single = Z.dim() == 2
    if single:
        Z = Z.unsqueeze(0)
    if Z.dim() != 3 or Z.shape[1] != Z.shape[2]:
        raise DimensionError(f"expected square (n,n) or (B,n,n), got {tuple(Z.shape)}")
    return embed(Z), Z.shape[1], single


def embed(Z):
    """torch complex (B,n,n) -> real fp64 embedding (B,2n,2n) on Z's device."""
    torch = _torch()
    A, B = Z.real.to(torch.float64), Z.imag.to(torch.float64)
    top = torch.cat([A, -B], dim=2)
    bot = torch.cat([B, A], dim=2)
    return torch.cat([top, bot], dim=1).contiguous()


def _complexify(out, n: int):
    from .engine import BatchReport, EvaluationReport
    if isinstance(out, EvaluationReport):
        out._cplx_n = n
        return out
    if isinstance(out, BatchReport):
        for rep in out:
            rep._cplx_n = n
        out.result = ComplexMatBatch(out.result, n)
        return out
    if isinstance(out, tuple):
        return tuple(_complexify(o, n) for o in out)
    if isinstance(out, MatBatch):
        return ComplexMatBatch(out, n)
    return out          # plans (plan_only) carry no matrix


def complex_aware(fn):
    """Entry-point decorator: complex inputs run on their embeddings inside
    a complex scope and come back as complex results."""
    @functools.wraps(fn)
    def wrapper(X, *args, **kw):
        cx = complex_input(X)
        if cx is None:
            return fn(X, *args, **kw)
        emb, n, single = cx
        if not isinstance(emb, MatBatch) and single:
            emb = emb[0]
        with _complex_scope(n):
            out = fn(emb, *args, **kw)
        return _complexify(out, n)
    return wrapper
