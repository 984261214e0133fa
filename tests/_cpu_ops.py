"""TEST DOUBLE for the SUMMA driver's device ops: the same call surface as
summa.DeviceOps, computed in plain float64 on CPU tensors (word plane 0;
higher planes stay zero).  Only the collective plumbing of the driver is
under test with it (gloo, world size 2); arithmetic parity of the real
kernels is covered by the GPU tests."""
import math

import numpy as np
import torch

from paper_2312_17396_b200.coefficients import coeff_words
from paper_2312_17396_b200.precision import FP32, MatBatch


class _Op:
    def __init__(self, mat):
        self.mat = mat


class CpuOps:
    device = torch.device("cpu")
    host_double = True     # no digit planes: one prepared Y per level format

    def prepare(self, A, side, fmt, exp=0):
        if A.fmt == fmt and not exp:
            return _Op(A)
        B = self.empty(fmt, A.rows, A.cols)
        self.convert(A, B, exp)
        return _Op(B)

    def gemm_op(self, L, R, C):
        self.gemm(L.mat, R.mat, C)

    def panel_start(self, grid, A, side, fmt, k_total):
        """The dd panel gathered by the grid (no digit planes on the host)."""
        pend = grid.row_panel_start(A) if side == 0 else grid.col_panel_start(A)
        ops = self

        class _P:
            def finish(self_):
                return ops.prepare(pend.panel_finish(), side, fmt)
        return _P()

    def concat_rows(self, ops_):
        return _Op(MatBatch(torch.cat([o.mat.data for o in ops_], dim=2), ops_[0].mat.fmt))

    def horner_op(self, Y, phi, fmt_level, Bprev, out, ey=0, ei=0, eo=0):
        self.horner_step(Y.mat, phi.mat, Bprev, out, ey, ei, eo)

    def empty(self, fmt, rows, cols):
        m = MatBatch.empty(fmt, 1, rows, cols, device="cpu")
        m.data.zero_()
        return m

    @staticmethod
    def _v(A):
        return A.data[0, 0].double()

    @staticmethod
    def _set(A, v):
        A.data.zero_()
        A.data[0, 0] = v.to(A.data.dtype)

    def convert(self, src, dst, exp=0):
        self._set(dst, self._v(src) * 2.0 ** exp)

    def gemm(self, A, B, C):
        self._set(C, self._v(A) @ self._v(B))

    def coeffs(self, series, ctx):
        return torch.tensor(coeff_words(series, ctx)).sum(dim=1)

    def assemble_dist(self, powers, m, coeffs, blocks, row0, col0):
        s = len(powers)
        r = m // s
        full = m // s
        rows, cols = powers[0].rows, powers[0].cols
        ii = torch.arange(rows)[:, None] + row0
        jj = torch.arange(cols)[None, :] + col0
        eye = (ii == jj).double()
        cs = torch.zeros((1, r + 2, cols), dtype=torch.float64)
        for i in range(r + 1):
            hi = s - 1 if i < full else m - s * full
            acc = coeffs[s * i] * eye
            for j in range(1, hi + 1):
                acc = coeffs[s * i + j] * self._v(powers[j - 1]) + acc
            self._set(blocks[i], acc)
            cs[0, i] = acc.abs().sum(dim=0)
        cs[0, r + 1] = self._v(powers[s - 1]).abs().sum(dim=0)
        return cs

    def colmax(self, colsums):
        return colsums.max(dim=2).values

    def horner_step(self, Y, phi, Bprev, out, ey=0, ei=0, eo=0):
        t = (self._v(Y) @ self._v(phi)) * 2.0 ** (-(ey + ei))
        self._set(out, (self._v(Bprev) + t) * 2.0 ** eo)

    def scalar_top(self, bm_words, fmt_top, Y, Bprev, out, eo=0):
        bm = float(sum(bm_words))
        self._set(out, (self._v(Bprev) + bm * self._v(Y)) * 2.0 ** eo)
