"""Out-of-bounds write guards for the hand-written kernels (TMA / tcgen05
GEMMs with staged epilogues, digit splits, block assembly, conversions).

compute-sanitizer is closed on the GPU pool this build runs on, so memory
safety is checked the other way round: every output lives inside a larger
allocation filled with a canary bit pattern (guard zones before and after
the buffer, padding columns between rows of strided outputs), inputs are
guarded the same way, and after each launch every byte outside the
footprint the ABI allows the kernel to write must still hold the canary.
Shapes are ragged (n = 200: not a multiple of the 128-row / 32-byte tiles)
and batched, with a selection list, so edge tiles and partial TMA boxes are
exercised."""
import ctypes

import numpy as np
import pytest

from _util import synth

pytestmark = pytest.mark.gpu

CANARY = 0x5A
G = 1 << 16          # guard bytes on each side


class Guarded:
    """A tensor of `shape`/`dtype` carved out of a canary-filled byte
    buffer; pad_cols extra canary columns after every row."""

    def __init__(self, torch, shape, dtype, pad_cols=0):
        self.torch = torch
        esz = torch.empty((), dtype=dtype).element_size()
        rows = int(np.prod(shape[:-1])) if len(shape) > 1 else 1
        ld = shape[-1] + pad_cols
        nbytes = rows * ld * esz
        self.raw = torch.full((nbytes + 2 * G,), CANARY, dtype=torch.uint8, device="cuda")
        body = self.raw[G:G + nbytes].view(dtype).view(*shape[:-1], ld)
        self.t = body[..., :shape[-1]]
        self.pad_cols = pad_cols
        self.ld, self.esz = ld, esz
        self.nbytes = nbytes

    def check(self, what):
        torch = self.torch
        raw = self.raw.cpu().numpy()
        assert (raw[:G] == CANARY).all(), f"{what}: write before the buffer"
        assert (raw[G + self.nbytes:] == CANARY).all(), f"{what}: write after the buffer"
        if self.pad_cols:
            body = raw[G:G + self.nbytes].reshape(-1, self.ld * self.esz)
            assert (body[:, (self.ld - self.pad_cols) * self.esz:] == CANARY).all(), f"{what}: write into row padding"


def _mat(torch, fmt, batch, rows, cols, pad_cols=0):
    from paper_2312_17396_b200.precision import FORMAT_WORDS, MatBatch
    dt = torch.float32 if fmt == 7 else torch.float64
    g = Guarded(torch, (FORMAT_WORDS[fmt], batch, rows, cols), dt, pad_cols)
    g.t.zero_()
    return g, MatBatch(g.t, fmt)


def _slices(torch, S, batch, rows, k, db):
    from paper_2312_17396_b200 import _lib
    sl = _lib.Slices(S, batch, rows, k, "cuda", db)
    gd = Guarded(torch, tuple(sl.digits.shape), torch.int8)
    ge = Guarded(torch, tuple(sl.exps.shape), torch.int32)
    sl.digits, sl.exps = gd.t, ge.t
    return sl, (gd, ge)


@pytest.mark.parametrize("fmt", [15, 31])
def test_guarded_split_gemm_horner(cuda, fmt):
    import torch
    from paper_2312_17396_b200 import _lib, gemm_engine as ge
    from paper_2312_17396_b200.precision import MatBatch
    h = _lib.handle_for()
    n, B = 200, 3
    X = np.stack([synth(n, 1.0, 60 + b) for b in range(B)])
    gx, A = _mat(torch, fmt, B, n, n, pad_cols=24)
    A.data[0].copy_(torch.from_numpy(X))
    if fmt == 31:
        A.data[1].copy_(torch.from_numpy(X * 2.0 ** -60))
    sel = torch.tensor([2, 0], dtype=torch.int32, device="cuda")
    for db in (7, 8):
        S = h.slices_for(fmt, db)
        rows_s, grs = _slices(torch, S, B, n, n, db)
        cols_s, gcs = _slices(torch, S, B, n, n, db)
        c = _lib.cmat(A)
        h._check(h.lib.mpps_slice(h.h, ctypes.byref(c), 0, ctypes.byref(rows_s.c()), None, 0), "slice rows")
        h._check(h.lib.mpps_slice(h.h, ctypes.byref(c), 1, ctypes.byref(cols_s.c()), None, 0), "slice cols")
        torch.cuda.synchronize()
        for g in grs + gcs:
            g.check(f"slice db={db}")
        gc_, C = _mat(torch, fmt, B, n, n, pad_cols=40)
        h.gemm_sliced(rows_s, cols_s, S, C)
        gs_, Cs = _mat(torch, fmt, B, n, n, pad_cols=8)
        h.gemm_sliced(rows_s, cols_s, S, Cs, sel)
        gb, Bp = _mat(torch, fmt, B, n, n, pad_cols=16)
        Bp.data[0].copy_(torch.from_numpy(X))
        go, Out = _mat(torch, fmt, B, n, n, pad_cols=32)
        h.horner_step_sliced(rows_s, cols_s, S, Bp, Out, sel, None, None, None, fmt_in=fmt)
        torch.cuda.synchronize()
        for g, what in ((gc_, "gemm"), (gs_, "gemm sel"), (go, "horner out"), (gb, "horner Bprev"),
                        (gx, "operand")):
            g.check(f"{what} db={db}")
        # selected members untouched outside the selection
        assert (Cs.data[:, 1] == 0).all() and (Out.data[:, 1] == 0).all()
        # the strided guarded product equals a plain contiguous one
        ref = MatBatch.empty(fmt, B, n, device="cuda")
        h.gemm_sliced(h.slice(MatBatch(A.data.contiguous(), fmt), 0, S, None, db),
                      h.slice(MatBatch(A.data.contiguous(), fmt), 1, S, None, db), S, ref)
        assert torch.equal(ref.data, C.data)


def test_guarded_assembly_convert_norms(cuda):
    import torch
    import paper_2312_17396_b200 as m
    from paper_2312_17396_b200 import _lib
    from paper_2312_17396_b200.coefficients import coeff_words
    from paper_2312_17396_b200.precision import MatBatch
    h = _lib.handle_for()
    n, B, s = 200, 3, 6
    ctx = m.PrecisionCtx(31)
    series = m.taylor_exp_coeffs(30)
    X = np.stack([synth(n, 1.0, 70 + b) for b in range(B)])
    powers = []
    for k in range(1, s + 1):
        g, P = _mat(torch, 31, B, n, n, pad_cols=8)
        P.data[0].copy_(torch.from_numpy(X * (0.5 ** k)))
        powers.append((g, P))
    cw = coeff_words(series, ctx)
    r = 30 // s
    # two-pass mixed assembly (B_0, B_1 dd, the rest fp64) + norms
    blocks = [_mat(torch, 31 if k < 2 else 15, B, n, n, pad_cols=16) for k in range(r)]
    gn = Guarded(torch, (B, r + 1), torch.float64)
    if h.assemble_hc_n_supported(-1, s, 30, r):
        h.assemble_blocks_hc_n([p for _, p in powers], 30, cw, [b for _, b in blocks], gn.t)
    # one-pass dd assembly (B_r unstored)
    dd = [_mat(torch, 31, B, n, n, pad_cols=4) for _ in range(r)] + [_mat(torch, 31, 1, 1, 1)]
    gn2 = Guarded(torch, (B, r + 2), torch.float64)
    h.assemble_blocks_hc([p for _, p in powers], 30, cw, [b for _, b in dd], gn2.t, True)
    # conversions with an exponent list, into strided outputs
    gf, F = _mat(torch, 7, B, n, n, pad_cols=12)
    ge_ = Guarded(torch, (B,), torch.int32)
    ge_.t.copy_(torch.tensor([3, -2, 0], dtype=torch.int32))
    h.convert(powers[0][1], F, None, ge_.t)
    gq, Q = _mat(torch, 63, B, n, n, pad_cols=12)
    h.convert(powers[1][1], Q)
    gnn = Guarded(torch, (B,), torch.float64)
    h.one_norm(powers[2][1], gnn.t)
    torch.cuda.synchronize()
    for g, _ in powers:
        g.check("powers (read only)")
    for g, _ in blocks + dd:
        g.check("blocks")
    for g in (gn, gn2, gf, ge_, gq, gnn):
        g.check("convert / norms")
