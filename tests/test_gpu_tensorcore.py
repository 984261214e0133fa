"""Tensor-core (INT8 tcgen05) multiword GEMM by exact operand splitting vs
the SIMT error-free-transform GEMM and the MPFR oracle: same normwise
accuracy class (c n u |A||B|), for fp64 (8 digit planes), dd (16), qd (31);
square, ragged and rectangular shapes, batched."""
from fractions import Fraction

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _words_of(fmt, A, rng):
    if fmt == 15:
        return A[None]
    lo = A * 2.0 ** -60 * rng.standard_normal(A.shape)
    w = [A, lo]
    if fmt == 63:
        w += [lo * 2.0 ** -60, lo * 2.0 ** -121]
    return np.stack(w)


@pytest.mark.parametrize("db", [7, 8])
@pytest.mark.parametrize("fmt,bits", [(15, 53), (31, 106), (63, 212)])
@pytest.mark.parametrize("shape", [(64, 64, 64), (70, 45, 33), (256, 256, 256), (130, 96, 300)])
def test_tc_gemm_vs_oracle(cuda, oracle_lib, fmt, bits, shape, db):
    import torch
    from paper_2312_17396_b200 import _lib, ops
    M, N, K = shape
    rng = np.random.default_rng(M + N + K + fmt)
    A = rng.standard_normal((M, K)) * np.exp(rng.uniform(-3, 3, (M, 1)))
    B = rng.standard_normal((K, N)) * np.exp(rng.uniform(-3, 3, (1, N)))
    Aw, Bw = _words_of(fmt, A, rng), _words_of(fmt, B, rng)
    h = _lib.handle_for()
    Ad, Bd = ops.from_numpy(Aw, fmt), ops.from_numpy(Bw, fmt)
    S = h.slices_for(fmt, db)
    assert S == {7: {15: 8, 31: 16, 63: 31}, 8: {15: 8, 31: 14, 63: 28}}[db][fmt]
    sa, sb = h.slice(Ad, 0, S, None, db), h.slice(Bd, 1, S, None, db)
    from paper_2312_17396_b200.precision import MatBatch
    C = MatBatch.empty(fmt, 1, M, N, device=cuda)
    h.gemm_sliced(sa, sb, S, C)
    got = C.data[:, 0].cpu().numpy()
    # oracle on the square embedding (orc_matmul is square)
    n = max(M, N, K)
    Ap = np.zeros((Aw.shape[0], n, n)); Ap[:, :M, :K] = Aw
    Bp = np.zeros((Bw.shape[0], n, n)); Bp[:, :K, :N] = Bw
    Co = oracle_lib.matmul(Ap, Bp, bits)[:, :M, :N]
    absAB = np.abs(A) @ np.abs(B)
    u = Fraction(1, 2 ** bits)
    for _ in range(200):
        i, j = rng.integers(0, M), rng.integers(0, N)
        g = sum(Fraction(float(x)) for x in got[:, i, j])
        o = sum(Fraction(float(x)) for x in Co[:, i, j])
        assert abs(g - o) <= 4 * K * u * Fraction(float(absAB[i, j])), (i, j, float(g - o), float(absAB[i, j]))


def test_abi_gemm_and_horner_step_on_plain_matrices(cuda):
    """mpps_gemm / mpps_horner_step (the C-ABI operator entry points on plain
    matrices: the library splits into stream-ordered scratch itself) equal
    the explicit split + sliced-kernel path bit for bit, with a selection."""
    import torch
    from paper_2312_17396_b200 import _lib
    from paper_2312_17396_b200.precision import MatBatch
    h = _lib.handle_for()
    B, n = 8, 200
    X = MatBatch.empty(31, B, n, device=cuda)
    X.data[0].normal_()
    X.data[1] = X.data[0] * 2.0 ** -55
    C1 = MatBatch.zeros(31, B, n, device=cuda)
    C2 = MatBatch.zeros(31, B, n, device=cuda)
    sel = torch.tensor([5, 1, 2], dtype=torch.int32, device=cuda)
    h.gemm(X, X, C1, sel)
    S = h.slices_for(31, 8)
    h.gemm_sliced(h.slice(X, 0, S, sel, 8), h.slice(X, 1, S, sel, 8), S, C2, sel)
    assert torch.equal(C1.data, C2.data)
    assert C1.data[:, 0].abs().sum() == 0 and C1.data[:, 5].abs().sum() > 0
    P = MatBatch.empty(15, B, n, device=cuda)
    P.data.normal_()
    Bp = MatBatch.empty(31, B, n, device=cuda)
    Bp.data.normal_()
    O1 = MatBatch.zeros(15, B, n, device=cuda)
    O2 = MatBatch.zeros(15, B, n, device=cuda)
    Xf = MatBatch(X.data[:1].clone(), 15)
    h.horner_step(Xf, P, Bp, O1)
    S = h.slices_for(15, 8)
    h.horner_step_sliced(h.slice(Xf, 0, S, None, 8), h.slice(P, 1, S, None, 8), S, Bp, O2, fmt_in=15)
    assert torch.equal(O1.data, O2.data)


@pytest.mark.parametrize("fmt,B,n", [(15, 3, 96), (31, 2, 200), (31, 1, 1024), (63, 1, 64), (7, 2, 128)])
def test_mat_mul_propagates_non_finite_entries(cuda, fmt, B, n):
    """mat_mul (precision.py:160-184) of an operand with a NaN / Inf entry: row i of the
    product is non-finite for a bad A[i, k], column j for a bad B[k, j] (the digit splits
    answer a non-finite row / column maximum with an Inf scale instead of cutting finite
    digits out of it); every other entry is bit-identical to the product of the clean
    operands (row and column scales are independent)."""
    import torch
    from paper_2312_17396_b200 import _lib
    from paper_2312_17396_b200.precision import MatBatch
    h = _lib.handle_for()
    torch.manual_seed(fmt + n)
    A = MatBatch.empty(fmt, B, n, device=cuda)
    Bm = MatBatch.empty(fmt, B, n, device=cuda)
    for M in (A, Bm):
        M.data[0].normal_()
        for w in range(1, M.words):
            M.data[w] = M.data[0] * 2.0 ** (-55 * w) if fmt != 7 else 0
    C0 = MatBatch.zeros(fmt, B, n, device=cuda)
    h.gemm(A, Bm, C0)
    assert torch.isfinite(C0.data).all()
    bad_rows = [(0, 2, 3, float("nan")), (B - 1, n - 1, 0, float("inf"))]
    bad_cols = [(0, 1, 4, float("-inf")), (B - 1, 7, n - 2, float("nan"))]
    A2, B2 = MatBatch(A.data.clone(), fmt), MatBatch(Bm.data.clone(), fmt)
    for b, i, k, v in bad_rows:
        A2.data[0, b, i, k] = v
    for b, k, j, v in bad_cols:
        B2.data[0, b, k, j] = v
    C = MatBatch.zeros(fmt, B, n, device=cuda)
    h.gemm(A2, B2, C)
    clean = torch.ones((B, n, n), dtype=torch.bool, device=cuda)
    for b, i, _, _ in bad_rows:
        assert not torch.isfinite(C.data[0, b, i, :]).any()
        clean[b, i, :] = False
    for b, _, j, _ in bad_cols:
        assert not torch.isfinite(C.data[0, b, :, j]).any()
        clean[b, :, j] = False
    for w in range(C.words):
        assert torch.equal(C.data[w][clean], C0.data[w][clean])


def test_tc_digit_width_rules(cuda):
    """8-bit digits: operands of one product must share the width; K beyond
    the exact-int32 limit is refused; every digit lies in [-128, 127] and the
    planes reproduce the value (checked through a GEMM with the identity)."""
    import torch
    from paper_2312_17396_b200 import _lib
    from paper_2312_17396_b200.precision import MatBatch
    h = _lib.handle_for()
    A = MatBatch.empty(31, 1, 64, device=cuda)
    A.data[0].normal_()
    A.data[1] = A.data[0] * 2.0 ** -60
    s7, s8 = h.slice(A, 0, 16, None, 7), h.slice(A, 1, 14, None, 8)
    C = MatBatch.empty(31, 1, 64, device=cuda)
    with pytest.raises(ValueError, match="7- and 8-bit"):
        h.gemm_sliced(s7, s8, 14, C)
    assert int(s8.digits.min()) >= -128 and int(s8.digits.max()) <= 127
    assert int(s8.digits[0].abs().max()) <= 65
    I = MatBatch.zeros(31, 1, 64, device=cuda)
    I.data[0, 0] = torch.eye(64, dtype=torch.float64, device=cuda)
    h.gemm_sliced(h.slice(A, 0, 14, None, 8), h.slice(I, 1, 14, None, 8), 14, C)
    d = (C.data[0] - A.data[0]) + (C.data[1] - A.data[1])
    assert (d.abs() <= 2.0 ** -104 * A.data[0].abs().amax(dim=-1, keepdim=True)).all()
    assert h.max_k_8bit() == 4800


@pytest.mark.parametrize("n", [96, 256])
@pytest.mark.parametrize("side", [0, 1])
@pytest.mark.parametrize("fmt,S", [(31, 14), (15, 8), (7, 4), (31, 8), (31, 4)])
def test_fixed_point_split_exact(cuda, side, fmt, S, n):
    """8-bit fixed-point split (fixed_biased_fast): every entry's digit planes
    reproduce round(v 2^(F-e)) to within one unit of 2^(e-F), F = 6 + 8(S-1),
    over entries spanning ~2^-200 .. 1 of their row/column maximum, signs,
    zeros and normalised dd low words.  n = 256 takes the register-resident
    row split (whole 16-byte-aligned rows of 128/256 entries)."""
    import torch
    from paper_2312_17396_b200 import _lib
    from paper_2312_17396_b200.precision import MatBatch
    h = _lib.handle_for()
    rng = np.random.default_rng(7 + S + fmt + side + n)
    hi = rng.standard_normal((n, n)) * 2.0 ** rng.integers(-200, 1, (n, n)).astype(float)
    hi[rng.random((n, n)) < 0.05] = 0.0
    hi[:, 3] *= 2.0 ** 40          # a column / row with a large maximum
    if fmt == 7:
        hi = hi.astype(np.float32).astype(np.float64)
    words = [hi]
    if fmt == 31:
        lo = np.where(hi != 0, hi * 2.0 ** -54 * rng.uniform(-1, 1, hi.shape), 0.0)
        lo = (hi + lo) - hi            # representable, |lo| <= ulp(hi)/2
        words = [hi, lo]
    A = MatBatch.empty(fmt, 1, n, device=cuda)
    for w, x in enumerate(words):
        A.data[w, 0] = torch.from_numpy(x).to(A.data.dtype)
    sl = h.slice(A, side, S, None, 8)
    dig = sl.digits[:, 0].cpu().numpy().astype(np.int64)      # (S, rpad, kpad)
    ex = sl.exps[0].cpu().numpy()
    F = 6 + 8 * (S - 1)
    for _ in range(300):
        i, k = int(rng.integers(0, n)), int(rng.integers(0, n))
        r, c = (i, k) if side == 0 else (k, i)     # row-split rows are A rows; col-split rows are A columns
        v = sum(Fraction(float(words[w][r, c])) for w in range(len(words)))
        V = sum(int(dig[s, i, k]) << (8 * (S - 1 - s)) for s in range(S))
        exact = v * Fraction(2) ** (F - int(ex[i]))
        assert abs(V - exact) <= 1, (side, i, k, float(V - exact))


_NT128_SCRIPT = r'''
import sys, numpy as np, torch
sys.path.insert(0, sys.argv[1])
from paper_2312_17396_b200 import _lib
from paper_2312_17396_b200.precision import MatBatch
h = _lib.handle_for()
rng = np.random.default_rng(3)
B, M, N = 3, 200, 300
out = {}
for K, S, fo in ((2080, 2, 7), (2080, 3, 15), (2080, 4, 31), (2080, 2, 31), (4160, 2, 7), (4160, 3, 31),
                 (4160, 4, 31)):
    Y = MatBatch(torch.from_numpy(rng.standard_normal((1, B, M, K))).cuda(), 15)
    P = MatBatch(torch.from_numpy(rng.standard_normal((1, B, K, N))).cuda(), 15)
    Bp = MatBatch(torch.from_numpy(rng.standard_normal((2, B, M, N)) * np.array([1, 2.0 ** -60])[:, None, None, None]).cuda(), 31)
    o = MatBatch.zeros(fo, B, M, N, device="cuda")
    sel = torch.tensor([2, 0], dtype=torch.int32, device="cuda")
    ei = torch.tensor([3, -1, 2], dtype=torch.int32, device="cuda")
    eo = torch.tensor([-2, 0, 1], dtype=torch.int32, device="cuda")
    h.horner_step_sliced(h.slice(Y, 0, S, None, 8), h.slice(P, 1, S, None, 8), S, Bp, o, sel, None, ei, eo, fmt_in=fo)
    out[f"{K}_{S}_{fo}"] = o.data.double().cpu().numpy()
np.savez(sys.argv[2], **out)
'''


def test_nt128_few_plane_horner_matches_nt32(cuda, tmp_path):
    """The 128-column few-plane Horner tiles (K >= 2048, S <= 4, chunked
    staged epilogue; 128-byte K boxes for S <= 3 at K >= 4096) give the same
    bits as the 32-column tiles (MPPS_OZ_NT128_K=0) and as the 32-byte-box
    128-column kernel (MPPS_OZ_WIDE=0), with ragged M / N / K, a selection
    and level exponents; separate processes (the switches are read once)."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    script = tmp_path / "nt.py"
    script.write_text(_NT128_SCRIPT)
    res = {}
    for tag, env in (("wide", {}), ("narrow", {"MPPS_OZ_NT128_K": "0", "MPPS_OZ_WIDE": "0"}),
                     ("tma128", {"MPPS_OZ_WIDE": "0"})):
        f = tmp_path / f"{tag}.npz"
        subprocess.check_call([sys.executable, str(script), root, str(f)], env=dict(os.environ, **env))
        res[tag] = dict(np.load(f))
    for k in res["wide"]:
        assert np.array_equal(res["wide"][k], res["narrow"][k]), k
        assert np.array_equal(res["wide"][k], res["tma128"][k]), k
        assert np.abs(res["wide"][k][:, 1]).sum() == 0 and np.abs(res["wide"][k][:, 0]).sum() > 0


_WIDE_SCRIPT = r'''
import sys, numpy as np, torch
sys.path.insert(0, sys.argv[1])
from paper_2312_17396_b200 import _lib
from paper_2312_17396_b200.precision import MatBatch
h = _lib.handle_for()
rng = np.random.default_rng(4)
out = {}
for (M, K, N, db, fmt) in ((384, 4160, 512, 8, 31), (256, 4096, 320, 7, 31), (200, 4160, 384, 8, 15)):
    A = MatBatch(torch.from_numpy(rng.standard_normal((2, 2, M, K)) * np.array([1, 2.0 ** -55])[:, None, None, None]).cuda(), 31)
    Bm = MatBatch(torch.from_numpy(rng.standard_normal((2, 2, K, N)) * np.array([1, 2.0 ** -57])[:, None, None, None]).cuda(), 31)
    S = h.slices_for(fmt, db)
    C = MatBatch.zeros(fmt, 2, M, N, device="cuda")
    h.gemm_sliced(h.slice(A, 0, S, None, db), h.slice(Bm, 1, S, None, db), S, C)
    out[f"{M}_{db}_{fmt}"] = C.data.cpu().numpy()
np.savez(sys.argv[2], **out)
'''


def test_wide_kernel_cluster_multicast_matches(cuda, tmp_path):
    """The 128-byte-box GEMMs (K >= 4096: dd, and the 8-plane fp64 product
    with 64-column tiles) with 2-CTA clusters multicasting the A planes give
    the same bits as one CTA per tile (MPPS_OZ_WIDE_MC=0) and as the 32-byte
    box kernels (MPPS_OZ_WIDE=0); 8- and 7-bit digits, batch 2, ragged K."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    script = tmp_path / "w.py"
    script.write_text(_WIDE_SCRIPT)
    res = {}
    for tag, env in (("mc", {}), ("solo", {"MPPS_OZ_WIDE_MC": "0"}), ("tma", {"MPPS_OZ_WIDE": "0"})):
        f = tmp_path / f"{tag}.npz"
        subprocess.check_call([sys.executable, str(script), root, str(f)], env=dict(os.environ, **env))
        res[tag] = dict(np.load(f))
    for k in res["mc"]:
        assert np.array_equal(res["mc"][k], res["solo"][k]), k
        assert np.array_equal(res["mc"][k], res["tma"][k]), k
        assert np.abs(res["mc"][k]).sum() > 0


_PW16_SCRIPT = r'''
import sys, numpy as np, torch
sys.path.insert(0, sys.argv[1])
from paper_2312_17396_b200 import _lib
from paper_2312_17396_b200.precision import MatBatch
h = _lib.handle_for()
rng = np.random.default_rng(5)
out = {}
dd = np.array([1, 2.0 ** -56])[:, None, None, None]
# plain dd products (mode 0): one plane per ring slot (K < 1024) and two (K >= 1024), ragged M / N / K,
# a paired output view (column offset inside a wider buffer) and a batch selection
for (B, M, K, N) in ((3, 200, 288, 300), (2, 384, 1056, 160), (1, 128, 2080, 512)):
    A = MatBatch(torch.from_numpy(rng.standard_normal((2, B, M, K)) * dd).cuda(), 31)
    Bm = MatBatch(torch.from_numpy(rng.standard_normal((2, B, K, N)) * dd).cuda(), 31)
    C = MatBatch.zeros(31, B, M, N, device="cuda")
    sel = torch.tensor(list(range(B))[::-1][: max(1, B - 1)], dtype=torch.int32, device="cuda")
    h.gemm_sliced(h.slice(A, 0, 14, None, 8), h.slice(Bm, 1, 14, None, 8), 14, C, sel)
    out[f"g_{M}_{K}_{N}"] = C.data.cpu().numpy()
wide = torch.zeros((2, 2, 256, 512), dtype=torch.float64, device="cuda")
A = MatBatch(torch.from_numpy(rng.standard_normal((2, 2, 256, 256)) * dd).cuda(), 31)
sa, sb = h.slice(A, 0, 14, None, 8), h.slice(A, 1, 14, None, 8)
h.gemm_sliced(sa, sb, 14, MatBatch(wide[:, :, :, 256:], 31))
out["g_view"] = wide.cpu().numpy()
# fused Horner levels (mode 1): every plane count of the level kernels, fp32 / fp64 / dd outputs,
# fp64 (1 word) and dd (2 words) B_prev, level exponents, selection, ragged shapes
B, M, N = 3, 200, 300
for K in (288, 1056):
    Y = MatBatch(torch.from_numpy(rng.standard_normal((2, B, M, K)) * dd).cuda(), 31)
    P = MatBatch(torch.from_numpy(rng.standard_normal((2, B, K, N)) * dd).cuda(), 31)
    ys = h.slice(Y, 0, 14, None, 8)
    for S, fo, fp in ((2, 7, 15), (2, 15, 15), (2, 31, 31), (3, 7, 31), (3, 15, 15), (3, 31, 31), (5, 15, 15),
                      (5, 31, 31), (6, 15, 31), (6, 31, 31), (10, 31, 31), (12, 31, 31), (14, 31, 31)):
        w = 2 if fp == 31 else 1
        Bp = MatBatch(torch.from_numpy(rng.standard_normal((w, B, M, N)) * dd[:w]).cuda(), fp)
        o = MatBatch.zeros(fo, B, M, N, device="cuda")
        sel = torch.tensor([2, 0], dtype=torch.int32, device="cuda")
        ey = torch.tensor([1, 0, -2], dtype=torch.int32, device="cuda")
        ei = torch.tensor([3, -1, 2], dtype=torch.int32, device="cuda")
        eo = torch.tensor([-2, 0, 1], dtype=torch.int32, device="cuda")
        h.horner_step_sliced(ys, h.slice(P, 1, S, None, 8), S, Bp, o, sel, ey, ei, eo, fmt_in=fo)
        out[f"h_{K}_{S}_{fo}_{fp}"] = o.data.double().cpu().numpy()
np.savez(sys.argv[2], **out)
'''


def test_persistent_kernel_matches_tile_per_cta_kernels(cuda, tmp_path):
    """The persistent 128-byte-box kernel (oz_gemm_pw16_kernel: dd products at
    K < 4096 and the fused Horner levels) gives the same bits as the
    tile-per-CTA ring / TMA kernels (MPPS_OZ_PW16=0): ragged M / N / K, one
    and two planes per ring slot, one and two accumulator sets, an output
    view inside a wider buffer, selections, level exponents, fp32 / fp64 / dd
    outputs, 1- and 2-word B_prev; separate processes (the switch is read
    once)."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    script = tmp_path / "p.py"
    script.write_text(_PW16_SCRIPT)
    res = {}
    for tag, env in (("pw16", {}), ("tiles", {"MPPS_OZ_PW16": "0"})):
        f = tmp_path / f"{tag}.npz"
        subprocess.check_call([sys.executable, str(script), root, str(f)], env=dict(os.environ, **env))
        res[tag] = dict(np.load(f))
    assert len(res["pw16"]) == 4 + 2 * 13
    for k in res["pw16"]:
        assert np.array_equal(res["pw16"][k], res["tiles"][k]), k
        assert np.abs(res["pw16"][k]).sum() > 0, k
    # rows of unselected members and the left half of the view stay untouched
    assert np.abs(res["pw16"]["g_view"][..., :256]).sum() == 0
    assert np.abs(res["pw16"]["h_288_2_7_15"][:, 1]).sum() == 0
