"""Decimal matrix I/O (precision.py:252-341) against the reference's own text
(tests/golden/io_reference.json, oracle/make_golden_io.py): writing the
same values gives the identical JSON / CSV text, reading the reference's
text gives exactly the reference's values (words), and write -> read is the
identity.  CPU only (MatBatch on host memory)."""
import json
import os
from fractions import Fraction

import numpy as np
import pytest

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def cases():
    with open(os.path.join(GOLD, "io_reference.json")) as f:
        return json.load(f)["cases"]


def _matrix(case):
    import torch
    from paper_2312_17396_b200 import ComplexMatBatch, MatBatch, matio
    d = case["digits"]
    fmt = matio.storage_format(d)
    W = {matio.FP64: 1, matio.DD: 2, matio.QD: 4}[fmt]
    words = case["words"]
    n = len(words)
    R = np.array([[e[0][:W] for e in row] for row in words]).transpose(2, 0, 1)
    I = np.array([[e[1][:W] for e in row] for row in words]).transpose(2, 0, 1)
    assert all(x == 0 for row in words for e in row for part in e for x in part[W:])
    if not I.any():
        return MatBatch(torch.from_numpy(np.ascontiguousarray(R[:, None])), fmt)
    E = np.zeros((W, 1, 2 * n, 2 * n))
    E[:, 0, :n, :n] = R
    E[:, 0, n:, n:] = R
    E[:, 0, n:, :n] = I
    E[:, 0, :n, n:] = -I
    return ComplexMatBatch(MatBatch(torch.from_numpy(E), fmt), n)


@pytest.mark.parametrize("case", cases(), ids=lambda c: c["name"])
def test_writer_matches_reference_text(case):
    from paper_2312_17396_b200 import matio
    A = _matrix(case)
    assert matio.matrix_to_json(A, case["digits"]) == case["json"]
    assert matio.matrix_to_csv(A, case["digits"]) == case["csv"]


@pytest.mark.parametrize("case", cases(), ids=lambda c: c["name"])
def test_reader_gives_reference_values(case):
    from paper_2312_17396_b200 import ComplexMatBatch, matio
    want = _matrix(case)
    for got in (matio.matrix_from_json(case["json"], device="cpu"), matio.matrix_from_csv(case["csv"], device="cpu")):
        assert type(got) is type(want)
        if isinstance(want, ComplexMatBatch):
            assert got.n == want.n
            assert np.array_equal(got.emb.data.numpy(), want.emb.data.numpy())
        else:
            assert np.array_equal(got.data.numpy(), want.data.numpy())


def test_roundtrip_and_errors():
    import torch
    from paper_2312_17396_b200 import MatBatch, matio
    rng = np.random.default_rng(3)
    hi = rng.standard_normal((4, 4)) * 10.0 ** rng.integers(-20, 20, (4, 4))
    lo = hi * 2.0 ** -60 * rng.standard_normal((4, 4))
    A = MatBatch(torch.from_numpy(np.stack([hi, lo])[:, None].copy()), matio.DD)
    # dd values carry up to 106 bits: printing 33 digits and re-reading at
    # 103 bits gives the 103-bit rounding of each entry
    B = matio.matrix_from_json(matio.matrix_to_json(A), device="cpu")
    C = matio.matrix_from_json(matio.matrix_to_json(B), device="cpu")
    assert np.array_equal(B.data.numpy(), C.data.numpy())
    for i in range(4):
        for j in range(4):
            a = Fraction(float(hi[i, j])) + Fraction(float(lo[i, j]))
            b = Fraction(float(B.data[0, 0, i, j])) + Fraction(float(B.data[1, 0, i, j]))
            assert abs(a - b) <= abs(a) * Fraction(1, 2 ** 102)
    with pytest.raises(ValueError):
        matio.matrix_from_csv("1,2\n3,4\n")
    with pytest.raises(ValueError):
        matio.matrix_from_json(json.dumps({"n_rows": 2, "n_cols": 2, "decimal_digits": 15, "entries": ["1"]}))
    with pytest.raises(ValueError):
        matio.matrix_from_json(json.dumps({"n_rows": 1, "n_cols": 1, "decimal_digits": 15, "entries": ["1+2"]}))
