"""CPU model of the tensor-core epilogue's diagonal recombination
(csrc/ozaki.cuh::combine_dd): sum_d D_d 2^-(12 + DB d) of the int32 diagonal
accumulators through integer carries and two FastTwoSums must be a normalised
double-double within 2^-105 of the exact sum -- for random, extreme and
heavily cancelling accumulators, 7- and 8-bit digits, every compiled plane
count.  Python floats are IEEE doubles with round-to-nearest, so the model
executes the kernel's operations bit for bit."""
import math
import random
import struct
from fractions import Fraction

import pytest


def _as_double(bits):
    return struct.unpack("<d", struct.pack("<Q", bits))[0]


def _u52_scaled(m, q, bias=0.0):
    assert 0 <= m < (1 << 52)
    return _as_double(((1075 - q) << 52) | m) - (2.0 ** (52 - q) + bias)


def combine_dd(D, S, DB):
    NG, WB = (S + 2) // 3, 3 * DB
    G = []
    for g in range(NG):
        d0 = 3 * g
        v = D[d0] << (2 * DB)
        if d0 + 1 < S:
            v += D[d0 + 1] << DB
        if d0 + 2 < S:
            v += D[d0 + 2]
        G.append(v)
    if NG == 1:
        return float(G[0]) * 2.0 ** -(12 + DB * 2), 0.0
    dig, c = [0] * NG, 0
    for g in range(NG - 1, 0, -1):
        t = G[g] + c
        dig[g] = t & ((1 << WB) - 1)
        c = t >> WB
    q0 = 12 + DB * 2
    p0 = _u52_scaled(G[0] + c + (1 << 51), q0, 2.0 ** (51 - q0))
    p = []
    for k in range((NG - 1 + 1) // 2):
        a = 1 + 2 * k
        if a + 1 < NG:
            p.append(_u52_scaled((dig[a] << WB) | dig[a + 1], 12 + DB * (3 * (a + 1) + 2)))
        else:
            p.append(_u52_scaled(dig[a], 12 + DB * (3 * a + 2)))
    s = p0 + p[0]
    lo = p[0] - (s - p0)
    if len(p) == 2:
        lo += p[1]
    if len(p) == 3:
        lo += p[1] + p[2]
    hi = s + lo
    return hi, lo - (hi - s)


def exact(D, S, DB):
    return sum(Fraction(D[d]) / (1 << (12 + DB * d)) for d in range(S))


def check(D, S, DB):
    hi, lo = combine_dd(D, S, DB)
    V = exact(D, S, DB)
    got = Fraction(hi) + Fraction(lo)
    assert abs(got - V) <= abs(V) / (1 << 105), (S, DB, D)
    if hi != 0.0:
        assert abs(lo) <= math.ulp(hi) / 2, (S, DB, D)      # normalised
        assert hi == float(V) or abs(Fraction(hi) - V) <= Fraction(math.ulp(hi)) / 2
    else:
        assert lo == 0.0 and V == 0


PLANES = {8: (2, 3, 4, 5, 6, 8, 10, 12, 14), 7: (4, 8, 16)}


@pytest.mark.parametrize("DB", (7, 8))
def test_combine_dd_random_and_extreme(DB):
    rng = random.Random(1234 + DB)
    lim = (1 << 31) - 1
    for S in PLANES[DB]:
        for _ in range(400):
            check([rng.randint(-lim, lim) for _ in range(S)], S, DB)
        for _ in range(200):      # small accumulators (short K)
            check([rng.randint(-(1 << rng.randint(0, 30)), 1 << rng.randint(0, 30)) for _ in range(S)], S, DB)
        check([lim] * S, S, DB)
        check([-lim - 1] * S, S, DB)
        check([0] * S, S, DB)
        for d in range(S):        # a single nonzero diagonal
            for v in (1, -1, lim, -lim - 1):
                check([v if i == d else 0 for i in range(S)], S, DB)


@pytest.mark.parametrize("DB", (7, 8))
def test_combine_dd_cancellation(DB):
    """Leading diagonals that cancel against the carries of the following
    ones (the sum is many orders below its largest term)."""
    rng = random.Random(99 + DB)
    for S in PLANES[DB]:
        if S < 3:
            continue
        for _ in range(300):
            D = [0] * S
            k = rng.randint(1, S - 1)
            # D_{k-1} 2^-DB(k-1) = -(D_k 2^-DB k) up to a residue
            D[k] = rng.randint(-(1 << 30), 1 << 30) << DB >> DB << DB   # multiple of 2^DB
            D[k - 1] = -(D[k] >> DB) + rng.choice((0, 0, 1, -1))
            for j in range(k + 1, S):
                D[j] = rng.randint(-(1 << 31) + 1, (1 << 31) - 1) if rng.random() < 0.7 else 0
            check(D, S, DB)
        # top = -1 with the lower digits all ones: the sum is -1 unit of the last place
        D = [0] * S
        D[0] = -1
        for j in range(1, S):
            D[j] = (1 << DB) - 1
        D[S - 1] = (1 << DB) - 1
        check(D, S, DB)
