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


def _two_sum(a, b):
    s = a + b
    bb = s - a
    return s, (a - (s - bb)) + (b - bb)


def combine_qd(D, S, DB):
    """csrc/ozaki.cuh::combine_qd, operation for operation."""
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
    dig, c = [0] * NG, 0
    for g in range(NG - 1, 0, -1):
        t = G[g] + c
        dig[g] = t & ((1 << WB) - 1)
        c = t >> WB
    q0 = 12 + DB * 2
    NP = 1 + NG // 2
    p = [_u52_scaled(G[0] + c + (1 << 51), q0, 2.0 ** (51 - q0))]
    for K in range(1, NP):
        a = 2 * K - 1
        if a + 1 < NG:
            p.append(_u52_scaled((dig[a] << WB) | dig[a + 1], 12 + DB * (3 * (a + 1) + 2)))
        else:
            p.append(_u52_scaled(dig[a], 12 + DB * (3 * a + 2)))
    for i in range(NP - 1, 0, -1):
        s = p[i - 1] + p[i]
        p[i] = p[i] - (s - p[i - 1])
        p[i - 1] = s
    for k in (1, 2):
        for i in range(NP - 1, 0, -1):
            p[i - 1], p[i] = _two_sum(p[i - 1], p[i])
    q = [p[0], p[1], p[2], 0.0]
    for i in range(NP - 1, 2, -1):
        q[3] += p[i]
    for _ in range(3):
        for i in range(3):
            if q[i] == 0.0:
                q[i], q[i + 1] = q[i + 1], 0.0
    return tuple(q)


def check_qd(D, S, DB):
    w = combine_qd(D, S, DB)
    V = exact(D, S, DB)
    got = sum(Fraction(x) for x in w)
    assert abs(got - V) <= abs(V) / (1 << 205), (S, DB, D)
    # word 0 is the value rounded to double (the digit splits take row / column maxima from
    # it) and word 1 lies below its last place; the lower words may overlap one another
    # mildly, as after mp::qd_renorm's three sweeps -- the sum is what the kernels use
    if V != 0:
        assert w[0] != 0.0 and abs(Fraction(w[0]) - V) <= Fraction(math.ulp(w[0])) / 2
        assert abs(w[1]) <= math.ulp(w[0]) / 2, (S, DB, D, w)
    nz = [x for x in w if x != 0.0]
    for a, b in zip(nz, nz[1:]):
        assert abs(b) < abs(a), (S, DB, D, w)
    # a zero word is followed only by zeros (no information behind a gap)
    seen_zero = False
    for x in w:
        if x == 0.0:
            seen_zero = True
        else:
            assert not seen_zero, (S, DB, D, w)


@pytest.mark.parametrize("DB,S", [(8, 28), (7, 31), (8, 12), (8, 10)])
def test_combine_qd(DB, S):
    rng = random.Random(4321 + DB + S)
    lim = (1 << 31) - 1
    for _ in range(400):
        check_qd([rng.randint(-lim, lim) for _ in range(S)], S, DB)
    for _ in range(200):
        check_qd([rng.randint(-(1 << rng.randint(0, 30)), 1 << rng.randint(0, 30)) for _ in range(S)], S, DB)
    check_qd([lim] * S, S, DB)
    check_qd([-lim - 1] * S, S, DB)
    check_qd([0] * S, S, DB)
    for d in range(S):
        for v in (1, -1, lim, -lim - 1):
            check_qd([v if i == d else 0 for i in range(S)], S, DB)
    for _ in range(300):          # cancelling leading diagonals
        D = [0] * S
        k = rng.randint(1, S - 1)
        D[k] = rng.randint(-(1 << 30), 1 << 30) >> DB << DB
        D[k - 1] = -(D[k] >> DB) + rng.choice((0, 0, 1, -1))
        for j in range(k + 1, S):
            D[j] = rng.randint(-lim, lim) if rng.random() < 0.7 else 0
        check_qd(D, S, DB)
    D = [0] * S
    D[0] = -1
    for j in range(1, S):
        D[j] = (1 << DB) - 1
    check_qd(D, S, DB)
