"""Dev tool: the operator mat_mul (mpps_gemm on plain matrices, the library splits internally) at random
ragged M x K x N, formats, badly scaled rows / columns, zero rows, against the CPU oracle's mat_mul
(entrywise: |C - C_oracle| <= 4 K u |A| |B| + the digit-plane truncation term, below)."""
import sys, os, time
from fractions import Fraction
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle
from paper_2312_17396_b200 import _lib, ops
from paper_2312_17396_b200.precision import MatBatch

N_ = int(sys.argv[1]) if len(sys.argv) > 1 else 60
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 0)
h = _lib.handle_for()
bad = 0
t0 = time.time()

def words_of(fmt, A):
    if fmt in (7, 15):
        return (A.astype(np.float32).astype(np.float64) if fmt == 7 else A)[None]
    lo = A * 2.0 ** -60 * rng.standard_normal(A.shape)
    w = [A, lo]
    if fmt == 63:
        w += [lo * 2.0 ** -60, lo * 2.0 ** -121]
    return np.stack(w)

for it in range(N_):
    fmt, bits = [(7, 24), (15, 53), (31, 106), (63, 212)][int(rng.integers(4))]
    M, K, N = (int(x) for x in rng.integers(1, 260 if fmt != 63 else 120, size=3))
    spread = float(rng.uniform(0, 40))
    A = rng.standard_normal((M, K)) * np.exp(rng.uniform(-spread, spread, (M, 1)))
    B = rng.standard_normal((K, N)) * np.exp(rng.uniform(-spread, spread, (1, N)))
    if rng.integers(3) == 0:
        A[int(rng.integers(M))] = 0.0
        B[:, int(rng.integers(N))] = 0.0
    if rng.integers(3) == 0:      # entries far below their row maximum
        A *= np.exp(rng.uniform(-30, 0, A.shape))
    Aw, Bw = words_of(fmt, A), words_of(fmt, B)
    tag = f"#{it} fmt={fmt} {M}x{K}x{N} spread=e^{spread:.0f}"
    try:
        Ad, Bd = ops.from_numpy(Aw, fmt), ops.from_numpy(Bw, fmt)
        C = MatBatch.empty(fmt, 1, M, N, device="cuda")
        h.gemm(Ad, Bd, C)
        got = C.data[:, 0].double().cpu().numpy()
        n = max(M, N, K)
        Ap = np.zeros((Aw.shape[0], n, n)); Ap[:, :M, :K] = Aw
        Bp = np.zeros((Bw.shape[0], n, n)); Bp[:, :K, :N] = Bw
        Co = oracle.matmul(Ap, Bp, bits)[:, :M, :N]
        absAB = np.abs(Aw[0]) @ np.abs(Bw[0])
        u = Fraction(1, 2 ** bits)
        worst = 0.0
        for _ in range(60):
            i, j = int(rng.integers(M)), int(rng.integers(N))
            g = sum(Fraction(float(x)) for x in got[:, i, j])
            o = sum(Fraction(float(x)) for x in Co[:, i, j])
            # entrywise 4 K u |A| |B|, plus the digit-plane truncation: every operand entry is cut at
            # 2^-(8 S - 2) of its ROW (column) maximum, so an entry far below that maximum carries
            # fewer bits than its own format (the scheme's error is normwise per row and column)
            S = {7: 4, 15: 8, 31: 14, 63: 28}[fmt]
            trunc = 2 * K * Fraction(1, 2 ** (8 * S - 2)) * Fraction(float(np.abs(Aw[0][i]).max())) * Fraction(float(np.abs(Bw[0][:, j]).max()))
            lim = 4 * K * u * Fraction(float(absAB[i, j])) + trunc
            if abs(g - o) > lim:
                bad += 1
                print("VALUE", tag, (i, j), float(g - o), float(lim), flush=True)
                break
    except Exception as e:
        bad += 1
        print("EXC", tag, type(e).__name__, str(e)[:200], flush=True)
print(f"{N_} products, {bad} failures, {time.time() - t0:.0f} s")
