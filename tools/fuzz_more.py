"""Dev tool: random scaling-and-squaring exponentials and Pade pairs: batch == singles bitwise, exp(A) exp(-A)
close to I; SUMMA on a 1 x 1 grid (NCCL, one rank) against the CPU oracle at random ragged sizes."""
import sys, os, time, socket
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import oracle
import paper_2312_17396_b200 as mp
from paper_2312_17396_b200 import summa
from paper_2312_17396_b200.precision import MatBatch
from _util import synth

N = int(sys.argv[1]) if len(sys.argv) > 1 else 40
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 0)
bad = 0
t0 = time.time()
for it in range(N):
    d = int(rng.choice([15, 31]))
    n = int(rng.integers(2, 80))
    B = int(rng.integers(2, 6))
    norms = 10.0 ** rng.uniform(-2, 2.5, size=B)
    A = np.stack([synth(n, float(norms[b]), int(rng.integers(1 << 30))) for b in range(B)])
    ctx = mp.PrecisionCtx(d)
    tag = f"#{it} expm d={d} n={n} B={B} lognorms={np.round(np.log10(norms), 1)}"
    try:
        reps = mp.expm_ss(A, ctx)
        b = int(rng.integers(B))
        solo = mp.expm_ss(A[b], ctx)
        if not torch.equal(solo.result.data[:, 0], reps.result.data[:, b]):
            bad += 1
            print("INVARIANCE", tag, b, flush=True)
        if norms[b] < 30:
            E = reps.result.data[:, b].double().sum(0).cpu().numpy()
            Em = mp.expm_ss(-A[b], ctx).result.data[:, 0].double().sum(0).cpu().numpy()
            res = np.abs(E @ Em - np.eye(n)).sum(axis=0).max()
            cond = np.abs(E).sum(axis=0).max() * np.abs(Em).sum(axis=0).max()
            if not res <= 1e3 * n * max(10.0 ** -d, 2.3e-16) * cond:     # fp64 check of the product
                bad += 1
                print("INVERSE", tag, b, res, cond, flush=True)
    except Exception as e:
        bad += 1
        print("EXC", tag, type(e).__name__, str(e)[:200], flush=True)
    k = int(rng.integers(2, 20))
    X = np.stack([synth(n, float(10.0 ** rng.uniform(-3, 0.8)), int(rng.integers(1 << 30))) for b in range(B)])
    tag = f"#{it} pade d={d} n={n} B={B} k={k}"
    try:
        num, den = mp.ps_mixed_pade(X, k, ctx)
        b = int(rng.integers(B))
        n1, d1 = mp.ps_mixed_pade(X[b], k, ctx)
        if not (torch.equal(n1.result.data[:, 0], num.result.data[:, b]) and torch.equal(d1.result.data[:, 0], den.result.data[:, b])):
            bad += 1
            print("INVARIANCE", tag, b, flush=True)
    except Exception as e:
        bad += 1
        print("EXC", tag, type(e).__name__, str(e)[:200], flush=True)
print(f"{N} expm + Pade rounds, {bad} failures, {time.time() - t0:.0f} s")

import torch.distributed as dist
s = socket.socket(); s.bind(("127.0.0.1", 0)); port = s.getsockname()[1]; s.close()
dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1)
grid = summa.ProcessGrid(1, 1)
bad2 = 0
for it in range(max(4, N // 4)):
    n = int(rng.integers(3, 200))
    m = int(rng.integers(4, 30))
    norm = float(10.0 ** rng.uniform(-2, 0.7))
    X = synth(n, norm, int(rng.integers(1 << 30)))
    ctx = mp.PrecisionCtx(31)
    series = mp.taylor_exp_coeffs(m)
    tag = f"#{it} summa n={n} m={m} norm={norm:.3g}"
    try:
        blk = MatBatch(torch.from_numpy(X).cuda()[None, None].contiguous().view(1, 1, n, n), mp.FP64)
        Xdd = MatBatch.empty(31, 1, n, device="cuda")
        from paper_2312_17396_b200 import _lib
        _lib.handle_for().convert(blk, Xdd)
        res = summa.ps_mixed_dist(Xdd, series, ctx, grid, summa.DeviceOps())
        ref = oracle.ps_eval(X, series.coeffs, 31)
        if tuple(res.digits) != tuple(ref.digits):
            bad2 += 1
            print("SCHEDULE", tag, res.digits, ref.digits, flush=True)
            continue
        diff, refn = ref.compare(res.block.data[:, 0].double().cpu().numpy())
        pabs = float(sum(abs(c) * norm ** k for k, c in enumerate(series.coeffs)))
        if not diff <= 10 * max(m // int(np.ceil(np.sqrt(m))), 1) * n * 1e-31 * max(refn, pabs):
            bad2 += 1
            print("VALUE", tag, diff / refn, flush=True)
    except Exception as e:
        bad2 += 1
        print("EXC", tag, type(e).__name__, str(e)[:200], flush=True)
dist.destroy_process_group()
print(f"summa 1x1: {bad2} failures")
