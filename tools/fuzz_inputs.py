"""Dev tool: the same matrices through different input forms -- fp64 arrays (graphed path), working-format
MatBatch inputs (eager path), complex arrays with a zero imaginary part, complex batches vs singles."""
import sys, os, time
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import paper_2312_17396_b200 as mp
from paper_2312_17396_b200 import _lib
from paper_2312_17396_b200.precision import MatBatch
from _util import synth

N = int(sys.argv[1]) if len(sys.argv) > 1 else 60
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 0)
bad = 0
t0 = time.time()
def words(rep):
    r = rep.result
    return r.data.double() if hasattr(r, "data") else None
for it in range(N):
    d = int(rng.choice([15, 31, 63]))
    n = int(rng.integers(2, 60 if d < 63 else 30))
    B = int(rng.integers(2, 5))
    m = int(rng.integers(2, 36))
    norms = 10.0 ** rng.uniform(-3, 0.9, size=B)
    X = np.stack([synth(n, float(norms[b]), int(rng.integers(1 << 30))) for b in range(B)])
    ctx = mp.PrecisionCtx(d)
    tag = f"#{it} d={d} n={n} B={B} m={m}"
    try:
        a = mp.ps_mixed_exp(X, m, ctx)
        wa = a.result.data.double()
        refn = wa[0].abs().sum(dim=1).amax(dim=1)       # (B,) one-norms of the leading words
        # working-format MatBatch input
        Xw = MatBatch.empty(ctx.fmt if ctx.fmt != 7 else 15, B, n, device="cuda")
        Xf = MatBatch(torch.from_numpy(X).cuda().unsqueeze(0), 15)
        _lib.handle_for().convert(Xf, Xw)
        b_ = mp.ps_mixed_exp(Xw, m, ctx)
        wb = b_.result.data.double()
        for b in range(B):
            if tuple(a[b].plan.level_digits) != tuple(b_[b].plan.level_digits):
                bad += 1; print("SCHEDULE matbatch", tag, b, a[b].plan.level_digits, b_[b].plan.level_digits, flush=True)
        diff = (wa - wb).sum(0).abs().sum(dim=1).amax(dim=1)
        tol = 10 * max(a[0].plan.r, 1) * n * 10.0 ** -d
        pabs = torch.tensor([float(sum(abs(c) * float(norms[b]) ** k for k, c in enumerate(mp.taylor_exp_coeffs(m).coeffs))) for b in range(B)], device="cuda", dtype=torch.float64)
        if not bool((diff <= tol * torch.maximum(refn, pabs)).all()):
            bad += 1; print("VALUE matbatch", tag, (diff / refn).tolist(), tol, flush=True)
        # complex input with zero imaginary part == real input (values), complex batch == singles (bits)
        if d <= 31:
            Xc = X.astype(np.complex128)
            c_ = mp.ps_mixed_exp(Xc, m, ctx)
            cz = c_.result.to_numpy() if hasattr(c_.result, "to_numpy") else None
            Xi = X + 1j * np.stack([synth(n, float(norms[b]) * 0.5, int(rng.integers(1 << 30))) for b in range(B)])
            ci = mp.ps_mixed_exp(Xi, m, ctx)
            b = int(rng.integers(B))
            cs = mp.ps_mixed_exp(Xi[b], m, ctx)
            ra, rb = ci[b].result, cs.result
            da = ra.emb.data if hasattr(ra, "emb") else ra.data
            db = rb.emb.data if hasattr(rb, "emb") else rb.data
            if not torch.equal(da.reshape(-1), db.reshape(-1)):
                bad += 1; print("INVARIANCE complex", tag, b, flush=True)
    except Exception as e:
        bad += 1
        print("EXC", tag, type(e).__name__, str(e)[:200], flush=True)
print(f"{N} cases, {bad} failures, {time.time() - t0:.0f} s")
