"""Per-tile phase timeline of the persistent dd GEMM (oz_gemm_pw16_kernel; dev tool):
MMA issue start / end (issuer thread), accumulators complete, TMEM released, tile stored
(epilogue warp 2), from mpps_debug_oz_trace (8 slots per tile)."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2312_17396_b200 import _lib
from paper_2312_17396_b200.precision import MatBatch

h = _lib.handle_for()
flags = int(sys.argv[1]) if len(sys.argv) > 1 else 0
h.lib.mpps_debug_oz_flags(flags)
print("debug flags", flags)
for B, n in ((64, 256), (16, 1024)):
    A = MatBatch.empty(31, B, n, device="cuda"); A.data.normal_(); A.data[1:] *= 1e-17
    C = MatBatch.empty(31, B, n, device="cuda")
    sa, sb = h.slice(A, 0, 14, None, 8), h.slice(A, 1, 14, None, 8)
    nt = B * (n // 128) * (n // 32)
    buf = torch.zeros(nt * 8, dtype=torch.int64, device="cuda")
    h.gemm_sliced(sa, sb, 14, C); torch.cuda.synchronize()
    h.lib.mpps_debug_oz_trace(buf.data_ptr())
    h.gemm_sliced(sa, sb, 14, C); torch.cuda.synchronize()
    h.lib.mpps_debug_oz_trace(None)
    t = buf.view(nt, 8).cpu().numpy().astype(np.float64)
    t0 = t[:, 0].min()
    i0, i1, full, rel, done, sm = (t[:, k] - (t0 if k < 5 else 0) for k in range(6))
    print(f"B={B} n={n}: span {(done.max())/1e3:.1f} us over {nt} tiles")
    print(f"  MMA issue {np.median(i1 - i0)/1e3:.2f} us; drain (issue end -> accumulators complete) {np.median(full - i1)/1e3:.2f} us; "
          f"accumulators complete -> TMEM released {np.median(rel - full)/1e3:.2f} us; released -> stored {np.median(done - rel)/1e3:.2f} us")
    # per SM: next tile's issue start after this tile's release
    lag, per = [], []
    for m in np.unique(sm):
        idx = np.where(sm == m)[0]
        o = idx[np.argsort(i0[idx])]
        lag += list(i0[o][1:] - rel[o][:-1])
        per += list(i0[o][1:] - i0[o][:-1])
    print(f"  released -> next tile's first MMA issued {np.median(lag)/1e3:.2f} us; tile period {np.median(per)/1e3:.2f} us")

# fused Horner levels (mode 1): phi (row-split, S planes) x Y (column-split) + B_prev
B, n = 64, 256
Y = MatBatch.empty(31, B, n, device="cuda"); Y.data.normal_(); Y.data[1:] *= 1e-17
Bp = MatBatch.empty(31, B, n, device="cuda"); Bp.data.normal_(); Bp.data[1:] *= 1e-17
ysb = h.slice(Y, 1, 14, None, 8)
for S, fin, fout in ((10, 31, 31), (5, 15, 31), (2, 7, 15), (2, 7, 7)):
    Pm = MatBatch.empty(fin, B, n, device="cuda"); Pm.data.normal_()
    if Pm.words > 1:
        Pm.data[1:] *= 1e-17
    out = MatBatch.empty(fout, B, n, device="cuda")
    ps = h.slice(Pm, 0, S, None, 8)
    nt = B * (n // 128) * (n // 32)
    buf = torch.zeros(nt * 8, dtype=torch.int64, device="cuda")
    fn = lambda: h.horner_step_sliced(ps, ysb, S, Bp, out, fmt_in=fin)
    fn(); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); fn(); b.record(); torch.cuda.synchronize()
    h.lib.mpps_debug_oz_trace(buf.data_ptr())
    fn(); torch.cuda.synchronize()
    h.lib.mpps_debug_oz_trace(None)
    t = buf.view(nt, 8).cpu().numpy().astype(np.float64)
    t0 = t[:, 0].min()
    i0, i1, full, rel, done, sm = (t[:, k] - (t0 if k < 5 else 0) for k in range(6))
    per = []
    for m in np.unique(sm):
        idx = np.where(sm == m)[0]
        o = idx[np.argsort(done[idx])]
        per += list(done[o][1:] - done[o][:-1])
    print(f"Horner S={S} -> fmt {fout}: {a.elapsed_time(b)*1e3:.1f} us; MMA issue {np.median(i1 - i0)/1e3:.2f} us; "
          f"acc complete -> released {np.median(rel - full)/1e3:.2f} us; released -> stored {np.median(done - rel)/1e3:.2f} us; "
          f"issue end -> acc seen by the epilogue {np.median(full - i1)/1e3:.2f} us; tile period {np.median(per)/1e3:.2f} us")
