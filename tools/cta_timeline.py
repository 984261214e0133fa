"""Per-CTA phase timeline of the TMA tensor-core GEMMs (dev tool).
Uses mpps_debug_oz_trace: start, setup done, MMAs done, end (globaltimer)."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2312_17396_b200 import _lib
from paper_2312_17396_b200.precision import MatBatch

h = _lib.handle_for()
lib = h.lib
B, n = 64, 256


def run(label, fn, nctas):
    buf = torch.zeros(nctas * 8, dtype=torch.int64, device="cuda")
    fn(); torch.cuda.synchronize()
    lib.mpps_debug_oz_trace(buf.data_ptr())
    fn(); torch.cuda.synchronize()
    lib.mpps_debug_oz_trace(None)
    t = buf.view(nctas, 8).cpu().numpy()
    t0 = t[:, 0].min()
    st, su, dn, en, sm = (t[:, i] - (t0 if i < 4 else 0) for i in range(5))
    span = en.max()
    per_sm = np.bincount(sm.astype(np.int64), minlength=148)
    print(f"{label}: span {span/1e3:.1f} us, CTAs {nctas}, per-SM CTAs {per_sm.min()}..{per_sm.max()}; "
          f"setup {np.median(su - st)/1e3:.2f} us, mainloop {np.median(dn - su)/1e3:.2f} us, "
          f"epilogue {np.median(en - dn)/1e3:.2f} us, CTA total {np.median(en - st)/1e3:.2f} us; "
          f"start-time spread: first wave ends {np.sort(en)[147]/1e3:.1f} us", flush=True)
    if t[:, 5].any():
        c5, c6, c7 = (t[:, i] - t0 for i in (5, 6, 7))
        print(f"    epilogue (thread 64): combine {np.median(c5 - dn)/1e3:.2f} us, sync {np.median(c6 - c5)/1e3:.2f} us, "
              f"store {np.median(c7 - c6)/1e3:.2f} us, exit sync {np.median(en - c7)/1e3:.2f} us", flush=True)
    # gaps between consecutive CTAs of one SM
    gaps = []
    for m in np.unique(sm):
        idx = np.where(sm == m)[0]
        o = idx[np.argsort(st[idx])]
        gaps += list(st[o][1:] - en[o][:-1])
    if gaps:
        print(f"    gap between consecutive CTAs of an SM: median {np.median(gaps)/1e3:.2f} us", flush=True)
    # concurrency: average CTAs resident
    ev = np.concatenate([np.stack([st, np.ones_like(st)], 1), np.stack([en, -np.ones_like(en)], 1)])
    ev = ev[np.argsort(ev[:, 0], kind="stable")]
    conc = np.cumsum(ev[:, 1])
    dt = np.diff(ev[:, 0])
    print(f"    mean resident CTAs {np.sum(conc[:-1] * dt) / span:.1f}", flush=True)


Y = MatBatch.empty(31, B, n, device="cuda"); Y.data.normal_(); Y.data[1:] *= 1e-17
P = MatBatch.empty(7, B, n, device="cuda"); P.data.normal_()
P64 = MatBatch.empty(15, B, n, device="cuda"); P64.data.normal_()
Bp = MatBatch.empty(31, B, n, device="cuda"); Bp.data.normal_(); Bp.data[1:] *= 1e-17
o32 = MatBatch.empty(7, B, n, device="cuda")
o64 = MatBatch.empty(15, B, n, device="cuda")
o128 = MatBatch.empty(31, B, n, device="cuda")
ys = h.slice(Y, 0, 16)
ysb = h.slice(Y, 1, 16)
ps4, ps8 = h.slice(P, 1, 4), h.slice(P64, 1, 8)
nct = B * (n // 128) * (n // 32)
ys14, ysb14 = h.slice(Y, 0, 14, None, 8), h.slice(Y, 1, 14, None, 8)
run("S=14 (8-bit) gemm dd", lambda: h.gemm_sliced(ys14, ysb14, 14, o128), nct)
run("S=14 (8-bit) horner dd", lambda: h.horner_step_sliced(ys14, ysb14, 14, Bp, o128, fmt_in=31), nct)
if len(sys.argv) > 1:
    sys.exit(0)
run("S=16 gemm dd", lambda: h.gemm_sliced(ys, ysb, 16, o128), nct)
run("S=16 horner dd", lambda: h.horner_step_sliced(ys, ysb, 16, Bp, o128, fmt_in=31), nct)
run("S=8 horner fp64", lambda: h.horner_step_sliced(ys, ps8, 8, Bp, o64, fmt_in=15), nct)
run("S=4 gemm fp32", lambda: h.gemm_sliced(ys, ps4, 4, o32), nct)
run("S=4 horner fp32", lambda: h.horner_step_sliced(ys, ps4, 4, Bp, o32, fmt_in=7), nct)

for flags, lab in ((1, "feed only"), (2, "MMA only")):
    lib.mpps_debug_oz_flags(flags)
    run(f"S=16 gemm dd [{lab}]", lambda: h.gemm_sliced(ys, ysb, 16, o128), nct)
    run(f"S=4 gemm fp32 [{lab}]", lambda: h.gemm_sliced(ys, ps4, 4, o32), nct)
lib.mpps_debug_oz_flags(0)
Yb = MatBatch.empty(31, 16, 1024, device="cuda"); Yb.data.normal_(); Yb.data[1:] *= 1e-17
ob = MatBatch.empty(31, 16, 1024, device="cuda")
yb0, yb1 = h.slice(Yb, 0, 16), h.slice(Yb, 1, 16)
nb = 16 * 8 * 32
for flags, lab in ((0, "normal"), (1, "feed only"), (2, "MMA only")):
    lib.mpps_debug_oz_flags(flags)
    run(f"S=16 gemm dd n=1024 [{lab}]", lambda: h.gemm_sliced(yb0, yb1, 16, ob), nb)
lib.mpps_debug_oz_flags(0)
