"""Persistent dd GEMM diagnostics: full / feed-only (no MMAs) / no epilogue /
MMA+feed only, per MPPS_OZ_PERS mode (dev tool)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2312_17396_b200 import _lib
from paper_2312_17396_b200.precision import MatBatch

h = _lib.handle_for()
for B, n in ((64, 256), (16, 1024)):
    A = MatBatch.empty(31, B, n, device="cuda")
    A.data.normal_()
    A.data[1:] *= 1e-17
    C = MatBatch.empty(31, B, n, device="cuda")
    sa, sb = h.slice(A, 0, 16), h.slice(A, 1, 16)
    for flags, what in ((0, "full"), (1, "no MMA"), (4, "no epilogue"), (5, "feed only")):
        h.lib.mpps_debug_oz_flags(flags)
        h.gemm_sliced(sa, sb, 16, C)
        torch.cuda.synchronize()
        best = 1e9
        for _ in range(5):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(); h.gemm_sliced(sa, sb, 16, C); b.record(); torch.cuda.synchronize()
            best = min(best, a.elapsed_time(b))
        print(f"pers={os.environ.get('MPPS_OZ_PERS', '2')} B={B} n={n} {what}: {best*1e3:.1f} us", flush=True)
    h.lib.mpps_debug_oz_flags(0)
