"""qd (28 planes of 8 bits) GEMM under the kernel selected by MPPS_OZ_WIDE (dev tool)."""
import os, sys, hashlib
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2312_17396_b200 import _lib
from paper_2312_17396_b200.precision import MatBatch
h = _lib.handle_for()
for B, n in ((4, 1024), (1, 2048)):
    torch.manual_seed(2)
    A = MatBatch.empty(63, B, n, device="cuda")
    A.data.normal_()
    for w in range(1, 4):
        A.data[w] *= 1e-17 ** w
    C = MatBatch.empty(63, B, n, device="cuda")
    sa, sb = h.slice(A, 0, 28, None, 8), h.slice(A, 1, 28, None, 8)
    h.gemm_sliced(sa, sb, 28, C)
    torch.cuda.synchronize()
    sha = hashlib.sha1(C.data.cpu().numpy().tobytes()).hexdigest()[:12]
    best = 1e9
    for _ in range(5):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); h.gemm_sliced(sa, sb, 28, C); b.record(); torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b))
    print(f"wide={os.environ.get('MPPS_OZ_WIDE', '1')} mc={os.environ.get('MPPS_OZ_WIDE_MC', '1')} B={B} n={n}: {best*1e3:.1f} us "
          f"{2.0*B*n**3*406/(best*1e-3)/1e12:.0f} TOPS sha {sha}", flush=True)
