"""8-bit 14-plane dd GEMM under the kernel selected by MPPS_OZ_PW16 / MPPS_OZ_WIDE (dev tool):
time (CUDA events, best of 7), debug-flag variants and a checksum of the result bits so that
runs of different kernels can be compared for bitwise equality."""
import os, sys, hashlib
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2312_17396_b200 import _lib
from paper_2312_17396_b200.precision import MatBatch

h = _lib.handle_for()
tag = f"wide={os.environ.get('MPPS_OZ_WIDE', '1')} pw16={os.environ.get('MPPS_OZ_PW16', '1')}"
flagsets = ((0, "full"),) if "flags" not in sys.argv else ((0, "full"), (1, "no MMA (feed + epilogue)"), (2, "no loads (MMA + epilogue)"), (4, "no epilogue"), (5, "feed only"))
SHAPES = ((1, 8192),) if "big" in sys.argv else ((64, 256), (16, 1024), (4, 2048))
for B, n in SHAPES:
    torch.manual_seed(1)
    A = MatBatch.empty(31, B, n, device="cuda")
    A.data.normal_()
    A.data[1:] *= 1e-17
    C = MatBatch.empty(31, B, n, device="cuda")
    sa, sb = h.slice(A, 0, 14, None, 8), h.slice(A, 1, 14, None, 8)
    for flags, what in flagsets:
        h.lib.mpps_debug_oz_flags(flags)
        C.data.zero_()
        h.gemm_sliced(sa, sb, 14, C)
        torch.cuda.synchronize()
        digest = hashlib.sha1(C.data.cpu().numpy().tobytes()).hexdigest()[:12] if flags == 0 else "-"
        best = 1e9
        for _ in range(7):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(); h.gemm_sliced(sa, sb, 14, C); b.record(); torch.cuda.synchronize()
            best = min(best, a.elapsed_time(b))
        tops = 2.0 * B * n ** 3 * 105 / (best * 1e-3) / 1e12
        print(f"{tag} B={B} n={n} {what}: {best*1e3:.1f} us  {tops:.0f} TOPS  sha {digest}", flush=True)
    h.lib.mpps_debug_oz_flags(0)
