"""Microbenchmark of the GEMM kernels (dev tool): times mpps_gemm per format
with CUDA events.  MPPS_LIB selects an alternative build for A/B tests."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2312_17396_b200 import _lib
from paper_2312_17396_b200.precision import MatBatch


def bench(fmt, B, n, reps=5):
    h = _lib.handle_for()
    A = MatBatch.empty(fmt, B, n, device="cuda")
    A.data.normal_()
    if A.words > 1:
        A.data[1:] *= 1e-17
    C = MatBatch.empty(fmt, B, n, device="cuda")
    h.gemm(A, A, C)
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        h.gemm(A, A, C)
        b.record()
        torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b) * 1e-3)
    tf = 2.0 * B * n ** 3 / best / 1e12
    print(f"{os.path.basename(_lib.LIB_PATH)} fmt={fmt} B={B} n={n}: {best*1e3:.3f} ms  {tf:.3f} TFLOP/s logical",
          flush=True)


if __name__ == "__main__" and len(sys.argv) == 1:
    for fmt, B, n in ((31, 64, 256), (31, 1, 2048), (31, 16, 1024), (15, 64, 256), (15, 1, 4096), (7, 64, 256),
                      (7, 1, 4096), (63, 1, 1024)):
        bench(fmt, B, n)


def bench_tc(fmt, B, n, reps=5):
    h = _lib.handle_for()
    A = MatBatch.empty(fmt, B, n, device="cuda")
    A.data.normal_()
    if A.words > 1:
        A.data[1:] *= 1e-17
    C = MatBatch.empty(fmt, B, n, device="cuda")
    S = h.slices_for(fmt)
    sa, sb = h.slice(A, 0, S), h.slice(A, 1, S)
    h.gemm_sliced(sa, sb, S, C)
    torch.cuda.synchronize()

    def t(fn):
        best = 1e9
        for _ in range(reps):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            fn()
            b.record()
            torch.cuda.synchronize()
            best = min(best, a.elapsed_time(b) * 1e-3)
        return best
    tg = t(lambda: h.gemm_sliced(sa, sb, S, C))
    ts = t(lambda: (h.slice(A, 0, S), h.slice(A, 1, S)))
    tf = 2.0 * B * n ** 3 / tg / 1e12
    pairs = S * (S + 1) // 2
    tops = 2.0 * B * n ** 3 * pairs / tg / 1e12
    print(f"TC fmt={fmt} S={S} B={B} n={n}: gemm {tg*1e3:.3f} ms ({tf:.2f} TFLOP/s logical, {tops:.0f} int8 TOPS), "
          f"slicing A+B {ts*1e3:.3f} ms", flush=True)


if __name__ == "__main__" and len(sys.argv) > 1 and sys.argv[1] == "tc":
    for fmt, B, n in ((31, 64, 256), (31, 16, 1024), (31, 1, 2048), (31, 1, 8192), (15, 64, 256), (15, 1, 4096),
                      (63, 1, 1024), (63, 1, 2048)):
        bench_tc(fmt, B, n)
