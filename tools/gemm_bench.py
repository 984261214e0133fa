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
    from paper_2312_17396_b200 import gemm_engine
    db = gemm_engine.digit_bits_for(h, n)
    S = h.slices_for(fmt, db)
    sa, sb = h.slice(A, 0, S, None, db), h.slice(A, 1, S, None, db)
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
    ts = t(lambda: (h.slice(A, 0, S, None, db), h.slice(A, 1, S, None, db)))
    tf = 2.0 * B * n ** 3 / tg / 1e12
    pairs = S * (S + 1) // 2
    tops = 2.0 * B * n ** 3 * pairs / tg / 1e12
    print(f"TC fmt={fmt} S={S} B={B} n={n}: gemm {tg*1e3:.3f} ms ({tf:.2f} TFLOP/s logical, {tops:.0f} int8 TOPS), "
          f"slicing A+B {ts*1e3:.3f} ms", flush=True)


if __name__ == "__main__" and len(sys.argv) > 1 and sys.argv[1] == "tc":
    for fmt, B, n in ((31, 64, 256), (31, 16, 1024), (31, 1, 2048), (31, 1, 8192), (15, 64, 256), (15, 1, 4096),
                      (63, 1, 1024), (63, 1, 2048)):
        bench_tc(fmt, B, n)


if __name__ == "__main__" and len(sys.argv) > 1 and sys.argv[1] == "sweep":
    # fixed per-tile cost vs per-K-step cost of the TC kernels
    for fmt in (7, 15, 31):
        for B, n in ((64, 64), (64, 128), (64, 256), (64, 512), (16, 1024), (4, 2048)):
            bench_tc(fmt, B, n)


if __name__ == "__main__" and len(sys.argv) > 1 and sys.argv[1] == "horner":
    # fused Horner step vs plain GEMM on the same slices (cfg2 fp32 level)
    h = _lib.handle_for()
    B, n = 64, 256
    Y = MatBatch.empty(31, B, n, device="cuda"); Y.data.normal_(); Y.data[1:] *= 1e-17
    P = MatBatch.empty(7, B, n, device="cuda"); P.data.normal_()
    Bp = MatBatch.empty(31, B, n, device="cuda"); Bp.data.normal_(); Bp.data[1:] *= 1e-17
    out = MatBatch.empty(7, B, n, device="cuda")
    for SA, fo in ((16, 7), (4, 7)):
        ys = h.slice(Y, 0, SA)
        ps = h.slice(P, 1, 4)
        e_in = torch.zeros(B, dtype=torch.int32, device="cuda")
        e_out = torch.zeros(B, dtype=torch.int32, device="cuda")

        def t(fn, reps=10):
            fn(); torch.cuda.synchronize()
            best = 1e9
            for _ in range(reps):
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(); fn(); b.record(); torch.cuda.synchronize()
                best = min(best, a.elapsed_time(b))
            return best * 1e3
        print(f"Y planes {SA}: gemm_sliced S=4 {t(lambda: h.gemm_sliced(ys, ps, 4, out)):.1f} us; "
              f"horner no exps {t(lambda: h.horner_step_sliced(ys, ps, 4, Bp, out, fmt_in=7)):.1f} us; "
              f"horner exps {t(lambda: h.horner_step_sliced(ys, ps, 4, Bp, out, None, None, e_in, e_out, fmt_in=7)):.1f} us",
              flush=True)


if __name__ == "__main__" and len(sys.argv) > 1 and sys.argv[1] == "horner32":
    # fp32 Horner level: SIMT FFMA kernel vs INT8 tensor cores (S = 4)
    h = _lib.handle_for()
    B, n = 64, 256
    Y = MatBatch.empty(31, B, n, device="cuda"); Y.data.normal_(); Y.data[1:] *= 1e-17
    Y32 = MatBatch.empty(7, B, n, device="cuda"); h.convert(Y, Y32)
    P = MatBatch.empty(7, B, n, device="cuda"); P.data.normal_()
    Bp = MatBatch.empty(31, B, n, device="cuda"); Bp.data.normal_(); Bp.data[1:] *= 1e-17
    out = MatBatch.empty(7, B, n, device="cuda")
    ys, ps = h.slice(Y, 0, 16), h.slice(P, 1, 4)

    def t(fn, reps=10):
        fn(); torch.cuda.synchronize()
        best = 1e9
        for _ in range(reps):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(); fn(); b.record(); torch.cuda.synchronize()
            best = min(best, a.elapsed_time(b))
        return best * 1e3
    print(f"fp32 level: simt horner {t(lambda: h.horner_step(Y32, P, Bp, out)):.1f} us "
          f"(+ convert Y {t(lambda: h.convert(Y, Y32)):.1f} us); tc horner {t(lambda: h.horner_step_sliced(ys, ps, 4, Bp, out, fmt_in=7)):.1f} us "
          f"(+ slice phi {t(lambda: h.slice(P, 1, 4)):.1f} us); simt gemm {t(lambda: h.gemm(Y32, P, out)):.1f} us", flush=True)
    Y64 = MatBatch.empty(15, B, n, device="cuda"); h.convert(Y, Y64)
    P64 = MatBatch.empty(15, B, n, device="cuda"); P64.data.normal_()
    o64 = MatBatch.empty(15, B, n, device="cuda")
    ps8 = h.slice(P64, 1, 8)
    print(f"fp64 level: simt horner {t(lambda: h.horner_step(Y64, P64, Bp, o64)):.1f} us; "
          f"tc horner {t(lambda: h.horner_step_sliced(ys, ps8, 8, Bp, o64, fmt_in=15)):.1f} us", flush=True)


if __name__ == "__main__" and len(sys.argv) > 1 and sys.argv[1] == "big":
    for fmt, B, n in ((31, 1, 8192), (63, 1, 2048), (31, 16, 1024), (31, 64, 256)):
        bench_tc(fmt, B, n, reps=3)


if __name__ == "__main__" and len(sys.argv) > 1 and sys.argv[1] == "group":
    # raster group size, interleaved in one process (per-process variance)
    import itertools
    shapes = ((31, 1, 8192), (63, 1, 2048), (31, 16, 1024), (31, 64, 256))
    G = (1, 2, 4, 8, 16)
    h = _lib.handle_for()
    res = {}
    setups = {}
    for fmt, B, n in shapes:
        A = MatBatch.empty(fmt, B, n, device="cuda"); A.data.normal_()
        if A.words > 1:
            A.data[1:] *= 1e-17
        C = MatBatch.empty(fmt, B, n, device="cuda")
        S = h.slices_for(fmt)
        setups[(fmt, B, n)] = (h.slice(A, 0, S), h.slice(A, 1, S), S, C)
    for rep in range(3):
        for g in G:
            h.lib.mpps_debug_oz_flags(g << 8)
            for key, (sa, sb, S, C) in setups.items():
                h.gemm_sliced(sa, sb, S, C); torch.cuda.synchronize()
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(); h.gemm_sliced(sa, sb, S, C); b.record(); b.synchronize()
                res.setdefault((key, g), []).append(a.elapsed_time(b))
    h.lib.mpps_debug_oz_flags(0)
    for key in setups:
        print(key, " ".join(f"G={g}:{min(res[(key, g)]):.3f}ms" for g in G), flush=True)
