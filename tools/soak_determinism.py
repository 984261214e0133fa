"""Dev tool: run every tensor-core kernel class many times on the same operands (while a second
stream keeps the GPU busy with copies, to vary the timing) and require bit-identical results --
a missed barrier or a ring-slot race in the TMA / MMA / epilogue pipelines shows up as a checksum
that changes between launches."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2312_17396_b200 import _lib
from paper_2312_17396_b200.precision import MatBatch

h = _lib.handle_for()
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 100
side = torch.cuda.Stream()
noise_a = torch.empty(64 << 20, dtype=torch.uint8, device="cuda")
noise_b = torch.empty(64 << 20, dtype=torch.uint8, device="cuda")


def mk(fmt, B, rows, cols=None):
    M = MatBatch.empty(fmt, B, rows, cols, device="cuda")
    M.data[0].normal_()
    for w in range(1, M.words):
        M.data[w] = M.data[0] * 2.0 ** (-53 * w) * 0.37
    return M


def soak(label, fn, out):
    fn(); torch.cuda.synchronize()
    ref = out.data.clone()
    bad = 0
    for i in range(reps):
        if i % 3 == 0:
            with torch.cuda.stream(side):
                noise_b.copy_(noise_a)
        out.data.zero_()
        fn()
        if not torch.equal(out.data, ref):
            bad += 1
    torch.cuda.synchronize()
    print(f"{label}: {reps} launches, {bad} differing", flush=True)
    return bad


total = 0
for fmt, B, n, db in ((31, 64, 256, 8), (31, 16, 1024, 8), (31, 3, 200, 8), (31, 1, 4096, 8), (63, 2, 512, 8), (63, 1, 1024, 8),
                      (15, 8, 512, 8), (31, 1, 8192, 8)):
    S = h.slices_for(fmt, db)
    A = mk(fmt, B, n)
    C = MatBatch.empty(fmt, B, n, device="cuda")
    sa, sb = h.slice(A, 0, S, None, db), h.slice(A, 1, S, None, db)
    total += soak(f"gemm fmt={fmt} B={B} n={n} S={S}", lambda: h.gemm_sliced(sa, sb, S, C), C)
    del A, C, sa, sb
# fused Horner levels at cfg2 / cfg3 shapes and a cfg5-shaped few-plane level
for B, n in ((64, 256), (16, 1024), (1, 4096)):
    Y = mk(31, B, n)
    ysb = h.slice(Y, 1, 14, None, 8)
    Bp = mk(31, B, n)
    for S, fin, fout in ((10, 31, 31), (5, 15, 31), (2, 7, 15), (2, 7, 7), (3, 7, 7)):
        Pm = mk(fin, B, n)
        out = MatBatch.empty(fout, B, n, device="cuda")
        ps = h.slice(Pm, 0, S, None, 8)
        total += soak(f"horner B={B} n={n} S={S} -> fmt {fout}", lambda: h.horner_step_sliced(ps, ysb, S, Bp, out, fmt_in=fin), out)
print("TOTAL differing", total)
sys.exit(1 if total else 0)
