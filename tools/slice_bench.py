"""Time the digit-plane slicing kernels (dd, 64 x 256^2 and 16 x 1024^2)."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2312_17396_b200 import _lib
from paper_2312_17396_b200.precision import MatBatch

h = _lib.handle_for()
for fmt, S, db in ((31, 16, 7), (31, 14, 8), (15, 8, 7), (15, 8, 8), (7, 4, 7), (7, 4, 8)):
  for B, n in ((64, 256), (16, 1024)):
    A = MatBatch.empty(fmt, B, n, device="cuda"); A.data.normal_()
    if A.words > 1:
        A.data[1:] *= 1e-17
    res = []
    for side in (0, 1):
        h.slice(A, side, S, None, db); torch.cuda.synchronize()
        best = 1e9
        for _ in range(10):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(); h.slice(A, side, S, None, db); b.record(); b.synchronize()
            best = min(best, a.elapsed_time(b))
        res.append(best * 1e3)
    print(f"fmt={fmt} S={S} db={db} B={B} n={n}: rows {res[0]:.1f} us, cols {res[1]:.1f} us", flush=True)
