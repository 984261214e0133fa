"""One tensor-core GEMM config, a few launches (for ncu captures):
python tools/one_gemm.py FMT B N [reps]   (MPPS_OZ_WIDE / MPPS_OZ_PW16 select the kernel)"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2312_17396_b200 import _lib
from paper_2312_17396_b200.precision import MatBatch

fmt, B, n = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 2
h = _lib.handle_for()
A = MatBatch.empty(fmt, B, n, device="cuda")
A.data.normal_()
if A.words > 1:
    A.data[1:] *= 1e-17
C = MatBatch.empty(fmt, B, n, device="cuda")
from paper_2312_17396_b200 import gemm_engine
db = gemm_engine.digit_bits_for(h, n)       # the engine's digit width for this K
S = h.slices_for(fmt, db)
sa, sb = h.slice(A, 0, S, None, db), h.slice(A, 1, S, None, db)
for _ in range(reps):
    h.gemm_sliced(sa, sb, S, C)
torch.cuda.synchronize()
print("ok")
