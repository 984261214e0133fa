"""fp64-precision product (8 planes of 8 bits) at K = 8192 (cfg5's Y = Z^5): dev tool."""
import os, sys, hashlib
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2312_17396_b200 import _lib
from paper_2312_17396_b200.precision import MatBatch
h = _lib.handle_for()
n = 8192
torch.manual_seed(3)
A = MatBatch.empty(31, 1, n, device="cuda"); A.data.normal_(); A.data[1:] *= 1e-17
C = MatBatch.empty(15, 1, n, device="cuda")
sa, sb = h.slice(A, 0, 8, None, 8), h.slice(A, 1, 8, None, 8)
h.gemm_sliced(sa, sb, 8, C); torch.cuda.synchronize()
sha = hashlib.sha1(C.data.cpu().numpy().tobytes()).hexdigest()[:12]
best = 1e9
for _ in range(5):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); h.gemm_sliced(sa, sb, 8, C); b.record(); torch.cuda.synchronize()
    best = min(best, a.elapsed_time(b))
print(f"{os.path.basename(_lib.LIB_PATH)}: fp64 product 8192^3, 8 planes: {best:.3f} ms {2.0*n**3*36/(best*1e-3)/1e12:.0f} TOPS sha {sha}")
