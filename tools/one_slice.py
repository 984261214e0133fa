"""Run the cfg2 dd digit splits (rows and columns, 14 planes, 8-bit digits, 64 x 256^2) a few
times: the ncu target for slice_rows_kernel<2,14> / slice_cols_kernel<2,14>."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2312_17396_b200 import _lib
from paper_2312_17396_b200.precision import MatBatch

h = _lib.handle_for()
A = MatBatch.empty(31, 64, 256, device="cuda"); A.data.normal_()
A.data[1:] *= 1e-17
for _ in range(3):
    h.slice(A, 0, 14, None, 8)
    h.slice(A, 1, 14, None, 8)
torch.cuda.synchronize()
print("ok")
