"""tcgen05.mma kind::i8 cost per instruction vs N (M = 128, K = 32)."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2312_17396_b200 import _lib

h = _lib.handle_for()
scratch = torch.zeros(16, dtype=torch.int32, device="cuda")
iters = 20000
clk = 1.965e9
cases = [(n, 1) for n in (32, 64, 128, 256)] + [(n, -a) for n in (32, 64, 96, 128) for a in (2, 4)] + [(256, -2)]
for n, nacc in cases:
    arg = n | ((nacc - 1) << 16) if nacc > 0 else n | ((-nacc - 1) << 24)
    h.lib.mpps_debug_probe_i8mma_n(h.h, 148, 100, arg, scratch.data_ptr())
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    h.lib.mpps_debug_probe_i8mma_n(h.h, 148, iters, arg, scratch.data_ptr())
    b.record(); b.synchronize()
    t = a.elapsed_time(b) * 1e-3
    ops = 2.0 * 128 * n * 32 * iters * 148 * (-nacc if nacc < 0 else 1)
    print(f"N={n:3d} accumulators={nacc}: {t / iters * clk / (-nacc if nacc < 0 else 1):7.1f} clk/instr (aggregate), {ops / t / 1e12:7.0f} TOPS", flush=True)
