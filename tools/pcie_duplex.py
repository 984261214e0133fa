"""Pinned host <-> device copy rates alone and concurrently (dev tool): the cfg2 e2e stream moves
32 MiB up and 64 MiB down per step; this is its ceiling."""
import torch, time
up_b, dn_b = 32 << 20, 64 << 20
hu = torch.empty(up_b // 8, dtype=torch.float64).pin_memory(); du = torch.empty_like(hu, device="cuda")
hd = torch.empty(dn_b // 8, dtype=torch.float64).pin_memory(); dd = torch.empty_like(hd, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def run(up, dn, reps=20):
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    s1.wait_stream(torch.cuda.current_stream()); s2.wait_stream(torch.cuda.current_stream())
    for _ in range(reps):
        if up:
            with torch.cuda.stream(s1): du.copy_(hu, non_blocking=True)
        if dn:
            with torch.cuda.stream(s2): hd.copy_(dd, non_blocking=True)
    torch.cuda.current_stream().wait_stream(s1); torch.cuda.current_stream().wait_stream(s2)
    b.record(); b.synchronize()
    return a.elapsed_time(b) / reps
for _ in range(2):
    tu, td, tb = run(True, False), run(False, True), run(True, True)
    print(f"H2D 32 MiB {tu:.3f} ms ({up_b/tu/1e6:.1f} GB/s); D2H 64 MiB {td:.3f} ms ({dn_b/td/1e6:.1f} GB/s); both concurrently "
          f"{tb:.3f} ms per step -> ceiling {64/tb*1e3:.0f} evals/s")
