"""Pinned D2H / H2D copy bandwidth on this box (the e2e floor of the
height-map read-back): python tools/gpu/pcie_bw.py"""
import torch

d = torch.empty(537 << 20, dtype=torch.uint8, device="cuda")
for mb in (1, 8, 67, 537):
    n = mb << 20
    h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    for name, (dst, src) in (("D2H", (h, d[:n])), ("H2D", (d[:n], h))):
        for _ in range(2):
            dst.copy_(src, non_blocking=True)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = max(1, 2000 // mb)
        a.record()
        for _ in range(reps):
            dst.copy_(src, non_blocking=True)
        b.record()
        torch.cuda.synchronize()
        ms = a.elapsed_time(b) / reps
        print(f"{name} {mb:4d} MiB: {ms:.3f} ms  {n / ms / 1e6:.1f} GB/s")
