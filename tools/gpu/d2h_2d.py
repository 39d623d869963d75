"""D2H rate: one 1-D 800 MB copy vs 16 column-strip 2-D copies (10001 rows x 5000 B, pitch 80008 B) of the same map."""
import sys, time
sys.path.insert(0, '.')
import torch
from paper_2603_28160_b200 import _native
lib = _native.lib()
rows, cols = 10001, 10001
d = torch.empty(rows * cols, dtype=torch.float64, device="cuda")
h = torch.empty(rows * cols, dtype=torch.float64, pin_memory=True)
sp = _native.stream_ptr()
for rep in range(3):
    torch.cuda.synchronize(); t = time.perf_counter()
    h.copy_(d, non_blocking=True); torch.cuda.synchronize()
    t1 = time.perf_counter() - t
    for k in (16, 8, 4):
        w = [(cols * q) // k for q in range(k + 1)]
        torch.cuda.synchronize(); t = time.perf_counter()
        for q in range(k):
            _native.check(lib.msurf_copy2d_d2h(h.data_ptr() + w[q] * 8, cols * 8, d.data_ptr() + w[q] * 8, cols * 8,
                                               (w[q + 1] - w[q]) * 8, rows, sp))
        torch.cuda.synchronize()
        t2 = time.perf_counter() - t
        print(f"1-D {8 * rows * cols / t1 / 1e9:.1f} GB/s   {k} strips 2-D {8 * rows * cols / t2 / 1e9:.1f} GB/s")
