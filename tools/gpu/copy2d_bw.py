"""D2H bandwidth of 2-D copies (rows x width bytes, source / destination
pitch = the full row-major map) into pinned memory, as the strip-pipelined
heights read-back issues them: python tools/gpu/copy2d_bw.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

from paper_2603_28160_b200 import _native  # noqa: E402

lib = _native.lib()
rows, cols = 10000, 10000
dev = torch.empty(rows * cols, dtype=torch.float64, device="cuda")
host = torch.empty(rows * cols, dtype=torch.float64, pin_memory=True)
st = torch.cuda.current_stream()
sp = int(st.cuda_stream)
pitch = cols * 8
for w in (625, 1250, 2500, 5000, 10000):
    nstrip = cols // w
    for rep in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for q in range(nstrip):
            off = q * w * 8
            _native.check(lib.msurf_copy2d_d2h(host.data_ptr() + off, pitch, dev.data_ptr() + off, pitch, w * 8,
                                               rows, sp))
        e1.record()
        torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    print(f"strip width {w:6d} cols ({w * 8} B rows) x {nstrip:2d} strips: {ms:.3f} ms, {rows * cols * 8 / ms / 1e6:.1f} GB/s")
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
host.copy_(dev, non_blocking=True)
e1.record()
torch.cuda.synchronize()
print(f"1-D copy: {e0.elapsed_time(e1):.3f} ms")
