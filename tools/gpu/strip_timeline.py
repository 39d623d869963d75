"""Timeline of one strip-pipelined e2e step (config 4 / 5): host wall marks
and device events (launch start, each strip's decode done on the launch
stream, copies done on the copy stream): python tools/gpu/strip_timeline.py 4"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

from paper_2603_28160_b200 import _native, configs, planner  # noqa: E402
from paper_2603_28160_b200.engine import SweepBatch  # noqa: E402
from paper_2603_28160_b200.grid import _copy_stream  # noqa: E402

c = int(sys.argv[1]) if len(sys.argv) > 1 else 4
cfg, ext, meta = configs.FACTORIES[c]()
for rep in range(4):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    p = planner.plan(cfg, ext)
    t1 = time.perf_counter()
    b = SweepBatch([(p, 0, p.grid.n)])
    t2 = time.perf_counter()
    side = _copy_stream(torch, b.dev)
    sptr = int(side.cuda_stream)
    host = torch.empty(b.keys.shape, dtype=torch.float64, pin_memory=True)
    s0 = b.surfs[0]
    pitch = (s0.j_hi - s0.j_lo + 1) * 8
    hp, dp = host.data_ptr(), b.keys.data_ptr()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev0.record()
    marks = []

    def strip_done(q, c0, w, r0, r1, stream):
        _native.check(b.lib.msurf_stream_wait(sptr, stream))
        e = torch.cuda.Event(enable_timing=True)
        e.record(side)  # copy q may start
        off = r0 * pitch + c0 * 8
        _native.check(b.lib.msurf_copy2d_d2h(hp + off, pitch, dp + off, pitch, w * 8, r1 - r0, sptr))
        marks.append(e)

    b.launch_by_strip(strip_done)
    t3 = time.perf_counter()
    end = torch.cuda.Event(enable_timing=True)
    end.record(side)
    end.synchronize()
    t4 = time.perf_counter()
    starts = [ev0.elapsed_time(e) for e in marks]
    print(f"config {c} rep {rep}: plan {1e3 * (t1 - t0):.2f} batch {1e3 * (t2 - t1):.2f} enqueue {1e3 * (t3 - t2):.2f} "
          f"wall {1e3 * (t4 - t0):.2f} ms; device: first copy may start {starts[0]:.2f}, last {starts[-1]:.2f}, "
          f"copies done {ev0.elapsed_time(end):.2f} ms ({len(marks)} copies)")
