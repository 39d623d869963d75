"""Sweep ONE rank's feed strip of a config as the N-GPU split would (for
per-kernel profiling of narrow strips): python tools/gpu/strip_rank.py 5 8 3 [reps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

from paper_2603_28160_b200 import configs, planner, sharded  # noqa: E402
from paper_2603_28160_b200.engine import SweepBatch  # noqa: E402

c, n, r = (int(a) for a in sys.argv[1:4])
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 3
cfg, ext, _ = configs.FACTORIES[c]()
p = planner.plan(cfg, ext)
lo, hi = sharded.strip_bounds(p.grid.n + 1, n)[r]
b = SweepBatch([(p, lo, hi)])
sp = torch.cuda.current_stream().cuda_stream
for _ in range(2):
    b.launch()
torch.cuda.synchronize()
ts = []
for _ in range(reps):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    b.launch_fill(sp)
    e0.record()
    b.launch_sweep(sp)
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
ts.sort()
print(f"config {c} N={n} rank {r} cols [{lo}, {hi}]: sweep median {ts[len(ts) // 2]:.3f} ms")
