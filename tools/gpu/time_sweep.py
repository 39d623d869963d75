"""Time the sweep launch alone for a config with the library in MSURF_LIB."""
import sys, os
sys.path.insert(0, '.')
import torch
from paper_2603_28160_b200 import configs, planner
from paper_2603_28160_b200.engine import SweepBatch
c = int(sys.argv[1]) if len(sys.argv) > 1 else 2
cfg, ext, meta = getattr(configs, f"config{c}")()
p = planner.plan(cfg, ext)
b = SweepBatch([(p, 0, p.grid.n)])
sp = torch.cuda.current_stream().cuda_stream
for _ in range(3):
    b.launch()
torch.cuda.synchronize()
ts = []
for _ in range(10):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    b.launch_fill(sp); e0.record(); b.launch_sweep(sp); e1.record(); torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
ts.sort()
print(f"SWEEP {os.environ.get('MSURF_LIB','default')} config {c}: median {ts[5]:.4f} ms min {ts[0]:.4f} ms")
