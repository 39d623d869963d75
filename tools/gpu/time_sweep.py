"""Time the production sweep launch alone for one BASELINE config (config 3 =
the 256-set batch) — also the target command of the ncu full captures:
    python tools/gpu/time_sweep.py 5 [reps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

from paper_2603_28160_b200 import configs, planner  # noqa: E402
from paper_2603_28160_b200.engine import SweepBatch  # noqa: E402

c = int(sys.argv[1]) if len(sys.argv) > 1 else 5
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
if c == 3:
    from paper_2603_28160_b200.dataset import ParameterRange, apply_sample, uniform_sample

    base, ext, meta = configs.config3_base()
    ranges = [ParameterRange(n, lo, hi) for n, lo, hi in meta["ranges"]]
    smp = uniform_sample(ranges, meta["count"], meta["seed"])
    pairs = [apply_sample(base, ext, [r.name for r in ranges], smp[i], meta["steps_per_rev"])
             for i in range(meta["count"])]
    plans = planner.plan_many([a for a, _ in pairs], [b for _, b in pairs])
else:
    cfg, ext, meta = configs.FACTORIES[c]()
    plans = [planner.plan(cfg, ext)]
b = SweepBatch([(p, 0, p.grid.n) for p in plans])
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
print(f"SWEEP config {c}: median {ts[len(ts) // 2]:.4f} ms min {ts[0]:.4f} ms over {reps}")
