"""Lane-slot utilisation of the staged phase-2 units (build with
-DMSURF_STAGE_STATS, load via MSURF_LIB): useful (step, chunk) pairs / (units x 64)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

from paper_2603_28160_b200 import configs, planner  # noqa: E402
from paper_2603_28160_b200.engine import SweepBatch  # noqa: E402

for c in (5, 2):
    cfg, ext, _ = configs.FACTORIES[c]()
    p = planner.plan(cfg, ext)
    b = SweepBatch([(p, 0, p.grid.n)])
    b.launch()
    torch.cuda.synchronize()
    ctr, _ = b.counters()
    slots, useful = int(ctr[0][2]), int(ctr[0][3])
    print(f"config {c}: units x 64 = {slots}, live (step, chunk) pairs = {useful}, utilisation {useful / max(slots, 1):.3f}; "
          f"live rows {int(ctr[0][0])}, points evaluated {int(ctr[0][1])}")
