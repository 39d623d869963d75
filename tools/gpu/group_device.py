"""Device time of one config-3 launch group (fill + sweep + decode) vs the
group size, alone and with a concurrent 64 MiB pinned D2H on a side stream
(what the e2e pipeline overlaps it with):  python tools/gpu/group_device.py"""
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2603_28160_b200 import planner  # noqa: E402
from paper_2603_28160_b200.engine import SweepBatch  # noqa: E402

meta, mine, _ = bench.config3_plans(0, 1)
cf = [c for c, _ in mine]
ex = [e for _, e in mine]
plans = planner.plan_many(cf, ex)
side = torch.cuda.Stream()
src = torch.empty(64 << 20, dtype=torch.uint8, device="cuda")
dst = torch.empty(64 << 20, dtype=torch.uint8, pin_memory=True)
for g in (16, 32, 64, 128, 256):
    b = SweepBatch([(p, 0, p.grid.n) for p in plans[:g]])
    for copy in (False, True):
        ts = []
        for rep in range(8):
            torch.cuda.synchronize()
            if copy:
                with torch.cuda.stream(side):
                    for _ in range(3):
                        dst.copy_(src, non_blocking=True)
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
            b.launch(events=ev)
            torch.cuda.synchronize()
            if rep >= 2:
                ts.append(ev[0].elapsed_time(ev[3]))
        print(f"group {g:3d} sets{' + D2H' if copy else '       '}: {statistics.median(ts):.3f} ms "
              f"({1e3 * statistics.median(ts) / g:.1f} us/set), launches {b.launches_per_run}")
    del b
