"""Per-statement host time of the batched launch path (config 3 groups of 32
planned sets): SweepBatch.__init__, _launch_results, Arena.upload.
    python tools/gpu/launch_profile.py"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2603_28160_b200 import _native, engine, planner  # noqa: E402
from tools.linetime import timed_copy  # noqa: E402

meta, mine, _ = bench.config3_plans(0, 1)
cf = [c for c, _ in mine]
ex = [e for _, e in mine]
pf, prep = timed_copy(planner, "_plan_ext_group_native")
planner._plan_ext_group_native = pf
for _ in range(2):
    for g in range(8):
        planner.plan_many(cf[32 * g:32 * g + 32], ex[32 * g:32 * g + 32], 1, 1)
prep(16)
groups = [planner.plan_many(cf[32 * g:32 * g + 32], ex[32 * g:32 * g + 32], 1, 1) for g in range(8)]
reports = []
for owner, name in ((engine, "_launch_results"), (engine.SweepBatch, "__init__"), (_native.Arena, "upload")):
    f, rep = timed_copy(owner, name, engine if owner is not _native.Arena else _native)
    setattr(owner, name, f)
    reports.append(rep)
for g in groups * 2:
    engine._launch_results(g, "device", prefetch=True)
torch.cuda.synchronize()
for r in reports:
    r(1)  # reset
n = 0
for _ in range(5):
    for g in groups:
        engine._launch_results(g, "device", prefetch=True)
        n += 1
    torch.cuda.synchronize()
for r in reports:
    r(n)
