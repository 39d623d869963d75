"""cProfile of the per-launch-group host work (_launch_results) for config 3."""
import sys, time
sys.path.insert(0, '.')
import torch
from paper_2603_28160_b200 import planner
from paper_2603_28160_b200.engine import _launch_results
import bench

base, ext, meta, ranges, mine, plans, total = bench.config3_workload(0, 1)
cfgs = [c for c, _ in mine]; exts = [e for _, e in mine]
groups = [planner.plan_many(cfgs[a:a + 32], exts[a:a + 32], 1) for a in range(0, 256, 32)]
keep = []
for it in range(3):
    keep.append([_launch_results(g, "device", False, True) for g in groups]); torch.cuda.synchronize()
    keep = keep[-2:]
ts = []
for it in range(5):
    t = time.perf_counter()
    keep.append([_launch_results(g, "device", False, True) for g in groups])
    ts.append((time.perf_counter() - t) / len(groups))
    torch.cuda.synchronize(); keep = keep[-2:]
print("host ms per _launch_results(32):", [round(1e3 * x, 3) for x in ts])
t = time.perf_counter()
for _ in range(5):
    planner.plan_many(cfgs[:32], exts[:32], 1)
print("plan_many(32, threads=1) ms:", round((time.perf_counter() - t) / 5 * 1e3, 3))
import cProfile, pstats
pr = cProfile.Profile(); pr.enable()
for it in range(3):
    keep.append([_launch_results(g, "device", False, True) for g in groups])
    torch.cuda.synchronize(); keep = keep[-2:]
pr.disable()
pstats.Stats(pr).sort_stats('tottime').print_stats(25)
