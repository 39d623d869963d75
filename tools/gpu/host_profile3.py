"""Host cost of SweepBatch for a 32-surface launch group (config 3 sets)."""
import sys, time
sys.path.insert(0, '.')
import torch
import bench
from paper_2603_28160_b200 import planner, engine
base, ext, meta, ranges, mine, plans, total = bench.config3_workload(0, 1)
ps = plans[:32]
for _ in range(3):
    engine.SweepBatch([(p, 0, p.grid.n) for p in ps])
torch.cuda.synchronize()
t = time.perf_counter()
for _ in range(20):
    b = engine.SweepBatch([(p, 0, p.grid.n) for p in ps])
torch.cuda.synchronize()
print(f"SweepBatch(32) {1e3 * (time.perf_counter() - t) / 20:.3f} ms")
t = time.perf_counter()
for _ in range(20):
    planner.plan_many([c for c, _ in mine[:32]], [e for _, e in mine[:32]], threads=1)
print(f"plan_many(32) {1e3 * (time.perf_counter() - t) / 20:.3f} ms")
import cProfile, pstats
pr = cProfile.Profile(); pr.enable()
for _ in range(20):
    b = engine.SweepBatch([(p, 0, p.grid.n) for p in ps])
pr.disable(); pstats.Stats(pr).sort_stats('tottime').print_stats(14)
