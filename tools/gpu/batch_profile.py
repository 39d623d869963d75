"""cProfile (cumulative) of planner.plan + SweepBatch.__init__ on config 2,
and of simulate_batch's per-group host work on config 3 (GPU box)."""
import cProfile, pstats, sys
sys.path.insert(0, '.')
import torch
from paper_2603_28160_b200 import configs, engine, planner
cfg, ext, meta = configs.config2()
p = planner.plan(cfg, ext)
for _ in range(20):
    engine.SweepBatch([(p, 0, p.grid.n)])
torch.cuda.synchronize()
pr = cProfile.Profile(); pr.enable()
for _ in range(200):
    p = planner.plan(cfg, ext)
    engine.SweepBatch([(p, 0, p.grid.n)])
pr.disable(); torch.cuda.synchronize()
pstats.Stats(pr).sort_stats('cumulative').print_stats(30)
import bench
base, ext3, meta3, ranges, mine, plans, total = bench.config3_workload(0, 1)
ps = plans[:32]
for _ in range(3):
    engine._launch_results(ps, "device", False, True)
torch.cuda.synchronize()
pr = cProfile.Profile(); pr.enable()
for _ in range(10):
    engine._launch_results(ps, "device", False, True)
    torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats('tottime').print_stats(25)
