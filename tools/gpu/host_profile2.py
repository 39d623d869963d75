import sys, time
sys.path.insert(0, '.')
import torch
import paper_2603_28160_b200 as ms
from paper_2603_28160_b200 import configs, planner, engine
cfg, ext, meta = configs.config2()
p = planner.plan(cfg, ext)
for _ in range(5):
    b = engine.SweepBatch([(p, 0, p.grid.n)]); b.launch()
torch.cuda.synchronize()
import cProfile, pstats
pr = cProfile.Profile(); pr.enable()
for _ in range(100):
    b = engine.SweepBatch([(p, 0, p.grid.n)])
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    b.launch(events=ev)
    torch.cuda.synchronize()
pr.disable(); pstats.Stats(pr).sort_stats('tottime').print_stats(25)
