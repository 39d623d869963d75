"""Host-side cost of simulate() on config 2 (no sync inside)."""
import sys, time
sys.path.insert(0, '.')
import torch
import paper_2603_28160_b200 as ms
from paper_2603_28160_b200 import configs, planner, engine
cfg, ext, meta = configs.config2()
for _ in range(5):
    ms.simulate(cfg, ext).field.heights
torch.cuda.synchronize()
N = 50
acc = {}
def tick(k, t0):
    acc[k] = acc.get(k, 0.0) + time.perf_counter() - t0
for _ in range(N):
    t0 = time.perf_counter(); p = planner.plan(cfg, ext); tick("plan", t0)
    t0 = time.perf_counter(); b = engine.SweepBatch([(p, 0, p.grid.n)]); tick("SweepBatch.__init__", t0)
    t0 = time.perf_counter(); ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]; b.launch(events=ev); tick("launch", t0)
    t0 = time.perf_counter(); torch.cuda.synchronize(); tick("gpu wait", t0)
for k, v in acc.items():
    print(f"{k:24s} {1e3 * v / N:.4f} ms")
import cProfile, pstats
pr = cProfile.Profile(); pr.enable()
for _ in range(N):
    b = engine.SweepBatch([(p, 0, p.grid.n)])
pr.disable(); pstats.Stats(pr).sort_stats('tottime').print_stats(12)
