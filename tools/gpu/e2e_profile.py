"""Break down the e2e (public API) step time on the GPU box."""
import sys, time
sys.path.insert(0, '.')
import torch
import paper_2603_28160_b200 as ms
from paper_2603_28160_b200 import configs, planner
from paper_2603_28160_b200.engine import SweepBatch

cfg, ext, meta = configs.config2()
def t():
    torch.cuda.synchronize(); return time.perf_counter()
for it in range(6):
    t0 = t(); p = planner.plan(cfg, ext); t1 = t()
    b = SweepBatch([(p, 0, p.grid.n)]); t2 = t()
    b.launch(); t3 = t()
    small, mach = b.counters(); t4 = t()
    f = ms.HeightField(p.grid, p.initial_height, device=b.heights()[0])
    am = ms.areal_metrics(f, uncut="exclude"); t5 = t()
    prs = ms.profile_roughness(f, every=64, uncut="exclude"); t6 = t()
    h = f.heights; t7 = t()
    print(f"plan {1e3*(t1-t0):.3f} batch(upload) {1e3*(t2-t1):.3f} launch+sweep {1e3*(t3-t2):.3f} counters {1e3*(t4-t3):.3f} "
          f"areal {1e3*(t5-t4):.3f} profiles {1e3*(t6-t5):.3f} d2h {1e3*(t7-t6):.3f} total {1e3*(t7-t0):.3f} ms")
# the public path exactly as bench e2e (no syncs between)
for it in range(6):
    t0 = time.perf_counter()
    res = ms.simulate(cfg, ext); ta = time.perf_counter()
    am = ms.areal_metrics(res.field, uncut="exclude"); tb = time.perf_counter()
    prs = ms.profile_roughness(res.field, every=64, uncut="exclude"); tc = time.perf_counter()
    hh = res.field.heights; td = time.perf_counter()
    print(f"e2e simulate {1e3*(ta-t0):.3f} areal {1e3*(tb-ta):.3f} profiles {1e3*(tc-tb):.3f} heights {1e3*(td-tc):.3f} total {1e3*(td-t0):.3f}")
import cProfile, pstats
pr = cProfile.Profile(); pr.enable()
for _ in range(20):
    res = ms.simulate(cfg, ext); am = ms.areal_metrics(res.field, uncut="exclude"); prs = ms.profile_roughness(res.field, every=64, uncut="exclude"); hh = res.field.heights
pr.disable()
pstats.Stats(pr).sort_stats('cumulative').print_stats(25)
