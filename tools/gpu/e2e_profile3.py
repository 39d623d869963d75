"""Break down the batched (config 3) e2e step on the GPU box."""
import sys, time
sys.path.insert(0, '.')
import torch
import paper_2603_28160_b200 as ms
from paper_2603_28160_b200 import planner
from paper_2603_28160_b200.engine import _launch_results
import bench

base, ext, meta, ranges, mine, plans, total = bench.config3_workload(0, 1)
cfgs = [c for c, _ in mine]; exts = [e for _, e in mine]
def t():
    torch.cuda.synchronize(); return time.perf_counter()
for it in range(4):
    t0 = t(); ps = planner.plan_many(cfgs, exts); t1 = t()
    out = _launch_results(ps, "device"); t2 = t()
    mets = ms.areal_metrics_batch([o.field for o in out], uncut=meta["uncut"]); t3 = t()
    d2h = 0
    for o in out:
        d2h += o.field.heights.nbytes
    t4 = t()
    print(f"plan_many {1e3*(t1-t0):.2f} upload+sweep {1e3*(t2-t1):.2f} metrics {1e3*(t3-t2):.2f} heights {1e3*(t4-t3):.2f} ({d2h/1e6:.0f} MB) total {1e3*(t4-t0):.2f} ms")
print("--- simulate_batch pipeline")
for chunk in (None, 16, 32, 256):
    for it in range(3):
        t0 = t()
        out = ms.simulate_batch(cfgs, exts, chunk=chunk); ta = time.perf_counter()
        mets = ms.areal_metrics_batch([o.field for o in out], uncut=meta["uncut"]); tb = time.perf_counter()
        d2h = sum(o.field.heights.nbytes for o in out); tc = time.perf_counter()
        torch.cuda.synchronize(); td = time.perf_counter()
        print(f"chunk {chunk}: simulate_batch {1e3*(ta-t0):.2f} metrics {1e3*(tb-ta):.2f} heights {1e3*(tc-tb):.2f} total {1e3*(td-t0):.2f} ms")
import cProfile, pstats
for chunk in (32, 256):
    pr = cProfile.Profile(); pr.enable()
    for _ in range(3):
        out = ms.simulate_batch(cfgs, exts, chunk=chunk)
        torch.cuda.synchronize()
    pr.disable()
    print("=== chunk", chunk)
    pstats.Stats(pr).sort_stats('tottime').print_stats(14)
