"""Timeline of the config 2 e2e step (public API): host milestones and device
events, ms from step start."""
import sys, time
sys.path.insert(0, '.')
import torch
import paper_2603_28160_b200 as ms
from paper_2603_28160_b200 import configs

name = next((a for a in sys.argv[1:] if a.startswith("config")), "config2")
cfg, ext, meta = getattr(configs, name)()
if "noprefetch" in sys.argv[1:]:
    from paper_2603_28160_b200 import engine, planner
    ms.simulate = lambda c, e: engine._launch_results([planner.plan(c, e)], "device", False, prefetch=False)[0]
every, uncut = 64, "exclude"


def ev():
    e = torch.cuda.Event(enable_timing=True); e.record(); return e


for it in range(8):
    torch.cuda.synchronize()
    start = ev(); t0 = time.perf_counter()
    res = ms.simulate(cfg, ext); ta = time.perf_counter(); ea = ev()
    am = ms.areal_metrics(res.field, uncut=uncut); tb = time.perf_counter(); eb = ev()
    prs = ms.profile_roughness(res.field, every=every, uncut=uncut); tc = time.perf_counter(); ec = ev()
    hh = res.field.heights; td = time.perf_counter(); ed = ev()
    torch.cuda.synchronize()
    if it < 3:
        continue
    f = lambda t: 1e3 * (t - t0)
    print(f"host: simulate ret {f(ta):.3f} areal ret {f(tb):.3f} profiles ret {f(tc):.3f} heights ret {f(td):.3f} | "
          f"device at: simulate-ret {start.elapsed_time(ea):.3f} areal-ret {start.elapsed_time(eb):.3f} "
          f"profiles-ret {start.elapsed_time(ec):.3f} heights-ret {start.elapsed_time(ed):.3f} | "
          f"main_loop (sweep launch) {1e3 * res.main_loop_seconds:.3f}")
