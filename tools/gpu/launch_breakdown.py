"""Where the host time of one simulate() launch goes (config N):
    python tools/gpu/launch_breakdown.py 1"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

from paper_2603_28160_b200 import _native, configs, engine, planner  # noqa: E402

c = int(sys.argv[1]) if len(sys.argv) > 1 else 1
cfg, ext, meta = configs.FACTORIES[c]()
T = {}


def timed(obj, name, key):
    f = getattr(obj, name)

    def w(*a, **k):
        t0 = time.perf_counter()
        try:
            return f(*a, **k)
        finally:
            T[key] = T.get(key, 0.0) + time.perf_counter() - t0
    setattr(obj, name, w)


timed(engine.SweepBatch, "__init__", "SweepBatch.__init__")
timed(engine.SweepBatch, "launch", "SweepBatch.launch")
timed(engine.SweepBatch, "launch_by_strip", "SweepBatch.launch_by_strip")
timed(_native.Arena, "upload", "Arena.upload")
timed(engine, "_take_events", "_take_events")
for rep in range(8):
    T.clear()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    p = planner.plan(cfg, ext)
    t1 = time.perf_counter()
    res = engine._launch_results([p], "device", prefetch=True)[0]
    t2 = time.perf_counter()
    torch.cuda.synchronize()
    print(f"config {c} rep {rep}: plan {1e3 * (t1 - t0):.3f} launch_results {1e3 * (t2 - t1):.3f} ms | " +
          " ".join(f"{k} {1e3 * v:.3f}" for k, v in T.items()))
