"""Host-side timeline of simulate_batch on config 3 (256 sets): per launch
group the planning, packing/upload, launch and result-wrapping times, and the
whole call with areal_metrics_batch and every map read back.
    python tools/gpu/batch_breakdown.py"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

import paper_2603_28160_b200 as ms  # noqa: E402
from paper_2603_28160_b200 import configs, engine, planner  # noqa: E402
from paper_2603_28160_b200.dataset import ParameterRange, apply_sample, uniform_sample  # noqa: E402

base, ext, meta = configs.config3_base()
ranges = [ParameterRange(n, lo, hi) for n, lo, hi in meta["ranges"]]
smp = uniform_sample(ranges, meta["count"], meta["seed"])
pairs = [apply_sample(base, ext, [r.name for r in ranges], smp[i], meta["steps_per_rev"]) for i in range(256)]
cfgs, exts = [a for a, _ in pairs], [b for _, b in pairs]
T = {}


def timed(obj, name, key):
    f = getattr(obj, name)

    def w(*a, **k):
        t0 = time.perf_counter()
        try:
            return f(*a, **k)
        finally:
            T.setdefault(key, []).append(time.perf_counter() - t0)
    setattr(obj, name, w)


timed(engine, "plan_many", "plan_many")
timed(engine.SweepBatch, "__init__", "SweepBatch.__init__")
timed(engine.SweepBatch, "launch", "SweepBatch.launch")
timed(engine, "_launch_results", "_launch_results")
for rep in range(5):
    T.clear()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    out = ms.simulate_batch(cfgs, exts)
    t1 = time.perf_counter()
    mets = ms.areal_metrics_batch([o.field for o in out], uncut="exclude")
    t2 = time.perf_counter()
    n = sum(o.field.heights.nbytes for o in out)
    t3 = time.perf_counter()
    torch.cuda.synchronize()
    t4 = time.perf_counter()
    print(f"rep {rep}: simulate_batch {1e3 * (t1 - t0):.2f} areal {1e3 * (t2 - t1):.2f} heights {1e3 * (t3 - t2):.2f} "
          f"sync {1e3 * (t4 - t3):.2f} total {1e3 * (t4 - t0):.2f} ms ({n / 1e6:.0f} MB) | " +
          " ".join(f"{k} n={len(v)} sum {1e3 * sum(v):.2f} max {1e3 * max(v):.2f}" for k, v in T.items()))
