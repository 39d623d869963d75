"""Host-side breakdown of one e2e step (public API) for a config:
    python tools/gpu/e2e_breakdown.py 1"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

import paper_2603_28160_b200 as ms  # noqa: E402
from paper_2603_28160_b200 import configs, planner  # noqa: E402
from paper_2603_28160_b200.engine import SweepBatch, _launch_results  # noqa: E402

c = int(sys.argv[1]) if len(sys.argv) > 1 else 1
cfg, ext, meta = configs.FACTORIES[c]()
for rep in range(6):
    torch.cuda.synchronize()
    t = [time.perf_counter()]
    p = planner.plan(cfg, ext)
    t.append(time.perf_counter())
    res = _launch_results([p], "device", prefetch=True)[0]
    t.append(time.perf_counter())
    am = ms.areal_metrics(res.field, uncut="exclude")
    t.append(time.perf_counter())
    prs = ms.profile_roughness(res.field, every=64, uncut="exclude")
    t.append(time.perf_counter())
    h = res.field.heights
    t.append(time.perf_counter())
    torch.cuda.synchronize()
    t.append(time.perf_counter())
    d = [1e3 * (b - a) for a, b in zip(t, t[1:])]
    print(f"config {c} rep {rep}: plan {d[0]:.3f} launch {d[1]:.3f} areal {d[2]:.3f} profiles {d[3]:.3f} "
          f"heights {d[4]:.3f} sync {d[5]:.3f} total {sum(d):.3f} ms")
