"""Device time of the eager public-API launch (simulate: fill + sweep +
decode between the launch's own events) vs the captured pipeline step, for
one config: python tools/gpu/eager_vs_graph.py 5"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

import paper_2603_28160_b200 as ms  # noqa: E402
from paper_2603_28160_b200 import configs, engine, planner  # noqa: E402

c = int(sys.argv[1]) if len(sys.argv) > 1 else 5
cfg, ext, meta = configs.FACTORIES[c]()
for label, kw in (("simulate (strip-pipelined D2H)", {}),):
    for i in range(6):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = ms.simulate(cfg, ext)
        h = r.field.heights
        t1 = time.perf_counter()
        print(f"{label} rep {i}: wall {1e3 * (t1 - t0):.3f} ms, device fill+sweep+decode "
              f"{1e3 * r.main_loop_seconds:.3f} ms")
p = planner.plan(cfg, ext)
for i in range(4):
    torch.cuda.synchronize()
    res = engine._launch_results([p], "device", prefetch=False)[0]
    torch.cuda.synchronize()
    print(f"_launch_results no prefetch rep {i}: device {1e3 * res.main_loop_seconds:.3f} ms")
