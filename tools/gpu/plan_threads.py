"""Native batched planning time per 32-set group vs native thread count (host of the GPU box)."""
import os, sys, time
sys.path.insert(0, '.')
import bench
from paper_2603_28160_b200 import planner as P
base, ext3, meta3, ranges, mine, plans, total = bench.config3_workload(0, 1)
cfgs = [c for c, _ in mine]; exts = [e for _, e in mine]
print("cpus", os.cpu_count(), "affinity", len(os.sched_getaffinity(0)))
for nt in (1, 2, 4, 8, 16):
    P._plan_ext_group_native(cfgs[:32], exts[:32], nt)
    t = time.perf_counter()
    for k in range(8):
        P._plan_ext_group_native(cfgs[32 * k:32 * k + 32], exts[32 * k:32 * k + 32], nt)
    print("native threads", nt, "ms per 32-set group %.3f" % ((time.perf_counter() - t) / 8 * 1e3))
