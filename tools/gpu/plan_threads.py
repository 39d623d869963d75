"""Native group planner cost vs host threads (config 3 groups of 32 sets), no GPU work:
    python tools/gpu/plan_threads.py"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2603_28160_b200 import planner  # noqa: E402

print("cpus", os.cpu_count(), "affinity", len(os.sched_getaffinity(0)))
try:
    print("cpu.max", open("/sys/fs/cgroup/cpu.max").read().strip())
except OSError:
    pass
meta, mine, _ = bench.config3_plans(0, 1)
cf = [c for c, _ in mine]
ex = [e for _, e in mine]
for nt in (1, 2, 4, 8):
    for _ in range(3):
        planner.plan_many(cf[:32], ex[:32], 1, nt)
    t = time.perf_counter()
    for g in range(8):
        planner.plan_many(cf[32 * g:32 * g + 32], ex[32 * g:32 * g + 32], 1, nt)
    print(f"native threads {nt}: 8 groups of 32 sets planned in {1e3 * (time.perf_counter() - t):.2f} ms")
