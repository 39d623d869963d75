"""Host timeline of one config-3 e2e step (simulate_batch + areal_metrics_batch
+ heights): wall-clock spans of the planner / launcher functions per thread.
    python tools/gpu/e2e_timeline.py [reps]"""
import os
import sys
import threading
import time

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2603_28160_b200 as ms  # noqa: E402
from paper_2603_28160_b200 import _native, engine, grid, planner, roughness  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
SPANS = []
LOCK = threading.Lock()


def wrap(obj, name, label):
    f = getattr(obj, name)

    def w(*a, **k):
        t0 = time.perf_counter()
        try:
            return f(*a, **k)
        finally:
            with LOCK:
                SPANS.append((threading.get_ident(), label, t0, time.perf_counter()))
    setattr(obj, name, w)


wrap(planner, "_plan_ext_group_native", "plan_group")
wrap(planner, "chunk_f32", "chunk_f32")
wrap(planner, "chunk_zfloor", "chunk_zfloor")
wrap(engine.SweepBatch, "__init__", "SweepBatch.init")
GPU_EV = []


def _launch_ev(f):
    def w(self, *a, **k):
        r = f(self, *a, **k)
        e = torch.cuda.Event(enable_timing=True)
        e.record()
        GPU_EV.append(("sweep+decode done", e))
        return r
    return w


engine.SweepBatch.launch = _launch_ev(engine.SweepBatch.launch)
wrap(engine.SweepBatch, "launch", "launch")
wrap(_native.Arena, "upload", "upload")
wrap(engine, "_launch_results", "launch_results")
wrap(roughness, "areal_metrics_batch", "areal_batch")
meta, mine, _ = bench.config3_plans(0, 1)
lib = _native.lib()
for nm in ("msurf_plan_geometry_many", "msurf_plan_finish_many"):
    wrap(lib, nm, nm)

for rep in range(reps + 3):
    SPANS.clear()
    GPU_EV.clear()
    torch.cuda.synchronize()
    g0 = torch.cuda.Event(enable_timing=True)
    g0.record()
    t0 = time.perf_counter()
    out = ms.simulate_batch([c for c, _ in mine], [e for _, e in mine], prefetch=os.environ.get("PREFETCH", "1") == "1")
    t1 = time.perf_counter()
    ms.areal_metrics_batch([o.field for o in out], uncut=meta["uncut"])
    t2 = time.perf_counter()
    a_ev = torch.cuda.Event(enable_timing=True)
    a_ev.record()
    d_ev = torch.cuda.Event(enable_timing=True)
    d_ev.record(grid._copy_stream(torch, torch.device("cuda", torch.cuda.current_device())))
    GPU_EV.append(("all heights D2H done", d_ev))
    GPU_EV.append(("areal done", a_ev))
    for o in out:
        o.field.heights
    t3 = time.perf_counter()
    torch.cuda.synchronize()
    t4 = time.perf_counter()
    if rep < 3:
        continue
    print(f"rep {rep}: simulate_batch {1e3 * (t1 - t0):.2f} areal {1e3 * (t2 - t1):.2f} heights {1e3 * (t3 - t2):.2f} "
          f"sync {1e3 * (t4 - t3):.2f} total {1e3 * (t4 - t0):.2f} ms")
    for lab, e in GPU_EV:
        try:
            print(f"   GPU {lab:26s} at {g0.elapsed_time(e):8.3f}")
        except RuntimeError:
            print(f"   GPU {lab:26s} (event without timing)")
    tids = {}
    for tid, lab, a, b in sorted(SPANS, key=lambda s: s[2]):
        k = tids.setdefault(tid, len(tids))
        print(f"   T{k} {lab:28s} {1e3 * (a - t0):8.3f} -> {1e3 * (b - t0):8.3f}  ({1e3 * (b - a):.3f})")
