"""Config 3 e2e (simulate_batch + areal_metrics_batch + heights) over the
pipeline knobs: plan workers, first-group size/threads, group size."""
import itertools, sys, time
sys.path.insert(0, '.')
import numpy as np
import torch
import paper_2603_28160_b200 as ms
from paper_2603_28160_b200 import engine
import bench

base, ext, meta, ranges, mine, plans, total = bench.config3_workload(0, 1)
cfgs = [c for c, _ in mine]; exts = [e for _, e in mine]


def step(chunk):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    out = ms.simulate_batch(cfgs, exts, chunk=chunk)
    mets = ms.areal_metrics_batch([o.field for o in out], uncut=meta["uncut"])
    hs = [o.field.heights for o in out]
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) * 1e3, out


keep = []
for _ in range(4):
    keep.append(step(32)[1]); keep = keep[-2:]
rows = []
grid = [(w, 0, 1, c, nt) for w in (0, 1) for c in (16, 32, 64) for nt in (1, 2, 4, 8)]
ivs = [0.005]
for workers, first, fthr, chunk, nthr, iv in [g + (iv,) for iv in ivs for g in grid]:
    engine.PIPELINE_PLAN_THREADS, engine.PIPELINE_FIRST_CHUNK, engine.PIPELINE_FIRST_THREADS = workers, first, fthr
    engine.PIPELINE_NATIVE_THREADS = nthr
    ts = []
    for _ in range(6):
        t, o = step(chunk); keep.append(o); keep = keep[-2:]; ts.append(t)
    rows.append((float(np.median(ts[1:])), workers, first, fthr, chunk, nthr, iv))
    print(f"iv {iv} workers {workers} first {first} first_threads {fthr} chunk {chunk} native {nthr}: median {rows[-1][0]:.2f} ms "
          f"(min {min(ts[1:]):.2f})", flush=True)
print("best", sorted(rows)[:3])
