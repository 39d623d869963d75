"""Host-side split of the config 2 e2e path (GPU box): each piece of
simulate() / profile_roughness() timed alone with perf_counter, GPU idle."""
import sys
import time

sys.path.insert(0, '.')
import numpy as np
import torch

import paper_2603_28160_b200 as ms
from paper_2603_28160_b200 import _native, configs, engine, planner, roughness

cfg, ext, meta = configs.config2()
uncut, every = meta["uncut"], meta.get("profiles_every", 64)
res = ms.simulate(cfg, ext)
f = res.field
torch.cuda.synchronize()
acc = {}


def tick(k, t0):
    acc[k] = acc.get(k, 0.0) + time.perf_counter() - t0
    return time.perf_counter()


N = 50
for it in range(N + 5):
    if it == 5:
        acc.clear()
    torch.cuda.synchronize()
    t = time.perf_counter()
    p = planner.plan(cfg, ext)
    t = tick("plan", t)
    b = engine.SweepBatch([(p, 0, p.grid.n)])
    t = tick("SweepBatch", t)
    st = torch.cuda.current_stream()
    sp = int(st.cuda_stream)
    t = tick("stream ptr", t)
    b.launch_fill(sp)
    t = tick("launch_fill", t)
    b.launch_sweep(sp)
    t = tick("launch_sweep", t)
    b.launch_decode(sp)
    t = tick("launch_decode", t)
    e0, e3 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    e3.record()
    t = tick("2 events", t)
    side = torch.cuda.Stream()
    t = tick("new stream", t)
    host = torch.empty(b.keys.shape, dtype=torch.float64, pin_memory=True)
    t = tick("pinned empty", t)
    host.copy_(b.keys.view(torch.float64), non_blocking=True)
    t = tick("d2h enqueue", t)
    fld = ms.HeightField(p.grid, p.initial_height, device=b.heights()[0])
    t = tick("HeightField", t)
    torch.cuda.synchronize()
    t = time.perf_counter()
    idx = list(range(0, 1001, 64))
    starts = [i * 1001 for i in idx]
    stt = torch.from_numpy(np.asarray(starts, dtype=np.int64)).pin_memory().to("cuda", non_blocking=True)
    t = tick("prof: starts H2D", t)
    rows = roughness._profiles_device(fld.device_heights(), 1, 0, starts, 1001, 1,
                                      roughness._field_sentinel(torch, fld, stt.device), True)
    t = tick("prof: _profiles_device", t)
    rr = _native.readback(rows).reshape(len(idx), 8)
    t = tick("prof: readback", t)
    out = [roughness._finish_profile(r, i, "exclude") for r, i in zip(rr, idx)]
    t = tick("prof: finish x16", t)
    am = ms.areal_metrics(fld, uncut="exclude")
    t = tick("areal_metrics", t)
for k, v in acc.items():
    print(f"{k:26s} {1e6 * v / N:8.1f} us")
