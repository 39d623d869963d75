"""Round-trip latency of the post-sweep public calls on an idle GPU (config 2
field): areal_metrics, profile_roughness, one readback, one pin_memory."""
import sys
import time

sys.path.insert(0, '.')
import numpy as np
import torch

import paper_2603_28160_b200 as ms
from paper_2603_28160_b200 import _native, configs

cfg, ext, meta = configs.config2()
uncut, every = meta["uncut"], meta.get("profiles_every", 64)
res = ms.simulate(cfg, ext)
f = res.field
ms.areal_metrics(f, uncut=uncut)
torch.cuda.synchronize()
small = torch.zeros(16, dtype=torch.float64, device="cuda")


def timeit(name, fn, n=200):
    for _ in range(10):
        fn()
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(n):
        fn()
    torch.cuda.synchronize()
    print(f"{name:28s} {1e6 * (time.perf_counter() - t) / n:8.1f} us")


timeit("areal_metrics", lambda: ms.areal_metrics(f, uncut=uncut))
timeit("profile_roughness", lambda: ms.profile_roughness(f, every=every, uncut=uncut))
timeit("readback(16 doubles)", lambda: _native.readback(small))
starts = np.arange(16, dtype=np.int64)
timeit("pin_memory+H2D", lambda: torch.from_numpy(starts).pin_memory().to("cuda", non_blocking=True))
timeit("torch.empty dev", lambda: torch.empty(128, dtype=torch.float64, device="cuda"))
ev = torch.cuda.Event()
timeit("event record+sync", lambda: (ev.record(), ev.synchronize()))
timeit("simulate (host part)", lambda: ms.simulate(cfg, ext), n=30)
