"""Where Arena.upload's time goes for a config-3 launch group (host side):
python tools/gpu/upload_prof.py"""
import ctypes
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2603_28160_b200 import _native, planner  # noqa: E402
from paper_2603_28160_b200.engine import SweepBatch  # noqa: E402

T = {}


def upload(self, device, fill_structs=None):
    t = [time.perf_counter()]
    dev = torch.empty(max(self.size, 1), dtype=torch.uint8, device=device)
    base = dev.data_ptr()
    t.append(time.perf_counter())
    extra = fill_structs(base) if fill_structs else []
    t.append(time.perf_counter())
    stage = torch.empty(max(self.size, 1), dtype=torch.uint8, pin_memory=True)
    hp = stage.data_ptr()
    t.append(time.perf_counter())
    for off, a in self._parts:
        if a is not None and a.nbytes:
            ctypes.memmove(hp + off, a.ctypes.data, a.nbytes)
    for off, b in extra:
        b = b if isinstance(b, np.ndarray) else np.frombuffer(b, dtype=np.uint8)
        ctypes.memmove(hp + off, b.ctypes.data, b.nbytes)
    t.append(time.perf_counter())
    dev.copy_(stage, non_blocking=True)
    t.append(time.perf_counter())
    for off, tt in self._direct:
        dev[off: off + tt.numel()].copy_(tt, non_blocking=True)
    t.append(time.perf_counter())
    for k, (a, b) in enumerate(zip(t, t[1:])):
        T.setdefault(k, []).append(1e3 * (b - a))
    T.setdefault("parts", []).append(len(self._parts))
    T.setdefault("size", []).append(self.size)
    return dev


_native.Arena.upload = upload
meta, mine, _ = bench.config3_plans(0, 1)
cfgs, exts = [c for c, _ in mine], [e for _, e in mine]
for rep in range(12):
    plans = planner.plan_many(cfgs[:32], exts[:32], 1, 8)
    t0 = time.perf_counter()
    b = SweepBatch([(p, 0, p.grid.n) for p in plans])
    t1 = time.perf_counter()
    T.setdefault("init", []).append(1e3 * (t1 - t0))
    torch.cuda.synchronize()
names = {0: "dev alloc", 1: "fill_structs", 2: "pinned alloc", 3: "memmoves", 4: "staged copy_", 5: "direct copies"}
for k, v in T.items():
    v = v[4:]
    print(f"{names.get(k, k):14s} median {sorted(v)[len(v) // 2]:.3f}")
