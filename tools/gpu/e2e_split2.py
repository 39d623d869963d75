"""Config 2 e2e (public API, as bench.py times it): wall split per call with
no extra syncs, plus a cProfile of the host side."""
import cProfile
import pstats
import sys
import time

sys.path.insert(0, '.')
import torch

import paper_2603_28160_b200 as ms
from paper_2603_28160_b200 import configs

cfg, ext, meta = configs.config2()
uncut, every = meta["uncut"], meta.get("profiles_every", 64)


def once(split):
    t0 = time.perf_counter()
    res = ms.simulate(cfg, ext)
    t1 = time.perf_counter()
    am = ms.areal_metrics(res.field, uncut=uncut)
    t2 = time.perf_counter()
    prs = ms.profile_roughness(res.field, every=every, uncut=uncut)
    t3 = time.perf_counter()
    hh = res.field.heights
    torch.cuda.synchronize()
    t4 = time.perf_counter()
    if split is not None:
        for k, v in zip(("simulate", "areal", "profiles", "heights", "total"), (t1 - t0, t2 - t1, t3 - t2, t4 - t3, t4 - t0)):
            split[k] = split.get(k, 0.0) + v


for _ in range(5):
    once(None)
torch.cuda.synchronize()
split = {}
N = 30
for _ in range(N):
    once(split)
print(" ".join(f"{k} {1e3 * v / N:.3f}" for k, v in split.items()), "ms")
pr = cProfile.Profile()
pr.enable()
for _ in range(N):
    once(None)
pr.disable()
pstats.Stats(pr).sort_stats('tottime').print_stats(25)
