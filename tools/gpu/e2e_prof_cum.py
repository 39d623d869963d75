"""cProfile (cumulative) of one small-surface public-API step:
python tools/gpu/e2e_prof_cum.py 1 [reps]"""
import cProfile
import os
import pstats
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

import paper_2603_28160_b200 as ms  # noqa: E402
from paper_2603_28160_b200 import configs  # noqa: E402

c = int(sys.argv[1]) if len(sys.argv) > 1 else 1
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 300
cfg, ext, meta = configs.FACTORIES[c]()


def step():
    res = ms.simulate(cfg, ext)
    ms.areal_metrics(res.field, uncut=meta["uncut"])
    ms.profile_roughness(res.field, every=meta.get("profiles_every", 64), uncut=meta["uncut"])
    return res.field.heights


for _ in range(10):
    step()
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
for _ in range(reps):
    step()
torch.cuda.synchronize()
pr.disable()
st = pstats.Stats(pr)
st.sort_stats("cumulative").print_stats(45)
