"""cProfile of the e2e public-API step (bench.py's e2e leg) for one config:
    python tools/gpu/e2e_profile.py 1 [reps]"""
import cProfile
import os
import pstats
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2603_28160_b200 as ms  # noqa: E402
from paper_2603_28160_b200 import configs  # noqa: E402

if os.environ.get("SWITCH_INTERVAL"):
    sys.setswitchinterval(float(os.environ["SWITCH_INTERVAL"]))
c = int(sys.argv[1]) if len(sys.argv) > 1 else 1
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 50
if c == 3:
    import bench

    meta, mine, _ = bench.config3_plans(0, 1)

    def step():
        out = ms.simulate_batch([c for c, _ in mine], [e for _, e in mine])
        ms.areal_metrics_batch([o.field for o in out], uncut=meta["uncut"])
        return [o.field.heights for o in out]
else:
    cfg, ext, meta = configs.FACTORIES[c]()

    def step():
        res = ms.simulate(cfg, ext)
        ms.areal_metrics(res.field, uncut=meta["uncut"])
        ms.profile_roughness(res.field, every=meta.get("profiles_every", 64), uncut=meta["uncut"])
        return res.field.heights


for _ in range(5):
    step()
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(reps):
    step()
torch.cuda.synchronize()
print(f"config {c}: {1e3 * (time.perf_counter() - t0) / reps:.3f} ms per e2e step (no profiler)")
if os.environ.get("NO_PROFILE"):
    sys.exit(0)
pr = cProfile.Profile()
pr.enable()
for _ in range(reps):
    step()
torch.cuda.synchronize()
pr.disable()
st = pstats.Stats(pr)
st.sort_stats("tottime").print_stats(35)
