"""Concurrent kernel timeline of one device step (CUPTI activity through
torch.profiler: kernels are NOT serialised, unlike an ncu launch list):
per kernel name the launches, summed and mean duration; GPU busy coverage
(union of kernel intervals) and mean concurrency over the step.
    python tools/gpu/kernel_timeline.py [config] [steps]"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2603_28160_b200 import configs  # noqa: E402
from paper_2603_28160_b200.engine import SweepBatch  # noqa: E402
from paper_2603_28160_b200.pipeline import SurfacePipeline  # noqa: E402
from paper_2603_28160_b200.planner import plan  # noqa: E402

cid = int(sys.argv[1]) if len(sys.argv) > 1 else 5
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
cfg, ext, meta = configs.FACTORIES[cid]()
p = plan(cfg, ext)
b = SweepBatch([(p, 0, p.grid.n)])
pipe = SurfacePipeline(b, every=meta.get("profiles_every", 64), uncut=meta["uncut"])
if os.environ.get("NO_GRAPH") != "1":
    pipe.capture()
for _ in range(3):
    pipe.run()
torch.cuda.synchronize()
from torch.profiler import ProfilerActivity, profile  # noqa: E402

with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(steps):
        pipe.run()
    torch.cuda.synchronize()
out = os.path.join(ROOT, "gpurun_out", f"trace_c{cid}.json")
os.makedirs(os.path.dirname(out), exist_ok=True)
prof.export_chrome_trace(out)
ev = [e for e in json.load(open(out))["traceEvents"] if e.get("cat") == "kernel"]
ev.sort(key=lambda e: e["ts"])
t0, t1 = ev[0]["ts"], max(e["ts"] + e["dur"] for e in ev)
by = {}
for e in ev:
    n = e["name"].replace("(anonymous namespace)::", "").split("(")[0][:60]
    d = by.setdefault(n, [0, 0.0])
    d[0] += 1
    d[1] += e["dur"]
busy, cur_s, cur_e = 0.0, None, None
for e in ev:
    s, f = e["ts"], e["ts"] + e["dur"]
    if cur_e is None or s > cur_e:
        if cur_e is not None:
            busy += cur_e - cur_s
        cur_s, cur_e = s, f
    else:
        cur_e = max(cur_e, f)
busy += cur_e - cur_s
span = t1 - t0
print(f"config {cid}: {steps} steps span {span / 1e3:.3f} ms ({span / steps / 1e3:.3f} ms/step), "
      f"kernel-busy {busy / span:.3f} of the span, mean concurrency {sum(e['dur'] for e in ev) / busy:.2f}")
for n, (c, d) in sorted(by.items(), key=lambda kv: -kv[1][1]):
    print(f"  {d / 1e3 / steps:8.3f} ms/step  {c // steps:5d} launches/step  mean {d / c:8.2f} us  {n}")
