import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
from paper_2603_28160_b200 import configs, planner, engine
cfg, ext, _ = configs.config5()
p = planner.plan(cfg, ext)
for trig in ("device", "host"):
    b = engine.SweepBatch([(p, 0, p.grid.n)], trig=trig)
    b.launch(); torch.cuda.synchronize()
    ref = b.heights()[0].clone()
    b2 = engine.SweepBatch([(p, 0, p.grid.n)], trig=trig)
    hostbuf = torch.empty(b2.keys.shape, dtype=torch.float64, pin_memory=True)
    b2.launch_by_strip(lambda *a: None)
    torch.cuda.synchronize()
    got = b2.heights()[0]
    d = (got != ref)
    print(trig, "launch vs launch_by_strip differing nodes", int(d.sum()))
    if int(d.sum()):
        idx = torch.nonzero(d.view(p.grid.m + 1, -1))
        print(" rows", idx[:, 0].min().item(), idx[:, 0].max().item(), "cols", idx[:, 1].min().item(), idx[:, 1].max().item())
    b3 = engine.SweepBatch([(p, 0, p.grid.n)], trig=trig)
    b3.launch(); torch.cuda.synchronize()
    print(trig, "launch vs launch", int((b3.heights()[0] != ref).sum()))
