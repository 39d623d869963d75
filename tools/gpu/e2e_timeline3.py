"""Timeline of the batched (config 3) e2e step: host milestones and device
events per launch group (sweep done, heights D2H done), ms from step start."""
import sys, time
sys.path.insert(0, '.')
import torch
import paper_2603_28160_b200 as ms
from paper_2603_28160_b200 import engine, grid
import bench

base, ext, meta, ranges, mine, plans, total = bench.config3_workload(0, 1)
cfgs = [c for c, _ in mine]; exts = [e for _, e in mine]
log = []
orig = engine._launch_results


def traced(plans, trig, diagnostics=False, prefetch=False):
    h0 = time.perf_counter()
    out = orig(plans, trig, diagnostics, prefetch)
    h1 = time.perf_counter()
    ev = torch.cuda.Event(enable_timing=True); ev.record()
    side = grid._copy_stream(torch, torch.device("cuda", 0))
    done = torch.cuda.Event(enable_timing=True); done.record(side)  # after the group's heights D2H
    log.append((h0, h1, ev, done))
    return out


engine._launch_results = traced
sb_init = engine.SweepBatch.__init__
sb_times = []


def timed_init(self, *a, **k):
    t = time.perf_counter()
    sb_init(self, *a, **k)
    sb_times.append(time.perf_counter() - t)


engine.SweepBatch.__init__ = timed_init
from paper_2603_28160_b200 import roughness
enq = roughness._areal_enqueue
mev = []


def timed_enqueue(*a, **k):
    e0 = torch.cuda.Event(enable_timing=True); e0.record()
    enq(*a, **k)
    e1 = torch.cuda.Event(enable_timing=True); e1.record()
    mev.append((time.perf_counter(), e0, e1))


roughness._areal_enqueue = timed_enqueue
for chunk in (32, 64):
    for it in range(4):
        log.clear(); sb_times.clear(); mev.clear()
        torch.cuda.synchronize()
        start = torch.cuda.Event(enable_timing=True); start.record()
        t0 = time.perf_counter()
        out = ms.simulate_batch(cfgs, exts, chunk=chunk); ta = time.perf_counter()
        m0 = torch.cuda.Event(enable_timing=True); m0.record()
        mets = ms.areal_metrics_batch([o.field for o in out], uncut=meta["uncut"]); tb = time.perf_counter()
        m1 = torch.cuda.Event(enable_timing=True); m1.record()
        hs = [o.field.heights for o in out]; tc = time.perf_counter()
        torch.cuda.synchronize(); td = time.perf_counter()
        if it < 2:
            continue
        print(f"chunk {chunk}: host simulate_batch {1e3*(ta-t0):.2f} metrics ret {1e3*(tb-t0):.2f} "
              f"heights ret {1e3*(tc-t0):.2f} end {1e3*(td-t0):.2f}; device metrics start {start.elapsed_time(m0):.2f} "
              f"end {start.elapsed_time(m1):.2f}")
        print("  metric runs (host enqueue, device start..end):",
              " ".join(f"[{1e3*(h-t0):.2f}: {start.elapsed_time(a):.2f}..{start.elapsed_time(b):.2f}]" for h, a, b in mev))
        for k, (h0, h1, ev, done) in enumerate(log):
            dd = f"{start.elapsed_time(done):.2f}" if done is not None else "-"
            print(f"  group {k}: host launch {1e3*(h0-t0):.2f}..{1e3*(h1-t0):.2f} (SweepBatch {1e3*sb_times[k]:.2f})"
                  f"  device decode done {start.elapsed_time(ev):.2f}  D2H done {dd}")
