"""One-GPU projection of the N-GPU feed-strip decomposition.

For each config and N in (1, 2, 4, 8), every rank's strip job is run on this
one GPU, one after another, exactly as that rank would run it (SweepBatch over
its node columns, StripPipeline step: fill, sweep, decode, areal + profile
partials; the all-reduces are no-ops without a process group). Reported per
rank: device step and sweep time (CUDA events, median of K, L2 flushed
between steps), live (step, tooth, pass) rows and evaluated points. The
projected N-GPU step is the max over ranks plus the measured NCCL latency of
the three tiny all-reduces (not measurable here; stated separately).

    python tools/gpu/project_strips.py [--configs 2 4 5] [--steps 5] > gpurun_out/project.jsonl
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", type=int, nargs="+", default=[2, 4, 5])
    ap.add_argument("--ns", type=int, nargs="+", default=[1, 2, 4, 8])
    ap.add_argument("--steps", type=int, default=5)
    args = ap.parse_args()
    import torch

    from paper_2603_28160_b200 import configs, sharded
    from paper_2603_28160_b200.engine import SweepBatch
    from paper_2603_28160_b200.planner import plan as make_plan

    dev = torch.device("cuda", 0)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    for cid in args.configs:
        if cid == 3:
            project_batch(args, dev, flush)
            continue
        cfg, ext, meta = configs.FACTORIES[cid]()
        p = make_plan(cfg, ext)
        base_ms = None
        for n in args.ns:
            ranks = []
            for r, (lo, hi) in enumerate(sharded.strip_bounds(p.grid.n + 1, n)):
                b = SweepBatch([(p, lo, hi)])
                pipe = sharded.StripPipeline(b, every=meta.get("profiles_every", 64), uncut=meta["uncut"])
                pipe.capture()
                for _ in range(2):
                    pipe.run()
                torch.cuda.synchronize()
                st, sw = [], []
                for _ in range(args.steps):
                    flush.fill_(1)
                    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
                    pipe.run(events=ev)
                    torch.cuda.synchronize()
                    st.append(ev[0].elapsed_time(ev[3]))
                    sw.append(ev[1].elapsed_time(ev[2]))
                ctr, mach = b.counters()
                ranks.append({"rank": r, "cols": [lo, hi], "step_ms": statistics.median(st),
                              "sweep_ms": statistics.median(sw), "live_rows": int(ctr[0][0]),
                              "points_evaluated": int(ctr[0][1]), "sub_strips": b.surfs[0].n_strips,
                              "sweep_launches": b.launches_per_run})
                del pipe, b
                torch.cuda.empty_cache()
            mx = max(x["step_ms"] for x in ranks)
            if n == 1:
                base_ms = mx
            rec = {"config": meta["name"], "n": n, "max_rank_step_ms": mx,
                   "max_rank_sweep_ms": max(x["sweep_ms"] for x in ranks),
                   "sum_live_rows": sum(x["live_rows"] for x in ranks),
                   "sum_points_evaluated": sum(x["points_evaluated"] for x in ranks),
                   "projected_speedup": base_ms / mx if base_ms else None, "ranks": ranks}
            print(json.dumps(rec), flush=True)


def project_batch(args, dev, flush):
    """Config 3 (256 parameter sets) sharded by set as bench.py does at N > 1:
    every rank's sets as one SweepBatch (fill + sweep + decode) on this
    GPU, one rank after another; max over ranks."""
    import torch

    import bench
    from paper_2603_28160_b200.engine import SweepBatch

    base_ms = None
    for n in args.ns:
        ranks = []
        for r in range(n):
            meta, _, plans = bench.config3_plans(r, n)
            b = SweepBatch([(p, 0, p.grid.n) for p in plans])
            st = []
            for k in range(args.steps + 2):
                flush.fill_(1)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                b.launch()
                e1.record()
                torch.cuda.synchronize()
                if k >= 2:
                    st.append(e0.elapsed_time(e1))
            ctr, _ = b.counters()
            ranks.append({"rank": r, "sets": len(plans), "step_ms": statistics.median(st),
                          "points_evaluated": int(sum(c[1] for c in ctr))})
            del b
            torch.cuda.empty_cache()
        mx = max(x["step_ms"] for x in ranks)
        if n == 1:
            base_ms = mx
        print(json.dumps({"config": "config3", "n": n, "max_rank_step_ms": mx,
                          "note": "fill + sweep + decode per rank's sets (parameter-set shards, no communication)",
                          "projected_speedup": base_ms / mx if base_ms else None, "ranks": ranks}), flush=True)


if __name__ == "__main__":
    main()
