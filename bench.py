"""Benchmark of the B200 FSM hot path (BASELINE.json metric: edge-point
updates/s and surfaces/s at 1/2/4/8 B200, % of roofline).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 5] [--impl ours|reference]

A "step" is one pass of the hot path over one surface: Z-map init, the
sweep of every (pass, step, tooth, edge point), key decode, areal roughness
(two passes) and Ra/Rz of every 64th feed profile. The default workload is
BASELINE configs[4] (config 5: 3-flute ball-end raster, 16 passes, 4096^2
nodes, 4.67e10 edge-point updates per surface), the largest configuration
that fits one GPU; at N=1 the line also carries ``per_config`` with the same
measurement for configs 1-4 (config 3 = the 256-set batch). N>1 (one rank
per GPU, NCCL) shards the surface into feed-direction strips: the total work
is fixed ("scaling": "strong") and the only collective is the all-reduce of
the partial roughness moments. ``--gpus N`` without torchrun's environment
re-launches itself under torch.distributed.run with N ranks (and fails if
fewer than N GPUs are visible).

``value`` is device-timed (CUDA events, inputs resident in HBM, L2 flushed
between steps, max over ranks); ``e2e`` goes through the public API
(simulate + areal_metrics + profile_roughness + the height map read back)
with host planning and host<->device copies inside the timed region.
``--impl reference`` times the reference algorithm's CPU restatement
(oracle/, all host threads) on a bounded sample of the same workload; it
imports nothing from the product package.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import socket
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "edge-point updates/s"
UNIT = "updates/s"
# algorithmic FP64 operations per evaluated edge point:
# REF 6 mul + 6 add, EXT 4 mul + 4 add, EXT+tilt 6 mul + 6 add (u, v, x', y',
# z' of the tilt model), plus the cell location 2 x [sub, div, add, floor]
FLOPS_PER_POINT = {0: 20, 1: 16, 2: 20}
FLOPS_PER_ROW = 2 * 60 + 32  # 2*C_trig + 32, C_trig ~ 60 ops (double-double sincos)
DEFAULT_CONFIG = 5
BASELINE_INDEX = {1: 0, 2: 1, 3: 2, 4: 3, 5: 4}


def _env_int(k, d):
    try:
        return int(os.environ.get(k, d))
    except ValueError:
        return d


def _local_device() -> int:
    import torch

    local = _env_int("LOCAL_RANK", 0)
    n = torch.cuda.device_count()
    return local % n if n else local


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 200 ms during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap,power.draw")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []
        self.thread = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm, mx, reasons = [], None, set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for nm, v in zip(names, parts[2:6]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return json.load(fh)
    except OSError:
        return {}


def profiled_traffic(cfg_name):
    """dram bytes per sweep launch from the committed ncu capture (profiles/)."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as fh:
            ent = json.load(fh).get(cfg_name)
        return None if ent is None else ent["dram_bytes_per_sweep_launch"]
    except (OSError, ValueError):
        return None


# ---------------------------------------------------------------- CPU legs
# Only oracle/ code runs here: the workloads come from oracle/workloads.py
# (equal to the product's configs field by field, tests/test_host_cpu.py).
def oracle_workload(cfg_id: int):
    from oracle import workloads as W

    if cfg_id not in W.FACTORIES:
        raise SystemExit(f"--config {cfg_id}: choose one of 1..5")
    return W.FACTORIES[cfg_id]()


def describe_oracle(cfg_id, cfg, ext, meta, xp, world):
    g = cfg.grid
    return {
        "workload": f"{meta['name']} (BASELINE configs[{BASELINE_INDEX[cfg_id]}])",
        "tool": f"{'ball' if ext.profile == 'ball' else 'flat(insert D=2R)'} R={cfg.tool.insert_radius_mm} "
                f"Z={cfg.tool.tooth_count}",
        "grid_nodes": [g.m + 1, g.n + 1], "spacing_mm": g.spacing_mm,
        "edge_points": xp.points, "time_steps_per_pass": xp.steps, "passes": len(xp.pass_x0),
        "steps_per_rev": round(2 * math.pi / (xp.omega * xp.dt)),
        "edge_point_updates_per_surface": xp.trajectory_points,
        "outputs": "heights + Sa/Sq/Sp/Sv/Sz/Ssk/Sku + Ra/Rz every 64th feed profile (uncut cells excluded)",
        "parallelism": f"feed strips x{world}" if world > 1 else "single GPU",
        "l2": "flushed between timed steps (256 MiB write)",
    }


def cpu_sample(cfg, ext, target_s: float = 12.0, threads: int | None = None):
    """The same workload on the host cores with the CPU restatement of the
    reference algorithm (oracle/fsm_ext_oracle.py, all threads). If the whole
    surface fits in ~2.5 x target_s it is run in full; otherwise a bounded
    sample: 16 step windows spread over the first pass, grown until the
    sample takes about target_s."""
    from oracle import fsm_ext_oracle as xorc

    threads = threads or os.cpu_count() or 1
    xp = xorc.ext_plan(cfg, ext)
    steps = xp.steps
    n_win = 16

    def run(win_len, passes=1):
        wins = [(int(round((k + 0.5) * steps / n_win - win_len / 2)),
                 int(round((k + 0.5) * steps / n_win + win_len / 2))) for k in range(n_win)]
        t0 = time.perf_counter()
        _, _, ctr, _ = xorc.ext_sweep(cfg, ext, workers=threads, windows=wins, pass_limit=passes)
        return ctr["trajectory_points"], time.perf_counter() - t0

    win = max(8, steps // 400)
    pts, dt = run(win)
    rate = pts / dt
    if dt < 0.05 * target_s:  # pilot too short to trust: one larger pilot
        win = min(steps // n_win, win * 8)
        pts, dt = run(win)
        rate = pts / dt
    if xp.trajectory_points / rate <= 2.5 * target_s:
        t0 = time.perf_counter()
        _, _, ctr, _ = xorc.ext_sweep(cfg, ext, workers=threads)
        dt = time.perf_counter() - t0
        pts = ctr["trajectory_points"]
        what = f"the full workload ({pts} edge-point updates in {dt:.2f} s"
    else:
        while dt < 0.5 * target_s and win < steps // n_win:
            win = min(steps // n_win, int(win * max(2.0, 0.7 * target_s / max(dt, 1e-3))))
            pts, dt = run(win)
        what = (f"first pass, {n_win} step windows x {win} steps spread over {steps} steps "
                f"({pts} edge-point updates in {dt:.2f} s")
    return {"value": pts / dt, "unit": UNIT, "cores": threads, "kind": "port",
            "sample": what + f", oracle/fsm_ext_oracle.py, {threads} threads)"}


def cpu_sample_batch(target_s: float, threads: int | None = None, n_sets: int = 4):
    """Config 3 on the host: the CPU restatement on `n_sets` of the 256
    parameter sets (bounded windows each), mean update rate."""
    import numpy as np

    from oracle import workloads as W

    sets, _, _ = W.config3_sets()
    rates = [cpu_sample(c, e, target_s=target_s / n_sets, threads=threads)["value"] for c, e in sets[:n_sets]]
    return {"value": float(np.mean(rates)), "unit": UNIT, "cores": threads or os.cpu_count(), "kind": "port",
            "sample": f"{n_sets} of the 256 parameter sets, 16 step windows each, oracle/fsm_ext_oracle.py, "
                      "mean edge-point-update rate"}


def config3_points():
    from oracle import fsm_ext_oracle as xorc
    from oracle import workloads as W

    sets, _, meta = W.config3_sets()
    return sum(xorc.ext_plan(c, e).trajectory_points for c, e in sets), meta


def run_reference(args, rank, world):
    """Reference arm: the reference algorithm's CPU restatement (oracle/, no
    product code) on the host cores, on a bounded sample per step."""
    if rank != 0:
        return
    from oracle import fsm_ext_oracle as xorc

    threads = os.cpu_count() or 1
    vals, sample = [], None
    if args.config == 3:
        total, meta = config3_points()
        for i in range(args.warmup + args.steps):
            cb = cpu_sample_batch(args.cpu_seconds, threads)
            if i >= args.warmup:
                vals.append(cb["value"])
                sample = cb
        v = statistics.median(vals)
        config = {"workload": "config3 (BASELINE configs[2]): 256 parameter sets, batched",
                  "edge_point_updates_per_batch": total}
        surfaces = meta["count"] * v / total
        ms_step = 1e3 * total / v
    else:
        cfg, ext, meta = oracle_workload(args.config)
        xp = xorc.ext_plan(cfg, ext)
        for i in range(args.warmup + args.steps):
            cb = cpu_sample(cfg, ext, target_s=args.cpu_seconds, threads=threads)
            if i >= args.warmup:
                vals.append(cb["value"])
                sample = cb
        v = statistics.median(vals)
        config = describe_oracle(args.config, cfg, ext, meta, xp, 1)
        surfaces = v / xp.trajectory_points
        ms_step = 1e3 * xp.trajectory_points / v
    sample = dict(sample, value=v)
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": config, "surfaces_per_s": surfaces, "cpu_baseline": sample,
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "reference_impl": "oracle/fsm_ext_oracle.py (the reference's engine.py:215-313 sweep restated "
                              "in NumPy, plus the BASELINE extensions), all host threads; imports no product code"}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------- GPU legs
_PEAKS = {}


def device_peaks():
    """Measured once per process on this GPU (msurf_microbench): 0 = fp64
    DADD/DMUL issue rate; 3 / 4 = RED.MIN lanes/s, random addresses / one
    256-byte run per warp instruction (32 MiB table); 32 + L = warp RED.MIN
    instructions/s when each touches L distinct 128-byte lines."""
    if not _PEAKS:
        import ctypes

        from paper_2603_28160_b200 import _native

        lib = _native.lib()
        r = ctypes.c_double(0.0)
        for w in (0, 3, 4, *range(33, 65)):
            _native.check(lib.msurf_microbench(w, ctypes.byref(r)))
            _PEAKS[w] = r.value
    return _PEAKS


def red_lines(batch):
    """This workload's own RED.MIN stream, shaped: one traced launch
    (MSURF_SWEEP_TRACE) histogrammed by distinct 128-byte lines per warp RED
    instruction (SweepBatch.red_lines)."""
    return batch.red_lines()


def mb_shape_sectors(L):
    """32-byte sectors one warp RED.MIN of msurf_microbench(32 + L) touches:
    lane l updates key (l // L) of line (l % L), lanes with l // L >= 16 idle
    (mb_atomic_lines_kernel)."""
    per_line = [0] * L
    for lane in range(32):
        if lane // L < 16:
            per_line[lane % L] += 1
    return sum(-(-k // 4) for k in per_line)


def roofline(flops, atomics, sweep_ms, lines, kernel_name):
    """The north star's roofline = the slower of fp64 issue and atomic
    traffic, each as the time the path's minimum work needs at the measured
    peak rate of its unit:
    * t_fp64 = algorithmic fp64 ops / the DADD/DMUL issue rate (microbench 0);
    * t_red = the 32-byte sector updates the sweep's RED.MIN stream performs
      (its traced warp REDs, each counted by the distinct sectors it touches)
      / the peak L2 atomic sector-update rate (the best RED.MIN shape of
      microbench 32+L, sectors/s). Sectors, not lines: across the measured
      shapes the L2 atomic throughput is nearly constant per sector update
      (1.2-1.9e11 /s) while the line-update rate spans 4x, and a 4x4-node
      blocked Z-map that cut config 4's lines per RED by 30 % left its sweep
      time unchanged.
    ``bound`` is the larger term and ``frac`` = that term / the measured
    sweep time. The shape-priced RED time (each warp RED at the measured rate
    for its line count, random placement) is reported beside it."""
    pk = device_peaks()
    t = sweep_ms * 1e-3
    t_fp64 = flops / pk[0]
    terms = {"t_sweep_ms": sweep_ms, "t_fp64_ms": t_fp64 * 1e3, "frac_fp64": t_fp64 / t,
             "red_synthetic_peaks_per_s": {"warp_run_32MiB": pk[4], "random_32MiB": pk[3]},
             "reds": atomics, "red_achieved_per_s": atomics / t}
    t_red = None
    if lines is not None and lines["records"] > 0:
        hist = lines["hist"]
        scale = lines["records_issued"] / lines["records"]
        line_updates = scale * sum(L * hist[L] for L in range(33))
        peak_L = max(range(1, 33), key=lambda L: pk[32 + L] * L)
        peak_lines = pk[32 + peak_L] * peak_L
        t_lines = line_updates / peak_lines
        hs = lines.get("hist_sectors") or [0] * 33
        sector_updates = scale * sum(S * hs[S] for S in range(33))
        peak_S = max(range(1, 33), key=lambda L: pk[32 + L] * mb_shape_sectors(L))
        peak_sectors = pk[32 + peak_S] * mb_shape_sectors(peak_S)
        t_red = sector_updates / peak_sectors
        t_shape = scale * sum(hist[L] / pk[32 + L] for L in range(1, 33))
        terms.update({"t_red_ms": t_red * 1e3, "frac_red": t_red / t, "sector_updates": sector_updates,
                      "peak_sector_updates_per_s": peak_sectors, "peak_shape_lines_for_sectors": peak_S,
                      "achieved_sector_updates_per_s": sector_updates / t,
                      "red_sectors_hist": hs,
                      "red_sector_rate_by_lines_per_s": {L: pk[32 + L] * mb_shape_sectors(L)
                                                         for L in (1, 2, 4, 8, 16, 32)},
                      "t_red_lines_ms": t_lines * 1e3, "line_updates": line_updates,
                      "peak_line_updates_per_s": peak_lines, "peak_shape_lines": peak_L,
                      "achieved_line_updates_per_s": line_updates / t,
                      "t_red_shape_priced_ms": t_shape * 1e3,
                      "red_records": lines["records_issued"], "red_lanes_traced": lines["lanes"],
                      "red_trace_truncated": lines["truncated"],
                      "mean_lines_per_red_instr": line_updates / max(1, lines["records_issued"]),
                      "red_lines_hist": hist,
                      "red_instr_rate_by_lines_per_s": {L: pk[32 + L] for L in (1, 2, 4, 8, 16, 32)},
                      "red_note": "every warp-wide RED.MIN of one sweep traced (MSURF_SWEEP_TRACE) and counted "
                                  "by the distinct 32-B sectors (t_red) and 128-B lines (t_red_lines) it updates"})
    bound = "fp64" if t_red is None or t_fp64 >= t_red else "atomic"
    if bound == "fp64":
        out = {"bound": "fp64", "achieved": flops / t / 1e12, "peak": pk[0] / 1e12, "unit": "TFLOP/s",
               "frac": t_fp64 / t}
    else:
        out = {"bound": "atomic", "achieved": terms["achieved_sector_updates_per_s"] / 1e9,
               "peak": terms["peak_sector_updates_per_s"] / 1e9, "unit": "G sector-updates/s (L2 RED.MIN)",
               "frac": t_red / t}
    out.update({"kernel": kernel_name, "sweep_ms": sweep_ms, "terms": terms,
                "peak_source": "measured in this run: fp64 = msurf_microbench(0) non-FMA DADD/DMUL issue rate "
                               "(MEASURED_PEAKS.json has no FP64 entry); atomic = best L2 RED.MIN sector-update rate "
                               "over msurf_microbench(32+L) shapes"})
    return out


def diag_counters(batch):
    """Per-point diagnostics (deposits, atomics) from one extra UNTIMED launch
    of the counting sweep variant (MSURF_SWEEP_DIAG); the timed steps run the
    production variant, which does not count them."""
    import torch

    batch.diagnostics = True
    batch.launch()
    torch.cuda.synchronize()
    ctr, _ = batch.counters()
    batch.diagnostics = False
    return ctr


def timed_steps(pipe, args, flush, dev_index, barrier):
    """W untimed steps, then K timed steps (CUDA events around each stage,
    L2 flushed between steps), clocks sampled during the timed region."""
    import torch

    for _ in range(args.warmup):
        pipe.run()
    torch.cuda.synchronize()
    clocks = ClockSampler(dev_index)
    clocks.start()
    step_ms, sweep_ms = [], []
    barrier()
    torch.cuda.synchronize()
    for _ in range(args.steps):
        flush.fill_(1)
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        pipe.run(events=ev)
        torch.cuda.synchronize()
        step_ms.append(ev[0].elapsed_time(ev[3]))
        sweep_ms.append(ev[1].elapsed_time(ev[2]))
    barrier()
    torch.cuda.synchronize()
    return step_ms, sweep_ms, clocks.stop()


def measure_surface(cfg_id, args, rank, world, with_cpu):
    """One single-surface config: device step (graphs, resident inputs),
    roofline of the sweep, e2e through the public API, CPU baseline."""
    import numpy as np
    import torch

    import paper_2603_28160_b200 as ms
    from paper_2603_28160_b200 import configs, sharded
    from paper_2603_28160_b200.engine import SweepBatch
    from paper_2603_28160_b200.pipeline import SurfacePipeline
    from paper_2603_28160_b200.planner import plan as make_plan
    from oracle import fsm_ext_oracle as xorc

    dist = torch.distributed
    local = _local_device()
    dev = torch.device("cuda", local)
    cfg, ext, meta = configs.FACTORIES[cfg_id]()
    p = make_plan(cfg, ext)
    uncut = meta["uncut"]
    every = meta.get("profiles_every", 64)
    j_lo, j_hi = sharded.strip_bounds(p.grid.n + 1, world)[rank]
    batch = SweepBatch([(p, j_lo, j_hi)])
    if world == 1:
        pipe = SurfacePipeline(batch, every=every, uncut=uncut)
        if not args.no_graph:
            pipe.capture()  # three CUDA graphs: fill | sweep | decode + reductions
    else:
        pipe = sharded.StripPipeline(batch, every=every, uncut=uncut)
        if not args.no_graph:
            pipe.capture()  # five CUDA graphs; the three all-reduces stay eager between them
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)

    def barrier():
        if world > 1:
            dist.barrier()

    step_ms, sweep_ms, clk = timed_steps(pipe, args, flush, local, barrier)
    launches = pipe.launches_per_run * args.steps
    ctr, machined = batch.counters()
    am, prs = pipe.collect()[0] if world == 1 else pipe.collect()
    dctr = diag_counters(batch)
    lines = red_lines(batch) if not args.no_red_trace else None

    tot = torch.tensor([sum(step_ms), sum(sweep_ms)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(tot, op=dist.ReduceOp.MAX)
    ms_per_step = float(tot[0]) / args.steps
    sweep_avg = float(tot[1]) / args.steps
    p_total = p.trajectory_points
    value = p_total / (ms_per_step * 1e-3)

    mode = p.mode
    # engaged rows (SURVEY P_eng) from the counting launch: the production
    # variant's tile pre-cull skips whole tiles before it counts them
    evald, live, engaged = int(ctr[0][1]), int(ctr[0][0]), int(dctr[0][4])
    flops = FLOPS_PER_POINT[mode] * evald + FLOPS_PER_ROW * live
    # the production sweep's RED count (its trace); the DIAG launch counts the
    # oracle's P_in without the stock-height cull, so its atomics are higher
    atomics = int(lines["lanes"]) if lines else int(dctr[0][3])
    roof = roofline(flops, atomics, sweep_avg, lines, "sweep_kernel<MODE>")
    roof.update({
        "traffic": profiled_traffic(meta["name"]), "flops_per_launch": flops,
        "flops_model": f"{FLOPS_PER_POINT[mode]} x points_evaluated + {FLOPS_PER_ROW} x live rows",
        "survey_def": {"note": "SURVEY 8(d) unit count P_eng: every point of each row whose whole-tooth box "
                               "meets the window; the kernel's chunk cull evaluates only points_evaluated of "
                               "them, which is what the fp64 term is computed on",
                       "P_eng": engaged * p.points, "engaged_rows": engaged},
        "points_evaluated": evald, "live_rows": live, "deposits": int(dctr[0][2]), "atomics": atomics,
        "diag_note": "deposits (P_in, the oracle's count) from one extra untimed MSURF_SWEEP_DIAG launch without "
                     "the stock-height cull; atomics = RED.MIN of the production sweep (its trace)",
        "hbm": {"bytes_per_step": 24 * (p.grid.m + 1) * (j_hi - j_lo + 1),
                "peak_gbs": measured_peaks().get("hbm_gbs")},
    })
    del pipe, flush, batch

    # ---- e2e through the public API with host buffers
    e2e_ms = []
    h2d = d2h = 0
    for i in range(args.warmup + args.steps):
        barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        if world == 1:
            res = ms.simulate(cfg, ext)
            am2 = ms.areal_metrics(res.field, uncut=uncut)
            prs2 = ms.profile_roughness(res.field, every=every, uncut=uncut)
            hh = res.field.heights
            h2d = res._launch.batch.h2d_bytes
        else:
            sres = sharded.simulate_strip(cfg, ext, rank, world)
            am2 = sharded.areal_metrics_strip(sres, uncut=uncut)
            prs2 = sharded.profile_roughness_strip(sres, every=every, uncut=uncut)
            hh = sres.heights.cpu().numpy()
            h2d = sres.batch.h2d_bytes
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        if i >= args.warmup:
            e2e_ms.append(dt * 1e3)
        d2h = hh.nbytes + 8 * (9 + 8 * len(prs2) + 5)
        del hh
    et = torch.tensor([sum(e2e_ms)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(et, op=dist.ReduceOp.MAX)
    e2e_step = float(et[0]) / args.steps
    e2e = {"value": p_total / (e2e_step * 1e-3), "unit": UNIT, "h2d_bytes_per_step": int(h2d),
           "d2h_bytes_per_step": int(d2h), "ms_per_step": e2e_step, "steps_ms": [round(x, 4) for x in e2e_ms],
           "api": "simulate + areal_metrics + profile_roughness + HeightField.heights"
           if world == 1 else "sharded.simulate_strip + areal/profile all-reduce + strip read-back"}

    cpu = None
    if with_cpu and world == 1 and rank == 0 and not args.no_cpu_baseline:
        ocfg, oext, _ = oracle_workload(cfg_id)
        cpu = cpu_sample(ocfg, oext, target_s=args.cpu_seconds)
    xp = xorc.ext_plan(*oracle_workload(cfg_id)[:2])
    assert xp.trajectory_points == p_total
    ok_prs = [q for q in prs if not isinstance(q, Exception)]
    return {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": describe_oracle(cfg_id, cfg, ext, meta, xp, world),
        "surfaces_per_s": 1e3 / ms_per_step,
        "roofline": roof, "cpu_baseline": cpu, "e2e": e2e,
        "gpu_launches": launches, "clocks": clk,
        "metrics": {"Sa_um": am.sa_um, "Sq_um": am.sq_um, "Sz_um": am.sz_um, "Ssk": am.ssk,
                    "Sku": am.sku, "cells": am.cell_count,
                    "Ra_um_mean": float(np.mean([q.ra_um for q in ok_prs])) if ok_prs else None,
                    "Rz_um_mean": float(np.mean([q.rz_um for q in ok_prs])) if ok_prs else None,
                    "profiles": len(prs)},
        "machined_cells_rank0": int(machined[0]),
    }


def config3_plans(rank, world):
    """BASELINE configs[2]: 256 parameter sets from default_rng(0), uniform
    (dataset.uniform_sample), sharded by parameter set across ranks."""
    from paper_2603_28160_b200 import configs, sharded
    from paper_2603_28160_b200.dataset import ParameterRange, apply_sample, uniform_sample
    from paper_2603_28160_b200.planner import plan_many

    base, ext, meta = configs.config3_base()
    ranges = [ParameterRange(n, lo, hi) for n, lo, hi in meta["ranges"]]
    samples = uniform_sample(ranges, meta["count"], meta["seed"])
    names = [r.name for r in ranges]
    all_cfgs = [apply_sample(base, ext, names, samples[i], meta["steps_per_rev"]) for i in range(meta["count"])]
    mine = all_cfgs[sharded.batch_slice(meta["count"], rank, world)]
    plans = plan_many([c for c, _ in mine], [e for _, e in mine])
    return meta, mine, plans


def measure_batch(args, rank, world, with_cpu):
    """Batched dataset mode (config 3): every parameter set of this rank in
    ONE sweep launch (+ fill/decode/reductions), value = all ranks' edge-point
    updates / max-rank step time; surfaces/s alongside."""
    import numpy as np
    import torch

    import paper_2603_28160_b200 as ms
    from paper_2603_28160_b200.engine import SweepBatch
    from paper_2603_28160_b200.pipeline import SurfacePipeline

    dist = torch.distributed
    local = _local_device()
    dev = torch.device("cuda", local)
    meta, mine, plans = config3_plans(rank, world)
    total_points, _ = config3_points()
    batch = SweepBatch([(p, 0, p.grid.n) for p in plans])
    pipe = SurfacePipeline(batch, every=None, uncut=meta["uncut"])
    if not args.no_graph:
        pipe.capture()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)

    def barrier():
        if world > 1:
            dist.barrier()

    step_ms, sweep_ms, clk = timed_steps(pipe, args, flush, local, barrier)
    launches = pipe.launches_per_run * args.steps
    ctr, machined = batch.counters()
    res = pipe.collect()
    dctr = diag_counters(batch)
    lines = red_lines(batch) if not args.no_red_trace else None
    tot = torch.tensor([sum(step_ms), sum(sweep_ms)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(tot, op=dist.ReduceOp.MAX)
    ms_step = float(tot[0]) / args.steps
    sweep_avg = float(tot[1]) / args.steps
    value = total_points / (ms_step * 1e-3)
    evald, live, engaged = int(ctr[:, 1].sum()), int(ctr[:, 0].sum()), int(dctr[:, 4].sum())
    npts = plans[0].points
    mode = plans[0].mode
    flops = FLOPS_PER_POINT[mode] * evald + FLOPS_PER_ROW * live
    atomics = int(lines["lanes"]) if lines else int(dctr[:, 3].sum())
    roof = roofline(flops, atomics, sweep_avg, lines, "sweep_kernel<MODE> (listed, persistent)")
    roof.update({"traffic": profiled_traffic(meta["name"]), "flops_per_launch": flops,
                 "survey_def": {"P_eng": engaged * npts, "engaged_rows": engaged},
                 "points_evaluated": evald, "live_rows": live, "deposits": int(dctr[:, 2].sum()),
                 "atomics": atomics,
                 "diag_note": "deposits/atomics from one extra untimed launch with MSURF_SWEEP_DIAG"})
    del pipe, flush, batch
    # e2e: public batched API with host planning, one H2D, metrics + every height map read back
    e2e_ms = []
    d2h = h2d = 0
    for i in range(args.warmup + args.steps):
        barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        out = ms.simulate_batch([c for c, _ in mine], [e for _, e in mine])
        ms.areal_metrics_batch([o.field for o in out], uncut=meta["uncut"])
        d2h = 0
        for o in out:
            d2h += o.field.heights.nbytes
        torch.cuda.synchronize()
        if i >= args.warmup:
            e2e_ms.append((time.perf_counter() - t0) * 1e3)
        h2d = sum(b.h2d_bytes for b in {id(o._launch.batch): o._launch.batch for o in out}.values())
        del out
    et = torch.tensor([sum(e2e_ms)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(et, op=dist.ReduceOp.MAX)
    e2e_step = float(et[0]) / args.steps
    cpu = None
    if with_cpu and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_sample_batch(args.cpu_seconds)
    ok = [m for m, _ in res if not isinstance(m, Exception)]
    return {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": "config3 (BASELINE configs[2]): 256 parameter sets, batched",
                       "sets": meta["count"], "sets_this_rank": len(plans), "grid_nodes": [512, 512],
                       "spacing_mm": 0.004, "edge_points": npts, "steps_per_rev": meta["steps_per_rev"],
                       "edge_point_updates_per_batch": total_points,
                       "parallelism": f"parameter-set shards x{world}" if world > 1 else "single GPU",
                       "l2": "flushed between timed steps (256 MiB write)"},
            "surfaces_per_s": meta["count"] / (ms_step * 1e-3),
            "roofline": roof, "cpu_baseline": cpu,
            "e2e": {"value": total_points / (e2e_step * 1e-3), "unit": UNIT,
                    "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
                    "ms_per_step": e2e_step, "steps_ms": [round(x, 3) for x in e2e_ms],
                    "api": "simulate_batch + areal_metrics_batch + heights"},
            "gpu_launches": launches, "clocks": clk,
            "metrics": {"surfaces_ok": len(ok), "Sa_um_mean": float(np.mean([m.sa_um for m in ok])) if ok else None}}


def compact(line):
    """The per-config summary carried inside the headline line."""
    r = line["roofline"]
    return {"workload": line["config"]["workload"], "value": line["value"], "unit": line["unit"],
            "ms_per_step": line["ms_per_step"], "surfaces_per_s": line["surfaces_per_s"],
            "e2e": {k: line["e2e"][k] for k in ("value", "unit", "ms_per_step", "h2d_bytes_per_step",
                                                 "d2h_bytes_per_step")},
            "roofline": {k: r[k] for k in ("bound", "achieved", "peak", "unit", "frac", "sweep_ms", "traffic",
                                           "terms")},
            "cpu_baseline": line["cpu_baseline"], "gpu_launches": line["gpu_launches"],
            "clocks": line["clocks"], "metrics": line["metrics"]}


def run_ours(args, rank, world):
    import torch

    def measure(cfg_id, with_cpu=True):
        if cfg_id == 3:
            out = measure_batch(args, rank, world, with_cpu)
        else:
            out = measure_surface(cfg_id, args, rank, world, with_cpu)
        torch.cuda.synchronize()
        torch.cuda.empty_cache()
        return out

    line = measure(args.config)
    if world == 1 and not args.no_per_config:
        line["per_config"] = {}
        for k in sorted(BASELINE_INDEX):
            if k != args.config:
                line["per_config"][f"config{k}"] = compact(measure(k))
        line["per_config_note"] = ("the same measurement (device step, sweep roofline, e2e through the public API, "
                                   "CPU baseline) for the other BASELINE configs; the headline is the largest "
                                   "single-GPU configuration")
    if rank == 0:
        print(json.dumps(line), flush=True)


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def spawn_ranks(args) -> int:
    """`bench.py --gpus N` outside torchrun: re-launch under
    torch.distributed.run with N ranks (one per GPU, NCCL), after checking
    that N GPUs are visible."""
    import torch

    have = torch.cuda.device_count()
    if have < args.gpus:
        print(json.dumps({"error": f"--gpus {args.gpus} requested but only {have} CUDA device(s) visible"}),
              flush=True)
        return 2
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), os.path.abspath(__file__),
           *sys.argv[1:]]
    print("+ " + " ".join(cmd), file=sys.stderr, flush=True)
    return subprocess.call(cmd, env=env)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=DEFAULT_CONFIG)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-per-config", action="store_true", help="headline config only")
    ap.add_argument("--no-red-trace", action="store_true", help="skip the RED trace (atomic roof term)")
    ap.add_argument("--no-graph", action="store_true", help="launch the step without CUDA graphs")
    args = ap.parse_args()
    if args.config not in BASELINE_INDEX:
        raise SystemExit(f"--config {args.config}: choose one of 1..5")
    world = _env_int("WORLD_SIZE", 1)
    rank = _env_int("RANK", 0)
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        raise SystemExit(spawn_ranks(args))
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    if world > 1:
        import torch
        import torch.distributed as dist

        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        torch.cuda.set_device(_local_device())
        # MSURF_DIST_BACKEND=gloo lets the N>1 path be exercised with several
        # ranks on one GPU (functional check only; NCCL needs one GPU per rank)
        dist.init_process_group(os.environ.get("MSURF_DIST_BACKEND", "nccl"))
    else:
        import torch

        torch.cuda.set_device(_local_device())
    try:
        run_ours(args, rank, world)
    finally:
        if world > 1:
            import torch.distributed as dist

            dist.destroy_process_group()


if __name__ == "__main__":
    main()
