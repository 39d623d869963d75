"""Build container only (reads /root/reference): the reference's own
millsurf.simulate against the oracle port that bench.py --impl reference
times, on the same reference-representable golden configurations, same
worker counts — heights must be equal and the timings show the port is a
faithful stand-in for the reference's CPU throughput.
    python tools/ref_vs_port_cpu.py"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402

import golden_io  # noqa: E402
import millsurf  # noqa: E402
from oracle import fsm_oracle as orc  # noqa: E402


def ref_config(d, **over):
    t, p, g = d["tool"], d["process"], d["grid"]
    tool = millsurf.ToolDefinition(
        cutting_diameter_mm=t["cutting_diameter_mm"], insert_radius_mm=t["insert_radius_mm"],
        tooth_count=t["tooth_count"], radial_rake_rad=t["radial_rake_rad"], axial_rake_rad=t["axial_rake_rad"],
        runouts_mm=tuple(tuple(r) for r in t["runouts_mm"]))
    proc = millsurf.ProcessParameters(
        angular_velocity_rad_s=p["angular_velocity_rad_s"], feed_speed_mm_s=p["feed_speed_mm_s"],
        feed_per_tooth_mm=p["feed_per_tooth_mm"], depth_of_cut_mm=p["depth_of_cut_mm"], phase_rad=p["phase_rad"],
        initial_position_mm=tuple(p["initial_position_mm"]), spindle_speed_rpm=p["spindle_speed_rpm"],
        cutting_speed_m_min=p["cutting_speed_m_min"])
    grid = millsurf.GridSpec(spacing_mm=g["spacing_mm"], x_min_mm=g["x_min_mm"], y_min_mm=g["y_min_mm"], m=g["m"],
                             n=g["n"])
    kw = dict(tool=tool, process=proc, grid=grid, edge_point_count=d["edge_point_count"],
              max_step_angle_rad=d["max_step_angle_rad"], time_step_s=d["time_step_s"],
              span_s=tuple(d["span_s"]) if d["span_s"] is not None else None, record_trajectory=False,
              worker_count=d["worker_count"])
    kw.update(over)
    return millsurf.SimulationConfig(**kw)


for name in ("config1_ref", "table6_3", "small_0"):
    d = golden_io.load(name)["config"]
    for w in (1, 16):
        t0 = time.perf_counter()
        r = millsurf.simulate(ref_config(d, worker_count=w))
        t1 = time.perf_counter()
        h, _, _, _ = orc.sweep(golden_io.product_config(d, worker_count=w, record_trajectory=False), workers=w)
        t2 = time.perf_counter()
        print(f"{name:12s} workers={w:2d}: reference {t1 - t0:7.3f} s, oracle port {t2 - t1:7.3f} s, "
              f"heights equal {np.array_equal(np.asarray(r.field.heights), h)}, points {r.trajectory_points:.3g}")
