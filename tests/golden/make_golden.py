"""Generate the golden fixtures under tests/golden/ from the REAL reference.

Runs only in the build container, where the reference package is mounted
read-only at /root/reference/pkg (it does not exist on the GPU box, which only
reads the committed .npz files). Usage:

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

Cases (all reference-representable, i.e. computed by ``millsurf.simulate``):
  * ``small_<seed>``: helpers.small_random_config seeds 0-4 (test_engine.py:127-137)
    and 1000-1019 (acceptance criterion 1, test_acceptance.py:50-57), with the
    trajectory record;
  * ``tiny``: test_engine.py:20-27 tiny_config;
  * ``cusp``: helpers.front_cut_config(0.6, 0.002) (acceptance criterion 2);
  * ``runout``: front_cut_config(0.5, 0.004, runouts (0,0),(0,0.009)) (criterion 3);
  * ``table6_3``: test_acceptance.py:207-222 condition 3 at dt=1e-4 (bench_10x5 geometry);
  * ``config1_ref``: the BASELINE config-1 analog without helix.
Heights are stored in full for grids up to 200k nodes, otherwise as a SHA-256
of the fp64 buffer plus every 37th row. Roughness (areal over the largest
machined rectangle, helpers.machined_rect_roi; feed-profile Ra) is stored from
millsurf.areal_metrics / line_roughness. LHS draws (dataset.py:91-105) too.
"""

from __future__ import annotations

import hashlib
import json
import math
import os
import sys

import numpy as np

REF = "/root/reference/pkg"
sys.dont_write_bytecode = True
sys.path.insert(0, os.path.join(REF, "src"))
sys.path.insert(0, os.path.join(REF, "tests"))

import millsurf  # noqa: E402
from millsurf import (  # noqa: E402
    GridSpec, ParameterRange, SimulationConfig, ToolDefinition, areal_metrics,
    derive_kinematics, extract_profile, lhs_sample, line_roughness, simulate,
)
import helpers  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))
FULL_LIMIT = 200_000


def cfg_to_dict(cfg: SimulationConfig) -> dict:
    t, p, g = cfg.tool, cfg.process, cfg.grid
    return {
        "tool": {
            "cutting_diameter_mm": t.cutting_diameter_mm, "insert_radius_mm": t.insert_radius_mm,
            "tooth_count": t.tooth_count, "radial_rake_rad": t.radial_rake_rad,
            "axial_rake_rad": t.axial_rake_rad, "runouts_mm": [list(r) for r in t.runouts_mm],
        },
        "process": {
            "angular_velocity_rad_s": p.angular_velocity_rad_s, "feed_speed_mm_s": p.feed_speed_mm_s,
            "feed_per_tooth_mm": p.feed_per_tooth_mm, "depth_of_cut_mm": p.depth_of_cut_mm,
            "phase_rad": p.phase_rad, "initial_position_mm": list(p.initial_position_mm),
            "spindle_speed_rpm": p.spindle_speed_rpm, "cutting_speed_m_min": p.cutting_speed_m_min,
        },
        "grid": {"spacing_mm": g.spacing_mm, "x_min_mm": g.x_min_mm, "y_min_mm": g.y_min_mm,
                 "m": g.m, "n": g.n},
        "edge_point_count": cfg.edge_point_count,
        "max_step_angle_rad": cfg.max_step_angle_rad,
        "time_step_s": cfg.time_step_s,
        "span_s": list(cfg.span_s) if cfg.span_s is not None else None,
        "record_trajectory": cfg.record_trajectory,
        "worker_count": cfg.worker_count,
    }


def config1_ref() -> SimulationConfig:
    """BASELINE config 1 (reference analog, helix omitted): 4 teeth, D=10,
    R=5, a_p=1, 3000 rpm, fz=0.05, N=200, 3600 steps/rev, 20 revs, 200x200
    nodes at 10 um, x0=0, start y=-2 (SURVEY Appendix B pins)."""
    tool = ToolDefinition(cutting_diameter_mm=10.0, insert_radius_mm=5.0, tooth_count=4)
    proc = derive_kinematics(tooth_count=4, cutting_diameter_mm=10.0, depth_of_cut_mm=1.0,
                             spindle_speed_rpm=3000.0, feed_per_tooth_mm=0.05,
                             initial_position_mm=(0.0, -2.0, 0.0))
    grid = GridSpec(spacing_mm=0.01, x_min_mm=-0.995, y_min_mm=0.0, m=199, n=199)
    omega = proc.angular_velocity_rad_s
    dt = (2.0 * math.pi / 3600.0) / omega
    return SimulationConfig(tool=tool, process=proc, grid=grid, edge_point_count=200,
                            time_step_s=dt, span_s=(0.0, 20.0 * (2.0 * math.pi) / omega),
                            worker_count=os.cpu_count() or 1)


def table6_3() -> SimulationConfig:
    proc = derive_kinematics(tooth_count=2, cutting_diameter_mm=10.0, depth_of_cut_mm=0.5,
                             cutting_speed_m_min=170.0, feed_per_tooth_mm=0.6,
                             initial_position_mm=(0.0, None, 0.0))
    grid = GridSpec.from_extents(0.01, (-5.0, 5.0), (0.0, 5.0))
    return SimulationConfig(tool=helpers.case1_tool(), process=proc, grid=grid,
                            edge_point_count=40, time_step_s=1e-4, worker_count=os.cpu_count() or 1)


def tiny() -> SimulationConfig:
    tool = helpers.case1_tool()
    process = helpers.case1_process(x0=0.0)
    grid = GridSpec.from_extents(0.05, (-0.5, 0.5), (0.0, 0.5))
    return SimulationConfig(tool=tool, process=process, grid=grid, edge_point_count=7,
                            time_step_s=2e-4, record_trajectory=True, worker_count=1)


def roughness_payload(field) -> dict:
    out = {}
    roi = helpers.machined_rect_roi(field)
    out["roi"] = list(roi) if roi is not None else None
    if roi is not None:
        i_lo, j_lo, i_hi, j_hi = roi
        if (i_hi - i_lo + 1) * (j_hi - j_lo + 1) >= 4:
            am = areal_metrics(field, roi=roi)
            out["areal"] = am.to_json_dict()
            if j_hi - j_lo >= 1:
                idx = (i_lo + i_hi) // 2
                prof = extract_profile(field, "feed", index=idx, roi=roi)
                out["profile_index"] = idx
                out["Ra"] = line_roughness(prof)
    try:
        out["areal_full"] = areal_metrics(field).to_json_dict()
    except millsurf.DomainError as exc:
        out["areal_full_error"] = str(exc)
    return out


def save_case(name: str, cfg: SimulationConfig) -> None:
    res = simulate(cfg)
    h = res.field.heights
    payload = {
        "config_json": json.dumps(cfg_to_dict(cfg)),
        "counters_json": json.dumps({
            "time_steps": res.time_steps, "trajectory_points": res.trajectory_points,
            "cells_updated": res.cells_updated, "initial_height": res.field.initial_height_mm,
        }),
        "roughness_json": json.dumps(roughness_payload(res.field)),
        "sha256": np.array(hashlib.sha256(h.tobytes()).hexdigest()),
    }
    if h.size <= FULL_LIMIT:
        payload["heights"] = h
    else:
        arr = res.field.as_array()
        payload["row_stride"] = np.array(37)
        payload["rows_sampled"] = np.ascontiguousarray(arr[::37])
    if res.trajectory is not None:
        n = len(res.trajectory)
        tr = res.trajectory
        payload["traj"] = np.stack([tr.t_s[:n], tr.tooth[:n].astype(np.float64),
                                    tr.x_mm[:n], tr.y_mm[:n], tr.z_mm[:n]])
    np.savez_compressed(os.path.join(OUT, f"{name}.npz"), **payload)
    print(name, res.time_steps, res.trajectory_points, res.cells_updated, h.size)


def save_lhs() -> None:
    names = ["cutting_speed_m_min", "feed_per_tooth_mm", "depth_of_cut_mm",
             "grid_spacing_mm", "radial_rake_deg", "phase_deg"]
    bounds = [(100.0, 250.0), (0.2, 0.7), (0.1, 0.5), (0.005, 0.05), (-2.0, 2.0), (0.0, 180.0)]
    ranges = [ParameterRange(nm, lo, hi) for nm, (lo, hi) in zip(names, bounds)]
    out = {}
    for count, seed in ((1, 0), (7, 3), (37, 5), (256, 0)):
        out[f"lhs_{count}_{seed}"] = lhs_sample(ranges, count, seed)
    out["bounds"] = np.array(bounds)
    np.savez_compressed(os.path.join(OUT, "lhs.npz"), **out)


def main() -> None:
    for seed in list(range(5)) + list(range(1000, 1020)):
        save_case(f"small_{seed}", helpers.small_random_config(seed))
    save_case("tiny", tiny())
    save_case("cusp", helpers.front_cut_config(feed_per_tooth_mm=0.6, spacing_mm=0.002))
    save_case("runout", helpers.front_cut_config(feed_per_tooth_mm=0.5, spacing_mm=0.004,
                                                 runouts=((0.0, 0.0), (0.0, 0.009))))
    save_case("table6_3", table6_3())
    save_case("config1_ref", config1_ref())
    save_lhs()


if __name__ == "__main__":
    main()
