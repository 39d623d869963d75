"""Load the committed golden fixtures (tests/golden/*.npz) and rebuild the
configurations they were produced from, as plain attribute namespaces (for
the oracle) or as product dataclasses (for the product path)."""

from __future__ import annotations

import glob
import hashlib
import json
import os
from types import SimpleNamespace

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def case_names():
    names = [os.path.basename(p)[:-4] for p in glob.glob(os.path.join(GOLDEN, "*.npz"))]
    return sorted(n for n in names if n != "lhs")


def load(name):
    z = np.load(os.path.join(GOLDEN, f"{name}.npz"))
    out = {k: z[k] for k in z.files}
    out["config"] = json.loads(str(out.pop("config_json")))
    out["counters"] = json.loads(str(out.pop("counters_json")))
    out["roughness"] = json.loads(str(out.pop("roughness_json")))
    out["sha256"] = str(out["sha256"])
    return out


def namespace_config(d, **over):
    t, p, g = d["tool"], d["process"], d["grid"]
    tool = SimpleNamespace(
        cutting_diameter_mm=t["cutting_diameter_mm"], insert_radius_mm=t["insert_radius_mm"],
        tooth_count=t["tooth_count"], radial_rake_rad=t["radial_rake_rad"],
        axial_rake_rad=t["axial_rake_rad"], runouts_mm=tuple(tuple(r) for r in t["runouts_mm"]))
    proc = SimpleNamespace(**{k: v for k, v in p.items()})
    proc.initial_position_mm = tuple(p["initial_position_mm"])
    grid = SimpleNamespace(spacing_mm=g["spacing_mm"], x_min_mm=g["x_min_mm"],
                           y_min_mm=g["y_min_mm"], m=g["m"], n=g["n"])
    grid.x_max_mm = g["x_min_mm"] + g["m"] * g["spacing_mm"]
    grid.y_max_mm = g["y_min_mm"] + g["n"] * g["spacing_mm"]
    cfg = SimpleNamespace(tool=tool, process=proc, grid=grid,
                          edge_point_count=d["edge_point_count"],
                          max_step_angle_rad=d["max_step_angle_rad"],
                          time_step_s=d["time_step_s"],
                          span_s=tuple(d["span_s"]) if d["span_s"] is not None else None,
                          record_trajectory=d["record_trajectory"],
                          worker_count=d["worker_count"])
    for k, v in over.items():
        setattr(cfg, k, v)
    return cfg


def product_config(d, **over):
    import paper_2603_28160_b200 as ms

    t, p, g = d["tool"], d["process"], d["grid"]
    tool = ms.ToolDefinition(
        cutting_diameter_mm=t["cutting_diameter_mm"], insert_radius_mm=t["insert_radius_mm"],
        tooth_count=t["tooth_count"], radial_rake_rad=t["radial_rake_rad"],
        axial_rake_rad=t["axial_rake_rad"], runouts_mm=tuple(tuple(r) for r in t["runouts_mm"]))
    proc = ms.ProcessParameters(
        angular_velocity_rad_s=p["angular_velocity_rad_s"], feed_speed_mm_s=p["feed_speed_mm_s"],
        feed_per_tooth_mm=p["feed_per_tooth_mm"], depth_of_cut_mm=p["depth_of_cut_mm"],
        phase_rad=p["phase_rad"], initial_position_mm=tuple(p["initial_position_mm"]),
        spindle_speed_rpm=p["spindle_speed_rpm"], cutting_speed_m_min=p["cutting_speed_m_min"])
    grid = ms.GridSpec(spacing_mm=g["spacing_mm"], x_min_mm=g["x_min_mm"], y_min_mm=g["y_min_mm"],
                       m=g["m"], n=g["n"])
    kw = dict(tool=tool, process=proc, grid=grid, edge_point_count=d["edge_point_count"],
              max_step_angle_rad=d["max_step_angle_rad"], time_step_s=d["time_step_s"],
              span_s=tuple(d["span_s"]) if d["span_s"] is not None else None,
              record_trajectory=d["record_trajectory"], worker_count=d["worker_count"])
    kw.update(over)
    return ms.SimulationConfig(**kw)


def heights_match(golden, heights):
    """Bitwise comparison against a golden entry (full array or SHA-256 + rows)."""
    h = np.ascontiguousarray(heights, dtype=np.float64)
    if "heights" in golden:
        return bool(np.array_equal(golden["heights"], h))
    return hashlib.sha256(h.tobytes()).hexdigest() == golden["sha256"]


def max_abs_diff(golden, heights, n1):
    h = np.asarray(heights, dtype=np.float64)
    if "heights" in golden:
        return float(np.max(np.abs(golden["heights"] - h)))
    stride = int(golden["row_stride"])
    return float(np.max(np.abs(golden["rows_sampled"] - h.reshape(-1, n1)[::stride])))
