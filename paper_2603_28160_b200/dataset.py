"""Batched parameter-set mode (surrogate-dataset production).

Sampling restates millsurf/dataset.py:91-105 (seeded Latin hypercube,
numpy PCG64 ``default_rng(seed)``, per dimension ``permutation`` then
``random``) so the same seed yields the same parameter table bit-for-bit;
``uniform_sample`` draws i.i.d. uniform columns (BASELINE config 3).
``generate_batch`` then sweeps every parameter set in the SAME kernel
launches (``simulate_batch``: one fill, one sweep per kinematics mode, one
decode) and reduces all areal metrics in two more launches; a sample whose
configuration is invalid is reported per row without aborting the batch
(dataset.py:155-185).
"""

from __future__ import annotations

import json
import math
from dataclasses import dataclass, replace

import numpy as np

from .engine import simulate_batch
from .errors import ConfigError, MillsurfError
from .extensions import Extensions
from .grid import GridSpec
from .kinematics import derive_kinematics
from .geometry import ToolDefinition
from .roughness import areal_metrics_batch

# reference names (dataset.py:36-48) + the extended-model parameters
REFERENCE_NAMES = ("cutting_speed_m_min", "spindle_speed_rpm", "feed_per_tooth_mm", "depth_of_cut_mm",
                   "phase_deg", "grid_spacing_mm", "radial_rake_deg", "axial_rake_deg",
                   "runout_radial_mm", "runout_axial_mm")
EXTENDED_NAMES = ("runout_offset_mm", "runout_phase_rad", "helix_angle_rad", "helix_angle_deg",
                  "tilt_rad", "vib_amplitude_mm")
PARAMETER_NAMES = REFERENCE_NAMES + EXTENDED_NAMES
_POSITIVE = {"cutting_speed_m_min", "spindle_speed_rpm", "feed_per_tooth_mm", "depth_of_cut_mm",
             "grid_spacing_mm"}


@dataclass(frozen=True)
class ParameterRange:
    """Closed interval of one named parameter (dataset.py:60-80 validation)."""

    name: str
    low: float
    high: float

    def __post_init__(self) -> None:
        if self.name not in PARAMETER_NAMES:
            raise ConfigError(f"unknown dataset parameter {self.name!r}; known: {', '.join(PARAMETER_NAMES)}")
        if not self.low < self.high:
            raise ConfigError(f"range for {self.name}: low {self.low} must be < high {self.high}")
        if self.name in _POSITIVE and self.low <= 0:
            raise ConfigError(f"range for {self.name}: bounds must be > 0, got low {self.low}")
        if self.name in ("radial_rake_deg", "axial_rake_deg") and (self.low <= -90 or self.high >= 90):
            raise ConfigError(f"range for {self.name}: must stay within (-90, 90) degrees")


def lhs_sample(ranges, count: int, seed: int) -> np.ndarray:
    """(count, dims) Latin hypercube, one sample per stratum per dimension."""
    if count < 1:
        raise ConfigError(f"sample count must be >= 1, got {count}")
    if not ranges:
        raise ConfigError("at least one parameter range is required")
    rng = np.random.default_rng(seed)
    out = np.empty((count, len(ranges)), dtype=np.float64)
    for d, prm in enumerate(ranges):
        strata = rng.permutation(count)
        offsets = rng.random(count)
        out[:, d] = prm.low + (prm.high - prm.low) * ((strata + offsets) / count)
    return out


def uniform_sample(ranges, count: int, seed: int) -> np.ndarray:
    """(count, dims) i.i.d. uniform draws, row-major from default_rng(seed).random."""
    if count < 1:
        raise ConfigError(f"sample count must be >= 1, got {count}")
    if not ranges:
        raise ConfigError("at least one parameter range is required")
    u = np.random.default_rng(seed).random((count, len(ranges)))
    lo = np.array([r.low for r in ranges])
    hi = np.array([r.high for r in ranges])
    return lo + (hi - lo) * u


def apply_sample(config, ext: Extensions | None, names, values, steps_per_rev: float | None = None):
    """Return (config, ext) with the sampled values applied (dataset.py:108-136
    semantics for the reference names: rpm/v_c and f_z re-derived canonically,
    run-outs applied to every tooth)."""
    ext = ext or Extensions()
    tool, proc, grid = config.tool, config.process, config.grid
    kin = {"rpm": proc.spindle_speed_rpm, "fz": proc.feed_per_tooth_mm, "vc": None,
           "ap": proc.depth_of_cut_mm, "phase": proc.phase_rad}
    tool_kw = {}
    ext_kw = {}
    runout_r = runout_a = None
    spacing = None
    for name, v in zip(names, values):
        v = float(v)
        if name == "spindle_speed_rpm":
            kin["rpm"], kin["vc"] = v, None
        elif name == "cutting_speed_m_min":
            kin["vc"], kin["rpm"] = v, None
        elif name == "feed_per_tooth_mm":
            kin["fz"] = v
        elif name == "depth_of_cut_mm":
            kin["ap"] = v
        elif name == "phase_deg":
            kin["phase"] = math.radians(v)
        elif name == "grid_spacing_mm":
            spacing = v
        elif name == "radial_rake_deg":
            tool_kw["radial_rake_rad"] = math.radians(v)
        elif name == "axial_rake_deg":
            tool_kw["axial_rake_rad"] = math.radians(v)
        elif name == "runout_radial_mm":
            runout_r = v
        elif name == "runout_axial_mm":
            runout_a = v
        elif name == "helix_angle_deg":
            ext_kw["helix_angle_rad"] = math.radians(v)
        elif name in EXTENDED_NAMES:
            ext_kw[name] = v
        else:
            raise ConfigError(f"unknown dataset parameter {name!r}")
    if runout_r is not None or runout_a is not None:
        tool_kw["runouts_mm"] = tuple((runout_r if runout_r is not None else p[0],
                                       runout_a if runout_a is not None else p[1]) for p in tool.runouts_mm)
    if tool_kw:
        tool = ToolDefinition(**{**tool.__dict__, **tool_kw})
    if spacing is not None:
        grid = GridSpec.from_extents(spacing, (grid.x_min_mm, grid.x_max_mm), (grid.y_min_mm, grid.y_max_mm))
    if kin["rpm"] is None and kin["vc"] is None:
        raise ConfigError("base process has no spindle speed")
    proc = derive_kinematics(tooth_count=tool.tooth_count, cutting_diameter_mm=tool.cutting_diameter_mm,
                             depth_of_cut_mm=kin["ap"], cutting_speed_m_min=kin["vc"],
                             spindle_speed_rpm=kin["rpm"], feed_per_tooth_mm=kin["fz"],
                             phase_rad=kin["phase"], initial_position_mm=proc.initial_position_mm)
    cfg = replace(config, tool=tool, process=proc, grid=grid)
    if steps_per_rev is not None:
        cfg = replace(cfg, time_step_s=(2.0 * math.pi / steps_per_rev) / proc.angular_velocity_rad_s)
    if ext_kw:
        ext = replace(ext, **ext_kw)
    return cfg, ext


@dataclass
class BatchRow:
    index: int
    params: dict
    status: str
    error: str | None
    metrics: dict | None
    metrics_error: str | None
    counters: dict | None


@dataclass
class BatchResult:
    samples: np.ndarray
    rows: list
    results: list
    device_seconds: float


def generate_batch(base_config, base_ext: Extensions | None, ranges, count: int, seed: int, *,
                   sampler: str = "lhs", steps_per_rev: float | None = None, roi=None,
                   uncut: str = "raise", sample_slice: slice | None = None, keep_fields: bool = True):
    """Sample ``count`` parameter sets, sweep them all in one batched launch,
    reduce all areal metrics in one batched launch. ``sample_slice`` selects
    the rows this process owns (parameter-set sharding across GPUs)."""
    if sampler == "lhs":
        samples = lhs_sample(ranges, count, seed)
    elif sampler == "uniform":
        samples = uniform_sample(ranges, count, seed)
    else:
        raise ConfigError(f"sampler must be 'lhs' or 'uniform', got {sampler!r}")
    names = [r.name for r in ranges]
    idx = list(range(count))[sample_slice] if sample_slice is not None else list(range(count))
    rows, cfgs, exts, ok_rows = [], [], [], []
    for i in idx:
        params = {n: float(samples[i, d]) for d, n in enumerate(names)}
        row = BatchRow(index=i, params=params, status="ok", error=None, metrics=None,
                       metrics_error=None, counters=None)
        try:
            c, e = apply_sample(base_config, base_ext, names, samples[i], steps_per_rev)
            cfgs.append(c)
            exts.append(e)
            ok_rows.append(row)
        except MillsurfError as exc:
            row.status, row.error = "failed", str(exc)
        rows.append(row)
    results = []
    dev_s = 0.0
    if cfgs:
        try:
            results = simulate_batch(cfgs, exts)
        except MillsurfError:
            # isolate per-sample failures (e.g. planning errors) like dataset.py:181-184
            results = []
            for row, c, e in zip(ok_rows, cfgs, exts):
                try:
                    results.extend(simulate_batch([c], [e]))
                except MillsurfError as exc:
                    row.status, row.error = "failed", str(exc)
            ok_rows = [r for r in ok_rows if r.status == "ok"]
        dev_s = sum(r.main_loop_seconds for r in results)
        mets = areal_metrics_batch([r.field for r in results], roi=roi, uncut=uncut)
        for row, res, met in zip(ok_rows, results, mets):
            row.counters = {"time_steps": res.time_steps, "trajectory_points": res.trajectory_points,
                            "cells_updated": res.cells_updated}
            if isinstance(met, Exception):
                row.metrics_error = str(met)
            else:
                row.metrics = met.to_json_dict()
    if not keep_fields:
        results = []
    return BatchResult(samples=samples, rows=rows, results=results, device_seconds=dev_s)


# ---------------------------------------------------------------- datasets
SCHEMA_VERSION = 1                      # dataset.py:31
RNG_NAME = "numpy-default-pcg64"        # dataset.py:32
# reference parameter -> (config block, key, keys cleared with it) (dataset.py:37-48)
_RAW_PATHS = {
    "cutting_speed_m_min": ("process", "cutting_speed_m_min", ("spindle_speed_rpm",)),
    "spindle_speed_rpm": ("process", "spindle_speed_rpm", ("cutting_speed_m_min",)),
    "feed_per_tooth_mm": ("process", "feed_per_tooth_mm", ("feed_speed_mm_min",)),
    "depth_of_cut_mm": ("process", "depth_of_cut_mm", ()),
    "phase_deg": ("process", "phase_deg", ("phase_rad",)),
    "grid_spacing_mm": ("grid", "spacing_mm", ()),
    "radial_rake_deg": ("tool", "radial_rake_deg", ("radial_rake_rad",)),
    "axial_rake_deg": ("tool", "axial_rake_deg", ("axial_rake_rad",)),
    # extended-model parameters land in the optional ``extensions`` block
    "runout_offset_mm": ("extensions", "runout_offset_mm", ()),
    "runout_phase_rad": ("extensions", "runout_phase_rad", ()),
    "helix_angle_rad": ("extensions", "helix_angle_rad", ()),
    "tilt_rad": ("extensions", "tilt_rad", ()),
    "vib_amplitude_mm": ("extensions", "vib_amplitude_mm", ()),
}
_RUNOUT_NAMES = ("runout_radial_mm", "runout_axial_mm")
# surfaces swept per launch group: bounds the HBM held by one group of Z-maps
DATASET_NODE_BUDGET = int(2.5e8)


@dataclass
class DatasetManifest:
    """dataset.py:83-88."""

    seed: int
    count: int
    rows: list
    path: object


def apply_overrides(base_raw: dict, names, values) -> dict:
    """Sampled values into a copy of the raw JSON config (dataset.py:108-136):
    sibling keys of a pair are cleared, run-outs rewrite every tooth's pair."""
    import copy

    raw = copy.deepcopy(base_raw)
    runout = {}
    for name, value in zip(names, values):
        value = float(value)
        if name in _RUNOUT_NAMES:
            runout[name] = value
            continue
        if name == "helix_angle_deg":
            name, value = "helix_angle_rad", math.radians(value)
        block, key, clears = _RAW_PATHS[name]
        blk = raw.setdefault(block, {})
        blk[key] = value
        for c in clears:
            blk.pop(c, None)
    if runout:
        tool = raw.setdefault("tool", {})
        pairs = tool.get("runouts_mm") or [[0.0, 0.0] for _ in range(tool.get("tooth_count", 1))]
        r = runout.get("runout_radial_mm")
        a = runout.get("runout_axial_mm")
        tool["runouts_mm"] = [[r if r is not None else p[0], a if a is not None else p[1]] for p in pairs]
    return raw


def _check_ranges_against_base(ranges, base_raw: dict) -> None:
    """dataset.py:139-152."""
    radius = base_raw.get("tool", {}).get("insert_radius_mm")
    if not isinstance(radius, (int, float)):
        return
    for prm in ranges:
        if prm.name == "depth_of_cut_mm" and prm.high > radius:
            raise ConfigError(f"range for depth_of_cut_mm: high {prm.high} exceeds insert radius {radius}")
        if prm.name in _RUNOUT_NAMES and max(abs(prm.low), abs(prm.high)) >= radius:
            raise ConfigError(f"range for {prm.name}: magnitude must stay below insert radius {radius}")


def _new_row(index: int, params: dict) -> dict:
    # key order of dataset.py:156-165 (the manifest bytes depend on it)
    return {"index": index, "params": params, "surface_file": f"sample_{index:05d}.srtf", "status": "ok",
            "error": None, "metrics": None, "metrics_error": None, "counters": None}


def _fail(row: dict, exc: Exception) -> None:
    row["status"], row["error"], row["surface_file"] = "failed", str(exc), None


def generate_dataset(ranges, count: int, seed: int, base_raw: dict, out_dir, workers: int = 1,
                     *, node_budget: int = DATASET_NODE_BUDGET) -> DatasetManifest:
    """LHS-sampled surfaces + SRTF files + JSON-lines manifest
    (dataset.py:188-241), with every parameter set of a launch group swept
    in ONE batched sweep launch and reduced in one batched metrics launch;
    each surface streams from HBM into its SRTF file. ``workers`` is accepted
    for compatibility (the result never depends on it, as in the reference).
    A failing sample is recorded in place and does not abort the batch."""
    from pathlib import Path

    from .config import config_from_dict
    from .engine import _launch_results
    from .planner import plan as make_plan
    from .roughness import areal_metrics_batch
    from .surface_io import write_surface

    config_from_dict(base_raw)  # fail fast on a broken base configuration
    _check_ranges_against_base(ranges, base_raw)
    samples = lhs_sample(ranges, count, seed)
    names = [p.name for p in ranges]
    out_dir = Path(out_dir)
    out_dir.mkdir(parents=True, exist_ok=True)
    manifest_path = out_dir / "manifest.jsonl"
    header = {"schema_version": SCHEMA_VERSION, "seed": seed, "count": count, "rng": RNG_NAME,
              "ranges": [{"name": p.name, "low": p.low, "high": p.high} for p in ranges],
              "base_config": base_raw}

    rows, planned = [], []
    for i in range(count):
        row = _new_row(i, {n: float(samples[i, d]) for d, n in enumerate(names)})
        rows.append(row)
        try:
            doc = config_from_dict(apply_overrides(base_raw, names, samples[i]))
            cfg = replace(doc.to_simulation_config(), worker_count=1, record_trajectory=False)
            planned.append((row, make_plan(cfg, doc.extensions)))
        except MillsurfError as exc:
            _fail(row, exc)

    # launch groups under the node budget; results are consumed group by group
    groups, cur, nodes = [], [], 0
    for item in planned:
        k = item[1].grid.node_count
        if cur and nodes + k > node_budget:
            groups.append(cur)
            cur, nodes = [], 0
        cur.append(item)
        nodes += k
    if cur:
        groups.append(cur)
    # the manifest is appended in index order as groups complete (header first,
    # one row per sample, flushed: a partial run leaves a valid prefix)
    with open(manifest_path, "w", encoding="utf-8") as fh:
        fh.write(json.dumps(header) + "\n")
        fh.flush()
        done = 0

        def emit(upto):
            nonlocal done
            for row in rows[done:upto]:
                fh.write(json.dumps(row) + "\n")
            fh.flush()
            done = max(done, upto)

        for g_idx, grp in enumerate(groups):
            results = _launch_results([p for _, p in grp], "device")
            mets = areal_metrics_batch([r.field for r in results])
            for (row, _), res, met in zip(grp, results, mets):
                try:
                    write_surface(res.field, out_dir / row["surface_file"])
                except MillsurfError as exc:
                    _fail(row, exc)
                    continue
                row["counters"] = {"time_steps": res.time_steps, "trajectory_points": res.trajectory_points,
                                   "cells_updated": res.cells_updated}
                if isinstance(met, MillsurfError):
                    row["metrics_error"] = str(met)
                else:
                    row["metrics"] = met.to_json_dict()
            nxt = groups[g_idx + 1][0][0]["index"] if g_idx + 1 < len(groups) else count
            emit(nxt)
        emit(count)
    return DatasetManifest(seed=seed, count=count, rows=rows, path=manifest_path)
