"""BASELINE WORKLOADS, ORACLE SIDE — TEST INFRASTRUCTURE ONLY.

The five BASELINE.json configurations restated as plain objects the CPU
oracle (``fsm_oracle`` / ``fsm_ext_oracle``) consumes, WITHOUT importing the
product package. ``bench.py --impl reference`` builds its workload here, so
the reference arm runs nothing of ``paper_2603_28160_b200`` (no product
Python, no ``libmsurf.so``); the fixture generator
``tests/golden/make_golden_configs.py`` uses it too.

Every pinned value is the one DESIGN.md §3.2 records ([B] = builder's
choice); ``tests/test_host_cpu.py::test_oracle_workloads_equal_product_configs``
checks field by field that these objects equal the product's
``paper_2603_28160_b200/configs.py`` (including the derived kinematics), so
both arms time the same workload.

Derived kinematics restate the reference's ``derive_kinematics``
(/root/reference/pkg/src/millsurf/kinematics.py:217-274): omega = 2 pi n/60,
v_f = f_z Z n/60, canonical in (rpm, f_z).
"""

from __future__ import annotations

import math
from dataclasses import dataclass, replace

import numpy as np


@dataclass(frozen=True)
class Tool:
    cutting_diameter_mm: float
    insert_radius_mm: float
    tooth_count: int
    radial_rake_rad: float = 0.0
    axial_rake_rad: float = 0.0
    runouts_mm: tuple = ()

    def __post_init__(self):
        if not self.runouts_mm:
            object.__setattr__(self, "runouts_mm", ((0.0, 0.0),) * self.tooth_count)


@dataclass(frozen=True)
class Process:
    angular_velocity_rad_s: float
    feed_speed_mm_s: float
    feed_per_tooth_mm: float
    depth_of_cut_mm: float
    phase_rad: float
    initial_position_mm: tuple
    spindle_speed_rpm: float
    cutting_speed_m_min: float


@dataclass(frozen=True)
class Grid:
    spacing_mm: float
    x_min_mm: float
    y_min_mm: float
    m: int
    n: int


@dataclass(frozen=True)
class Config:
    tool: Tool
    process: Process
    grid: Grid
    edge_point_count: int | None = None
    time_step_s: float | None = None
    max_step_angle_rad: float = math.radians(1.0)
    span_s: tuple | None = None
    worker_count: int = 1
    record_trajectory: bool = False


@dataclass(frozen=True)
class Ext:
    profile: str = "insert"
    helix_angle_rad: float = 0.0
    helix_ref_radius_mm: float | None = None
    runout_offset_mm: float = 0.0
    runout_phase_rad: float = 0.0
    tilt_rad: float = 0.0
    vib_amplitude_mm: float = 0.0
    vib_frequency_hz: float = 0.0
    vib_phase_rad: float = 0.0
    noise_sigma_mm: float = 0.0
    noise_corr_mm: float = 0.0
    noise_seed: int = 0
    passes: int = 1
    stepover_mm: float = 0.0
    force_extended: bool = False


def process(tooth_count, diameter, a_p, rpm, f_z, phase=0.0, initial=(0.0, None, 0.0)) -> Process:
    """kinematics.py:217-274 (rpm and f_z given)."""
    return Process(angular_velocity_rad_s=2.0 * math.pi * rpm / 60.0,
                   feed_speed_mm_s=f_z * tooth_count * rpm / 60.0, feed_per_tooth_mm=f_z,
                   depth_of_cut_mm=a_p, phase_rad=phase, initial_position_mm=initial,
                   spindle_speed_rpm=rpm, cutting_speed_m_min=math.pi * diameter * rpm / 1000.0)


def _dt(proc, steps_per_rev):
    return (2.0 * math.pi / steps_per_rev) / proc.angular_velocity_rad_s


def _centered(nodes_x, nodes_y, spacing, y_min=0.0):
    return Grid(spacing, -0.5 * (nodes_x - 1) * spacing, y_min, nodes_x - 1, nodes_y - 1)


def config1():
    tool = Tool(10.0, 5.0, 4)
    proc = process(4, 10.0, 1.0, 3000.0, 0.05, initial=(0.0, -2.0, 0.0))
    cfg = Config(tool, proc, Grid(0.01, -0.995, 0.0, 199, 199), edge_point_count=200,
                 time_step_s=_dt(proc, 3600),
                 span_s=(0.0, 20.0 * (2.0 * math.pi) / proc.angular_velocity_rad_s))
    return cfg, Ext(helix_angle_rad=math.radians(30.0)), {"name": "config1", "profiles_every": 64,
                                                          "uncut": "exclude"}


def config2():
    tool = Tool(6.0, 3.0, 2)
    proc = process(2, 6.0, 0.2, 6000.0, 0.08, initial=(-0.75, None, 0.0))
    cfg = Config(tool, proc, _centered(1000, 1000, 0.002), edge_point_count=500, time_step_s=_dt(proc, 7200))
    ext = Ext(profile="ball", helix_angle_rad=math.radians(30.0), tilt_rad=math.radians(15.0),
              runout_offset_mm=0.005, runout_phase_rad=math.radians(40.0), passes=6, stepover_mm=0.3)
    return cfg, ext, {"name": "config2", "profiles_every": 64, "uncut": "exclude"}


CONFIG3_RANGES = (("feed_per_tooth_mm", 0.02, 0.2), ("spindle_speed_rpm", 2000.0, 12000.0),
                  ("runout_offset_mm", 0.0, 0.010), ("runout_phase_rad", 0.0, 2.0 * math.pi),
                  ("helix_angle_deg", 20.0, 45.0))


def config3_base():
    tool = Tool(8.0, 4.0, 4)
    proc = process(4, 8.0, 0.5, 6000.0, 0.1)
    cfg = Config(tool, proc, _centered(512, 512, 0.004), edge_point_count=300)
    return cfg, Ext(helix_angle_rad=math.radians(30.0)), {
        "name": "config3", "count": 256, "seed": 0, "steps_per_rev": 3600, "ranges": CONFIG3_RANGES,
        "sampler": "uniform", "uncut": "exclude"}


def config3_sets():
    """All 256 parameter sets: default_rng(0).random((256, 5)) scaled to the
    ranges (row-major), applied as the product's dataset.apply_sample does
    for these names (rpm and f_z re-derived, dt from 3600 steps/rev)."""
    base, ext, meta = config3_base()
    lo = np.array([r[1] for r in CONFIG3_RANGES])
    hi = np.array([r[2] for r in CONFIG3_RANGES])
    u = np.random.default_rng(meta["seed"]).random((meta["count"], len(CONFIG3_RANGES)))
    samples = lo + (hi - lo) * u
    out = []
    for row in samples:
        fz, rpm, rho, lam, helix = (float(v) for v in row)
        proc = process(4, 8.0, base.process.depth_of_cut_mm, rpm, fz, base.process.phase_rad,
                       base.process.initial_position_mm)
        cfg = replace(base, process=proc, time_step_s=_dt(proc, meta["steps_per_rev"]))
        out.append((cfg, replace(ext, runout_offset_mm=rho, runout_phase_rad=lam,
                                 helix_angle_rad=math.radians(helix))))
    return out, samples, meta


def config4():
    tool = Tool(12.0, 6.0, 4)
    proc = process(4, 12.0, 1.0, 3000.0, 0.1)
    cfg = Config(tool, proc, _centered(10000, 10000, 0.001), edge_point_count=1000,
                 time_step_s=_dt(proc, 14400))
    ext = Ext(runout_offset_mm=0.003, vib_amplitude_mm=0.002, vib_frequency_hz=1.7 * 4 * 3000.0 / 60.0)
    return cfg, ext, {"name": "config4", "profiles_every": 64, "uncut": "exclude"}


def config5():
    tool = Tool(4.0, 2.0, 3)
    proc = process(3, 4.0, 0.1, 6000.0, 0.06, initial=(-1.5, None, 0.0))
    cfg = Config(tool, proc, _centered(4096, 4096, 0.001), edge_point_count=2000, time_step_s=_dt(proc, 14400))
    ext = Ext(profile="ball", tilt_rad=math.radians(10.0), runout_offset_mm=0.004, noise_sigma_mm=0.001,
              noise_corr_mm=0.020, noise_seed=0, passes=16, stepover_mm=0.2)
    return cfg, ext, {"name": "config5", "profiles_every": 64, "uncut": "exclude"}


FACTORIES = {1: config1, 2: config2, 4: config4, 5: config5}
