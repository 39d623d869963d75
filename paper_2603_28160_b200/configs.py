"""The five BASELINE.json workloads, pinned (DESIGN.md Appendix A lists every
value the BASELINE text leaves open, marked [B] below). Each factory returns
(SimulationConfig, Extensions, meta); meta names the roughness outputs.

Grid sizes "N x N" are NODE counts (the array shape), spacing as stated.
"Flat-end mill, radius R" is the reference's circular-insert cutter with
D = 2R and insert radius R (SURVEY.md §2.3 recommendation, keeps the
reference as a special case); "ball-end" is Extensions(profile="ball").
"""

from __future__ import annotations

import math

from .engine import SimulationConfig
from .extensions import Extensions
from .geometry import ToolDefinition
from .grid import GridSpec
from .kinematics import derive_kinematics


def _dt(proc, steps_per_rev):
    return (2.0 * math.pi / steps_per_rev) / proc.angular_velocity_rad_s


def _centered_grid(nodes_x, nodes_y, spacing, y_min=0.0):
    return GridSpec.from_nodes(spacing, -0.5 * (nodes_x - 1) * spacing, y_min, nodes_x, nodes_y)


def config1(helix: bool = True):
    """4-flute flat-end R=5 (D=10), helix 30 deg, fz 0.05, 3000 rpm, a_p 1,
    no runout, N=200, 3600 steps/rev, 20 revs (explicit span, x0=0, y0=-2 [B]),
    200x200 nodes at 10 um. helix=False is the reference-representable analog
    (tests/golden/config1_ref.npz)."""
    tool = ToolDefinition(cutting_diameter_mm=10.0, insert_radius_mm=5.0, tooth_count=4)
    proc = derive_kinematics(tooth_count=4, cutting_diameter_mm=10.0, depth_of_cut_mm=1.0,
                             spindle_speed_rpm=3000.0, feed_per_tooth_mm=0.05,
                             initial_position_mm=(0.0, -2.0, 0.0))
    om = proc.angular_velocity_rad_s
    cfg = SimulationConfig(tool=tool, process=proc, grid=GridSpec(0.01, -0.995, 0.0, 199, 199),
                           edge_point_count=200, time_step_s=_dt(proc, 3600),
                           span_s=(0.0, 20.0 * (2.0 * math.pi) / om))
    ext = Extensions(helix_angle_rad=math.radians(30.0)) if helix else None
    return cfg, ext, {"name": "config1", "profiles_every": 64, "uncut": "exclude"}


def config2():
    """2-flute ball-end R=3, helix 30 deg, lead tilt 15 deg, fz 0.08, runout
    5 um at 40 deg, 6 passes at 0.3 mm stepover (x0 = -0.75 + 0.3k [B]),
    1000x1000 nodes at 2 um, N=500, 7200 steps/rev; 6000 rpm [B], a_p 0.2 [B],
    auto-span per pass."""
    tool = ToolDefinition(cutting_diameter_mm=6.0, insert_radius_mm=3.0, tooth_count=2)
    proc = derive_kinematics(tooth_count=2, cutting_diameter_mm=6.0, depth_of_cut_mm=0.2,
                             spindle_speed_rpm=6000.0, feed_per_tooth_mm=0.08,
                             initial_position_mm=(-0.75, None, 0.0))
    cfg = SimulationConfig(tool=tool, process=proc, grid=_centered_grid(1000, 1000, 0.002),
                           edge_point_count=500, time_step_s=_dt(proc, 7200))
    ext = Extensions(profile="ball", helix_angle_rad=math.radians(30.0), tilt_rad=math.radians(15.0),
                     runout_offset_mm=0.005, runout_phase_rad=math.radians(40.0), passes=6,
                     stepover_mm=0.3)
    return cfg, ext, {"name": "config2", "profiles_every": 64, "uncut": "exclude"}


CONFIG3_RANGES = (("feed_per_tooth_mm", 0.02, 0.2), ("spindle_speed_rpm", 2000.0, 12000.0),
                  ("runout_offset_mm", 0.0, 0.010), ("runout_phase_rad", 0.0, 2.0 * math.pi),
                  ("helix_angle_deg", 20.0, 45.0))


def config3_base():
    """Batched: 256 sets, default_rng(0) i.i.d. uniform over CONFIG3_RANGES
    (column order [B]); 4-flute flat-end R=4 (D=8), a_p 0.5 [B], 512x512
    nodes at 4 um, N=300, 3600 steps/rev [B], auto-span."""
    tool = ToolDefinition(cutting_diameter_mm=8.0, insert_radius_mm=4.0, tooth_count=4)
    proc = derive_kinematics(tooth_count=4, cutting_diameter_mm=8.0, depth_of_cut_mm=0.5,
                             spindle_speed_rpm=6000.0, feed_per_tooth_mm=0.1,
                             initial_position_mm=(0.0, None, 0.0))
    cfg = SimulationConfig(tool=tool, process=proc, grid=_centered_grid(512, 512, 0.004),
                           edge_point_count=300)
    ext = Extensions(helix_angle_rad=math.radians(30.0))
    return cfg, ext, {"name": "config3", "count": 256, "seed": 0, "steps_per_rev": 3600,
                      "ranges": CONFIG3_RANGES, "sampler": "uniform", "uncut": "exclude"}


def config4():
    """4-flute flat-end R=6 (D=12), fz 0.1, runout 3 um (phase 0 [B]),
    radial vibration 2 um along X at 1.7 x tooth-passing frequency (phase 0
    [B]), 10000x10000 nodes at 1 um, N=1000, 14400 steps/rev, 3000 rpm [B],
    a_p 1 [B], auto-span."""
    tool = ToolDefinition(cutting_diameter_mm=12.0, insert_radius_mm=6.0, tooth_count=4)
    proc = derive_kinematics(tooth_count=4, cutting_diameter_mm=12.0, depth_of_cut_mm=1.0,
                             spindle_speed_rpm=3000.0, feed_per_tooth_mm=0.1,
                             initial_position_mm=(0.0, None, 0.0))
    cfg = SimulationConfig(tool=tool, process=proc, grid=_centered_grid(10000, 10000, 0.001),
                           edge_point_count=1000, time_step_s=_dt(proc, 14400))
    ext = Extensions(runout_offset_mm=0.003, vib_amplitude_mm=0.002,
                     vib_frequency_hz=1.7 * 4 * 3000.0 / 60.0)
    return cfg, ext, {"name": "config4", "profiles_every": 64, "uncut": "exclude"}


def config5():
    """3-flute ball-end R=2, fz 0.06, tilt 10 deg, runout 4 um (phase 0 [B]),
    edge-radius noise sigma 1 um, correlation 20 um, seed 0 [B], 16 passes
    at 0.2 mm (x0 = -1.5 + 0.2k [B]), 4096x4096 nodes at 1 um; N=2000 [B],
    14400 steps/rev [B], 6000 rpm [B], a_p 0.1 [B], auto-span. Outputs
    Sa/Sq/Sz/Ssk/Sku and Ra/Rz every 64 rows."""
    tool = ToolDefinition(cutting_diameter_mm=4.0, insert_radius_mm=2.0, tooth_count=3)
    proc = derive_kinematics(tooth_count=3, cutting_diameter_mm=4.0, depth_of_cut_mm=0.1,
                             spindle_speed_rpm=6000.0, feed_per_tooth_mm=0.06,
                             initial_position_mm=(-1.5, None, 0.0))
    cfg = SimulationConfig(tool=tool, process=proc, grid=_centered_grid(4096, 4096, 0.001),
                           edge_point_count=2000, time_step_s=_dt(proc, 14400))
    ext = Extensions(profile="ball", tilt_rad=math.radians(10.0), runout_offset_mm=0.004,
                     noise_sigma_mm=0.001, noise_corr_mm=0.020, noise_seed=0, passes=16,
                     stepover_mm=0.2)
    return cfg, ext, {"name": "config5", "profiles_every": 64, "uncut": "exclude"}


FACTORIES = {1: config1, 2: config2, 4: config4, 5: config5}
