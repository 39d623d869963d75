"""The native planner (csrc/msurf_plan.cpp via msurf_plan_geometry/finish)
against the NumPy statement of planner.py (MSURF_NATIVE_PLAN=0 semantics):
every plan array bitwise equal on the reference goldens, the extended-model
cases and the five BASELINE configurations. CPU only (the library loads
without a GPU)."""

import numpy as np
import pytest

import golden_io
from paper_2603_28160_b200 import configs, planner
from paper_2603_28160_b200.extensions import Extensions
from test_host_cpu import EXT_CASES, _ext_cfg

FIELDS = ["tooth_base", "tooth_rows", "px", "py", "pz", "zw", "zkey", "chunk_box", "pass_x0", "min_index",
          "pts", "chunk_circ", "tooth_box"]
SCALARS = ["mode", "teeth", "points", "steps", "dt", "t_start", "x0", "y0", "z0", "feed_speed", "omega",
           "initial_height", "half_length", "tilt_c", "tilt_s", "zoff", "vib_amp", "vib_omega", "vib_phase"]


def _both(cfg, ext=None):
    old = planner.NATIVE_PLAN
    try:
        planner.NATIVE_PLAN = False
        ref = planner.plan(cfg, ext)
        planner.NATIVE_PLAN = True
        nat = planner.plan(cfg, ext)
    finally:
        planner.NATIVE_PLAN = old
    return ref, nat


def _same(ref, nat):
    for f in SCALARS:
        a, b = getattr(ref, f), getattr(nat, f)
        assert np.float64(a).tobytes() == np.float64(b).tobytes(), (f, a, b)
    for f in FIELDS:
        a, b = np.ascontiguousarray(getattr(ref, f)), np.ascontiguousarray(getattr(nat, f))
        assert a.shape == b.shape and a.dtype == b.dtype, (f, a.shape, b.shape, a.dtype, b.dtype)
        assert a.tobytes() == b.tobytes(), (f, int(np.count_nonzero(a != b)))


@pytest.mark.parametrize("name", golden_io.case_names())
def test_native_plan_bitwise_on_goldens(name):
    g = golden_io.load(name)
    _same(*_both(golden_io.product_config(g["config"], record_trajectory=False)))


@pytest.mark.parametrize("case", sorted(EXT_CASES))
def test_native_plan_bitwise_extended(case):
    kw = EXT_CASES[case]
    _same(*_both(_ext_cfg(kw.get("profile", "insert")), Extensions(**kw)))


@pytest.mark.parametrize("n", [1, 2, 3, 4, 5])
def test_native_plan_bitwise_baseline_configs(n):
    cfg, ext, _ = getattr(configs, f"config{n}")() if n != 3 else configs.config3_base()[:3]
    _same(*_both(cfg, ext))


def test_native_plan_force_extended_and_odd_points():
    g = golden_io.load("small_2")
    cfg = golden_io.product_config(g["config"], record_trajectory=False)
    _same(*_both(cfg, Extensions(force_extended=True)))
    from dataclasses import replace
    for n in (2, 31, 33, 65):
        _same(*_both(replace(cfg, edge_point_count=n)))
        _same(*_both(replace(cfg, edge_point_count=n), Extensions(profile="ball", tilt_rad=0.1)))


def test_native_plan_bitwise_config3_samples():
    from paper_2603_28160_b200.dataset import ParameterRange, apply_sample, uniform_sample

    base, ext, meta = configs.config3_base()
    ranges = [ParameterRange(n, lo, hi) for n, lo, hi in meta["ranges"]]
    samples = uniform_sample(ranges, 6, meta["seed"])
    for row in samples:
        c, e = apply_sample(base, ext, [r.name for r in ranges], row, meta["steps_per_rev"])
        _same(*_both(c, e))
