"""Pin the CPU oracle (oracle/fsm_oracle.py) to the reference's own outputs.

The golden fixtures were produced by the real reference (tests/golden/
make_golden.py); the oracle must reproduce every height bit-exactly, the
counters exactly and the roughness numbers to 1e-12 relative."""

import math

import numpy as np
import pytest

import golden_io
from oracle import fsm_oracle as orc

CASES = golden_io.case_names()


@pytest.mark.parametrize("name", CASES)
def test_oracle_heights_bitexact(name):
    g = golden_io.load(name)
    cfg = golden_io.namespace_config(g["config"])
    h, plan, ctr, _ = orc.sweep(cfg, workers=min(8, orc.default_cpu_workers()))
    assert ctr["time_steps"] == g["counters"]["time_steps"]
    assert ctr["trajectory_points"] == g["counters"]["trajectory_points"]
    assert ctr["cells_updated"] == g["counters"]["cells_updated"]
    assert plan.initial_height == g["counters"]["initial_height"]
    assert golden_io.heights_match(g, h)


def _rel(a, b):
    return abs(a - b) / max(abs(b), 1e-300)


@pytest.mark.parametrize("name", CASES)
def test_oracle_roughness(name):
    g = golden_io.load(name)
    rough = g["roughness"]
    cfg = golden_io.namespace_config(g["config"])
    h, plan, _, _ = orc.sweep(cfg, workers=4)
    h2 = h.reshape(plan.m + 1, plan.n + 1)
    if rough.get("areal"):
        got = orc.areal_metrics(h2, plan.initial_height, roi=tuple(rough["roi"]))
        ref = rough["areal"]
        for k_got, k_ref in (("Sa", "Sa_um"), ("Sq", "Sq_um"), ("Sp", "Sp_um"), ("Sv", "Sv_um"),
                             ("Sz", "Sz_um"), ("Ssk", "Ssk"), ("Sku", "Sku")):
            if ref[k_ref] is None:
                assert got[k_got] is None
            else:
                assert _rel(got[k_got], ref[k_ref]) < 1e-12, (k_got, got[k_got], ref[k_ref])
        assert got["cell_count"] == ref["cell_count"]
    if "Ra" in rough:
        i_lo, j_lo, i_hi, j_hi = rough["roi"]
        prof = h2[rough["profile_index"], j_lo:j_hi + 1]
        assert _rel(orc.profile_roughness(prof, plan.initial_height)["Ra"], rough["Ra"]) < 1e-12
    if "areal_full_error" in rough:
        with pytest.raises(ValueError):
            orc.areal_metrics(h2, plan.initial_height)


def test_oracle_trajectory_argmin_pinned():
    # The per-(step, tooth) min-z point (engine.py:266-270) is reproducible from the plan.
    g = golden_io.load("tiny")
    cfg = golden_io.namespace_config(g["config"])
    p = orc.plan(cfg)
    tr = g["traj"]
    assert tr.shape[1] == p.steps * p.teeth
    for ki in range(p.teeth):
        assert np.all(tr[4][ki::p.teeth] == p.zw[ki][p.min_index[ki]])


def test_oracle_lhs_golden():
    z = np.load(golden_io.GOLDEN + "/lhs.npz")
    bounds = [tuple(b) for b in z["bounds"]]
    for key in z.files:
        if not key.startswith("lhs_"):
            continue
        _, count, seed = key.split("_")
        got = orc.lhs_sample(bounds, int(count), int(seed))
        assert np.array_equal(got, z[key])


def test_oracle_locate_kats():
    # surface_grid KATs (SPEC locate examples; test_surface_grid.py:42-67)
    assert orc.locate(0.012, 0.0, 0.01, 0.0, 0.0, 10, 10) == (1, 0)
    assert orc.locate(0.0, 0.0, 0.01, 0.0, 0.0, 10, 10) == (0, 0)
    assert orc.locate(-0.006, 0.0, 0.01, 0.0, 0.0, 10, 10) is None
    assert orc.locate(0.005, 0.0, 0.01, 0.0, 0.0, 10, 10) == (1, 0)  # boundary -> upper cell


def test_oracle_tool_geometry_kats():
    # test_tool_geometry.py:57-66: dL = 2.17945 at R=5, a_p=0.5; feed branch 0.3
    assert orc.effective_half_length(5.0, 0.5, 0.6) == pytest.approx(2.17945, abs=1e-5)
    assert orc.effective_half_length(5.0, 0.001, 0.6) == pytest.approx(0.3, abs=1e-12)
    assert math.isclose(orc.default_point_count(2.0, 0.01), 801)
