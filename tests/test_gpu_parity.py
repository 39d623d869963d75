"""GPU parity: the CUDA path (through the C ABI) against the reference goldens
and the CPU oracles. Heights: bit-exact (tolerance 0). Roughness: 1e-9
relative (north-star gate 0.1 %). Requires a B200 and the built libmsurf.so."""

import math
from types import SimpleNamespace as NS

import numpy as np
import pytest

import golden_io
import paper_2603_28160_b200 as ms
from oracle import fsm_ext_oracle as xorc
from oracle import fsm_oracle as orc
from test_host_cpu import EXT_CASES, _ext_cfg

pytestmark = pytest.mark.gpu
CASES = golden_io.case_names()
REL = 1e-9


def _rel(a, b):
    return abs(a - b) / max(abs(b), 1e-300)


@pytest.mark.parametrize("trig", ["device", "host"])
@pytest.mark.parametrize("name", CASES)
def test_heights_bitexact_vs_reference_goldens(name, trig):
    g = golden_io.load(name)
    cfg = golden_io.product_config(g["config"])
    res = ms.simulate(cfg, trig=trig)
    assert res.time_steps == g["counters"]["time_steps"]
    assert res.trajectory_points == g["counters"]["trajectory_points"]
    assert res.cells_updated == g["counters"]["cells_updated"]
    h = res.field.heights
    assert golden_io.heights_match(g, h), golden_io.max_abs_diff(g, h, cfg.grid.n + 1)
    if "traj" in g:
        tr = g["traj"]
        rec = res.trajectory
        assert rec is not None and len(rec) == tr.shape[1]
        assert np.array_equal(rec.t_s, tr[0]) and np.array_equal(rec.tooth, tr[1].astype(np.int64))
        assert np.array_equal(rec.z_mm, tr[4])
        if trig == "host":
            assert np.array_equal(rec.x_mm, tr[2]) and np.array_equal(rec.y_mm, tr[3])
        else:
            assert np.max(np.abs(rec.x_mm - tr[2])) < 1e-12 and np.max(np.abs(rec.y_mm - tr[3])) < 1e-12


@pytest.mark.parametrize("name", CASES)
def test_roughness_vs_reference_goldens(name):
    g = golden_io.load(name)
    rough = g["roughness"]
    res = ms.simulate(golden_io.product_config(g["config"]))
    if rough.get("areal"):
        am = ms.areal_metrics(res.field, roi=tuple(rough["roi"]))
        ref = rough["areal"]
        got = am.to_json_dict()
        for k in ("Sa_um", "Sq_um", "Sp_um", "Sv_um", "Sz_um", "Ssk", "Sku"):
            if ref[k] is None:
                assert got[k] is None
            else:
                assert _rel(got[k], ref[k]) < REL or abs(got[k] - ref[k]) < 1e-12, (k, got[k], ref[k])
        assert got["cell_count"] == ref["cell_count"]
    if "Ra" in rough:
        i_lo, j_lo, i_hi, j_hi = rough["roi"]
        prof = ms.extract_profile(res.field, "feed", index=rough["profile_index"], roi=tuple(rough["roi"]))
        assert _rel(ms.line_roughness(prof), rough["Ra"]) < REL
        pr = ms.profile_roughness(res.field, indices=[rough["profile_index"]], roi=tuple(rough["roi"]))[0]
        assert _rel(pr.ra_um, rough["Ra"]) < REL
    if "areal_full_error" in rough:
        with pytest.raises(ms.DomainError):
            ms.areal_metrics(res.field)
    elif "areal_full" in rough:
        am = ms.areal_metrics(res.field)
        assert _rel(am.sa_um, rough["areal_full"]["Sa_um"]) < REL


@pytest.mark.parametrize("case", sorted(EXT_CASES))
@pytest.mark.parametrize("trig", ["device", "host"])
def test_extended_model_bitexact_vs_ext_oracle(case, trig):
    kw = EXT_CASES[case]
    cfg = _ext_cfg(kw.get("profile", "insert"))
    res = ms.simulate(cfg, ms.Extensions(**kw), trig=trig, diagnostics=True)
    h_ref, p, ctr, _ = xorc.ext_sweep(cfg, NS(**kw), workers=4)
    h = res.field.heights
    assert res.trajectory_points == ctr["trajectory_points"]
    assert res.cells_updated == ctr["cells_updated"]
    assert np.array_equal(h, h_ref), float(np.max(np.abs(h - h_ref)))
    assert res.counters["deposits"] == ctr["deposits"]


def test_force_extended_equals_reference_on_goldens():
    for name in CASES:
        g = golden_io.load(name)
        cfg = golden_io.product_config(g["config"], record_trajectory=False)
        res = ms.simulate(cfg, ms.Extensions(force_extended=True))
        assert golden_io.heights_match(g, res.field.heights), name


def test_batched_equals_individual():
    names = ["small_0", "small_3", "tiny", "small_1004", "config1_ref"]
    cfgs = [golden_io.product_config(golden_io.load(n)["config"], record_trajectory=False) for n in names]
    batch = ms.simulate_batch(cfgs)
    for n, r in zip(names, batch):
        assert golden_io.heights_match(golden_io.load(n), r.field.heights), n


def test_batched_ext_same_shape_and_metrics():
    cfg = _ext_cfg("ball")
    exts = [ms.Extensions(profile="ball", helix_angle_rad=math.radians(20 + 5 * k),
                          runout_offset_mm=0.001 * k, runout_phase_rad=0.7 * k) for k in range(6)]
    batch = ms.simulate_batch([cfg] * 6, exts)
    mets = ms.areal_metrics_batch([b.field for b in batch], uncut="exclude")
    for e, b, m in zip(exts, batch, mets):
        kw = {k: getattr(e, k) for k in ("profile", "helix_angle_rad", "runout_offset_mm", "runout_phase_rad")}
        h_ref, p, _, _ = xorc.ext_sweep(cfg, NS(**kw), workers=2)
        assert np.array_equal(b.field.device_heights().cpu().numpy(), h_ref)
        exp = orc.areal_metrics(h_ref.reshape(p.m + 1, p.n + 1), p.initial_height, uncut="exclude")
        assert _rel(m.sa_um, exp["Sa"]) < REL and _rel(m.sku, exp["Sku"]) < REL


def test_areal_metrics_batch_mixed_runs_equal_per_field():
    """areal_metrics_batch over several launch groups (strided runs), a
    host-built field, a different grid and an uncut-stock field: every entry
    equals areal_metrics of that field alone (same kernels, one D2H)."""
    cfg = _ext_cfg("ball")
    exts = [ms.Extensions(profile="ball", helix_angle_rad=math.radians(15 + 4 * k)) for k in range(9)]
    batch = ms.simulate_batch([cfg] * 9, exts, chunk=4)  # launch groups of 4, 4, 1
    small = ms.simulate(golden_io.product_config(golden_io.load("small_3")["config"], record_trajectory=False))
    host = ms.HeightField(batch[0].field.spec, batch[0].field.initial_height_mm,
                          heights=batch[2].field.device_heights().cpu().numpy())
    stock = ms.HeightField(batch[0].field.spec, batch[0].field.initial_height_mm)
    fields = [b.field for b in batch[:5]] + [host, small.field, stock] + [b.field for b in batch[5:]]
    for uncut in ("exclude", "raise"):
        got = ms.areal_metrics_batch(fields, uncut=uncut)
        assert len(got) == len(fields)
        for f, g in zip(fields, got):
            try:
                exp = ms.areal_metrics(f, uncut=uncut)
            except ms.DomainError as exc:
                assert isinstance(g, ms.DomainError) and str(g) == str(exc)
                continue
            assert g == exp


def test_profiles_ra_rz_every_k_rows():
    kw = EXT_CASES["ball_noise"]
    cfg = _ext_cfg("ball")
    res = ms.simulate(cfg, ms.Extensions(**kw))
    h_ref, p, _, _ = xorc.ext_sweep(cfg, NS(**kw), workers=2)
    a2 = h_ref.reshape(p.m + 1, p.n + 1)
    prs = ms.profile_roughness(res.field, every=16, uncut="exclude")
    assert [q.index for q in prs] == list(range(0, p.m + 1, 16))
    for q in prs:
        exp = orc.profile_roughness(a2[q.index], p.initial_height, uncut="exclude")
        assert _rel(q.ra_um, exp["Ra"]) < REL and _rel(q.rz_um, exp["Rz"]) < REL


def test_no_engagement_and_edge_cases():
    g = golden_io.load("tiny")
    d = g["config"]
    proc = dict(d["process"])
    proc["initial_position_mm"] = [100.0, None, 0.0]
    d2 = dict(d, process=proc)
    res = ms.simulate(golden_io.product_config(d2))
    assert res.cells_updated == 0
    assert np.all(res.field.heights == res.field.initial_height_mm)
    with pytest.raises(ms.DomainError):
        ms.areal_metrics(res.field)
    # 1-cell grid, odd point counts, large N (> 2048 -> several mask words)
    for n_pts, spacing in ((2, 0.3), (33, 0.05), (2500, 0.004)):
        cfg = golden_io.product_config(d, edge_point_count=n_pts, record_trajectory=False,
                                       grid=ms.GridSpec(spacing, -0.2, 0.0, 1 if spacing == 0.3 else 40, 1 if spacing == 0.3 else 30))
        res = ms.simulate(cfg, diagnostics=True)
        h_ref, _, ctr, _ = orc.sweep(cfg, workers=2)
        assert np.array_equal(res.field.heights, h_ref)
        assert res.counters["deposits"] == ctr["deposits"]


def test_heightfield_device_roundtrip_and_merge():
    g = golden_io.load("small_3")
    cfg = golden_io.product_config(g["config"], record_trajectory=False)
    a = ms.simulate(cfg).field
    b = ms.simulate(cfg).field
    a.merge_min(b)
    assert golden_io.heights_match(g, a.heights)
    c = a.copy()
    assert np.array_equal(c.heights, a.heights)


@pytest.mark.parametrize("name", ["small_0", "small_1004", "table6_3", "config1_ref", "cusp", "runout"])
def test_l2_substrips_and_time_windows_bitexact(name):
    """Force many feed-direction sub-strips (each with its own time window)
    on one surface: the assembled map must equal the reference golden."""
    from paper_2603_28160_b200 import planner
    from paper_2603_28160_b200.engine import SweepBatch

    g = golden_io.load(name)
    cfg = golden_io.product_config(g["config"], record_trajectory=False)
    p = planner.plan(cfg)
    b = SweepBatch([(p, 0, p.grid.n)], l2_tile_bytes=(p.grid.m + 1) * 8 * 7)  # ~7 columns per sub-strip
    assert len(b.jobs) > 1
    b.launch()
    assert golden_io.heights_match(g, b.heights()[0].cpu().numpy())


@pytest.mark.parametrize("world", [2, 3])
def test_rank_strips_assemble_to_whole(world):
    """Strip sharding as run across GPUs (each rank: its columns, its time
    window), emulated sequentially on one GPU: strips assemble bit-exactly."""
    from paper_2603_28160_b200 import sharded

    kw = EXT_CASES["ball_tilt"]
    cfg = _ext_cfg("ball")
    ext = ms.Extensions(**kw)
    whole = ms.simulate(cfg, ext).field.heights.reshape(cfg.grid.m + 1, cfg.grid.n + 1)
    for r in range(world):
        sr = sharded.simulate_strip(cfg, ext, r, world)
        got = sr.heights.cpu().numpy().reshape(cfg.grid.m + 1, sr.j_hi - sr.j_lo + 1)
        assert np.array_equal(got, whole[:, sr.j_lo: sr.j_hi + 1])


_FORCE_NEAR_SCRIPT = r"""
import sys
sys.path.insert(0, {root!r}); sys.path.insert(0, {tests!r})
import numpy as np
import golden_io
import paper_2603_28160_b200 as ms
from test_host_cpu import EXT_CASES, _ext_cfg
from types import SimpleNamespace as NS
from oracle import fsm_ext_oracle as xorc
for name in ["small_0", "small_1004", "cusp", "runout", "table6_3"]:
    g = golden_io.load(name)
    res = ms.simulate(golden_io.product_config(g["config"], record_trajectory=False))
    assert golden_io.heights_match(g, res.field.heights), name
for case in ("ball_tilt", "vib_runout"):
    kw = EXT_CASES[case]
    cfg = _ext_cfg(kw.get("profile", "insert"))
    res = ms.simulate(cfg, ms.Extensions(**kw), diagnostics=True)
    h_ref, _, ctr, _ = xorc.ext_sweep(cfg, NS(**kw), workers=4)
    assert np.array_equal(res.field.heights, h_ref), case
    assert res.counters["deposits"] == ctr["deposits"], case
print("FORCE_NEAR_OK")
"""


def test_deferred_exact_path_bitexact():
    """libmsurf built with MSURF_FORCE_NEAR routes EVERY point through the
    deferred exact-index path (the one near-boundary points take): heights
    must still equal the reference goldens / extended oracle bit-exactly."""
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    lib = os.path.join(root, "tests", "native", "libmsurf_forcenear.so")
    if not os.path.exists(lib):
        pytest.fail("tests/native/libmsurf_forcenear.so missing: run __graft_entry__.build()")
    env = dict(os.environ, MSURF_LIB=lib)
    script = _FORCE_NEAR_SCRIPT.format(root=root, tests=os.path.join(root, "tests"))
    out = subprocess.run([sys.executable, "-c", script], env=env, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0 and "FORCE_NEAR_OK" in out.stdout, out.stderr[-3000:]


@pytest.mark.parametrize("case", ["ref", "ext", "tilt"])
def test_tile_list_path_equals_per_job_path(case, monkeypatch):
    """The batched launch pre-culls its tiles into a list walked by persistent
    CTAs; the single-job launch culls tiles inline. Same heights and the same
    row/point counters, also for narrow strip windows where most tiles die.
    (A tilt single job also runs capped — surface-cap cull, fewer rows and
    points — so the counters are compared with the cap off and the heights
    with it on as well.)"""
    from paper_2603_28160_b200 import engine, planner
    from paper_2603_28160_b200.engine import SweepBatch

    monkeypatch.setattr(engine, "ZCAP", False)

    if case == "ref":
        cfg, ext = golden_io.product_config(golden_io.load("small_3")["config"], record_trajectory=False), None
    elif case == "ext":
        cfg, ext = _ext_cfg("insert"), ms.Extensions(helix_angle_rad=math.radians(25), runout_offset_mm=0.002)
    else:
        cfg, ext = _ext_cfg("ball"), ms.Extensions(**EXT_CASES["ball_tilt"])
    p = planner.plan(cfg, ext)
    n = p.grid.n
    windows = [(0, n), (n // 3, n // 3 + 4), (n - 2, n)]
    for lo, hi in windows:
        one = SweepBatch([(p, lo, hi)])
        one.launch()
        many = SweepBatch([(p, lo, hi)] * 3)
        assert not any(many.group_per_job)  # three jobs of few tiles: the listed batched launch
        many.launch()
        h1 = one.heights()[0].cpu().numpy()
        c1, m1 = one.counters()
        cm, mm = many.counters()
        for k, h in enumerate(many.heights()):
            assert np.array_equal(h.cpu().numpy(), h1), (case, lo, hi, k)
            assert np.array_equal(cm[k], c1[0]) and mm[k] == m1[0], (case, lo, hi, k)
        monkeypatch.setattr(engine, "ZCAP", True)
        capped = SweepBatch([(p, lo, hi)])
        capped.launch()
        assert np.array_equal(capped.heights()[0].cpu().numpy(), h1), (case, lo, hi, "capped")
        assert int(capped.counters()[1][0]) == int(m1[0])
        monkeypatch.setattr(engine, "ZCAP", False)


@pytest.mark.parametrize("case", ["ball_tilt", "ball_noise", "vib_runout"])
@pytest.mark.parametrize("nodes,points", [((2, 2), 2), ((2, 40), 33), ((40, 2), 2), ((3, 2), 65), ((64, 65), 2)])
def test_extended_model_degenerate_grids_vs_ext_oracle(case, nodes, points):
    """Extended kinematics (capped tilt raster passes, edge noise, vibration)
    on degenerate grids — one cell, one cell row, one cell column, 3 x 2 — and the
    smallest / odd point counts: heights bit-exact and machined-cell counts
    equal to the extended oracle (host-libm trig)."""
    kw = EXT_CASES[case]
    cfg = _ext_cfg(kw.get("profile", "insert"))
    g = cfg.grid
    grid = ms.GridSpec.from_nodes(g.spacing_mm, g.x_min_mm + 0.37 * (g.m + 1 - nodes[0]) * g.spacing_mm,
                                  g.y_min_mm + 0.41 * (g.n + 1 - nodes[1]) * g.spacing_mm, nodes[0], nodes[1])
    from dataclasses import replace

    cfg = replace(cfg, grid=grid, edge_point_count=points)
    res = ms.simulate(cfg, ms.Extensions(**kw), trig="host")
    h_ref, _, ctr, _ = xorc.ext_sweep(cfg, NS(**kw), workers=2)
    assert np.array_equal(res.field.heights, h_ref), float(np.max(np.abs(res.field.heights - h_ref)))
    assert res.cells_updated == ctr["cells_updated"]
