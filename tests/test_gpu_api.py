"""GPU API tests mirroring the reference's own unit and acceptance tests
(pkg/tests/test_roughness.py, test_engine.py, test_acceptance.py criteria 2,
3, 5), run through the product's device reductions and sweep."""

import dataclasses
import math

import numpy as np
import pytest

import golden_io
import paper_2603_28160_b200 as ms
from paper_2603_28160_b200.roughness import LineProfile
from oracle import fsm_oracle as orc

pytestmark = pytest.mark.gpu


def field_from_um(z_um, sentinel_mm=1.0):
    m, n = z_um.shape[0] - 1, z_um.shape[1] - 1
    spec = ms.GridSpec(spacing_mm=0.01, x_min_mm=0.0, y_min_mm=0.0, m=m, n=n)
    return ms.HeightField(spec, sentinel_mm, np.ascontiguousarray(z_um / 1000.0).reshape(-1))


def brute_force(z_um):
    v = [float(x) for x in z_um.reshape(-1)]
    c = len(v)
    mean = sum(v) / c
    d = [x - mean for x in v]
    sq = math.sqrt(sum(x * x for x in d) / c)
    return (sum(abs(x) for x in d) / c, sq, max(d), -min(d),
            (sum(x ** 3 for x in d) / c) / sq ** 3, (sum(x ** 4 for x in d) / c) / sq ** 4)


class TestArealOnDevice:
    def test_flat(self):
        m = ms.areal_metrics(field_from_um(np.zeros((21, 21))))
        assert (m.sa_um, m.sq_um, m.sp_um, m.sv_um, m.sz_um) == (0.0, 0.0, 0.0, 0.0, 0.0)
        assert m.ssk is None and m.sku is None and m.cell_count == 441

    def test_two_level(self):
        z = np.ones((20, 20))
        z[:10] = -1.0
        m = ms.areal_metrics(field_from_um(z))
        for got, exp in ((m.sa_um, 1.0), (m.sq_um, 1.0), (m.sp_um, 1.0), (m.sv_um, 1.0), (m.sz_um, 2.0),
                         (m.ssk, 0.0), (m.sku, 1.0)):
            assert got == pytest.approx(exp, abs=1e-12)

    def test_sinusoid(self):
        row = np.sin(2.0 * np.pi * np.arange(100) / 100)
        m = ms.areal_metrics(field_from_um(np.tile(row, (100, 1))))
        assert m.sa_um == pytest.approx(2.0 / math.pi, rel=0.01)
        assert m.sq_um == pytest.approx(1.0 / math.sqrt(2.0), rel=0.01)
        assert m.sku == pytest.approx(1.5, rel=0.01)

    def test_brute_force(self):
        z = np.random.default_rng(21).normal(0.0, 3.0, (17, 23))
        m = ms.areal_metrics(field_from_um(z, sentinel_mm=10.0))
        for got, exp in zip((m.sa_um, m.sq_um, m.sp_um, m.sv_um, m.ssk, m.sku), brute_force(z)):
            assert got == pytest.approx(exp, rel=1e-12)

    def test_invariances(self):
        rng = np.random.default_rng(4)
        z = rng.normal(0.0, 2.0, (12, 12))
        a = ms.areal_metrics(field_from_um(z, sentinel_mm=50.0))
        b = ms.areal_metrics(field_from_um(z + 17.0, sentinel_mm=50.0))
        assert b.sa_um == pytest.approx(a.sa_um, rel=1e-9) and b.sku == pytest.approx(a.sku, rel=1e-6)
        r = ms.areal_metrics(field_from_um(-z, sentinel_mm=50.0))
        assert r.sp_um == pytest.approx(a.sv_um, rel=1e-12) and r.ssk == pytest.approx(-a.ssk, rel=1e-9)

    def test_uncut_and_roi_errors(self):
        field = ms.HeightField(ms.GridSpec(0.01, 0.0, 0.0, 4, 4), 1.0)
        with pytest.raises(ms.DomainError, match="unmachined"):
            ms.areal_metrics(field)
        f = field_from_um(np.zeros((5, 5)))
        with pytest.raises(ms.DomainError):
            ms.areal_metrics(f, roi=(0, 0, 9, 9))
        with pytest.raises(ms.DomainError):
            ms.areal_metrics(f, roi=(3, 0, 2, 4))
        with pytest.raises(ms.DomainError):
            ms.areal_metrics(f, leveling="median")

    def test_roi_subset(self):
        z = np.zeros((10, 10))
        z[2:5, 2:5] = 4.0
        sub = ms.areal_metrics(field_from_um(z), roi=(2, 2, 4, 4))
        assert sub.cell_count == 9 and sub.sa_um == 0.0
        assert ms.areal_metrics(field_from_um(z)).sa_um > 0.0

    def test_plane_leveling(self):
        rng = np.random.default_rng(8)
        z = rng.normal(0.0, 1.0, (15, 15))
        xi, yj = np.meshgrid(np.arange(15), np.arange(15), indexing="ij")
        a = ms.areal_metrics(field_from_um(z, sentinel_mm=99.0), leveling="plane")
        b = ms.areal_metrics(field_from_um(z + 0.5 * xi - 0.2 * yj, sentinel_mm=99.0), leveling="plane")
        assert b.sq_um == pytest.approx(a.sq_um, rel=1e-9)
        exp = orc.areal_metrics(z / 1000.0, 99.0, leveling="plane")
        for got, k in ((a.sa_um, "Sa"), (a.sq_um, "Sq"), (a.sp_um, "Sp"), (a.sv_um, "Sv"), (a.ssk, "Ssk"),
                       (a.sku, "Sku")):
            assert got == pytest.approx(exp[k], rel=1e-9, abs=1e-12)


class TestProfiles:
    def test_feed_center_and_pickfeed(self):
        f = field_from_um(np.zeros((11, 21)))
        p = ms.extract_profile(f, "feed")
        assert p.index == 5 and p.heights_mm.size == 21 and p.spacing_mm == 0.01
        assert ms.extract_profile(f, "pickfeed", index=0).heights_mm.size == 11
        with pytest.raises(ms.DomainError):
            ms.extract_profile(f, "diagonal")
        with pytest.raises(ms.DomainError):
            ms.extract_profile(f, "feed", index=20)

    def test_uncut_in_profile(self):
        field = ms.HeightField(ms.GridSpec(0.01, 0.0, 0.0, 4, 4), 1.0)
        field.heights[:] = 0.0
        field.heights[12] = 1.0
        with pytest.raises(ms.DomainError):
            ms.extract_profile(field, "feed", index=2)
        ms.extract_profile(field, "feed", index=1)

    def test_line_roughness(self):
        assert ms.line_roughness(LineProfile("feed", 0, np.arange(5.0), np.ones(5), 1.0)) == 0.0
        alt = LineProfile("feed", 0, np.arange(20.0), np.array([1e-3, -1e-3] * 10), 1.0)
        assert ms.line_roughness(alt) == pytest.approx(1.0, abs=1e-12)
        j = np.arange(1000)
        sin = LineProfile("feed", 0, j * 0.01, 1e-3 * np.sin(2 * np.pi * j / 100), 0.01)
        assert ms.line_roughness(sin) == pytest.approx(2.0 / math.pi, rel=0.01)
        with pytest.raises(ms.DomainError):
            ms.line_roughness(LineProfile("feed", 0, np.zeros(1), np.zeros(1), 1.0))


def _front_cut(feed, spacing, runouts=()):
    """helpers.front_cut_config restated with the product's types."""
    tool = ms.ToolDefinition(cutting_diameter_mm=10.0, insert_radius_mm=5.0, tooth_count=2, runouts_mm=runouts)
    margin = feed / 2.0 + 0.3
    y0 = -5.0 - margin
    proc = ms.derive_kinematics(tooth_count=2, cutting_diameter_mm=10.0, depth_of_cut_mm=0.5,
                                cutting_speed_m_min=170.0, feed_per_tooth_mm=feed, initial_position_mm=(0.0, y0, 0.0))
    half = ms.effective_half_length(5.0, 0.5, feed)
    dt = (spacing / (5.0 + half)) / proc.angular_velocity_rad_s
    grid = ms.GridSpec.from_extents(spacing, (-0.05, 0.05), (0.0, 5.0))
    t_end = (5.0 - 5.0 + margin - y0) / proc.feed_speed_mm_s
    return ms.SimulationConfig(tool=tool, process=proc, grid=grid, time_step_s=dt, span_s=(0.0, t_end))


def test_acceptance_cusp_height():
    """Criterion 2 (test_acceptance.py:99-111): scallop 9.008 um +- 0.4 at 2 um pitch."""
    res = ms.simulate(_front_cut(0.6, 0.002))
    p = ms.extract_profile(res.field, "feed")
    w = (p.positions_mm >= 0.25) & (p.positions_mm <= 4.75)
    measured = (p.heights_mm[w].max() - p.heights_mm[w].min()) * 1000.0
    expected = (5.0 - math.sqrt(25.0 - 0.09)) * 1000.0
    assert abs(measured - expected) <= 0.4


def test_acceptance_runout_period_shift():
    """Criterion 3 (test_acceptance.py:116-137): +9 um axial run-out on tooth 2
    moves the dominant feed-profile period from f_z to 2 f_z."""
    def dominant_period(h, spacing, lo, hi, frac=0.9):
        d = h - h.mean()
        n = d.size
        ac = np.correlate(d, d, "full")[n - 1:] / (n - np.arange(n))
        lags = np.arange(n) * spacing
        a, b = int(np.searchsorted(lags, lo)), int(np.searchsorted(lags, hi))
        wnd = ac[a:b]
        peaks = [k for k in range(1, wnd.size - 1) if wnd[k] >= wnd[k - 1] and wnd[k] >= wnd[k + 1] and wnd[k] > 0]
        strongest = max(wnd[k] for k in peaks)
        return float(lags[a + next(k for k in peaks if wnd[k] >= frac * strongest)])

    periods = []
    for runouts in ((), ((0.0, 0.0), (0.0, 0.009))):
        res = ms.simulate(_front_cut(0.5, 0.004, runouts))
        p = ms.extract_profile(res.field, "feed")
        w = (p.positions_mm >= 0.25) & (p.positions_mm <= 4.75)
        periods.append(dominant_period(p.heights_mm[w], 0.004, 0.15, 1.4))
    assert abs(periods[0] - 0.5) <= 5 * 0.004
    assert abs(periods[1] - 1.0) <= 5 * 0.004


def test_acceptance_metric_invariants_and_determinism():
    """Criterion 5 on simulated surfaces + bit-identical reruns (criterion 8 spirit)."""
    for name in ("small_1000", "small_1004", "small_1013", "cusp", "runout"):
        g = golden_io.load(name)
        cfg = golden_io.product_config(g["config"], record_trajectory=False)
        a = ms.simulate(cfg)
        b = ms.simulate(dataclasses.replace(cfg, worker_count=4))
        assert np.array_equal(a.field.heights, b.field.heights)
        roi = tuple(g["roughness"]["roi"])
        m1 = ms.areal_metrics(a.field, roi)
        m2 = ms.areal_metrics(b.field, roi)
        assert m1 == m2  # deterministic reductions: bit-identical metrics
        assert m1.sz_um == pytest.approx(m1.sp_um + m1.sv_um, abs=1e-9)
        assert m1.sq_um >= m1.sa_um * (1.0 - 1e-12)
        if m1.sku is not None:
            assert m1.sku >= (m1.ssk ** 2 + 1.0) * (1.0 - 1e-12)


def test_reduction_scratch_bound_at_max_blocks():
    """Every reduction entry point writes at most MSURF_WORK_DOUBLES scratch
    doubles per surface, even at the block cap (a 2049 x 2049 field uses all
    MSURF_RED_BLOCKS blocks): a guard region right after the scratch must be
    untouched (include/msurf.h contract)."""
    import torch

    from paper_2603_28160_b200 import _native

    lib = _native.lib()
    dev = torch.device("cuda", 0)
    rows = cols = 2049
    rng = np.random.default_rng(3)
    h = torch.tensor(rng.random(rows * cols) * 0.01, dtype=torch.float64, device=dev)
    sent = torch.tensor([1.0], dtype=torch.float64, device=dev)
    guard = 4096
    work = torch.full((_native.WORK_DOUBLES + guard,), 12345.0, dtype=torch.float64, device=dev)
    out = torch.zeros(64, dtype=torch.float64, device=dev)
    coef = torch.tensor([0.0, 0.0, 5.0], dtype=torch.float64, device=dev)
    sp = _native.stream_ptr()
    w, o = work.data_ptr(), out.data_ptr()
    args = (h.data_ptr(), cols, rows * cols, 1, 0, 0, rows, cols, sent.data_ptr(), 1)
    _native.check(lib.msurf_areal_pass1(*args, w, o, sp))
    _native.check(lib.msurf_areal_pass2(*args, o, w, o + 6 * 8, sp))
    _native.check(lib.msurf_areal_plane_pass1(*args, w, o + 16 * 8, sp))
    _native.check(lib.msurf_areal_plane_pass2(*args, coef.data_ptr(), w, o + 32 * 8, sp))
    torch.cuda.synchronize()
    assert bool(torch.all(work[_native.WORK_DOUBLES:] == 12345.0))
    assert int(out[3].item()) == rows * cols


@pytest.mark.gpu
def test_readback_mapped_matches_copy():
    """Small results come back through mapped page-locked memory (msurf_readback),
    also while a large D2H copy is in flight on a side stream."""
    import torch

    from paper_2603_28160_b200 import _native

    dev = torch.device("cuda", 0)
    big = torch.randn(1 << 24, dtype=torch.float64, device=dev)
    host = torch.empty(big.shape, dtype=torch.float64, pin_memory=True)
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        host.copy_(big, non_blocking=True)
    for n, dt in ((1, torch.float64), (10, torch.float64), (2560, torch.float64), (7, torch.int64),
                  (1 << 17, torch.float64), (3, torch.float32)):
        t = (torch.arange(n, device=dev) * 3 - 5).to(dt) / (1 if dt != torch.float64 else 7)
        got = _native.readback(t)
        assert got.dtype == t.cpu().numpy().dtype and got.shape == tuple(t.shape)
        assert np.array_equal(got, t.cpu().numpy())
    m = torch.arange(12, dtype=torch.float64, device=dev).reshape(3, 4)
    assert np.array_equal(_native.readback(m), m.cpu().numpy())
    side.synchronize()
    assert torch.equal(host[:100].to(dev), big[:100])


def test_fields_outlive_results_with_pooled_events():
    """A field keeps its prefetched heights after its SimulationResult is
    released: the launch's timing events go back to the pool and are
    re-recorded by later launches, the prefetch event is never pooled."""
    import gc

    cfg = _front_cut(0.6, 0.01)
    ref = ms.simulate(cfg)
    h_ref = ref.field.heights.copy()
    assert ref.main_loop_seconds > 0
    fields = []
    for _ in range(4):
        r = ms.simulate(cfg)
        fields.append(r.field)
        del r
        gc.collect()
    for _ in range(3):
        r2 = ms.simulate(cfg)
        assert r2.main_loop_seconds > 0
    for f in fields:
        assert np.array_equal(f.heights, h_ref)


def test_profile_roughness_cached_offsets_and_streams():
    """Profile offsets are cached per (device, stream, offsets): repeated
    calls, a second profile set and a second stream return the same results
    as the first call of each."""
    import torch

    f = ms.simulate(_front_cut(0.6, 0.01)).field
    a = ms.profile_roughness(f, every=2, uncut="exclude")
    assert ms.profile_roughness(f, every=2, uncut="exclude") == a
    c = ms.profile_roughness(f, every=3, uncut="exclude")
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        d = ms.profile_roughness(f, every=3, uncut="exclude")
        e = ms.profile_roughness(f, every=2, uncut="exclude")
    assert c == d and e == a
    assert len(a) == len(range(0, f.spec.m + 1, 2))
