"""The surface-cap path (engine.ZCAP: per-(pass, tooth) launches with a
per-tile height bound, sub-strips side by side on library streams, staged
two-kernel launches) is result-neutral: on a reduced config 5 cut into four
L2 sub-strips, every variant gives the uncapped heights bit for bit, in both
launch forms (launch(); launch_by_strip(), the e2e path with per-strip joins),
and the whole simulate() equals the extended oracle."""

from dataclasses import replace

import numpy as np
import pytest

import paper_2603_28160_b200 as ms
from paper_2603_28160_b200 import configs, engine, planner
from paper_2603_28160_b200.engine import SweepBatch
from oracle import fsm_ext_oracle as xorc

pytestmark = pytest.mark.gpu


def _reduced_config5():
    cfg, ext, _ = configs.config5()
    cfg = replace(cfg, grid=ms.GridSpec.from_nodes(0.001, -0.2555, 0.0, 512, 512), edge_point_count=600)
    cfg = replace(cfg, process=replace(cfg.process, initial_position_mm=(-0.2, None, 0.0)))
    return cfg, replace(ext, passes=3, stepover_mm=0.2)


def _heights(p, by_strip=False):
    b = SweepBatch([(p, 0, p.grid.n)])
    if by_strip:
        b.launch_by_strip(lambda *a: None)
    else:
        b.launch()
    out = b.heights()[0].cpu().numpy().copy()
    return out, b


@pytest.mark.parametrize("staged", [True, False])
@pytest.mark.parametrize("depth", [0, 1, 3])
def test_capped_variants_equal_uncapped(monkeypatch, staged, depth):
    cfg, ext = _reduced_config5()
    p = planner.plan(cfg, ext)
    quarter = (p.grid.m + 1) * (p.grid.n + 1) * 8 // 4 + 8
    monkeypatch.setattr(engine, "L2_TILE_BYTES", quarter)
    monkeypatch.setattr(engine, "ZCAP_L2_TILE_BYTES", quarter)
    monkeypatch.setattr(engine, "ZCAP", False)
    ref, b0 = _heights(p)
    assert b0.surfs[0].n_strips == 4 and all(q is None for s in b0.zc_seq for q in s)
    monkeypatch.setattr(engine, "ZCAP", True)
    monkeypatch.setattr(engine, "ZCAP_STAGED", staged)
    monkeypatch.setattr(engine, "ZCAP_DEPTH", depth)
    got, b1 = _heights(p)
    assert sum(q is not None for s in b1.zc_seq for q in s) == 4
    assert np.array_equal(got, ref), int(np.count_nonzero(got != ref))
    got2, _ = _heights(p, by_strip=True)
    assert np.array_equal(got2, ref), int(np.count_nonzero(got2 != ref))


def test_capped_simulate_equals_ext_oracle(monkeypatch):
    cfg, ext = _reduced_config5()
    p = planner.plan(cfg, ext)
    third = (p.grid.m + 1) * (p.grid.n + 1) * 8 // 3 + 8
    monkeypatch.setattr(engine, "L2_TILE_BYTES", third)
    monkeypatch.setattr(engine, "ZCAP_L2_TILE_BYTES", third)
    h_ref, _, ctr, _ = xorc.ext_sweep(cfg, ext, workers=8)
    res = ms.simulate(cfg, ext, trig="host")
    assert res._launch.batch.pipelined_strips()
    assert np.array_equal(res.field.heights, h_ref)
    assert res.cells_updated == ctr["cells_updated"]


def test_capped_many_mask_words_equal_uncapped(monkeypatch):
    """A tilt surface with 2500 edge points (79 chunks: two 64-bit chunk-mask
    words per step) through the staged capped path equals the uncapped sweep."""
    cfg, ext = _reduced_config5()
    cfg = replace(cfg, edge_point_count=2500)
    p = planner.plan(cfg, ext)
    assert (p.points + 31) // 32 > 64
    monkeypatch.setattr(engine, "ZCAP", False)
    ref, _ = _heights(p)
    monkeypatch.setattr(engine, "ZCAP", True)
    got, b = _heights(p)
    assert any(q is not None for s in b.zc_seq for q in s)
    assert np.array_equal(got, ref), int(np.count_nonzero(got != ref))


def test_progressive_row_release_equals_whole_strips(monkeypatch):
    """launch_by_strip with the last raster passes launched one call each
    (engine.PROGRESSIVE_PASSES): the node rows no later pass can reach are
    decoded and handed out early; the heights (device and the pinned host
    copy through simulate()) and the machined-cell count equal the
    whole-strip path, and rows really are released before the last pass."""
    cfg, ext, _ = configs.config5()
    cfg = replace(cfg, grid=ms.GridSpec.from_nodes(0.001, -1.0, 0.0, 2001, 256), edge_point_count=600)
    cfg = replace(cfg, process=replace(cfg.process, initial_position_mm=(-1.2, None, 0.0)))
    ext = replace(ext, passes=8, stepover_mm=0.3)
    p = planner.plan(cfg, ext)
    third = (p.grid.m + 1) * (p.grid.n + 1) * 8 // 3 + 8
    monkeypatch.setattr(engine, "L2_TILE_BYTES", third)
    monkeypatch.setattr(engine, "ZCAP_L2_TILE_BYTES", third)
    monkeypatch.setattr(engine, "PROGRESSIVE_PASSES", 0)
    ref, b0 = _heights(p, by_strip=True)
    assert b0.surfs[0].n_strips == 3 and b0.pipelined_strips()
    ref_cells = int(b0.counters()[1][0])
    monkeypatch.setattr(engine, "PROGRESSIVE_PASSES", 3)
    calls = []
    b = SweepBatch([(p, 0, p.grid.n)])
    b.launch_by_strip(lambda q, c0, w, r0, r1, st: calls.append((q, r0, r1)))
    got = b.heights()[0].cpu().numpy()
    assert np.array_equal(got, ref), int(np.count_nonzero(got != ref))
    assert int(b.counters()[1][0]) == ref_cells
    rows = p.grid.m + 1
    assert any(r1 < rows for _, _, r1 in calls)  # released before the last pass
    for q in range(3):  # each strip's rows exactly once, in order
        spans = [(r0, r1) for qq, r0, r1 in calls if qq == q]
        assert spans[0][0] == 0 and spans[-1][1] == rows
        assert all(a[1] == b_[0] for a, b_ in zip(spans, spans[1:]))
    res = ms.simulate(cfg, ext)
    assert np.array_equal(res.field.heights, ref)
    assert res.cells_updated == ref_cells
