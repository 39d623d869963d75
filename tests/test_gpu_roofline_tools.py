"""The bench's roofline instrumentation on the B200: the RED trace
(MSURF_SWEEP_TRACE, msurf_trace_arm) records exactly the production sweep's
RED.MIN stream, msurf_red_lines histograms every record, and the traced sweep
leaves the same heights. The traced (production) lanes are the counting
variant's RED.MIN minus those the stock-height cull removes (chunks whose
lowest point sits at the stock top: no-op deposits), so on a flat-end EXT
surface they agree to within a few per cent and never exceed it."""

import numpy as np
import pytest

from paper_2603_28160_b200 import planner
from paper_2603_28160_b200.engine import SweepBatch
import paper_2603_28160_b200 as ms
from test_host_cpu import EXT_CASES, _ext_cfg

pytestmark = pytest.mark.gpu


def test_red_trace_counts_the_sweeps_reds():
    cfg = _ext_cfg("insert")
    p = planner.plan(cfg, ms.Extensions(**EXT_CASES["vib_runout"]))
    b = SweepBatch([(p, 0, p.grid.n)])
    b.launch()
    ref = b.heights()[0].cpu().numpy().copy()
    b.diagnostics = True
    b.launch()
    ctr, _ = b.counters()
    atomics = int(ctr[0][3])
    b.diagnostics = False
    lines = b.red_lines()
    assert lines["records"] == lines["records_issued"] and not lines["truncated"]
    assert sum(lines["hist"]) == lines["records"] and lines["hist"][0] == 0
    assert 0.97 * atomics <= lines["lanes"] <= atomics and atomics > 0
    # a record touches at least ceil(lanes / 16) and at most its lanes' lines
    assert sum(L * n for L, n in enumerate(lines["hist"])) <= lines["lanes"]
    # sectors: every record once; at least as many sectors as lines, at most its lanes
    hs = lines["hist_sectors"]
    assert sum(hs) == lines["records"] and hs[0] == 0
    assert sum(L * n for L, n in enumerate(lines["hist"])) <= sum(S * n for S, n in enumerate(hs)) <= lines["lanes"]
    assert np.array_equal(b.heights()[0].cpu().numpy(), ref)  # the traced launch changes no result
