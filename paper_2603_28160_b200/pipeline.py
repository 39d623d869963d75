"""Resident-input surface pipeline: the whole hot path of one batch of
surfaces as a sync-free launch sequence (optionally captured in a CUDA graph).

    fill -> sweep -> decode -> areal pass1 -> areal pass2 -> profiles

Everything is preallocated, no host synchronisation sits between launches,
and ``collect()`` reads all results back with one D2H copy. This is what the
benchmark times as a "step"; ``simulate`` + ``areal_metrics`` is the same
work through the drop-in API (with host planning and copies per call).
"""

from __future__ import annotations

import numpy as np

from . import _native
from .engine import SweepBatch
from .errors import ConfigError
from .roughness import _finish_areal, _finish_profile


class SurfacePipeline:
    def __init__(self, batch: SweepBatch, every: int | None = 64, uncut: str = "exclude"):
        torch = _native.require_cuda()
        self.torch = torch
        self.lib = _native.lib()
        self.batch = batch
        s0 = batch.surfs[0]
        if not batch.same_shape or any(s.j_lo != 0 or s.j_hi != s.plan.grid.n for s in batch.surfs):
            raise ConfigError("SurfacePipeline needs whole, same-shape surfaces (use sharded.* for strips)")
        self.grid = s0.plan.grid
        self.n = batch.n
        self.uncut = uncut
        self.exclude = int(uncut == "exclude")
        g = self.grid
        self.ld = g.n + 1
        self.nodes = (g.m + 1) * (g.n + 1)
        self.rows_idx = list(range(0, g.m + 1, every)) if every else []
        dev = batch.dev
        n = self.n
        self.work = torch.empty(n * _native.WORK_DOUBLES, dtype=torch.float64, device=dev)
        self.out = torch.empty(n * 10 + max(1, n * len(self.rows_idx) * 8), dtype=torch.float64, device=dev)
        self.starts = torch.tensor([i * self.ld for i in self.rows_idx] or [0], dtype=torch.int64, device=dev)
        self.graph = None
        self.launches_per_run = batch.launches_per_run + 4 + (1 if self.rows_idx else 0)

    def _reduce(self, sp: int) -> None:
        lib, b = self.lib, self.batch
        h = b.keys.data_ptr()
        sent = b.base + b.sentinel_off
        o = self.out.data_ptr()
        n = self.n
        g = self.grid
        _native.check(lib.msurf_areal_pass1(h, self.ld, self.nodes, n, 0, 0, g.m + 1, g.n + 1, sent,
                                            self.exclude, self.work.data_ptr(), o, sp))
        _native.check(lib.msurf_areal_pass2(h, self.ld, self.nodes, n, 0, 0, g.m + 1, g.n + 1, sent,
                                            self.exclude, o, self.work.data_ptr(), o + n * 6 * 8, sp))
        if self.rows_idx:
            _native.check(lib.msurf_profiles(h, self.nodes, n, self.starts.data_ptr(), len(self.rows_idx),
                                             g.n + 1, 1, sent, self.exclude, None, o + n * 10 * 8, sp))

    def stages(self):
        """The step as three launch groups: (fill), (sweep), (decode + reductions)."""
        b = self.batch
        return [b.launch_fill, b.launch_sweep, lambda sp: (b.launch_decode(sp), self._reduce(sp))]

    def enqueue(self, events=None):
        """Launch the full step on the current stream; no host sync.
        ``events`` (4): before fill, after fill, after sweep, at the end."""
        st = self.torch.cuda.current_stream()
        sp = int(st.cuda_stream)
        for k, stage in enumerate(self.stages()):
            if events:
                events[k].record(st)
            stage(sp)
        if events:
            events[3].record(st)

    def capture(self):
        """Capture each stage into its own CUDA graph; run() replays them with
        optional events between stages (so the sweep is still timed alone)."""
        torch = self.torch
        self.enqueue()  # lazy module loading and allocator warm-up outside capture
        torch.cuda.synchronize()
        graphs = []
        for stage in self.stages():
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                stage(int(torch.cuda.current_stream().cuda_stream))
            graphs.append(g)
        self.graph = graphs
        return graphs

    def run(self, events=None):
        if self.graph is None:
            return self.enqueue(events)
        st = self.torch.cuda.current_stream()
        for k, g in enumerate(self.graph):
            if events:
                events[k].record(st)
            g.replay()
        if events:
            events[3].record(st)

    def collect(self):
        """One D2H: per surface (ArealMetrics | DomainError, [ProfileRoughness])."""
        a = _native.readback(self.out)
        n = self.n
        st1 = a[: n * 6].reshape(n, 6)
        st2 = a[n * 6: n * 10].reshape(n, 4)
        prof = a[n * 10: n * 10 + n * len(self.rows_idx) * 8].reshape(n, len(self.rows_idx), 8)
        res = []
        for s in range(n):
            try:
                am = _finish_areal(st1[s], st2[s], self.uncut)
            except Exception as exc:  # DomainError per sample
                am = exc
            prs = []
            for r, i in zip(prof[s], self.rows_idx):
                try:
                    prs.append(_finish_profile(r, i, self.uncut))
                except Exception as exc:
                    prs.append(exc)
            res.append((am, prs))
        return res
