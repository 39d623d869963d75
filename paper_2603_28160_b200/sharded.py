"""Multi-GPU: feed-direction strips for one large surface, parameter-set
shards for batches. One process per GPU (torchrun), torch.distributed over
NCCL for the only exchange the path has: the partial roughness moments.

Strip sharding: rank r owns node columns [j_lo, j_hi] of
the Z-map (all rows i) and holds only that (m+1) x (j_hi-j_lo+1) slab. The
sweep kernel's 2-D cull window is the strip, so each GPU evaluates only the
(step, tooth, 32-point chunk) work whose footprint meets its strip; heights
never cross GPUs. Roughness then needs two tiny all-reduces per output:
  areal:    stats1 = [sum z, max z, min z, n, n_uncut]  -> global mean
            moments = [sum|d|, sum d^2, sum d^3, sum d^4] around that mean
  profiles: [sum z, n, n_uncut, max z, min z] then [sum |z - mean|]
Batched runs shard by parameter set with no communication at all.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _native
from .errors import ConfigError, DomainError
from .extensions import Extensions
from .grid import GridSpec
from .planner import plan as make_plan
from .roughness import (ArealMetrics, ProfileRoughness, _finish_areal, _finish_profile,
                        _metrics_from_moments)

# column layouts of the reduced records (see include/msurf.h)
STATS1_SUM, STATS1_MAX, STATS1_MIN = (0, 3, 4), (1,), (2,)
PROF_SUM, PROF_MAX, PROF_MIN = (0, 1, 2), (3,), (4,)


def strip_bounds(nodes: int, world: int):
    """Contiguous, near-equal split of `nodes` feed-direction node columns."""
    if world < 1 or nodes < world:
        raise ConfigError(f"cannot split {nodes} columns over {world} ranks")
    cuts = [round(r * nodes / world) for r in range(world + 1)]
    return [(cuts[r], cuts[r + 1] - 1) for r in range(world)]


def batch_slice(count: int, rank: int, world: int) -> slice:
    """Parameter-set shard of a batch: contiguous block for rank."""
    lo = (count * rank) // world
    hi = (count * (rank + 1)) // world
    return slice(lo, hi)


def combine(t, sums, maxs, mins, group=None):
    """In-place all-reduce of a [k, c] record tensor whose columns are SUM,
    MAX or MIN quantities: two collectives (SUM on the sum columns, MAX on
    [max columns, -min columns])."""
    import torch
    import torch.distributed as dist

    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size(group) == 1:
        return t
    s = t[:, list(sums)].contiguous()
    dist.all_reduce(s, op=dist.ReduceOp.SUM, group=group)
    mm = torch.cat([t[:, list(maxs)], -t[:, list(mins)]], dim=1).contiguous()
    dist.all_reduce(mm, op=dist.ReduceOp.MAX, group=group)
    t[:, list(sums)] = s
    t[:, list(maxs)] = mm[:, : len(maxs)]
    t[:, list(mins)] = -mm[:, len(maxs):]
    return t


def make_allreduce(group=None):
    """Callable(tensor, kind) for roughness.areal_moments_device."""

    def ar(t, kind):
        if kind == "stats1":
            combine(t, STATS1_SUM, STATS1_MAX, STATS1_MIN, group)
        elif kind == "moments":
            combine(t, tuple(range(t.shape[1])), (), (), group)
        elif kind == "profiles1":
            combine(t, PROF_SUM, PROF_MAX, PROF_MIN, group)
        elif kind == "profiles2":
            combine(t, tuple(range(t.shape[1])), (), (), group)
        else:
            raise ValueError(kind)
        return t

    return ar


@dataclass
class StripResult:
    plan: object
    j_lo: int
    j_hi: int
    heights: object           # device fp64 (m+1) * (j_hi-j_lo+1), row-major
    counters: dict
    cells_updated: int
    main_loop_seconds: float
    batch: object


def simulate_strip(config, ext: Extensions | None, rank: int, world: int, trig: str = "device",
                   diagnostics: bool = False) -> StripResult:
    """Sweep this rank's feed-direction strip of one surface."""
    from .engine import SweepBatch, _counters_dict

    torch = _native.require_cuda()
    p = make_plan(config, ext)
    if p.record:
        raise ConfigError("record_trajectory is not supported under strip sharding")
    j_lo, j_hi = strip_bounds(p.grid.n + 1, world)[rank]
    b = SweepBatch([(p, j_lo, j_hi)], trig=trig, diagnostics=diagnostics)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    b.launch(events=ev)
    ctr, machined = b.counters()
    return StripResult(plan=p, j_lo=j_lo, j_hi=j_hi, heights=b.heights()[0],
                       counters=_counters_dict(ctr[0], diagnostics),
                       cells_updated=int(machined[0]), main_loop_seconds=ev[0].elapsed_time(ev[3]) * 1e-3,
                       batch=b)


def strip_roi(grid: GridSpec, roi, j_lo: int, j_hi: int):
    """Intersect a global inclusive ROI with a strip -> local (i_lo, jl_lo, rows, cols) or None."""
    if roi is None:
        roi = (0, 0, grid.m, grid.n)
    i_lo, a, i_hi, b = roi
    if not (0 <= i_lo <= i_hi <= grid.m and 0 <= a <= b <= grid.n):
        raise DomainError(f"roi {roi} outside grid [0, {grid.m}] x [0, {grid.n}] or empty")
    lo, hi = max(a, j_lo), min(b, j_hi)
    if lo > hi:
        return None
    return (i_lo, lo - j_lo, i_hi - i_lo + 1, hi - lo + 1)


def areal_metrics_strip(res: StripResult, roi=None, uncut: str = "raise", group=None) -> ArealMetrics:
    """Global areal metrics of a strip-sharded surface (two all-reduces)."""
    import torch

    lib = _native.lib()
    grid = res.plan.grid
    box = strip_roi(grid, roi, res.j_lo, res.j_hi)
    ld = res.j_hi - res.j_lo + 1
    dev = res.heights.device
    sent = torch.tensor([res.plan.initial_height], dtype=torch.float64, device=dev)
    work = torch.empty(_native.WORK_DOUBLES, dtype=torch.float64, device=dev)
    st1 = torch.zeros((1, 6), dtype=torch.float64, device=dev)
    st1[0, 1], st1[0, 2] = -np.inf, np.inf
    st2 = torch.zeros((1, 4), dtype=torch.float64, device=dev)
    sp = _native.stream_ptr()
    ex = int(uncut == "exclude")
    if box is not None:
        i_lo, jl, rows, cols = box
        _native.check(lib.msurf_areal_pass1(res.heights.data_ptr(), ld, 0, 1, i_lo, jl, rows, cols,
                                            sent.data_ptr(), ex, work.data_ptr(), st1.data_ptr(), sp))
    combine(st1, STATS1_SUM, STATS1_MAX, STATS1_MIN, group)
    st1[:, 5] = st1[:, 0] / st1[:, 3]  # global mean
    if box is not None:  # an all-excluded ROI yields n = 0 and is rejected on the host
        i_lo, jl, rows, cols = box
        _native.check(lib.msurf_areal_pass2(res.heights.data_ptr(), ld, 0, 1, i_lo, jl, rows, cols,
                                            sent.data_ptr(), ex, st1.data_ptr(), work.data_ptr(),
                                            st2.data_ptr(), sp))
    combine(st2, (0, 1, 2, 3), (), (), group)
    return _finish_areal(_native.readback(st1[0]), _native.readback(st2[0]), uncut)


def profile_roughness_strip(res: StripResult, every: int = 64, uncut: str = "raise", group=None):
    """Ra/Rz of every `every`-th feed profile (fixed i, all j) across strips."""
    import torch

    lib = _native.lib()
    grid = res.plan.grid
    ld = res.j_hi - res.j_lo + 1
    idx = list(range(0, grid.m + 1, every))
    dev = res.heights.device
    starts = torch.tensor([i * ld for i in idx], dtype=torch.int64, device=dev)
    sent = torch.tensor([res.plan.initial_height], dtype=torch.float64, device=dev)
    out = torch.empty(len(idx) * 8, dtype=torch.float64, device=dev)
    sp = _native.stream_ptr()
    ex = int(uncut == "exclude")
    _native.check(lib.msurf_profiles(res.heights.data_ptr(), 0, 1, starts.data_ptr(), len(idx), ld, 1,
                                     sent.data_ptr(), ex, None, out.data_ptr(), sp))
    first = out.view(-1, 8).clone()
    combine(first, PROF_SUM, PROF_MAX, PROF_MIN, group)
    first[:, 6] = first[:, 0] / first[:, 1]
    _native.check(lib.msurf_profiles(res.heights.data_ptr(), 0, 1, starts.data_ptr(), len(idx), ld, 1,
                                     sent.data_ptr(), ex, first.data_ptr(), out.data_ptr(), sp))
    sabs = out.view(-1, 8)[:, 5:6].contiguous()
    combine(sabs, (0,), (), (), group)
    first[:, 5:6] = sabs
    rows = _native.readback(first)
    return [_finish_profile(r, i, uncut) for r, i in zip(rows, idx)]


class StripPipeline:
    """Sync-free multi-GPU step for one strip-sharded surface: sweep of this
    rank's strip, then the roughness reductions with THREE small NCCL
    all-reduces per step (round 1: areal + profile sums, and their max/min;
    round 2: areal central moments + profile |d| sums). The device work
    between the collectives runs as three stages that ``capture()`` records as
    CUDA graphs (every buffer is preallocated, so replays reuse the captured
    addresses); the collectives stay eager between the replays. Results are
    read back by collect() after the timed region."""

    def __init__(self, batch, every: int = 64, uncut: str = "exclude", group=None):
        import torch

        self.torch = torch
        self.lib = _native.lib()
        self.batch = batch
        s = batch.surfs[0]
        self.plan, self.j_lo, self.j_hi = s.plan, s.j_lo, s.j_hi
        g = self.plan.grid
        self.ld = self.j_hi - self.j_lo + 1
        self.rows = g.m + 1
        self.uncut, self.exclude, self.group = uncut, int(uncut == "exclude"), group
        self.prof_idx = list(range(0, g.m + 1, every)) if every else []
        P = len(self.prof_idx)
        dev = batch.dev
        f64 = torch.float64
        self.work = torch.empty(_native.WORK_DOUBLES, dtype=f64, device=dev)
        self.st1 = torch.empty((1, 6), dtype=f64, device=dev)
        self.st2 = torch.empty((1, 4), dtype=f64, device=dev)
        self.prof = torch.empty((max(P, 1), 8), dtype=f64, device=dev)
        self.first = torch.empty((max(P, 1), 8), dtype=f64, device=dev)
        self.starts = torch.tensor([i * self.ld for i in self.prof_idx] or [0], dtype=torch.int64, device=dev)
        # collective buffers: round 1 sums [sum z, n, n_uncut] and extrema
        # [max z, -min z] of the areal record and every profile; round 2 moments
        self.sums = torch.empty((1 + P, 3), dtype=f64, device=dev)
        self.ext = torch.empty((1 + P, 2), dtype=f64, device=dev)
        self.mom = torch.empty(4 + P, dtype=f64, device=dev)
        self.P = P
        self.graphs = None
        self.launches_per_run = batch.launches_per_run + 4 + (2 if P else 0)

    def _allreduce(self, t, op):
        import torch.distributed as dist

        if dist.is_available() and dist.is_initialized() and dist.get_world_size(self.group) > 1:
            dist.all_reduce(t, op=op, group=self.group)

    def _stage_fill(self, sp):
        self.batch.launch_fill(sp)

    def _stage_sweep(self, sp):
        self.batch.launch_sweep(sp)

    def _stage_pack1(self, sp):
        """decode, areal pass 1, profile pass 1, pack round 1."""
        lib, b, P = self.lib, self.batch, self.P
        b.launch_decode(sp)
        h = b.keys.data_ptr()
        sent = b.base + b.sentinel_off
        _native.check(lib.msurf_areal_pass1(h, self.ld, 0, 1, 0, 0, self.rows, self.ld, sent, self.exclude,
                                            self.work.data_ptr(), self.st1.data_ptr(), sp))
        if P:
            _native.check(lib.msurf_profiles(h, 0, 1, self.starts.data_ptr(), P, self.ld, 1, sent,
                                             self.exclude, None, self.prof.data_ptr(), sp))
        self.sums[0:1, 0:1].copy_(self.st1[:, 0:1])
        self.sums[0:1, 1:3].copy_(self.st1[:, 3:5])
        self.ext[0:1, 0].copy_(self.st1[:, 1])
        self.torch.neg(self.st1[:, 2], out=self.ext[0:1, 1])
        if P:
            self.sums[1:].copy_(self.prof[:P, 0:3])
            self.ext[1:, 0].copy_(self.prof[:P, 3])
            self.torch.neg(self.prof[:P, 4], out=self.ext[1:, 1])

    def _stage_moments(self, sp):
        """unpack round 1 (global means), areal pass 2, profile pass 2, pack round 2."""
        lib, b, P = self.lib, self.batch, self.P
        self.st1[:, 0:1] = self.sums[0:1, 0:1]
        self.st1[:, 3:5] = self.sums[0:1, 1:3]
        self.st1[:, 1] = self.ext[0:1, 0]
        self.st1[:, 2] = -self.ext[0:1, 1]
        self.st1[:, 5] = self.st1[:, 0] / self.st1[:, 3]  # global mean
        if P:
            self.first[:P, 0:3] = self.sums[1:]
            self.first[:P, 3] = self.ext[1:, 0]
            self.first[:P, 4] = -self.ext[1:, 1]
            self.first[:P, 6] = self.first[:P, 0] / self.first[:P, 1]
        h = b.keys.data_ptr()
        sent = b.base + b.sentinel_off
        _native.check(lib.msurf_areal_pass2(h, self.ld, 0, 1, 0, 0, self.rows, self.ld, sent, self.exclude,
                                            self.st1.data_ptr(), self.work.data_ptr(), self.st2.data_ptr(), sp))
        if P:
            _native.check(lib.msurf_profiles(h, 0, 1, self.starts.data_ptr(), P, self.ld, 1, sent,
                                             self.exclude, self.first.data_ptr(), self.prof.data_ptr(), sp))
        self.mom[:4].copy_(self.st2.reshape(-1))
        if P:
            self.mom[4:].copy_(self.prof[:P, 5])

    def _stage_finish(self, sp):
        self.st2.copy_(self.mom[:4].view(1, 4))
        if self.P:
            self.first[: self.P, 5] = self.mom[4:]

    def _stages(self):
        return (self._stage_fill, self._stage_sweep, self._stage_pack1, self._stage_moments, self._stage_finish)

    def capture(self):
        """Record the five device stages as CUDA graphs (one warm-up run
        first, outside capture); the collectives between them stay eager."""
        torch = self.torch
        self.run()
        torch.cuda.synchronize()
        graphs = []
        for stage in self._stages():
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                stage(int(torch.cuda.current_stream().cuda_stream))
            graphs.append(g)
        self.graphs = graphs
        return graphs

    def run(self, events=None):
        """One step; ``events`` (4): start, after the fill, after the sweep, end."""
        import torch.distributed as dist

        torch = self.torch
        st = torch.cuda.current_stream()
        sp = int(st.cuda_stream)

        def stage(k):
            if self.graphs is None:
                self._stages()[k](sp)
            else:
                self.graphs[k].replay()

        if events:
            events[0].record(st)
        stage(0)
        if events:
            events[1].record(st)
        stage(1)
        if events:
            events[2].record(st)
        stage(2)
        self._allreduce(self.sums, dist.ReduceOp.SUM)
        self._allreduce(self.ext, dist.ReduceOp.MAX)
        stage(3)
        self._allreduce(self.mom, dist.ReduceOp.SUM)
        stage(4)
        if events:
            events[3].record(st)

    def collect(self):
        st1 = _native.readback(self.st1[0])
        st2 = _native.readback(self.st2[0])
        try:
            am = _finish_areal(st1, st2, self.uncut)
        except DomainError as exc:
            am = exc
        prs = []
        if self.P:
            rows = _native.readback(self.first[: self.P])
            for r, i in zip(rows, self.prof_idx):
                try:
                    prs.append(_finish_profile(r, i, self.uncut))
                except DomainError as exc:
                    prs.append(exc)
        return am, prs
