"""The FSM sweep on the GPU — drop-in for millsurf.engine (engine.py:63-485).

``simulate(config)`` plans on the host (planner.py), ships every per-surface
array to HBM in one copy, and runs three kernels from libmsurf.so on the
current stream: key fill (stock height), the sweep, and the key -> fp64
decode that also counts machined cells. ``simulate_batch`` runs many
parameter sets in the same three launches (the batched dataset mode).
The returned HeightField stays in HBM until its NumPy view is requested, so
``areal_metrics`` on it never leaves the device.

``main_loop_seconds`` is the device time of fill + sweep + decode measured
with CUDA events (the reference times its main loop plus the min-merge,
engine.py:329-342).
"""

from __future__ import annotations

import ctypes
import math
import threading
from dataclasses import dataclass, field, replace

import numpy as np

from . import _native
from .errors import ConfigError, MillsurfError
from .extensions import Extensions
from .grid import GridSpec, HeightField, TrajectoryRecord
from .planner import (DEVICE_FIELDS, MODE_EXT_TILT, MODE_REF, SweepPlan, chunk_f32, plan, plan_many, plan_zfloor, step_window,
                      time_step)

DEFAULT_MAX_STEP_ANGLE_RAD = math.radians(0.5)
# Z-map bytes one sweep job may cover: keeps its RED.MIN traffic in the
# 126 MB L2 (surfaces above this are cut into feed-direction sub-strips)
L2_TILE_BYTES = int(float(__import__("os").environ.get("MSURF_L2_TILE_MB", "48")) * (1 << 20))
# groups of at most this many jobs launch one msurf_sweep_job per job, provided
# each job fills the GPU several times over (>= ONE_JOB_MIN_TILES tiles: the L2
# sub-strips of one large surface); groups of many small surfaces take one
# batched launch (per-job launches would pay a grid tail per surface:
# config 3 in launch groups of 32 sets, 2.1 -> 1.2 ms per group)
ONE_JOB_LAUNCH_MAX = int(__import__("os").environ.get("MSURF_ONE_JOB_MAX", "32"))
ONE_JOB_MIN_TILES = int(__import__("os").environ.get("MSURF_ONE_JOB_MIN_TILES", "16384"))


# surface-cap cull (msurf_job.zcap) for tilt-mode by-value jobs: swept (pass,
# tooth) by (pass, tooth) with a per-tile upper bound of the current heights
# refreshed in between (MSURF_ZCAP=0 turns it off; result-neutral either way)
ZCAP = __import__("os").environ.get("MSURF_ZCAP", "1") != "0"
# eight-warp CTAs for capped launches (measured slower once launches overlap)
ZCAP_WIDE = __import__("os").environ.get("MSURF_ZCAP_WIDE", "0") != "0"
# slab budget of capped surfaces: their phase 1 repeats per slab, their RED
# stream is small (config 5 sweep with 48 / 72 / 96 / 160 MB slabs: 15.5 /
# 14.1 / 14.2 / 17.5 ms)
ZCAP_L2_TILE_BYTES = int(float(__import__("os").environ.get("MSURF_ZCAP_L2_TILE_MB", "72")) * (1 << 20))
ZCAP_MIN_JOBS = int(__import__("os").environ.get("MSURF_ZCAP_MIN_JOBS", "1"))  # capped jobs swept side by side
# sub-strips a capped surface is cut into at least (several jobs side by side
# keep more of the GPU busy than one job's (pass, tooth) chain)
ZCAP_MIN_STRIPS = int(__import__("os").environ.get("MSURF_ZCAP_MIN_STRIPS", "1"))
# overlapping (pass, tooth) launches per capped job. Measured on config 5 (3
# sub-strip jobs; sweep without caps 37.3 ms): single-kernel launches depth 1 /
# 2 / 3 / 4 -> 27.1 / 20.5 / 20.3 / 20.9 ms; staged two-kernel launches depth
# 1 / 2 / 3 -> 16.7 / 17.0 / 19.6 ms
ZCAP_DEPTH = int(__import__("os").environ.get("MSURF_ZCAP_DEPTH", "0"))  # 0: SweepBatch._capped_depth
# step-points of a (pass, tooth) launch above which it fills the GPU alone
ZCAP_LONG_LAUNCH = float(__import__("os").environ.get("MSURF_ZCAP_LONG_LAUNCH", "3e8"))
# capped launches as two kernels: phase 1 staged to HBM, phase 2 balanced over every warp
ZCAP_STAGED = __import__("os").environ.get("MSURF_ZCAP_STAGED", "1") != "0"
# strip-pipelined capped surfaces: the last PROGRESSIVE_PASSES raster passes
# are launched one call each, and after every call the node rows no later
# pass can reach are decoded and start crossing PCIe (0: whole strips only)
PROGRESSIVE_PASSES = int(__import__("os").environ.get("MSURF_PROGRESSIVE_PASSES", "3"))


def _per_job_launches(tiles) -> bool:
    live = [t for t in tiles if t]
    return len(live) <= 1 or (len(tiles) <= ONE_JOB_LAUNCH_MAX and min(live) >= ONE_JOB_MIN_TILES)
# launch-group size of large simulate_batch calls
BATCH_CHUNK = int(__import__("os").environ.get("MSURF_BATCH_CHUNK", "32"))
PIPELINE_PLAN_THREADS = int(__import__("os").environ.get("MSURF_PIPELINE_THREADS", "1"))
# size of the first launch group of a pipelined batch (the GPU starts sooner)
PIPELINE_FIRST_CHUNK = int(__import__("os").environ.get("MSURF_FIRST_CHUNK", "0"))
# native planner threads for the first group (planned while nothing else runs)
PIPELINE_FIRST_THREADS = int(__import__("os").environ.get("MSURF_FIRST_THREADS", "1"))
# threads of the native planning loops of every group (GIL released)
PIPELINE_NATIVE_THREADS = int(__import__("os").environ.get("MSURF_NATIVE_THREADS", "8"))

__all__ = ["SimulationConfig", "SimulationResult", "time_step", "simulate", "simulate_batch",
           "simulate_reference", "run_benchmark", "BenchmarkReport", "BenchmarkRow", "sweep_plans"]


@dataclass(frozen=True)
class SimulationConfig:
    """Same fields and defaults as millsurf.engine.SimulationConfig (engine.py:63-73).
    ``worker_count`` is accepted for compatibility; the GPU result does not
    depend on it (the reference guarantees the same, engine.py:316-317)."""

    tool: object
    process: object
    grid: GridSpec
    edge_point_count: int | None = None
    max_step_angle_rad: float = DEFAULT_MAX_STEP_ANGLE_RAD
    time_step_s: float | None = None
    span_s: tuple | None = None
    record_trajectory: bool = False
    worker_count: int = 1


class _Launch:
    """Device-side state of one asynchronous sweep launch: the batch (keeps
    every buffer alive), its events, and the small D2H read of the counters
    performed once, on first demand. Its events go back to a per-device pool
    when it is released (re-recording a finished or abandoned event is
    legal), so a simulate call does not pay cudaEventCreate."""

    def __init__(self, batch, events):
        self.batch, self.events = batch, events
        self._small = None

    def counters(self):
        if self._small is None:
            self._small = self.batch.counters()
        return self._small

    def device_seconds(self):
        self.events[3].synchronize()
        return self.events[0].elapsed_time(self.events[3]) * 1e-3

    def __del__(self):
        try:
            _give_events(self.batch.dev.index, (self.events[0], self.events[3]))
        except Exception:  # interpreter shutdown
            pass


class SimulationResult:
    """Same fields as millsurf.engine.SimulationResult (engine.py:76-83).
    ``simulate`` returns before the GPU finishes: ``cells_updated``,
    ``main_loop_seconds`` and ``counters`` synchronise on first access, the
    height field stays in HBM until ``field.heights`` is read."""

    def __init__(self, field, trajectory, time_steps, trajectory_points, cells_updated=None,
                 main_loop_seconds=None, counters=None, launch=None, index=0, share=1.0):
        self.field, self.trajectory = field, trajectory
        self.time_steps, self.trajectory_points = time_steps, trajectory_points
        self._cells, self._secs, self._ctrs = cells_updated, main_loop_seconds, counters
        self._launch, self._index, self._share = launch, index, share

    @property
    def cells_updated(self) -> int:
        if self._cells is None:
            self._cells = int(self._launch.counters()[1][self._index])
        return self._cells

    @property
    def main_loop_seconds(self) -> float:
        if self._secs is None:
            self._secs = self._launch.device_seconds() * self._share
        return self._secs

    @property
    def counters(self) -> dict:
        if self._ctrs is None:
            self._ctrs = _counters_dict(self._launch.counters()[0][self._index],
                                        self._launch.batch.diagnostics)
        return self._ctrs

    def __repr__(self) -> str:
        return (f"SimulationResult(time_steps={self.time_steps}, trajectory_points={self.trajectory_points}, "
                f"cells_updated={self.cells_updated})")


@dataclass
class _Surface:
    plan: SweepPlan
    j_lo: int
    j_hi: int
    key_off: int = 0          # element offset into the keys tensor
    nodes: int = 0
    n_strips: int = 1         # L2 sub-strips the surface is cut into
    strip_off: int = -1       # element offset into strip_keys (n_strips > 1)
    col0: list = field(default_factory=list)  # sub-strip column offsets from j_lo


def final_rows(p: SweepPlan, p_next: int) -> int:
    """Node rows [0, r) of a surface that no raster pass from p_next on can
    deposit into: pass q reaches x in x0_q +- (max|x_t| + max|y_t| over every
    tooth's tool-frame box + |vibration|) (the cap refresh's band, msurf.cu
    ZBand), located with two nodes of slack (launch_by_strip's progressive
    row release; tests/test_host_cpu.py checks it against the oracle's
    per-pass deposits)."""
    tb = np.asarray(p.tooth_box, dtype=np.float64).reshape(-1, 6)
    reach = float((np.maximum(np.abs(tb[:, 0]), np.abs(tb[:, 1])) +
                   np.maximum(np.abs(tb[:, 2]), np.abs(tb[:, 3]))).max()) + abs(p.vib_amp)
    x_lo = float(np.min(p.pass_x0[p_next:])) - reach
    r = int(math.floor((x_lo - p.grid.x_min_mm) / p.grid.spacing_mm)) - 2
    return max(0, min(p.grid.m + 1, r))


def _trig_tables(p: SweepPlan):
    """Host-libm tables (parity mode): exactly the reference's per-row trig
    (engine.py:240, 252-255) — np.cos/np.sin of base_K - omega*t."""
    t = p.t_start + np.arange(p.steps, dtype=np.float64) * p.dt
    tab = np.empty((p.steps, p.teeth, 2))
    for k in range(p.teeth):
        th = p.tooth_base[k] - p.omega * t
        tab[:, k, 0] = np.cos(th)
        tab[:, k, 1] = np.sin(th)
    vib = np.sin(p.vib_omega * t + p.vib_phase) if p.vib_amp != 0.0 else None
    return tab, vib


class SweepBatch:
    """A set of surfaces (plans, each with its owned column range [j_lo, j_hi])
    uploaded to HBM once and swept by ``launch()`` as many times as needed
    (the benchmark times repeated launches with inputs resident).

    Device layout: one uint8 arena holding every per-surface array, the job
    descriptors (msurf_job) and tile prefix sums, written by ONE H2D copy;
    one int64 tensor holding all surfaces' Z-maps back to back (u64 keys
    during the sweep, fp64 heights after the decode, in place). A surface
    larger than the L2 budget keeps its keys in a second tensor, sub-strip by
    sub-strip (each sweep job deposits into one contiguous slab), and its
    decode writes the row-major heights into the first."""

    def __init__(self, surfaces, trig: str = "device", device=None, l2_tile_bytes: int | None = None,
                 diagnostics: bool = False):
        torch = _native.require_cuda()
        self.torch = torch
        self.lib = _native.lib()
        if l2_tile_bytes is None:
            l2_tile_bytes = L2_TILE_BYTES
        # per-point deposit/atomic counters (MSURF_SWEEP_DIAG): off on the hot path
        self.diagnostics = bool(diagnostics)
        self.dev = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
        if trig not in ("device", "host"):
            raise ConfigError(f"trig must be 'device' or 'host', got {trig!r}")
        surfs = [_Surface(p, lo, hi) for p, lo, hi in surfaces]
        if not surfs:
            raise ConfigError("empty batch")
        total = 0
        strip_total = 0
        for s in surfs:
            s.key_off = total
            w = s.j_hi - s.j_lo + 1
            rows = s.plan.grid.m + 1
            s.nodes = rows * w
            total += s.nodes
            # surfaces above the L2 budget are cut into feed-direction sub-strips;
            # their keys live strip by strip (contiguous slab per sweep job) and the
            # decode writes the row-major heights (msurf_decode_strips)
            budget = l2_tile_bytes
            capped = ZCAP and s.plan.mode == MODE_EXT_TILT and s.plan.passes * s.plan.teeth > 1
            if capped:
                budget = max(budget, ZCAP_L2_TILE_BYTES)  # capped surfaces: fewer, larger slabs
            k = 1 if s.plan.record else max(1, min(w, -(-rows * w * 8 // budget)))
            if capped and not s.plan.record:
                k = max(k, min(ZCAP_MIN_STRIPS, max(1, w // 64)))
            s.n_strips = k
            s.col0 = [(w * q) // k for q in range(k + 1)]
            if k > 1:
                s.strip_off = strip_total
                strip_total += s.nodes
        self.surfs = surfs
        self.keys = torch.empty(max(total, 1), dtype=torch.int64, device=self.dev)
        self.strip_keys = torch.empty(strip_total, dtype=torch.int64, device=self.dev) if strip_total else None
        self.need_traj = [s.plan.record for s in surfs]
        traj_len = sum(s.plan.steps * s.plan.teeth * 3 for s, r in zip(surfs, self.need_traj) if r)
        self.traj = torch.empty(traj_len, dtype=torch.float64, device=self.dev) if traj_len else None

        ar = _native.Arena()
        offs = [None] * len(surfs)
        i = 0
        while i < len(surfs):
            p = surfs[i].plan
            grp = p.group
            if grp is not None and grp[0].owns(p, grp[1]):
                # a run of consecutive sets planned together: one slice per field
                g, b0 = grp
                k = i + 1
                while (k < len(surfs) and surfs[k].plan.group is not None and surfs[k].plan.group[0] is g
                       and surfs[k].plan.group[1] == b0 + (k - i) and g.owns(surfs[k].plan, b0 + (k - i))):
                    k += 1
                run = {}
                for f in DEVICE_FIELDS:
                    a = g.arrays[f]
                    run[f] = (ar.add(a[b0: b0 + (k - i)], pinned=g.pinned_sets(f, b0, k - i)), a[0].nbytes)
                for q in range(i, k):
                    offs[q] = {f: o + (q - i) * nb for f, (o, nb) in run.items()}
            else:
                k = i + 1
                offs[i] = dict(
                    tooth_base=ar.add(p.tooth_base.astype(np.float64, copy=False)),
                    tooth_rows=ar.add(p.tooth_rows.astype(np.float64, copy=False)),
                    pts=ar.add(p.pts.astype(np.float64, copy=False)),
                    tooth_box=ar.add(p.tooth_box.astype(np.float64, copy=False)),
                    chunk_circ=ar.add(p.chunk_circ.astype(np.float64, copy=False)),
                    chunk_f32=ar.add(chunk_f32(p.chunk_circ, p.tooth_box, plan_zfloor(p))),
                    pass_x0=ar.add(p.pass_x0.astype(np.float64, copy=False)),
                    min_index=ar.add(p.min_index.astype(np.int32, copy=False)),
                )
            for q in range(i, k):
                s, o = surfs[q], offs[q]
                if s.n_strips > 1:
                    o["col0"] = ar.add(np.asarray(s.col0, dtype=np.int64))
                    # per strip [0, w_q]: msurf_decode_strips over a row range of one strip
                    o["strip_w"] = ar.add(np.array([[0, s.col0[q + 1] - s.col0[q]] for q in range(s.n_strips)],
                                                   dtype=np.int64))
                # the trajectory record (engine.py:242-310) exposes the per-row
                # cos/sin themselves, and the reference defines it with the libm
                # values (simulate and simulate_reference records are identical,
                # test_engine.py:127-137): a record-keeping surface takes the
                # host-libm per-row table (O(steps x teeth)); the sweep stays on
                # the device either way
                if trig == "host" or s.plan.record:
                    tab, vib = _trig_tables(s.plan)
                    o["trig_table"] = ar.add(tab)
                    if vib is not None:
                        o["vib_table"] = ar.add(vib)
            i = k
        n = len(surfs)
        self.n = n
        self.sentinel_off = ar.add(np.array([s.plan.initial_height for s in surfs], dtype=np.float64))
        # counters [n][NUM_CTRS] then machined [n], contiguous: zeroed by one memset per launch
        self.ctr_off = ar.add(np.zeros(n * (_native.NUM_CTRS + 1), dtype=np.uint64))
        self.machined_off = self.ctr_off + n * _native.NUM_CTRS * 8
        # Jobs: each surface is cut into feed-direction sub-strips whose Z-map
        # slab fits in L2 (the RED.MIN traffic then stays on chip), each with
        # the time window whose footprint can reach it; sub-strips of one
        # surface are consecutive in the tile order so resident CTAs share one.
        tile_steps = self.lib.msurf_tile_steps()
        jobs = []  # (surface index, j_lo, j_hi, step_lo, step_hi)
        for i, s in enumerate(surfs):
            k = s.n_strips  # 1 when a trajectory record needs every step in one job
            for q in range(k):
                lo = s.j_lo + s.col0[q]
                hi = s.j_lo + s.col0[q + 1] - 1
                whole = k == 1 and s.j_lo == 0 and s.j_hi == s.plan.grid.n
                s_lo, s_hi = (0, s.plan.steps) if (whole or s.plan.record) else step_window(s.plan, lo, hi)
                if s_hi > s_lo:
                    jobs.append((i, lo, hi, s_lo, s_hi))
        self.jobs = jobs
        groups = {}
        for jn, jb in enumerate(jobs):
            groups.setdefault(surfs[jb[0]].plan.mode, []).append(jn)
        self.group_meta = []
        self.group_tiles = []
        self.group_host_jobs = []  # host copies of the descriptors (by-value launches)
        self.group_per_job = []
        for mode, jidx in sorted(groups.items()):
            tiles = [surfs[jobs[j][0]].plan.passes * surfs[jobs[j][0]].plan.teeth *
                     ((jobs[j][4] - jobs[j][3] + tile_steps - 1) // tile_steps) for j in jidx]
            per_job = _per_job_launches(tiles)
            if per_job:  # by-value launches: host descriptors only
                job_off = pre_off = None
            else:
                prefix = np.zeros(len(tiles) + 1, dtype=np.int64)
                np.cumsum(tiles, out=prefix[1:])
                job_off = ar.reserve(len(jidx) * _native.JOB_DTYPE.itemsize)  # written by fill()
                pre_off = ar.add(prefix)
            self.group_meta.append((mode, jidx, job_off, pre_off, sum(tiles),
                                    max(surfs[jobs[j][0]].plan.points for j in jidx)))
            self.group_tiles.append(tiles)
            self.group_per_job.append(per_job)
        keys_ptr = self.keys.data_ptr()
        strip_ptr = self.strip_keys.data_ptr() if self.strip_keys is not None else 0
        traj_ptr = self.traj.data_ptr() if self.traj is not None else 0
        self.traj_off = []
        toff = 0
        for s, r in zip(surfs, self.need_traj):
            self.traj_off.append(toff if r else None)
            if r:
                toff += s.plan.steps * s.plan.teeth * 3

        def fill(base):
            # descriptors as rows of a structured array with msurf_job's layout
            out = []
            for mode, jidx, job_off, _, _, _ in self.group_meta:
                rows = []
                for jn in jidx:
                    i, lo, hi, s_lo, s_hi = jobs[jn]
                    s, o, p = surfs[i], offs[i], surfs[i].plan
                    g = p.grid
                    if s.n_strips > 1:  # contiguous rows x (hi - lo + 1) slab of strip_keys
                        ld, kp = hi - lo + 1, strip_ptr + (s.strip_off + (g.m + 1) * (lo - s.j_lo)) * 8
                    else:
                        ld, kp = s.j_hi - s.j_lo + 1, keys_ptr + (s.key_off + (lo - s.j_lo)) * 8
                    # trajectory rows are written by the job that owns column j_lo of
                    # the surface and covers every step (REF mode records need no cull)
                    tr = (traj_ptr + self.traj_off[i] * 8) if (self.need_traj[i] and lo == s.j_lo) else 0
                    rows.append((
                        g.spacing_mm, g.x_min_mm, g.y_min_mm, g.m, g.n, lo, hi, ld, kp,
                        p.t_start, p.dt, p.steps, s_lo, s_hi, p.y0, p.feed_speed, p.omega,
                        base + o["tooth_base"], base + o["tooth_rows"], base + o["pts"], base + o["tooth_box"],
                        base + o["chunk_circ"], base + o["chunk_f32"], base + o["pass_x0"],
                        p.tilt_c, p.tilt_s, p.zoff, p.vib_amp, p.vib_omega, p.vib_phase,
                        base + o["trig_table"] if "trig_table" in o else 0,
                        base + o["vib_table"] if "vib_table" in o else 0,
                        tr, base + o["min_index"], base + self.ctr_off + i * _native.NUM_CTRS * 8, 0, 0,
                        p.teeth, p.points, p.passes, 0, 0, 0))
                arr = np.array(rows, dtype=_native.JOB_DTYPE)
                if job_off is not None:
                    out.append((job_off, arr.view(np.uint8)))
                self.group_host_jobs.append(arr)
            return out

        self.h2d_bytes = ar.size
        self.buf = ar.upload(self.dev, fill)
        self._fresh = True
        self.base = self.buf.data_ptr()
        self.offs = offs
        self.same_shape = len({s.nodes for s in surfs}) == 1
        # one fill / decode launch for the whole batch (no strip-layout surface)
        self.batched_fill = self.same_shape and all(s.n_strips == 1 for s in surfs)
        # msurf_sweep scratch (tile count + pre-culled tile list), shared by the
        # batched launch groups (they run in stream order)
        need = max((gm[4] for gm, pj in zip(self.group_meta, self.group_per_job) if not pj), default=0)
        self.sweep_scratch = torch.empty(need + 1, dtype=torch.int64, device=self.dev) if need else None
        sweeps = sum((sum(1 for t in tl if t) if pj else 1) for pj, tl in zip(self.group_per_job, self.group_tiles))
        self.zc_seq = self._build_zcap_sequences()
        # a capped job: per (pass, tooth) one sweep (staged: phase 1 + phase 2)
        # and one cap refresh, instead of one launch
        per = 3 if ZCAP_STAGED else 2
        extra = sum(per * q[0] - 1 for seqs in self.zc_seq for q in seqs if q is not None)
        self.launches_per_run = 2 * (1 if self.batched_fill else n) + sweeps + extra

    def _build_zcap_sequences(self):
        """Per launch group, per job: None, or the surface-cap state of a
        tilt-mode by-value job of more than one (pass, tooth): its launch
        count, cap tile array and stock pointer (msurf_sweep_jobs_capped)."""
        torch = self.torch
        out = []
        for g, (mode, jidx, _, _, _, _) in enumerate(self.group_meta):
            seqs = [None] * len(jidx)
            if ZCAP and self.group_per_job[g] and mode == MODE_EXT_TILT:
                host = self.group_host_jobs[g]
                for k, jn in enumerate(jidx):
                    i, lo, hi, _, _ = self.jobs[jn]
                    p = self.surfs[i].plan
                    if p.passes * p.teeth < 2 or not self.group_tiles[g][k]:
                        continue
                    rows, cols = p.grid.m + 1, hi - lo + 1
                    # written by the first cap refresh of every launch
                    ct = self.lib.msurf_zcap_tile()
                    zc = torch.empty(((rows + ct - 1) // ct) * ((cols + ct - 1) // ct), dtype=torch.float32,
                                     device=self.dev)
                    host[k]["zcap"] = zc.data_ptr()
                    # (launches, the cap tiles kept alive, the device stock height)
                    seqs[k] = (p.passes * p.teeth, zc, self.base + self.sentinel_off + 8 * i)
                # the (pass, tooth) launches of one job are short and underfill the
                # GPU: several jobs (L2 sub-strips) run side by side and each
                # keeps ceil(3 / jobs) launches in flight (measured, staged form,
                # 72 MB slabs: config 5 at N = 1 / 2 / 4 / 8 strips per GPU 14.5 /
                # 8.7 / 4.7 / 2.8 ms; config 2, one job: 0.59 vs 0.69 ms uncapped)
                if sum(q is not None for q in seqs) < ZCAP_MIN_JOBS:
                    for k, q in enumerate(seqs):
                        if q is not None:
                            host[k]["zcap"] = 0
                    seqs = [None] * len(jidx)
            out.append(seqs)
        return out

    def _capped_depth(self, g: int, ks) -> int:
        """Launches in flight per capped job: about three per GPU in total for
        short (pass, tooth) launches, which underfill the GPU on their own; two
        for long ones, which fill it, so that the caps each launch reads are
        fresher (measured: config 2, one job of ~1.3e8 step-points per launch,
        0.88 / 0.62 / 0.59 ms at 1 / 2 / 3 in flight; config 5, two jobs of
        ~6.4e8, 13.6 / 13.8 / 16.9 ms at 2 / 4 / 6)."""
        if ZCAP_DEPTH > 0:
            return max(1, min(ZCAP_DEPTH, 4))
        work = 0
        for k in ks:
            i, _, _, s_lo, s_hi = self.jobs[self.group_meta[g][1][k]]
            work = max(work, (s_hi - s_lo) * self.surfs[i].plan.points)
        total = 2 if work >= ZCAP_LONG_LAUNCH else 3
        return max(1, min(-(-total // len(ks)), 4))

    def _capped_stage(self, g: int, ks, depth: int, max_pts: int):
        """Staging buffer: one (job, in-flight launch) slot each, sized for the
        largest job (msurf_stage_bytes); reused across launches."""
        if not ZCAP_STAGED:
            return 0, 0
        # one buffer per (group, jobs, depth), kept for the batch's life: CUDA
        # graphs captured over a launch hold its address
        key = (g, tuple(ks), depth)
        if not hasattr(self, "_stages"):
            self._stages = {}
        if key not in self._stages:
            host = self.group_host_jobs[g]
            nb = ctypes.c_int64(0)
            each = 0
            for k in ks:
                _native.check(self.lib.msurf_stage_bytes(host[k:k + 1].ctypes.data, max_pts, ctypes.byref(nb)))
                each = max(each, (nb.value + 255) // 256 * 256)
            buf = self.torch.empty(each * len(ks) * depth, dtype=self.torch.uint8, device=self.dev)
            self._stages[key] = (buf, each)
        buf, each = self._stages[key]
        return buf.data_ptr(), each

    def _launch_capped(self, g: int, ks, mode: int, flag: int, max_pts: int, sp: int, split: bool = False,
                       passes=None, anchors=None):
        """Surface-cap jobs ks of by-value group g side by side
        (msurf_sweep_jobs_capped; staged two-kernel launches when
        ZCAP_STAGED). ``split``: one call per job, each forked from and joined
        into its own anchor stream (returned, in ks order) so the caller can
        wait for each job's slab separately; jobs still run side by side, the
        earlier ones at higher stream priority. ``passes`` = (p0, p1): only
        raster passes [p0, p1) of every job (the caps carry over between
        calls); ``anchors``: continue on these anchor streams (a previous
        split call's) instead of forking new ones from ``sp``."""
        host = self.group_host_jobs[g]
        wide = _native.SWEEP_WIDE if ZCAP_WIDE else 0
        depth = self._capped_depth(g, ks)
        stage, each = self._capped_stage(g, ks, depth, max_pts)
        stocks = np.array([self.zc_seq[g][k][-1] for k in ks], dtype=np.int64)
        if not split:
            for c0 in range(0, len(ks), 8):  # eight stream slots per call
                part = ks[c0:c0 + 8]
                arr = np.ascontiguousarray(host[part])
                st_p = stage + c0 * depth * each if stage else 0
                _native.check(self.lib.msurf_sweep_jobs_capped(arr.ctypes.data, len(part), mode | flag | wide, max_pts,
                                                               stocks[c0:].ctypes.data, depth, st_p, each, 0, sp))
            return None
        lib = self.lib
        out = []
        for n, k in enumerate(ks):
            if anchors is not None:
                anchor = anchors[n]
            else:
                anchor = lib.msurf_anchor_stream(n % 8)
                if not anchor:
                    raise MillsurfError("libmsurf: no anchor stream")
                _native.check(lib.msurf_stream_wait(anchor, sp))
            arr = host[k:k + 1].copy()  # a copy: the pass range edits must not touch the batch's descriptors
            if passes is not None:
                p0, p1 = passes
                arr["pass_x0"] += 8 * p0
                arr["passes"] = p1 - p0
            st_p = stage + n * depth * each if stage else 0
            _native.check(lib.msurf_sweep_jobs_capped(arr.ctypes.data, 1, mode | flag | wide, max_pts,
                                                      stocks[n:].ctypes.data, depth, st_p, each, n % 8, anchor))
            out.append(anchor)
        return out

    def _launch_job(self, g: int, k: int, mode: int, flag: int, max_pts: int, sp: int) -> None:
        """Job k of by-value launch group g (a surface-cap job through
        msurf_sweep_job_capped: (pass, tooth) launches with cap refreshes)."""
        lib, sz = self.lib, _native.JOB_DTYPE.itemsize
        job = self.group_host_jobs[g].ctypes.data + k * sz
        seq = self.zc_seq[g][k]
        if seq is None:
            _native.check(lib.msurf_sweep_job(job, mode | flag, max_pts, sp))
            return
        stock = seq[-1]
        wide = _native.SWEEP_WIDE if ZCAP_WIDE else 0
        _native.check(lib.msurf_sweep_job_capped(job, mode | flag | wide, max_pts, stock, sp))

    # ------------------------------------------------------------------
    def launch_fill(self, sp: int) -> None:
        """Zero the counters and initialise every Z-map to its stock height."""
        lib, base, keys_ptr = self.lib, self.base, self.keys.data_ptr()
        if self._fresh:  # the upload itself wrote zero counters
            self._fresh = False
        else:
            self.buf[self.ctr_off: self.ctr_off + self.n * (_native.NUM_CTRS + 1) * 8].zero_()
        if self.batched_fill:
            _native.check(lib.msurf_fill_keys(keys_ptr, self.surfs[0].nodes, self.n,
                                              base + self.sentinel_off, sp))
        else:
            for i, s in enumerate(self.surfs):
                dst = (self.strip_keys.data_ptr() + s.strip_off * 8) if s.n_strips > 1 else keys_ptr + s.key_off * 8
                _native.check(lib.msurf_fill_keys(dst, s.nodes, 1, base + self.sentinel_off + 8 * i, sp))

    def launch_sweep(self, sp: int) -> None:
        """One msurf_sweep launch per kinematics mode present in the batch."""
        lib, base = self.lib, self.base
        for g, (mode, idx, job_off, pre_off, n_tiles, max_pts) in enumerate(self.group_meta):
            flag = self._sweep_flag()
            if self.group_per_job[g]:
                # one job, or the L2 sub-strips of a large surface: one launch per job
                # with the descriptor passed by value (constant-bank operands); the
                # surface-cap jobs of the group run concurrently, one stream each
                capped = [k for k, t in enumerate(self.group_tiles[g]) if t and self.zc_seq[g][k] is not None]
                for k, t in enumerate(self.group_tiles[g]):
                    if t and self.zc_seq[g][k] is None:
                        self._launch_job(g, k, mode, flag, max_pts, sp)
                if capped:
                    self._launch_capped(g, capped, mode, flag, max_pts, sp)
                continue
            _native.check(lib.msurf_sweep(base + job_off, len(idx), base + pre_off, n_tiles, mode | flag,
                                          max_pts, self.sweep_scratch.data_ptr(), sp))

    def _sweep_flag(self) -> int:
        if self.diagnostics == "trace":
            return _native.SWEEP_TRACE
        return _native.SWEEP_DIAG if self.diagnostics else 0

    def red_lines(self, cap_bytes: int = 24 << 30):
        """Roofline helper (bench.py; not on the product path): trace every
        RED.MIN of one sweep of this batch (MSURF_SWEEP_TRACE launch, one
        record of 32 key offsets per warp-wide RED) and histogram the records
        by the number of distinct 128-byte lines each touches
        (msurf_red_sectors). Returns {"hist": [33 counts], "hist_sectors": [33
        counts, by distinct 32-byte sectors], "records",
        "records_issued", "lanes" (active lanes = RED.MIN of the production
        sweep, all records), "truncated"}; a truncated trace (above
        ``cap_bytes``) histograms the first records in issue order. None when
        the surfaces' keys do not share one buffer."""
        torch, lib = self.torch, self.lib
        if self.strip_keys is not None and any(s.n_strips == 1 for s in self.surfs):
            return None
        base = self.strip_keys if self.strip_keys is not None else self.keys
        free, _ = torch.cuda.mem_get_info(self.dev)
        cap = int(min(cap_bytes, free // 2)) // 128
        trace = torch.empty(max(cap, 1) * 32, dtype=torch.int32, device=self.dev)
        ctr = torch.zeros(2, dtype=torch.int64, device=self.dev)
        hist = torch.zeros(66, dtype=torch.int64, device=self.dev)  # lines [0, 33), sectors [33, 66)
        _native.check(lib.msurf_trace_arm(trace.data_ptr(), cap, ctr.data_ptr(), base.data_ptr()))
        prev, self.diagnostics = self.diagnostics, "trace"
        try:
            self.launch()
        finally:
            self.diagnostics = prev
        torch.cuda.synchronize(self.dev)
        issued, lanes = (int(v) for v in ctr.cpu())
        n_rec = min(issued, cap)
        _native.check(lib.msurf_red_sectors(trace.data_ptr(), n_rec, hist.data_ptr(), hist.data_ptr() + 33 * 8,
                                            _native.stream_ptr()))
        h = [int(v) for v in hist.cpu()]
        del trace
        torch.cuda.empty_cache()
        return {"hist": h[:33], "hist_sectors": h[33:], "records": n_rec, "records_issued": issued, "lanes": lanes,
                "truncated": issued > cap}

    def launch_decode(self, sp: int) -> None:
        """Keys -> fp64 heights in place, machined-cell counts."""
        lib, base, keys_ptr = self.lib, self.base, self.keys.data_ptr()
        if self.batched_fill:
            _native.check(lib.msurf_decode(keys_ptr, self.surfs[0].nodes, self.n, base + self.sentinel_off,
                                           base + self.machined_off, sp))
        else:
            for i, s in enumerate(self.surfs):
                if s.n_strips > 1:
                    _native.check(lib.msurf_decode_strips(
                        self.strip_keys.data_ptr() + s.strip_off * 8, keys_ptr + s.key_off * 8, s.plan.grid.m + 1,
                        s.j_hi - s.j_lo + 1, s.n_strips, base + self.offs[i]["col0"],
                        base + self.sentinel_off + 8 * i, base + self.machined_off + 8 * i, sp))
                    continue
                _native.check(lib.msurf_decode(keys_ptr + s.key_off * 8, s.nodes, 1,
                                               base + self.sentinel_off + 8 * i,
                                               base + self.machined_off + 8 * i, sp))

    def launch(self, stream=None, events=None):
        """Enqueue fill -> sweep(s) -> decode on ``stream`` (default: the
        current stream; async). ``events`` = (start, after_fill, after_sweep,
        end) CUDA events, optional, recorded on the same stream."""
        sp = _native.stream_ptr(stream)
        ev = events if events else (None, None, None, None)
        if stream is None and any(e is not None for e in ev):
            # the stream object once, by explicit device (Event.record() with no
            # stream resolves the current device through torch's availability
            # checks on every call)
            stream = self.torch.cuda.current_stream(self.dev)

        def mark(e):
            if e is not None:
                e.record(stream)

        mark(ev[0])
        self.launch_fill(sp)
        mark(ev[1])
        self.launch_sweep(sp)
        mark(ev[2])
        self.launch_decode(sp)
        mark(ev[3])

    def pipelined_strips(self) -> bool:
        """ONE strip-layout surface whose sub-strips are swept job by job: each
        strip can be decoded, and its heights copied out, as soon as its own
        sweep is done (launch_by_strip)."""
        return (self.n == 1 and self.surfs[0].n_strips > 1 and len(self.group_meta) == 1
                and self.group_per_job[0])

    def launch_by_strip(self, strip_done, events=None):
        """Same work and results as launch(), ordered strip by strip on the
        current stream: fill, then per sub-strip q its sweep job and its
        decode (msurf_decode_strips over that strip alone), then
        ``strip_done(q, c0, w, r0, r1, stream)`` (node rows [r0, r1) of
        columns [c0, c0 + w) are final once the raw ``stream``'s work so far
        is done: the caller enqueues their D2H, which then overlaps the later
        sweeps). Surface-cap strips run side by side; with PROGRESSIVE_PASSES
        their last passes are launched one call each and the rows no later
        pass can reach are released after each. ``events`` = (start, -, -, end)."""
        if not self.pipelined_strips():
            raise ConfigError("launch_by_strip needs one strip-layout surface with per-job sweeps")
        lib, base = self.lib, self.base
        sp = _native.stream_ptr()
        ev = events if events else (None, None, None, None)
        s, i = self.surfs[0], 0
        cs = self.torch.cuda.current_stream(self.dev)
        if ev[0] is not None:
            ev[0].record(cs)
        self.launch_fill(sp)
        mode, jidx, _, _, _, max_pts = self.group_meta[0]
        flag = self._sweep_flag()
        ptr, sz = self.group_host_jobs[0].ctypes.data, _native.JOB_DTYPE.itemsize
        by_lo = {}
        for k, jn in enumerate(jidx):
            by_lo.setdefault(self.jobs[jn][1], []).append(k)
        rows, w_all = s.plan.grid.m + 1, s.j_hi - s.j_lo + 1
        covered = sum(len(by_lo.get(s.j_lo + s.col0[q], ())) for q in range(s.n_strips))
        if covered != len(jidx):
            raise ConfigError(f"launch_by_strip: {len(jidx) - covered} sweep jobs start at no strip boundary")
        # surface-cap jobs run side by side (one joined call) before the strip loop:
        # their decodes and copies then follow, no longer overlapping the sweep
        capped = [k for k, t in enumerate(self.group_tiles[0]) if t and self.zc_seq[0][k] is not None]
        anchor_of = {}
        done_rows = [0] * s.n_strips
        strip_of = {k: q for q in range(s.n_strips) for k in by_lo.get(s.j_lo + s.col0[q], ())}

        def release(q, r1, stream):
            # decode node rows [done, r1) of strip q on `stream`, then hand them out
            r0 = done_rows[q]
            if r1 <= r0:
                return
            c0, w = s.col0[q], s.col0[q + 1] - s.col0[q]
            _native.check(lib.msurf_decode_strips(
                self.strip_keys.data_ptr() + (s.strip_off + rows * c0 + r0 * w) * 8,
                self.keys.data_ptr() + (s.key_off + r0 * w_all + c0) * 8, r1 - r0, w_all, 1,
                base + self.offs[i]["strip_w"] + 16 * q, base + self.sentinel_off + 8 * i,
                base + self.machined_off + 8 * i, stream))
            done_rows[q] = r1
            strip_done(q, c0, w, r0, r1, stream)

        if capped:
            # side by side, in strip order of stream priority; each strip's decode
            # and copy-out waits for that strip's own jobs only
            n_pass = s.plan.passes
            k_prog = min(PROGRESSIVE_PASSES, n_pass - 1)
            cuts = [0] + ([n_pass - k_prog + t for t in range(k_prog)] if k_prog > 0 else []) + [n_pass]
            anchors = None
            for c in range(len(cuts) - 1):
                p0, p1 = cuts[c], cuts[c + 1]
                anchors = self._launch_capped(0, capped, mode, flag, max_pts, sp, split=True,
                                              passes=(p0, p1) if len(cuts) > 2 else None, anchors=anchors)
                if p1 < n_pass:
                    r_fin = self._final_rows(s, p1)
                    for k, a in zip(capped, anchors):
                        release(strip_of[k], r_fin, a)
            anchor_of = dict(zip(capped, anchors))
        for q in range(s.n_strips):
            for k in by_lo.get(s.j_lo + s.col0[q], ()):
                if k in anchor_of:
                    _native.check(lib.msurf_stream_wait(sp, anchor_of[k]))
                elif self.group_tiles[0][k]:
                    self._launch_job(0, k, mode, flag, max_pts, sp)
            release(q, rows, sp)
        if ev[3] is not None:
            ev[3].record(cs)

    def _final_rows(self, s, p_next: int) -> int:
        return final_rows(s.plan, p_next)

    def heights(self):
        """fp64 views (valid after a launch) — one per surface."""
        h = self.keys.view(self.torch.float64)
        total = self.surfs[-1].key_off + self.surfs[-1].nodes
        # surfaces sit back to back: one split call instead of n slices
        return list(h[:total].split([s.nodes for s in self.surfs]))

    def sentinels_device(self):
        return self.buf[self.sentinel_off: self.sentinel_off + 8 * self.n].view(self.torch.float64)

    def counters(self):
        """(counters [n,4], machined [n]) on the host (synchronises)."""
        u64 = self.buf[self.ctr_off: self.ctr_off + self.n * (_native.NUM_CTRS + 1) * 8].view(self.torch.int64)
        a = _native.readback(u64)
        return a[: self.n * _native.NUM_CTRS].reshape(self.n, _native.NUM_CTRS), a[self.n * _native.NUM_CTRS:]

    def trajectories(self):
        out = []
        for s, r, o in zip(self.surfs, self.need_traj, self.traj_off):
            out.append(self.traj[o: o + s.plan.steps * s.plan.teeth * 3] if r else None)
        return out


def sweep_plans(surfaces, trig: str = "device", device=None, diagnostics: bool = True):
    """One-shot: upload, launch, collect. Returns (heights views, counters,
    machined, device_ms, trajectories, batch)."""
    torch = _native.require_cuda()
    b = SweepBatch(surfaces, trig=trig, device=device, diagnostics=diagnostics)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    b.launch(events=ev)
    small, machined = b.counters()
    return b.heights(), small, machined, ev[0].elapsed_time(ev[3]), b.trajectories(), b


def _counters_dict(row, diagnostics: bool = True) -> dict:
    """Sweep counters; deposits/atomics are None unless the launch counted
    them (``diagnostics=True``)."""
    return {"live_rows": int(row[0]), "points_evaluated": int(row[1]),
            "deposits": int(row[2]) if diagnostics else None,
            "atomics": int(row[3]) if diagnostics else None, "engaged_rows": int(row[4])}


def _build_trajectory(p: SweepPlan, traj_dev) -> TrajectoryRecord:
    xyz = traj_dev.cpu().numpy().reshape(p.steps * p.teeth, 3)
    rec = TrajectoryRecord(p.steps * p.teeth)
    t = p.t_start + np.arange(p.steps, dtype=np.float64) * p.dt   # engine.py:240
    rec.extend_block(np.repeat(t, p.teeth), np.tile(np.arange(1, p.teeth + 1, dtype=np.int64), p.steps),
                     xyz[:, 0].copy(), xyz[:, 1].copy(), xyz[:, 2].copy())
    return rec


def simulate(config: SimulationConfig, extensions: Extensions | None = None, *,
             trig: str = "device", diagnostics: bool = False) -> SimulationResult:
    """GPU FSM sweep with the reference's contract (engine.py:316-357).

    ``extensions`` selects the extended kinematics (extensions.py).
    ``trig='host'`` takes the per-(step, tooth) cos/sin from the host libm
    (exactly the reference's values) instead of the device's correctly
    rounded double-double sincos — the parity mode. ``diagnostics=True``
    also counts deposits and atomics (``result.counters``)."""
    p = plan(config, extensions)
    # the reference returns host heights: their D2H starts right after the
    # sweep and overlaps the caller's next launches (areal_metrics etc. run
    # on the device copy)
    return _launch_results([p], trig, diagnostics, prefetch=True)[0]


class _Inflight:
    """Pinned host buffers that raw strip D2H copies (msurf_copy2d_d2h, not
    visible to torch's pinned-memory cache) may still be writing: an entry is
    registered BEFORE its first copy is enqueued and released only once its
    completion event has been recorded and has passed, so the buffer cannot
    be recycled under a running DMA even if every field is dropped or the
    launch raises partway. Pruned on every launch; guarded by a lock."""

    _lock = threading.Lock()
    _entries = []  # [event | None, buffer]; event None = copies still being enqueued

    @classmethod
    def register(cls, buf):
        ent = [None, buf]
        with cls._lock:
            cls._prune_locked()
            cls._entries.append(ent)
        return ent

    @classmethod
    def seal(cls, ent, event):
        with cls._lock:
            ent[0] = event

    @classmethod
    def prune(cls):
        with cls._lock:
            cls._prune_locked()

    @classmethod
    def _prune_locked(cls):
        cls._entries[:] = [e for e in cls._entries if e[0] is None or not e[0].query()]
_EVENT_POOL = {}  # device index -> timing events of released launches (cudaEventCreate costs ~10 us)


def _take_events(torch, dev, n):
    pool = _EVENT_POOL.setdefault(dev.index, [])
    out = []
    while len(out) < n:
        try:
            out.append(pool.pop())  # atomic under the GIL; another thread may empty the pool first
        except IndexError:
            out.append(torch.cuda.Event(enable_timing=True))
    return out


def _give_events(dev_index, events):
    pool = _EVENT_POOL.get(dev_index)
    if pool is not None and len(pool) < 64:
        pool.extend(e for e in events if e is not None)


def _launch_results(plans, trig, diagnostics=False, prefetch=False):
    """Upload, launch asynchronously, wrap the fields (no host sync unless a
    trajectory record is requested). ``prefetch``: one D2H copy of the whole
    group's heights into one pinned buffer on a side stream, started right
    after the decode; each field's ``heights`` then only waits for it."""
    torch = _native.require_cuda()
    _Inflight.prune()
    b = SweepBatch([(p, 0, p.grid.n) for p in plans], trig=trig, diagnostics=diagnostics)
    # e0/e3 time the launch (main_loop_seconds) and are pooled; the prefetch's
    # event is fresh: the fields keep it after the launch object is released
    e0, e3 = _take_events(torch, b.dev, 2)
    ev = [e0, None, None, e3]
    host = None
    if prefetch and b.pipelined_strips():
        # a map above the L2 budget: each sub-strip's heights start crossing
        # PCIe (2-D copy into the row-major pinned map) as soon as that strip
        # is decoded, overlapping the sweeps of the later strips
        from .grid import _copy_stream

        side = _copy_stream(torch, b.dev)
        sptr = int(side.cuda_stream)
        host = torch.empty(b.keys.shape, dtype=torch.float64, pin_memory=True)
        s0 = b.surfs[0]
        pitch = (s0.j_hi - s0.j_lo + 1) * 8
        hp, dp, rows = host.data_ptr() + s0.key_off * 8, b.keys.data_ptr() + s0.key_off * 8, s0.plan.grid.m + 1

        def strip_done(q, c0, w, r0, r1, stream):
            _native.check(b.lib.msurf_stream_wait(sptr, stream))
            off = r0 * pitch + c0 * 8
            _native.check(b.lib.msurf_copy2d_d2h(hp + off, pitch, dp + off, pitch, w * 8, r1 - r0, sptr))

        # the raw 2-D copies are invisible to torch's pinned-memory cache: the
        # buffer stays referenced until they finish, even if every field is
        # dropped or a launch below raises after some copies were enqueued
        ent = _Inflight.register(host)
        done = torch.cuda.Event()
        try:
            b.launch_by_strip(strip_done, events=ev)
        finally:
            done.record(side)
            _Inflight.seal(ent, done)
        b.keys.record_stream(side)
        prefetch = False  # copies already enqueued
    else:
        b.launch(events=ev)
    lk = _Launch(b, ev)
    views, trajs = b.heights(), b.trajectories()
    sents = b.sentinels_device()
    if prefetch:
        from .grid import _copy_stream

        side = _copy_stream(torch, b.dev)
        side.wait_event(e3)  # e3 closes the decode on the launch stream
        host = torch.empty(b.keys.shape, dtype=torch.float64, pin_memory=True)
        with torch.cuda.stream(side):
            host.copy_(b.keys.view(torch.float64), non_blocking=True)
            done = torch.cuda.Event()
            done.record(side)
        b.keys.record_stream(side)
    out = []
    sent1 = sents.split(1)
    hosts = host[:views[-1].numel() + b.surfs[-1].key_off].split([s.nodes for s in b.surfs]) \
        if host is not None else None
    for i, (p, v, tr) in enumerate(zip(plans, views, trajs)):
        f = HeightField(p.grid, p.initial_height, device=v)
        f._dev_sentinel = sent1[i]
        if hosts is not None:
            f._set_prefetch(hosts[i], done)
        out.append(SimulationResult(field=f, trajectory=_build_trajectory(p, tr) if p.record else None,
                                    time_steps=p.steps, trajectory_points=p.trajectory_points,
                                    launch=lk, index=i, share=1.0 / len(plans)))
    return out


def simulate_batch(configs, extensions=None, *, trig: str = "device", diagnostics: bool = False,
                   chunk: int | None = None, prefetch: bool = True):
    """Batched mode: many parameter sets swept in the same kernel launches.
    ``extensions`` is None, one Extensions, or a list aligned with configs.

    Large batches run as a software pipeline of launch groups of ``chunk``
    sets (default: about 64 sets or 6e7 Z-map nodes): host planning of group
    k+1 overlaps the sweep of group k on the GPU, and each group's heights
    start streaming to pinned host memory (``prefetch``) as soon as its
    sweep is done, overlapping the later sweeps. Every group is one fill, one
    sweep per kinematics mode and one decode launch."""
    if isinstance(extensions, (list, tuple)):
        exts = list(extensions)
        if len(exts) != len(configs):
            raise ConfigError("extensions list must align with configs")
    else:
        exts = [extensions] * len(configs)
    if not configs:
        return []
    if chunk is None:
        chunk = BATCH_CHUNK if len(configs) >= 128 else max(4, -(-len(configs) // 4))
    first = min(chunk, PIPELINE_FIRST_CHUNK) if PIPELINE_FIRST_CHUNK > 0 else chunk
    bounds = [(0, min(len(configs), first))]
    bounds += [(lo, min(len(configs), lo + chunk)) for lo in range(bounds[0][1], len(configs), chunk)]
    if len(bounds) == 1:
        return _launch_results(plan_many(configs, exts), trig, diagnostics, prefetch)
    # launch groups are planned concurrently on host threads (one vectorised
    # plan per group) and launched in order as soon as each is ready, so the
    # GPU starts on group 0 while the host still plans the rest
    from concurrent.futures import ThreadPoolExecutor

    from .planner import PLAN_THREADS

    out = []
    # group 0 is planned right here with nothing else running (the GPU and the
    # heights' D2H start as early as possible); the rest are planned on worker
    # threads while the main thread launches, and launched in order
    first_plans = plan_many(configs[bounds[0][0]:bounds[0][1]], exts[bounds[0][0]:bounds[0][1]],
                            PIPELINE_FIRST_THREADS, PIPELINE_NATIVE_THREADS)
    with ThreadPoolExecutor(max_workers=min(PIPELINE_PLAN_THREADS, PLAN_THREADS, len(bounds) - 1)) as pool:
        futs = [pool.submit(plan_many, configs[lo:hi], exts[lo:hi], 1, PIPELINE_NATIVE_THREADS)
                for lo, hi in bounds[1:]]
        out.extend(_launch_results(first_plans, trig, diagnostics, prefetch))
        for f in futs:
            out.extend(_launch_results(f.result(), trig, diagnostics, prefetch))
    return out


def simulate_reference(config: SimulationConfig, extensions: Extensions | None = None, *,
                       diagnostics: bool = False) -> SimulationResult:
    """The reference's 'naive' kernel is its oracle (engine.py:360-406). On the
    GPU the same sweep runs in parity mode: trig from the host libm, so every
    input the reference rounds is bit-identical by construction."""
    return simulate(config, extensions, trig="host", diagnostics=diagnostics)


@dataclass(frozen=True)
class BenchmarkRow:
    scale: float
    trajectory_points: int
    t_reference_s: float
    t_optimized_s: float
    speedup: float


@dataclass
class BenchmarkReport:
    case_id: str
    rows: list = field(default_factory=list)

    def to_json_dict(self) -> dict:
        return {"case_id": self.case_id,
                "rows": [{"scale": r.scale, "trajectory_points": r.trajectory_points,
                          "t_reference_s": r.t_reference_s, "t_optimized_s": r.t_optimized_s,
                          "speedup": r.speedup} for r in self.rows]}

    def to_text(self) -> str:
        header = f"{'scale':>8} {'trajectory_points':>18} {'t_reference_s':>14} {'t_optimized_s':>14} {'speedup':>9}"
        lines = [f"case: {self.case_id}", header, "-" * len(header)]
        for r in self.rows:
            lines.append(f"{r.scale:>8g} {r.trajectory_points:>18d} {r.t_reference_s:>14.4f} "
                         f"{r.t_optimized_s:>14.4f} {r.speedup:>9.1f}")
        return "\n".join(lines)


def run_benchmark(config: SimulationConfig, sizes, case_id: str = "benchmark") -> BenchmarkReport:
    """engine.py:449-485 shape: per size multiplier, parity-mode run vs device-
    trig run, fields must agree exactly (a mismatch aborts)."""
    if not sizes:
        raise ConfigError("benchmark sizes must be non-empty")
    base_dt = time_step(config)
    rep = BenchmarkReport(case_id=case_id)
    for size in sizes:
        if size <= 0:
            raise ConfigError(f"benchmark size must be > 0, got {size}")
        scaled = replace(config, time_step_s=base_dt / size)
        opt = simulate(scaled)
        ref = simulate_reference(scaled)
        if not np.array_equal(opt.field.heights, ref.field.heights):
            raise MillsurfError(f"kernel mismatch at size {size}: device-trig and host-trig fields differ")
        rep.rows.append(BenchmarkRow(scale=size, trajectory_points=opt.trajectory_points,
                                     t_reference_s=ref.main_loop_seconds, t_optimized_s=opt.main_loop_seconds,
                                     speedup=ref.main_loop_seconds / opt.main_loop_seconds
                                     if opt.main_loop_seconds > 0 else math.inf))
    return rep
