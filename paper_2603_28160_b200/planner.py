"""Host-side sweep planning: SimulationConfig (+ Extensions) -> device arrays.

Restates the reference planner (engine.py:134-212, ``_plan``) for the
reference kinematics, and states the extended model (extensions.py) for the
rest. Everything here is O(teeth x edge points) NumPy on the host, done once
per surface; the O(steps x teeth x points) work runs on the GPU. Evaluation
order matches the reference expression by expression, so the device sweep
reproduces the reference's heights bit-for-bit.
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass, field

import numpy as np

from .errors import ConfigError, DomainError
from .extensions import Extensions
from .geometry import default_point_count, edge_coordinates, effective_half_length
from .kinematics import edge_to_tool_rows, tooth_base_angle

MODE_REF, MODE_EXT, MODE_EXT_TILT = 0, 1, 2
# planning arrays from libmsurf's native planner (msurf_plan.cpp, bitwise equal
# to the NumPy statement below, which stays the specification and is used when
# MSURF_NATIVE_PLAN=0; tests/test_native_plan_cpu.py compares the two)
NATIVE_PLAN = __import__("os").environ.get("MSURF_NATIVE_PLAN", "1") == "1"
CHUNK = 32  # edge points per warp
MAX_POINTS = 64 * 64 * 32  # mask words are bounded by the CTA's shared memory


def encode_keys(z: np.ndarray) -> np.ndarray:
    """Order-preserving fp64 -> u64 keys (the device's enc_key): -0 -> +0,
    negative values bit-inverted, non-negative ones with the sign bit set."""
    z = np.ascontiguousarray(z, dtype=np.float64) + 0.0
    b = z.view(np.uint64)
    neg = (b >> np.uint64(63)).astype(bool)
    return np.where(neg, ~b, b | np.uint64(1 << 63))


def decode_keys(k: np.ndarray) -> np.ndarray:
    k = np.ascontiguousarray(k, dtype=np.uint64)
    pos = (k >> np.uint64(63)).astype(bool)
    b = np.where(pos, k & np.uint64(0x7FFFFFFFFFFFFFFF), ~k)
    return b.view(np.float64)


def time_step(config) -> float:
    """Resolved dt: explicit, else min(step-angle guard, one-cell feed guard)
    (engine.py:86-98)."""
    if config.time_step_s is not None:
        if config.time_step_s <= 0:
            raise ConfigError(f"time_step_s must be > 0, got {config.time_step_s}")
        return config.time_step_s
    if config.max_step_angle_rad <= 0:
        raise ConfigError(f"max_step_angle_rad must be > 0, got {config.max_step_angle_rad}")
    by_angle = config.max_step_angle_rad / config.process.angular_velocity_rad_s
    by_feed = config.grid.spacing_mm / config.process.feed_speed_mm_s
    return min(by_angle, by_feed)


@dataclass
class SweepPlan:
    mode: int
    grid: object
    teeth: int
    points: int
    steps: int
    dt: float
    t_start: float
    x0: float
    y0: float
    z0: float
    feed_speed: float
    omega: float
    initial_height: float
    half_length: float
    tooth_base: np.ndarray            # (Z,)
    tooth_rows: np.ndarray            # (Z, 8) REF, zeros otherwise
    px: np.ndarray                    # REF (N,), EXT (Z, N)
    py: np.ndarray
    pz: np.ndarray
    zw: np.ndarray                    # (Z, N) z' (time-invariant unless tilt)
    zkey: np.ndarray                  # (Z, N) u64
    chunk_box: np.ndarray             # (Z, nchunk, 6) tool-frame boxes
    pass_x0: np.ndarray               # (P,)
    min_index: np.ndarray             # (Z,) int32
    tilt_c: float = 1.0
    tilt_s: float = 0.0
    zoff: float = 0.0
    vib_amp: float = 0.0
    vib_omega: float = 0.0
    vib_phase: float = 0.0
    record: bool = False
    pts: np.ndarray | None = None        # (Z, N, 4) device point records (msurf_job.pts)
    chunk_circ: np.ndarray | None = None # (Z, nchunk, 6) device cull records
    tooth_box: np.ndarray | None = None  # (Z, 6) whole-tooth tool-frame boxes
    extras: dict = field(default_factory=dict)
    group: tuple | None = None           # (PlanGroup, index) when planned by plan_many

    @property
    def passes(self) -> int:
        return int(self.pass_x0.shape[0])

    @property
    def trajectory_points(self) -> int:
        """steps x teeth x points x passes (engine.py:129-131)."""
        return self.steps * self.teeth * self.points * self.passes


def _chunk_circles(xt, yt, zt, tilt_c: float, tilt_s: float) -> np.ndarray:
    """Per tooth and 32-point chunk the device's cull record
    (xc, yc, rx, ry, yz, 0): tool-frame centre, the radius bounding the
    chunk's workpiece x-extent at any rotation, the radius of its y-extent
    after the lead tilt, and the tilt's z offset -sin(tau)*zc. A rotation by
    theta maps the chunk into x = c*xc + s*yc +- rx (+ x offset) and
    y = cos(tau)*(c*yc - s*xc) + yz +- ry (+ feed), which the kernel tests
    against the owned window widened by 1.5 cells (conservative)."""
    z_n, n = xt.shape
    nchunk = (n + CHUNK - 1) // CHUNK
    pad = nchunk * CHUNK - n
    def blk(a):
        full = np.concatenate([a, np.repeat(a[:, -1:], pad, axis=1)], axis=1) if pad else a
        return full.reshape(z_n, nchunk, CHUNK)
    bx, by, bz = blk(xt), blk(yt), blk(zt)
    xc = 0.5 * (bx.min(2) + bx.max(2))
    yc = 0.5 * (by.min(2) + by.max(2))
    zc = 0.5 * (bz.min(2) + bz.max(2))
    zr = 0.5 * (bz.max(2) - bz.min(2))
    rho = np.sqrt(((bx - xc[:, :, None]) ** 2 + (by - yc[:, :, None]) ** 2).max(2))
    rho = rho * (1.0 + 1e-12) + 1e-12
    out = np.zeros((z_n, nchunk, 6))
    out[:, :, 0], out[:, :, 1], out[:, :, 2] = xc, yc, rho
    out[:, :, 3] = tilt_c * rho + abs(tilt_s) * (zr * (1.0 + 1e-12) + 1e-12)
    out[:, :, 4] = -tilt_s * zc
    return out


def _chunk_boxes(xt: np.ndarray, yt: np.ndarray, zt: np.ndarray) -> np.ndarray:
    """Per tooth and 32-point chunk, tool-frame [xlo, xhi, ylo, yhi, zlo, zhi]."""
    z_n, n = xt.shape
    nchunk = (n + CHUNK - 1) // CHUNK
    pad = nchunk * CHUNK - n
    out = np.empty((z_n, nchunk, 6))
    for a, arr in enumerate((xt, yt, zt)):
        full = np.concatenate([arr, np.repeat(arr[:, -1:], pad, axis=1)], axis=1) if pad else arr
        blk = full.reshape(z_n, nchunk, CHUNK)
        out[:, :, 2 * a] = blk.min(axis=2)
        out[:, :, 2 * a + 1] = blk.max(axis=2)
    return out


def _span(config, margin: float):
    """Auto-span (engine.py:153-162) or explicit span (163-167); steps (170)."""
    grid, proc = config.grid, config.process
    x0, y0, z0 = proc.initial_position_mm
    dt = time_step(config)
    if config.span_s is None:
        y0 = grid.y_min_mm - margin
        t_start = 0.0
        t_end = (grid.y_max_mm + margin - y0) / proc.feed_speed_mm_s
    else:
        t_start, t_end = config.span_s
        if t_start < 0 or t_end <= t_start:
            raise ConfigError(f"span_s must satisfy 0 <= start < end, got {config.span_s}")
        if y0 is None:
            raise ConfigError("initial position y is required when span_s is explicit")
    if z0 is None:
        z0 = 0.0
    steps = int(math.floor((t_end - t_start) / dt)) + 1
    return dt, t_start, steps, x0, y0, z0


def edge_noise(teeth: int, n: int, sigma: float, corr: float, ds: float, seed: int) -> np.ndarray:
    """Per-flute edge-radius perturbation (Extensions.noise_*): white noise
    from default_rng(seed) of shape (teeth, n), smoothed along the edge by a
    Gaussian of std g = corr/(2 ds) samples (truncated at 4g), divided by
    sqrt(sum k^2) and scaled by sigma."""
    rng = np.random.default_rng(seed)
    white = rng.standard_normal((teeth, n))
    g = corr / (2.0 * ds)
    if g < 0.5:
        return sigma * white
    w = int(math.ceil(4.0 * g))
    k = np.exp(-0.5 * (np.arange(-w, w + 1, dtype=np.float64) / g) ** 2)
    norm = math.sqrt(float(np.sum(k * k)))
    out = np.empty((teeth, n))
    for t in range(teeth):
        out[t] = sigma * (np.convolve(white[t], k, mode="same") / norm)
    return out


def plan(config, ext: Extensions | None = None) -> SweepPlan:
    ext = ext or Extensions()
    tool, proc, grid = config.tool, config.process, config.grid
    if proc.depth_of_cut_mm > tool.insert_radius_mm:
        raise ConfigError(f"depth of cut {proc.depth_of_cut_mm} mm exceeds insert radius "
                          f"{tool.insert_radius_mm} mm")
    if getattr(config, "worker_count", 1) < 1:
        raise ConfigError(f"worker_count must be >= 1, got {config.worker_count}")
    passes = int(ext.passes)
    if ext.kinematic:
        p = _plan_ext(config, ext)
    else:
        p = _plan_ref(config)
    p.pass_x0 = np.array([p.x0 + k * ext.stepover_mm for k in range(passes)], dtype=np.float64)
    p.record = bool(getattr(config, "record_trajectory", False))
    if p.record and p.mode != MODE_REF:
        raise ConfigError("record_trajectory is defined for the reference kinematics only")
    _pack(p)
    _check_device_limits(p, grid)
    return p


def tilt_z_term(tilt_c, zt, zoff):
    """cos(tau)*zt + zoff, two roundings, canonical +0 (the fused tilt model's
    per-point constant: z' = fma(sin(tau), v, this))."""
    return (tilt_c * zt + zoff) + 0.0


def _pack_records(p: SweepPlan) -> None:
    """Per-(tooth, point) 32-byte records the device reads with one broadcast
    load per point (include/msurf.h msurf_job.pts)."""
    z_n, n = p.teeth, p.points
    rec = np.zeros((z_n, n, 4))
    kf = p.zkey.view(np.float64)
    if p.mode == MODE_REF:
        rec[:, :, 0] = p.px[None, :]
        rec[:, :, 1] = p.py[None, :]
        rec[:, :, 2] = p.pz[None, :]
        rec[:, :, 3] = kf
    elif p.mode == MODE_EXT:
        rec[:, :, 0], rec[:, :, 1], rec[:, :, 2] = p.px, p.py, kf
    else:
        # time-invariant parts of the fused tilt model:
        # sin(tau)*zt, and cos(tau)*zt + zoff (+0.0: never -0)
        rec[:, :, 0], rec[:, :, 1] = p.px, p.py
        rec[:, :, 2] = p.tilt_s * p.pz
        rec[:, :, 3] = tilt_z_term(p.tilt_c, p.pz, p.zoff)
    p.pts = rec


def _pack(p: SweepPlan) -> None:
    """Device records, bounding circles and whole-tooth boxes."""
    if p.pts is not None and p.chunk_circ is not None and p.tooth_box is not None:
        return  # the native planner produced them
    _pack_records(p)
    if p.mode == MODE_REF:
        xt = (p.tooth_rows[:, 0:1] * p.px[None, :] + p.tooth_rows[:, 1:2] * p.py[None, :]) \
            + p.tooth_rows[:, 2:3] * p.pz[None, :] + p.tooth_rows[:, 3:4]
        yt = (p.tooth_rows[:, 4:5] * p.px[None, :] + p.tooth_rows[:, 5:6] * p.py[None, :]) \
            + p.tooth_rows[:, 6:7] * p.pz[None, :] + p.tooth_rows[:, 7:8]
        p.chunk_circ = _chunk_circles(xt, yt, p.zw, 1.0, 0.0)
    else:
        p.chunk_circ = _chunk_circles(p.px, p.py, p.pz, p.tilt_c, p.tilt_s)
    b = p.chunk_box
    p.tooth_box = np.stack([b[:, :, 0].min(1), b[:, :, 1].max(1), b[:, :, 2].min(1), b[:, :, 3].max(1),
                            b[:, :, 4].min(1), b[:, :, 5].max(1)], axis=1)


def chunk_f32(chunk_circ: np.ndarray, tooth_box: np.ndarray, zfloor: np.ndarray | None = None) -> np.ndarray:
    """fp32 phase-1 cull records (msurf_job.chunk_f32): per tooth and chunk
    (xc, yc, rx, ry, yz, Rt, zfloor, zmargin), Rt = max|x| + max|y| + max|z| of
    the tooth box, zfloor = chunk_zfloor (0 when not given). The kernel widens
    its fp32 tests by 4e-6 (Rt + |offset|) + 1e-6 mm, which covers the fp32
    roundings of every term; for the z tests that margin,
    4e-6 (Rt + |zfloor|) + 1e-6, is precomputed here in fp64 and rounded up to
    fp32 (zmargin). Leading (set) axes are allowed: (..., Z, nchunk, 6) and
    (..., Z, 6)."""
    out = np.zeros(chunk_circ.shape[:-1] + (8,), dtype=np.float32)
    out[..., :5] = chunk_circ[..., :5]
    b = np.abs(tooth_box)
    rt = (np.maximum(b[..., 0], b[..., 1]) + np.maximum(b[..., 2], b[..., 3])
          + np.maximum(b[..., 4], b[..., 5]))
    out[..., 5] = rt[..., None]
    if zfloor is not None:
        out[..., 6] = zfloor
    zf = out[..., 6].astype(np.float64)
    mg = 4e-6 * (out[..., 5].astype(np.float64) + np.abs(zf)) + 1e-6
    m32 = mg.astype(np.float32)
    out[..., 7] = np.where(m32.astype(np.float64) < mg, np.nextafter(m32, np.float32(np.inf)), m32)
    return out


def chunk_zfloor(w: np.ndarray, rho: np.ndarray, tilt_s: float, stock) -> np.ndarray:
    """Per tooth and chunk (leading set axes allowed): the lowest workpiece z'
    any point of the chunk can reach at any spindle angle, minus the stock
    height. z' = sin(tau) v + w with w the point's angle-free part (tilt:
    cos(tau) zt + zoff; otherwise z' itself) and |v - v_centre| <= rho, the
    chunk's bounding-circle radius, so z' >= sin(tau) v_centre + zfloor +
    stock. The kernel skips a (step, chunk) whose bound is at or above the
    stock top: such evaluations can never lower a key below the initial
    height (a result-neutral cull)."""
    n = w.shape[-1]
    # per-chunk minima (the last chunk is partial; its padding would repeat the
    # last point, which leaves the minimum unchanged)
    wmin = np.minimum.reduceat(w, np.arange(0, n, CHUNK), axis=-1)
    stock = np.asarray(stock, dtype=np.float64).reshape(np.shape(stock) + (1,) * (wmin.ndim - np.ndim(stock)))
    return wmin - abs(tilt_s) * rho - stock


def plan_zfloor(p) -> np.ndarray:
    """chunk_zfloor of one plan (its records, circles and stock height)."""
    w = p.pts[..., 3] if p.mode == MODE_EXT_TILT else p.zw
    return chunk_zfloor(w, p.chunk_circ[..., 2], p.tilt_s if p.mode == MODE_EXT_TILT else 0.0, p.initial_height)


# msurf_job array fields, in the order SweepBatch packs them
DEVICE_FIELDS = ("tooth_base", "tooth_rows", "pts", "tooth_box", "chunk_circ", "chunk_f32", "pass_x0", "min_index")


class PlanGroup:
    """Device arrays of parameter sets planned together (plan_many): one
    (sets, ...) array per msurf_job field, each set's plan holding views
    ``arrays[name][b]``. SweepBatch packs a run of consecutive sets of one
    group as ONE slice per field instead of one small array per set."""

    __slots__ = ("arrays", "views", "pinned")

    def __init__(self, arrays: dict, pinned: dict | None = None):
        self.arrays = arrays
        self.views = [tuple(arrays[f][b] for f in DEVICE_FIELDS if f != "chunk_f32")
                      for b in range(len(arrays["pts"]))]
        # field -> the page-locked torch tensor (flat uint8) backing arrays[field]
        self.pinned = pinned or {}

    def pinned_sets(self, name: str, b0: int, count: int):
        """The page-locked bytes of sets [b0, b0 + count) of a field, or None
        (then SweepBatch stages the slice like any host array)."""
        t = self.pinned.get(name)
        if t is None:
            return None
        per = self.arrays[name][0].nbytes
        return t[b0 * per: (b0 + count) * per]

    def owns(self, p: "SweepPlan", b: int) -> bool:
        """True while the plan still holds this group's views (a plan whose
        arrays were replaced after planning is packed on its own)."""
        v = self.views[b]
        return (p.tooth_base is v[0] and p.tooth_rows is v[1] and p.pts is v[2] and p.tooth_box is v[3]
                and p.chunk_circ is v[4] and p.pass_x0 is v[5] and p.min_index is v[6])


def _check_device_limits(p: SweepPlan, grid) -> None:
    if p.points > MAX_POINTS:
        raise ConfigError(f"edge_point_count {p.points} exceeds the device limit {MAX_POINTS}")
    # bounds of the device's fast exact cell location (msurf.cu cell_fast):
    # node indices < 2^19 and grid origin within 2^20 cells of the frame origin
    if max(grid.m, grid.n) >= (1 << 19) - 2:
        raise ConfigError("grid axes must have fewer than 2^19 - 2 cells")
    if max(abs(grid.x_min_mm), abs(grid.y_min_mm)) / grid.spacing_mm >= float(1 << 20):
        raise ConfigError("grid origin too far from the workpiece frame origin (> 2^20 cells)")
    if (grid.m + 1) * (grid.n + 1) >= 1 << 31:
        raise ConfigError("grid has too many nodes for one device surface (>= 2^31)")


def reach_y(p: SweepPlan) -> float:
    """Upper bound of |y_w - ty| over every edge point and rotation (feed-
    direction reach of the footprint), from the device cull records."""
    c = p.chunk_circ
    rad = np.sqrt(c[:, :, 0] ** 2 + c[:, :, 1] ** 2)
    return float(np.max(abs(p.tilt_c) * rad + c[:, :, 3] + np.abs(c[:, :, 4]))) + 2.0 * p.grid.spacing_mm


def step_window(p: SweepPlan, j_lo: int, j_hi: int):
    """Steps [s_lo, s_hi) whose footprint can reach node columns [j_lo, j_hi]
    (each strip sweeps only the time steps that meet it).
    Conservative: the kernel's exact 2-D chunk cull still applies inside."""
    g = p.grid
    reach = reach_y(p) + 1.5 * g.spacing_mm
    y_lo = g.y_min_mm + j_lo * g.spacing_mm - reach
    y_hi = g.y_min_mm + j_hi * g.spacing_mm + reach
    t_lo = (y_lo - p.y0) / p.feed_speed
    t_hi = (y_hi - p.y0) / p.feed_speed
    s_lo = math.floor((t_lo - p.t_start) / p.dt) - 2
    s_hi = math.ceil((t_hi - p.t_start) / p.dt) + 3
    return max(0, min(p.steps, s_lo)), max(0, min(p.steps, s_hi))


def _native_arrays(mode, z_n, n, rows12, *, radius, half=0.0, kmax=0.0, profile=0, z0=0.0, tanb_over_r=0.0,
                   tilt_c=1.0, tilt_s=0.0, delta=None, runout_xy=None, zoff_fn=None):
    """Run msurf_plan_geometry + msurf_plan_finish; returns a dict of the plan
    arrays (and the (z_shift, max|zt|) statistics the caller's margin needs)."""
    from . import _native

    lib = _native.lib()
    rows12 = np.ascontiguousarray(rows12, dtype=np.float64)
    g = _native.MsurfGeomIn(mode=mode, teeth=z_n, points=n, profile=profile, radius=radius, half=half, kmax=kmax,
                            tan_beta_over_r=tanb_over_r, tilt_c=tilt_c, tilt_s=tilt_s, z0=z0,
                            rows=rows12.ctypes.data)
    keep = [rows12]
    if delta is not None:
        delta = np.ascontiguousarray(delta, dtype=np.float64)
        keep.append(delta)
        g.delta = delta.ctypes.data
    if runout_xy is not None:
        runout_xy = np.ascontiguousarray(runout_xy, dtype=np.float64)
        keep.append(runout_xy)
        g.runout_xy = runout_xy.ctypes.data
    shape = (n,) if mode == MODE_REF else (z_n, n)
    px, py, pz = np.empty(shape), np.empty(shape), np.empty(shape)
    stats = np.zeros(2)
    gp = ctypes.addressof(g)
    if lib.msurf_plan_geometry(gp, px.ctypes.data, py.ctypes.data, pz.ctypes.data, stats.ctypes.data):
        raise DomainError("native planner rejected the geometry")
    zoff = zoff_fn(float(stats[0]), float(stats[1])) if zoff_fn is not None else 0.0
    nchunk = (n + CHUNK - 1) // CHUNK
    out = dict(px=px, py=py, pz=pz, pts=np.empty((z_n, n, 4)), tooth_box=np.empty((z_n, 6)),
               chunk_circ=np.empty((z_n, nchunk, 6)), chunk_box=np.empty((z_n, nchunk, 6)),
               min_index=np.empty(z_n, dtype=np.int32), zw=np.empty((z_n, n)), zkey=np.empty((z_n, n), np.uint64),
               zoff=zoff)
    if lib.msurf_plan_finish(gp, px.ctypes.data, py.ctypes.data, pz.ctypes.data, zoff, out["pts"].ctypes.data,
                             out["tooth_box"].ctypes.data, out["chunk_circ"].ctypes.data,
                             out["chunk_box"].ctypes.data, out["min_index"].ctypes.data, out["zw"].ctypes.data,
                             out["zkey"].ctypes.data):
        raise DomainError("native planner rejected the geometry")
    return out


def _rows12(e) -> list:
    return [e[0][0], e[0][1], e[0][2], e[0][3], e[1][0], e[1][1], e[1][2], e[1][3],
            e[2][0], e[2][1], e[2][2], e[2][3]]


def _plan_ref(config) -> SweepPlan:
    """engine.py:134-212 restated."""
    tool, proc, grid = config.tool, config.process, config.grid
    half = effective_half_length(tool.insert_radius_mm, proc.depth_of_cut_mm,
                                 proc.feed_per_tooth_mm, tool.radial_rake_rad)
    n = config.edge_point_count
    if n is None:
        n = default_point_count(half, grid.spacing_mm)
    if n < 2:
        raise DomainError(f"point_count must be >= 2, got {n}")
    if half > tool.insert_radius_mm:
        raise DomainError(f"engaged half-length {half:.6g} mm exceeds the insert radius "
                          f"{tool.insert_radius_mm} mm (feed per tooth too large for this insert)")
    margin = tool.cutting_diameter_mm / 2.0 + half                  # engine.py:158
    dt, t_start, steps, x0, y0, z0 = _span(config, margin)
    z_n = tool.tooth_count
    if NATIVE_PLAN:
        es = [edge_to_tool_rows(tool, k) for k in range(1, z_n + 1)]
        a = _native_arrays(MODE_REF, z_n, n, [_rows12(e) for e in es], radius=tool.insert_radius_mm,
                           half=half, z0=z0)
        p = SweepPlan(
            mode=MODE_REF, grid=grid, teeth=z_n, points=n, steps=steps, dt=dt, t_start=t_start,
            x0=x0, y0=y0, z0=z0, feed_speed=proc.feed_speed_mm_s, omega=proc.angular_velocity_rad_s,
            initial_height=z0 + proc.depth_of_cut_mm, half_length=half,
            tooth_base=np.array([tooth_base_angle(proc.phase_rad, k, z_n) for k in range(1, z_n + 1)]),
            tooth_rows=np.array([_rows12(e)[:8] for e in es], dtype=np.float64).reshape(z_n, 8),
            px=a["px"], py=a["py"], pz=a["pz"], zw=a["zw"], zkey=a["zkey"], chunk_box=a["chunk_box"],
            pass_x0=np.array([x0]), min_index=a["min_index"])
        p.pts, p.chunk_circ, p.tooth_box = a["pts"], a["chunk_circ"], a["tooth_box"]
        return p
    xp, yp, zp = edge_coordinates(half, n, tool.insert_radius_mm)
    rows = np.zeros((z_n, 8))
    xt = np.empty((z_n, n))
    yt = np.empty((z_n, n))
    zw = np.empty((z_n, n))
    for k in range(1, z_n + 1):
        e = edge_to_tool_rows(tool, k)
        rows[k - 1] = [e[0][0], e[0][1], e[0][2], e[0][3], e[1][0], e[1][1], e[1][2], e[1][3]]
        tz = e[2][3] + z0                                           # engine.py:181-182
        zw[k - 1] = ((e[2][0] * xp + e[2][1] * yp) + e[2][2] * zp) + tz
        xt[k - 1] = ((e[0][0] * xp + e[0][1] * yp) + e[0][2] * zp) + e[0][3]
        yt[k - 1] = ((e[1][0] * xp + e[1][1] * yp) + e[1][2] * zp) + e[1][3]
    return SweepPlan(
        mode=MODE_REF, grid=grid, teeth=z_n, points=n, steps=steps, dt=dt, t_start=t_start,
        x0=x0, y0=y0, z0=z0, feed_speed=proc.feed_speed_mm_s, omega=proc.angular_velocity_rad_s,
        initial_height=z0 + proc.depth_of_cut_mm, half_length=half,
        tooth_base=np.array([tooth_base_angle(proc.phase_rad, k, z_n) for k in range(1, z_n + 1)]),
        tooth_rows=rows, px=xp, py=yp, pz=zp, zw=zw, zkey=encode_keys(zw),
        chunk_box=_chunk_boxes(xt, yt, zw), pass_x0=np.array([x0]),
        min_index=np.argmin(zw, axis=1).astype(np.int32),
    )


def _plan_ext(config, ext: Extensions) -> SweepPlan:
    """Extended model (extensions.py / DESIGN.md §3)."""
    tool, proc, grid = config.tool, config.process, config.grid
    r = tool.insert_radius_mm
    a_p = proc.depth_of_cut_mm
    tau = ext.tilt_rad
    z_n = tool.tooth_count
    if ext.profile == "insert":
        half = effective_half_length(r, a_p, proc.feed_per_tooth_mm, tool.radial_rake_rad)
        n = config.edge_point_count or default_point_count(half, grid.spacing_mm)
        if n < 2:
            raise DomainError(f"point_count must be >= 2, got {n}")
        arc = 2.0 * r * math.asin(min(1.0, half / r))
        base_margin = tool.cutting_diameter_mm / 2.0 + half
        if not NATIVE_PLAN:
            ex, ey, ez = edge_coordinates(half, n, r)
            nx = ex / r
            nz = -(r - ez) / r
    else:
        n = config.edge_point_count
        if n is None or n < 2:
            raise ConfigError("the ball profile needs edge_point_count >= 2")
        kmax = min(math.pi / 2.0, math.acos((r - a_p) / r) + abs(tau))
        arc = r * kmax
        half = r * math.sin(kmax)
        base_margin = half
        if not NATIVE_PLAN:
            kap = kmax * np.arange(n, dtype=np.float64) / (n - 1)
            kap[-1] = kmax
            nx = np.sin(kap)
            nz = -np.cos(kap)
            ex = r * nx
            ey = np.zeros(n)
            ez = r - r * np.cos(kap)
    sigma = ext.noise_sigma_mm
    if sigma != 0.0:
        delta = edge_noise(z_n, n, sigma, ext.noise_corr_mm, arc / (n - 1), int(ext.noise_seed))
    beta, rho, lam = ext.helix_angle_rad, ext.runout_offset_mm, ext.runout_phase_rad
    if beta != 0.0:
        r_ref = ext.helix_ref_radius_mm
        if r_ref is None:
            r_ref = tool.cutting_diameter_mm / 2.0 if ext.profile == "insert" else r
        tanb_over_r = math.tan(beta) / r_ref
    radial = None if ext.profile == "insert" else 0.0
    if NATIVE_PLAN:
        tilt = tau != 0.0
        tc, ts = math.cos(tau), math.sin(tau)
        amp = ext.vib_amplitude_mm
        offs = None
        if rho != 0.0:
            offs = []
            for k in range(1, z_n + 1):
                ang = lam + (2.0 * math.pi) * (k - 1) / z_n
                offs.append((rho * math.cos(ang), rho * math.sin(ang)))
        span = {}

        def zoff_fn(z_shift, zmax):
            margin = base_margin + (abs(rho) + abs(amp) + 5.0 * abs(sigma) + abs(ts) * zmax)
            span["v"] = _span(config, margin)
            return (span["v"][5] + (z_shift if tilt else 0.0)) + 0.0  # canonical: never -0

        a = _native_arrays(MODE_EXT_TILT if tilt else MODE_EXT, z_n, n,
                           [_rows12(edge_to_tool_rows(tool, k, radial_offset_mm=radial)) for k in range(1, z_n + 1)],
                           radius=r, half=half if ext.profile == "insert" else 0.0,
                           kmax=kmax if ext.profile != "insert" else 0.0,
                           profile=0 if ext.profile == "insert" else 1,
                           tanb_over_r=tanb_over_r if beta != 0.0 else 0.0, tilt_c=tc, tilt_s=ts,
                           delta=delta if sigma != 0.0 else None, runout_xy=offs, zoff_fn=zoff_fn)
        dt, t_start, steps, x0, y0, z0 = span["v"]
        p = SweepPlan(
            mode=MODE_EXT_TILT if tilt else MODE_EXT, grid=grid, teeth=z_n, points=n, steps=steps,
            dt=dt, t_start=t_start, x0=x0, y0=y0, z0=z0, feed_speed=proc.feed_speed_mm_s,
            omega=proc.angular_velocity_rad_s, initial_height=z0 + a_p, half_length=half,
            tooth_base=np.array([tooth_base_angle(proc.phase_rad, k, z_n) for k in range(1, z_n + 1)]),
            tooth_rows=np.zeros((z_n, 8)), px=a["px"], py=a["py"], pz=a["pz"], zw=a["zw"], zkey=a["zkey"],
            chunk_box=a["chunk_box"], pass_x0=np.array([x0]), min_index=a["min_index"],
            tilt_c=tc, tilt_s=ts, zoff=a["zoff"], vib_amp=amp,
            vib_omega=2.0 * math.pi * ext.vib_frequency_hz, vib_phase=ext.vib_phase_rad,
            extras={"base_margin": base_margin})
        p.pts, p.chunk_circ, p.tooth_box = a["pts"], a["chunk_circ"], a["tooth_box"]
        return p
    xt = np.empty((z_n, n))
    yt = np.empty((z_n, n))
    zt = np.empty((z_n, n))
    for k in range(1, z_n + 1):
        if sigma != 0.0:
            px = ex + delta[k - 1] * nx
            pz = ez + delta[k - 1] * nz
        else:
            px, pz = ex, ez
        py = ey
        e = edge_to_tool_rows(tool, k, radial_offset_mm=radial)
        qx = ((e[0][0] * px + e[0][1] * py) + e[0][2] * pz) + e[0][3]
        qy = ((e[1][0] * px + e[1][1] * py) + e[1][2] * pz) + e[1][3]
        qz = ((e[2][0] * px + e[2][1] * py) + e[2][2] * pz) + e[2][3]
        if beta != 0.0:
            psi = pz * tanb_over_r
            cps, sps = np.cos(psi), np.sin(psi)
            qx, qy = cps * qx + sps * qy, (-sps) * qx + cps * qy
        if rho != 0.0:
            ang = lam + (2.0 * math.pi) * (k - 1) / z_n
            qx = qx + rho * math.cos(ang)
            qy = qy + rho * math.sin(ang)
        xt[k - 1], yt[k - 1], zt[k - 1] = qx, qy, qz
    tilt = tau != 0.0
    tc, ts = math.cos(tau), math.sin(tau)
    z_shift = -float(np.min(tc * zt - abs(ts) * np.sqrt(xt * xt + yt * yt))) if tilt else 0.0
    amp = ext.vib_amplitude_mm
    margin = base_margin + (abs(rho) + abs(amp) + 5.0 * abs(sigma) + abs(ts) * float(np.max(np.abs(zt))))
    dt, t_start, steps, x0, y0, z0 = _span(config, margin)
    zoff = (z0 + z_shift) + 0.0  # canonical: never -0 (the device relies on it)
    zw = zt + zoff
    return SweepPlan(
        mode=MODE_EXT_TILT if tilt else MODE_EXT, grid=grid, teeth=z_n, points=n, steps=steps,
        dt=dt, t_start=t_start, x0=x0, y0=y0, z0=z0, feed_speed=proc.feed_speed_mm_s,
        omega=proc.angular_velocity_rad_s, initial_height=z0 + a_p, half_length=half,
        tooth_base=np.array([tooth_base_angle(proc.phase_rad, k, z_n) for k in range(1, z_n + 1)]),
        tooth_rows=np.zeros((z_n, 8)), px=xt, py=yt, pz=zt, zw=zw, zkey=encode_keys(zw),
        chunk_box=_chunk_boxes(xt, yt, zt), pass_x0=np.array([x0]),
        min_index=np.argmin(zw, axis=1).astype(np.int32),
        tilt_c=tc, tilt_s=ts, zoff=zoff, vib_amp=amp,
        vib_omega=2.0 * math.pi * ext.vib_frequency_hz, vib_phase=ext.vib_phase_rad,
        extras={"base_margin": base_margin},
    )


# ------------------------------------------------------------------ batches
def _ext_group_key(config, ext: Extensions):
    """Everything the extended model's per-point geometry depends on, except
    the per-sample helix angle and tool-axis runout (vectorised below)."""
    tool, proc, grid = config.tool, config.process, config.grid
    half = None
    if ext.profile == "insert":
        half = effective_half_length(tool.insert_radius_mm, proc.depth_of_cut_mm, proc.feed_per_tooth_mm,
                                     tool.radial_rake_rad)
    return (ext.profile, tool.cutting_diameter_mm, tool.insert_radius_mm, tool.tooth_count,
            tool.radial_rake_rad, tool.axial_rake_rad, tool.runouts_mm, proc.depth_of_cut_mm, half,
            config.edge_point_count, grid.spacing_mm, ext.tilt_rad, ext.noise_sigma_mm, ext.noise_corr_mm,
            ext.noise_seed, ext.helix_ref_radius_mm, bool(ext.helix_angle_rad != 0.0),
            bool(ext.runout_offset_mm != 0.0), int(ext.passes))


PLAN_THREADS = max(1, min(8, (__import__("os").cpu_count() or 1)))


_PINNED_OK = []  # [torch or None], decided once per process


def _pinned_empty(shape, dtype=np.float64):
    """(array, backing tensor): an uninitialised array in page-locked host
    memory from torch's caching host allocator when a CUDA device is present
    (decided once per process), else plain (array, None). An allocation
    failure (pinned memory exhausted) also falls back to pageable memory:
    SweepBatch then stages the array like any other."""
    if not _PINNED_OK:
        try:
            import torch

            _PINNED_OK.append(torch if torch.cuda.is_available() else None)
        except ImportError:
            _PINNED_OK.append(None)
    torch = _PINNED_OK[0]
    if torch is not None:
        nbytes = int(np.prod(shape)) * np.dtype(dtype).itemsize
        try:
            t = torch.empty(max(nbytes, 1), dtype=torch.uint8, pin_memory=True)
        except RuntimeError:
            t = None
        if t is not None:
            return t.numpy()[:nbytes].view(dtype).reshape(shape), t
    return np.empty(shape, dtype=dtype), None


def plan_many(configs, exts, threads: int | None = None, native_threads: int = 1):
    """plan() for many parameter sets. Extended-model sets that share their
    edge geometry are planned together with (sets, teeth, points) arrays —
    the same element-wise operations as plan(), so every array is bitwise
    identical to the per-set plan (tests/test_host_cpu.py) — which keeps host
    planning of a 256-set batch in the low milliseconds."""
    exts = [e or Extensions() for e in exts]
    out = [None] * len(configs)
    groups = {}
    for i, (c, e) in enumerate(zip(configs, exts)):
        if e.kinematic and getattr(c, "edge_point_count", None) and not getattr(c, "record_trajectory", False):
            try:
                groups.setdefault(_ext_group_key(c, e), []).append(i)
                continue
            except (ConfigError, DomainError):
                pass
        out[i] = plan(c, e)
    jobs = []
    for idx in groups.values():
        if len(idx) < 4:
            for i in idx:
                out[i] = plan(configs[i], exts[i])
            continue
        # sub-groups planned on host threads (NumPy releases the GIL inside
        # its element-wise kernels); each sub-group is the same vectorised
        # computation, so the arrays stay bitwise equal to per-set plan()
        # the native group planner spreads a group's sets over its own worker
        # pool (GIL released): one Python job per group; the NumPy statement
        # splits groups over Python threads instead
        if NATIVE_PLAN and threads is None:
            nthr, native_threads = 1, max(native_threads, PLAN_THREADS)
        else:
            nthr = PLAN_THREADS if threads is None else max(1, threads)
        step = max(4, -(-len(idx) // nthr))
        jobs.extend(idx[a: a + step] for a in range(0, len(idx), step))
    if jobs:
        def run(sub):
            fn = _plan_ext_group_native if NATIVE_PLAN else _plan_ext_group
            if fn is _plan_ext_group_native:  # native loops over sets on their own threads (GIL released)
                return sub, fn([configs[i] for i in sub], [exts[i] for i in sub], native_threads)
            return sub, fn([configs[i] for i in sub], [exts[i] for i in sub])

        if len(jobs) == 1:
            done = [run(jobs[0])]
        else:
            from concurrent.futures import ThreadPoolExecutor

            with ThreadPoolExecutor(max_workers=min(PLAN_THREADS if threads is None else threads, len(jobs))) as pool:
                done = list(pool.map(run, jobs))
        for sub, plans in done:
            for i, p in zip(sub, plans):
                out[i] = p
    return out


def _plan_ext_group_native(configs, exts, threads: int = 1):
    """_plan_ext for a group of parameter sets sharing their edge geometry:
    per-set scalars on the host, the arrays of every set in two native calls
    (msurf_plan_geometry_many / msurf_plan_finish_many); bitwise equal to
    per-set plan() (tests/test_native_plan_cpu.py)."""
    from . import _native

    lib = _native.lib()
    c0, e0 = configs[0], exts[0]
    tool, proc0 = c0.tool, c0.process
    r = tool.insert_radius_mm
    a_p = proc0.depth_of_cut_mm
    z_n = tool.tooth_count
    B = len(configs)
    tau = e0.tilt_rad
    tilt = tau != 0.0
    tc, ts = math.cos(tau), math.sin(tau)
    if e0.profile == "insert":
        half = effective_half_length(r, a_p, proc0.feed_per_tooth_mm, tool.radial_rake_rad)
        n = c0.edge_point_count or default_point_count(half, c0.grid.spacing_mm)
        if n < 2:
            raise DomainError(f"point_count must be >= 2, got {n}")
        arc = 2.0 * r * math.asin(min(1.0, half / r))
        base_margin = tool.cutting_diameter_mm / 2.0 + half
        kmax = 0.0
    else:
        n = c0.edge_point_count
        if n is None or n < 2:
            raise ConfigError("the ball profile needs edge_point_count >= 2")
        kmax = min(math.pi / 2.0, math.acos((r - a_p) / r) + abs(tau))
        arc = r * kmax
        half = r * math.sin(kmax)
        base_margin = half
    sigma = e0.noise_sigma_mm
    delta = None
    if sigma != 0.0:
        delta = np.ascontiguousarray(edge_noise(z_n, n, sigma, e0.noise_corr_mm, arc / (n - 1), int(e0.noise_seed)))
    radial = None if e0.profile == "insert" else 0.0
    rows = np.ascontiguousarray([_rows12(edge_to_tool_rows(tool, k, radial_offset_mm=radial))
                                 for k in range(1, z_n + 1)], dtype=np.float64)
    r_ref = e0.helix_ref_radius_mm
    if r_ref is None:
        r_ref = tool.cutting_diameter_mm / 2.0 if e0.profile == "insert" else r
    offs = np.zeros((B, z_n, 2))
    mode = MODE_EXT_TILT if tilt else MODE_EXT
    # the B msurf_geom_in records as one structured array (ctypes layout):
    # per-set scalars by columns instead of ~15 ctypes attribute writes per set
    ins = np.zeros(B, dtype=_native.GEOM_IN_DTYPE)
    ins["mode"], ins["teeth"], ins["points"] = mode, z_n, n
    ins["profile"] = 0 if e0.profile == "insert" else 1
    ins["radius"], ins["half"], ins["kmax"] = r, half if e0.profile == "insert" else 0.0, kmax
    ins["tan_beta_over_r"] = [math.tan(e.helix_angle_rad) / r_ref if e.helix_angle_rad != 0.0 else 0.0
                              for e in exts]
    ins["tilt_c"], ins["tilt_s"] = tc, ts
    ins["rows"] = rows.ctypes.data
    ins["delta"] = delta.ctypes.data if delta is not None else 0
    two_pi_k = [(2.0 * math.pi) * (k - 1) / z_n for k in range(1, z_n + 1)]
    base_ptr, stride = offs.ctypes.data, offs.strides[0]
    for b, e in enumerate(exts):
        rho, lam = e.runout_offset_mm, e.runout_phase_rad
        if rho != 0.0:
            for k in range(z_n):
                ang = lam + two_pi_k[k]
                offs[b, k, 0], offs[b, k, 1] = rho * math.cos(ang), rho * math.sin(ang)
            ins["runout_xy"][b] = base_ptr + b * stride
    px, py, pz = np.empty((B, z_n, n)), np.empty((B, z_n, n)), np.empty((B, z_n, n))
    stats = np.zeros((B, 2))
    if lib.msurf_plan_geometry_many(ins.ctypes.data, B, px.ctypes.data, py.ctypes.data, pz.ctypes.data,
                                    stats.ctypes.data, threads):
        raise DomainError("native planner rejected the geometry")
    spans, zoffs = [], np.empty(B)
    for b, (cfg, e) in enumerate(zip(configs, exts)):
        margin = base_margin + (abs(e.runout_offset_mm) + abs(e.vib_amplitude_mm) + 5.0 * abs(sigma)
                                + abs(ts) * float(stats[b, 1]))
        sp = _span(cfg, margin)
        spans.append(sp)
        zoffs[b] = (sp[5] + (float(stats[b, 0]) if tilt else 0.0)) + 0.0
    nchunk = (n + CHUNK - 1) // CHUNK
    # the largest device field (B x teeth x points x 32 B) is written straight
    # into page-locked memory: SweepBatch then copies it to HBM by DMA instead
    # of staging it through a host memmove on the launching thread
    pts, pts_pinned = _pinned_empty((B, z_n, n, 4))
    tbox = np.empty((B, z_n, 6))
    circ = np.empty((B, z_n, nchunk, 6))
    cbox = np.empty((B, z_n, nchunk, 6))
    mins = np.empty((B, z_n), dtype=np.int32)
    zw = np.empty((B, z_n, n))
    zkey = np.empty((B, z_n, n), dtype=np.uint64)
    if lib.msurf_plan_finish_many(ins.ctypes.data, B, px.ctypes.data, py.ctypes.data, pz.ctypes.data, zoffs.ctypes.data,
                                  pts.ctypes.data, tbox.ctypes.data, circ.ctypes.data, cbox.ctypes.data,
                                  mins.ctypes.data, zw.ctypes.data, zkey.ctypes.data, threads):
        raise DomainError("native planner rejected the geometry")
    n_pass = {int(e.passes) for e in exts}
    if len(n_pass) != 1:
        raise DomainError("a plan group needs one pass count")  # _ext_group_key includes it
    n_pass = n_pass.pop()
    tbase = np.array([[tooth_base_angle(cfg.process.phase_rad, k, z_n) for k in range(1, z_n + 1)]
                      for cfg in configs], dtype=np.float64)
    px0 = np.array([[spans[b][3] + k * e.stepover_mm for k in range(n_pass)]
                    for b, e in enumerate(exts)], dtype=np.float64)
    stock = np.array([sp[5] for sp in spans]) + a_p  # initial heights z0 + a_p
    zfl = chunk_zfloor(pts[..., 3] if tilt else zw, circ[..., 2], ts if tilt else 0.0, stock)
    grp = PlanGroup({"tooth_base": tbase, "tooth_rows": np.zeros((B, z_n, 8)), "pts": pts, "tooth_box": tbox,
                     "chunk_circ": circ, "chunk_f32": chunk_f32(circ, tbox, zfl), "pass_x0": px0,
                     "min_index": mins}, pinned={"pts": pts_pinned} if pts_pinned is not None else None)
    plans = []
    for b, (cfg, e) in enumerate(zip(configs, exts)):
        proc, grid = cfg.process, cfg.grid
        dt, t_start, steps, x0, y0, z0 = spans[b]
        v = grp.views[b]
        p = SweepPlan(
            mode=mode, grid=grid, teeth=z_n, points=n, steps=steps, dt=dt, t_start=t_start, x0=x0, y0=y0, z0=z0,
            feed_speed=proc.feed_speed_mm_s, omega=proc.angular_velocity_rad_s, initial_height=z0 + a_p,
            half_length=half, tooth_base=v[0], tooth_rows=v[1], px=px[b], py=py[b], pz=pz[b], zw=zw[b],
            zkey=zkey[b], chunk_box=cbox[b], pass_x0=v[5], min_index=v[6], tilt_c=tc, tilt_s=ts,
            zoff=float(zoffs[b]), vib_amp=e.vib_amplitude_mm, vib_omega=2.0 * math.pi * e.vib_frequency_hz,
            vib_phase=e.vib_phase_rad, extras={"base_margin": base_margin}, pts=v[2], chunk_circ=v[4],
            tooth_box=v[3], group=(grp, b))
        _check_device_limits(p, grid)
        plans.append(p)
    return plans


def _plan_ext_group(configs, exts):
    c0, e0 = configs[0], exts[0]
    # sample-independent part: one per-set plan() restated without helix/runout
    base = _plan_ext(c0, replace_ext(e0, helix_angle_rad=0.0, runout_offset_mm=0.0))
    tool = c0.tool
    z_n, n = base.teeth, base.points
    r = tool.insert_radius_mm
    B = len(configs)
    # rebuild the per-tooth tool-frame points before helix/runout (same ops as _plan_ext)
    if e0.profile == "insert":
        half = base.half_length
        ex, ey, ez = edge_coordinates(half, n, r)
        nx = ex / r
        nz = -(r - ez) / r
        arc = 2.0 * r * math.asin(min(1.0, half / r))
    else:
        kmax = min(math.pi / 2.0, math.acos((r - c0.process.depth_of_cut_mm) / r) + abs(e0.tilt_rad))
        kap = kmax * np.arange(n, dtype=np.float64) / (n - 1)
        kap[-1] = kmax
        nx = np.sin(kap)
        nz = -np.cos(kap)
        ex = r * nx
        ey = np.zeros(n)
        ez = r - r * np.cos(kap)
        arc = r * kmax
    sigma = e0.noise_sigma_mm
    if sigma != 0.0:
        delta = edge_noise(z_n, n, sigma, e0.noise_corr_mm, arc / (n - 1), int(e0.noise_seed))
    radial = None if e0.profile == "insert" else 0.0
    qx0 = np.empty((z_n, n))
    qy0 = np.empty((z_n, n))
    qz0 = np.empty((z_n, n))
    pzs = np.empty((z_n, n))
    for k in range(1, z_n + 1):
        if sigma != 0.0:
            px = ex + delta[k - 1] * nx
            pz = ez + delta[k - 1] * nz
        else:
            px, pz = ex, ez
        e = edge_to_tool_rows(tool, k, radial_offset_mm=radial)
        qx0[k - 1] = ((e[0][0] * px + e[0][1] * ey) + e[0][2] * pz) + e[0][3]
        qy0[k - 1] = ((e[1][0] * px + e[1][1] * ey) + e[1][2] * pz) + e[1][3]
        qz0[k - 1] = ((e[2][0] * px + e[2][1] * ey) + e[2][2] * pz) + e[2][3]
        pzs[k - 1] = pz
    qx = np.broadcast_to(qx0, (B, z_n, n))
    qy = np.broadcast_to(qy0, (B, z_n, n))
    if e0.helix_angle_rad != 0.0:
        r_ref = e0.helix_ref_radius_mm
        if r_ref is None:
            r_ref = tool.cutting_diameter_mm / 2.0 if e0.profile == "insert" else r
        tbr = np.array([math.tan(e.helix_angle_rad) / r_ref for e in exts])
        psi = pzs[None, :, :] * tbr[:, None, None]
        cps, sps = np.cos(psi), np.sin(psi)
        qx, qy = cps * qx + sps * qy, (-sps) * qx + cps * qy
    if e0.runout_offset_mm != 0.0:
        offx = np.empty((B, z_n))
        offy = np.empty((B, z_n))
        for b, e in enumerate(exts):
            for k in range(1, z_n + 1):
                ang = e.runout_phase_rad + (2.0 * math.pi) * (k - 1) / z_n
                offx[b, k - 1] = e.runout_offset_mm * math.cos(ang)
                offy[b, k - 1] = e.runout_offset_mm * math.sin(ang)
        qx = qx + offx[:, :, None]
        qy = qy + offy[:, :, None]
    xt = np.ascontiguousarray(qx)
    yt = np.ascontiguousarray(qy)
    zt = qz0
    tau = e0.tilt_rad
    tilt = tau != 0.0
    tc, ts = math.cos(tau), math.sin(tau)
    zmax = float(np.max(np.abs(zt)))
    if tilt:
        zsh = -np.min((tc * zt[None] - abs(ts) * np.sqrt(xt * xt + yt * yt)).reshape(B, -1), axis=1)
    plans = []
    boxes = _chunk_boxes(xt.reshape(B * z_n, n), yt.reshape(B * z_n, n),
                         np.broadcast_to(zt, (B, z_n, n)).reshape(B * z_n, n)).reshape(B, z_n, -1, 6)
    circs = _chunk_circles(xt.reshape(B * z_n, n), yt.reshape(B * z_n, n),
                           np.broadcast_to(zt, (B, z_n, n)).reshape(B * z_n, n), tc, ts).reshape(B, z_n, -1, 6)
    base_margin = base.extras.get("base_margin")
    tooth_box = np.stack([boxes[..., 0].min(2), boxes[..., 1].max(2), boxes[..., 2].min(2),
                          boxes[..., 3].max(2), boxes[..., 4].min(2), boxes[..., 5].max(2)], axis=2)
    spans = []
    zoffs = np.empty(B)
    for b, (cfg, e) in enumerate(zip(configs, exts)):
        z_shift = float(zsh[b]) if tilt else 0.0
        margin = base_margin + (abs(e.runout_offset_mm) + abs(e.vib_amplitude_mm) + 5.0 * abs(sigma)
                                + abs(ts) * zmax)
        sp = _span(cfg, margin)
        spans.append(sp)
        zoffs[b] = (sp[5] + z_shift) + 0.0
    zw_all = zt[None, :, :] + zoffs[:, None, None]
    keys_all = encode_keys(zw_all)
    minidx = np.argmin(zw_all, axis=2).astype(np.int32)
    rec = np.zeros((B, z_n, n, 4))
    rec[..., 0], rec[..., 1] = xt, yt
    if tilt:
        rec[..., 2] = ts * zt[None]
        rec[..., 3] = tilt_z_term(tc, zt[None], zoffs[:, None, None])
    else:
        rec[..., 2] = keys_all.view(np.float64)
    mode = MODE_EXT_TILT if tilt else MODE_EXT
    plans = []
    for b, (cfg, e) in enumerate(zip(configs, exts)):
        proc, grid = cfg.process, cfg.grid
        dt, t_start, steps, x0, y0, z0 = spans[b]
        p = SweepPlan(
            mode=mode, grid=grid, teeth=z_n, points=n, steps=steps,
            dt=dt, t_start=t_start, x0=x0, y0=y0, z0=z0, feed_speed=proc.feed_speed_mm_s,
            omega=proc.angular_velocity_rad_s, initial_height=z0 + proc.depth_of_cut_mm,
            half_length=base.half_length,
            tooth_base=np.array([tooth_base_angle(proc.phase_rad, k, z_n) for k in range(1, z_n + 1)]),
            tooth_rows=np.zeros((z_n, 8)), px=xt[b], py=yt[b], pz=zt, zw=zw_all[b], zkey=keys_all[b],
            chunk_box=boxes[b], pass_x0=np.array([x0 + k * e.stepover_mm for k in range(int(e.passes))],
                                                 dtype=np.float64),
            min_index=minidx[b], tilt_c=tc, tilt_s=ts, zoff=float(zoffs[b]), vib_amp=e.vib_amplitude_mm,
            vib_omega=2.0 * math.pi * e.vib_frequency_hz, vib_phase=e.vib_phase_rad)
        p.chunk_circ = circs[b]
        p.pts = rec[b]
        p.tooth_box = tooth_box[b]
        p.record = False
        _check_device_limits(p, grid)
        plans.append(p)
    return plans


def replace_ext(ext: Extensions, **kw) -> Extensions:
    from dataclasses import replace as _r

    return _r(ext, **kw)
