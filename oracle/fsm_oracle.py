"""CPU ORACLE — TEST INFRASTRUCTURE ONLY.

A plain NumPy restatement of the reference FSM path of arXiv 2603.28160
(reference package ``millsurf``, mounted read-only at /root/reference/pkg).
Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline
leg may import this module, and only as the checker / the timed CPU
baseline. The product (``paper_2603_28160_b200``) never imports it.

Parity status: PINNED. ``tests/golden/make_golden.py`` runs the real
reference (imported from /root/reference in the build container) on the
reference's own golden configurations (``helpers.small_random_config`` seeds
0-4 and 1000-1019, ``configs/bench_10x5.json`` geometry, the test_engine tiny
config, the config-1 analog) and commits heights, counters and roughness as
``tests/golden/*.npz``; ``tests/test_oracle_golden.py`` requires this module
to reproduce them bit-exactly.

Every function cites the reference lines it restates. Floating-point
evaluation order follows the reference exactly (NumPy never contracts to FMA),
which is what makes bitwise parity possible.
"""

from __future__ import annotations

import math
import os
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass

import numpy as np


class OracleDomainError(ValueError):
    """Mirrors millsurf.DomainError (errors.py:8-9)."""


class OracleConfigError(ValueError):
    """Mirrors millsurf.ConfigError (errors.py:12-13)."""


# ----------------------------------------------------------------- geometry
def effective_half_length(r, a_p, f_z, rake=0.0):
    """tool_geometry.py:109-136: max(half-chord at depth a_p, f_z/(2 cos rake))."""
    if a_p <= 0 or a_p > r or f_z <= 0 or abs(rake) >= math.pi / 2:
        raise OracleDomainError("effective_half_length domain")
    half_immersion = math.sqrt(r * r - (r - a_p) * (r - a_p))
    half_feed = f_z / (2.0 * math.cos(rake))
    return max(half_immersion, half_feed)


def default_point_count(half, spacing):
    """tool_geometry.py:139-143."""
    return max(2, math.ceil(4.0 * half / spacing) + 1)


def edge_arrays(r, half, n):
    """tool_geometry.py:167-174: uniform l in [-half, half], z = R - sqrt(R^2 - l^2)."""
    l = -half + (2.0 * half) * np.arange(n, dtype=np.float64) / (n - 1)
    l[0] = -half
    l[-1] = half
    x = l.copy()
    y = np.zeros(n)
    z = r - np.sqrt(r * r - l * l)
    return x, y, z


def edge_to_tool_rows(tool, k):
    """kinematics.py:85-99 (rake rotation + radial/axial placement of tooth k)."""
    cf = math.cos(tool.radial_rake_rad)
    sf = math.sin(tool.radial_rake_rad)
    cp = math.cos(tool.axial_rake_rad)
    sp = math.sin(tool.axial_rake_rad)
    runouts = tool.runouts_mm or ((0.0, 0.0),) * tool.tooth_count
    eps_r, eps_a = runouts[k - 1]
    tx = tool.cutting_diameter_mm / 2.0 + (k - 1) * eps_r
    tz = (k - 1) * eps_a
    return [
        [cf, sf * cp, sf * sp, tx],
        [-sf, cf * cp, cf * sp, 0.0],
        [0.0, -sp, cp, tz],
        [0.0, 0.0, 0.0, 1.0],
    ]


def tooth_base(phase, k, z_n):
    """kinematics.py:76: base = phase + (2*pi)*(k-1)/Z (evaluation order kept)."""
    return phase + (2.0 * math.pi) * (k - 1) / z_n


def time_step(cfg):
    """engine.py:86-98."""
    if cfg.time_step_s is not None:
        if cfg.time_step_s <= 0:
            raise OracleConfigError("time_step_s must be > 0")
        return cfg.time_step_s
    if cfg.max_step_angle_rad <= 0:
        raise OracleConfigError("max_step_angle_rad must be > 0")
    by_angle = cfg.max_step_angle_rad / cfg.process.angular_velocity_rad_s
    by_feed = cfg.grid.spacing_mm / cfg.process.feed_speed_mm_s
    return min(by_angle, by_feed)


@dataclass
class OraclePlan:
    """engine.py:110-131 (_Plan) restated with plain arrays."""

    m: int
    n: int
    spacing: float
    x_min: float
    y_min: float
    teeth: int
    points: int
    xp: np.ndarray
    yp: np.ndarray
    zp: np.ndarray
    rows: list          # per tooth 4x4 python floats
    zw: list            # per tooth (N,) z' (time-invariant, engine.py:181-182)
    x_range: list       # per tooth tool-frame x range (engine.py:183,190)
    y_range: list
    min_index: list
    dt: float
    t_start: float
    steps: int
    x0: float
    y0: float
    z0: float
    feed_speed: float
    omega: float
    phase: float
    initial_height: float
    half_length: float

    @property
    def trajectory_points(self):
        return self.steps * self.teeth * self.points


def plan(cfg) -> OraclePlan:
    """engine.py:134-212 (_plan): validation, edge, dt, span, steps, per-tooth rows."""
    tool, proc, grid = cfg.tool, cfg.process, cfg.grid
    if proc.depth_of_cut_mm > tool.insert_radius_mm:
        raise OracleConfigError("depth of cut exceeds insert radius")
    half = effective_half_length(tool.insert_radius_mm, proc.depth_of_cut_mm,
                                 proc.feed_per_tooth_mm, tool.radial_rake_rad)
    n_points = cfg.edge_point_count
    if n_points is None:
        n_points = default_point_count(half, grid.spacing_mm)
    if n_points < 2:
        raise OracleDomainError("point_count must be >= 2")
    if half > tool.insert_radius_mm:
        raise OracleDomainError("engaged half-length exceeds insert radius")
    xp, yp, zp = edge_arrays(tool.insert_radius_mm, half, n_points)
    dt = time_step(cfg)
    x0, y0, z0 = proc.initial_position_mm
    if cfg.span_s is None:
        margin = tool.cutting_diameter_mm / 2.0 + half          # engine.py:158
        y0 = grid.y_min_mm - margin
        t_start = 0.0
        y_max = grid.y_min_mm + grid.n * grid.spacing_mm                 # surface_grid.py:63-65
        t_end = (y_max + margin - y0) / proc.feed_speed_mm_s
    else:
        t_start, t_end = cfg.span_s
        if t_start < 0 or t_end <= t_start:
            raise OracleConfigError("bad span")
        if y0 is None:
            raise OracleConfigError("initial y required with explicit span")
    if z0 is None:
        z0 = 0.0
    steps = int(math.floor((t_end - t_start) / dt)) + 1                 # engine.py:170
    initial_height = z0 + proc.depth_of_cut_mm                           # engine.py:174
    rows, zws, xr, yr, mi = [], [], [], [], []
    for k in range(1, tool.tooth_count + 1):
        e = edge_to_tool_rows(tool, k)
        tz = e[2][3] + z0
        zw = ((e[2][0] * xp + e[2][1] * yp) + e[2][2] * zp) + tz
        xt = ((e[0][0] * xp + e[0][1] * yp) + e[0][2] * zp) + e[0][3]
        yt = ((e[1][0] * xp + e[1][1] * yp) + e[1][2] * zp) + e[1][3]
        rows.append(e)
        zws.append(zw)
        xr.append((float(xt.min()), float(xt.max())))
        yr.append((float(yt.min()), float(yt.max())))
        mi.append(int(np.argmin(zw)))
    return OraclePlan(
        m=grid.m, n=grid.n, spacing=grid.spacing_mm, x_min=grid.x_min_mm, y_min=grid.y_min_mm,
        teeth=tool.tooth_count, points=n_points, xp=xp, yp=yp, zp=zp, rows=rows, zw=zws,
        x_range=xr, y_range=yr, min_index=mi, dt=dt, t_start=t_start, steps=steps,
        x0=x0, y0=y0, z0=z0, feed_speed=proc.feed_speed_mm_s, omega=proc.angular_velocity_rad_s,
        phase=proc.phase_rad, initial_height=initial_height, half_length=half,
    )


# -------------------------------------------------------------------- sweep
_CHUNK_ELEMS = 2_000_000  # engine.py:58-60 (memory bound only, not results)


def _sweep_range(p: OraclePlan, lo_step, hi_step, heights, counters):
    """engine.py:215-313 (_run_step_range): per chunk of steps, per tooth:
    trig (252-255) -> composite coefficients (257-264) -> x-interval cull
    (272-287) -> affine (289-296) -> locate (298-300) -> np.minimum.at (301-305)."""
    m, n, dd = p.m, p.n, p.spacing
    n1 = n + 1
    win_lo = p.x_min - 1.5 * dd
    win_hi = p.x_min + m * dd + 1.5 * dd
    xp, yp, zp = p.xp, p.yp, p.zp
    chunk = max(64, _CHUNK_ELEMS // max(p.points, 1))
    deposits = 0
    s = lo_step
    while s < hi_step:
        e_s = min(s + chunk, hi_step)
        t = p.t_start + np.arange(s, e_s, dtype=np.float64) * p.dt
        ty = p.y0 + p.feed_speed * t
        for ki in range(p.teeth):
            e = p.rows[ki]
            th = tooth_base(p.phase, ki + 1, p.teeth) - p.omega * t
            c = np.cos(th)
            sn = np.sin(th)
            ns = -sn
            m00 = c * e[0][0] + sn * e[1][0]
            m01 = c * e[0][1] + sn * e[1][1]
            m02 = c * e[0][2] + sn * e[1][2]
            m03 = (c * e[0][3] + sn * e[1][3]) + p.x0
            m10 = ns * e[0][0] + c * e[1][0]
            m11 = ns * e[0][1] + c * e[1][1]
            m12 = ns * e[0][2] + c * e[1][2]
            m13 = (ns * e[0][3] + c * e[1][3]) + ty
            axl, axh = p.x_range[ki]
            ayl, ayh = p.y_range[ki]
            x_lo = np.minimum(c * axl, c * axh) + np.minimum(sn * ayl, sn * ayh) + p.x0
            x_hi = np.maximum(c * axl, c * axh) + np.maximum(sn * ayl, sn * ayh) + p.x0
            keep = np.flatnonzero((x_hi >= win_lo) & (x_lo <= win_hi))
            if keep.size == 0:
                continue
            a = [v[keep] for v in (m00, m01, m02, m03, m10, m11, m12, m13)]
            xw = a[0][:, None] * xp
            xw += a[1][:, None] * yp
            xw += a[2][:, None] * zp
            xw += a[3][:, None]
            yw = a[4][:, None] * xp
            yw += a[5][:, None] * yp
            yw += a[6][:, None] * zp
            yw += a[7][:, None]
            gi = np.floor((xw - p.x_min) / dd + 0.5)
            gj = np.floor((yw - p.y_min) / dd + 0.5)
            ok = (gi >= 0.0) & (gi <= m) & (gj >= 0.0) & (gj <= n)
            cnt = int(np.count_nonzero(ok))
            if cnt:
                deposits += cnt
                flat = gi[ok].astype(np.int64) * n1 + gj[ok].astype(np.int64)
                zv = np.broadcast_to(p.zw[ki], xw.shape)[ok]
                np.minimum.at(heights, flat, zv)
        s = e_s
    counters["deposits"] = counters.get("deposits", 0) + deposits


def sweep(cfg, workers=None, plan_obj=None):
    """engine.py:316-357 (simulate): contiguous time ranges per worker, one
    private field each, elementwise-min merge (339-341). Returns
    (heights (m+1)*(n+1) fp64, plan, counters, main_loop_seconds)."""
    import time as _time

    p = plan_obj if plan_obj is not None else plan(cfg)
    w = workers if workers is not None else getattr(cfg, "worker_count", 1)
    if w < 1:
        raise OracleConfigError("worker_count must be >= 1")
    w = min(w, p.steps) or 1
    bounds = [round(i * p.steps / w) for i in range(w + 1)]
    ranges = [(bounds[i], bounds[i + 1]) for i in range(w) if bounds[i] < bounds[i + 1]]
    fields = [np.full((p.m + 1) * (p.n + 1), p.initial_height) for _ in ranges]
    ctrs = [dict() for _ in ranges]
    t0 = _time.perf_counter()
    if len(ranges) == 1:
        _sweep_range(p, ranges[0][0], ranges[0][1], fields[0], ctrs[0])
    else:
        with ThreadPoolExecutor(max_workers=len(ranges)) as pool:
            list(pool.map(lambda a: _sweep_range(p, a[0][0], a[0][1], a[1], a[2]),
                          zip(ranges, fields, ctrs)))
    h = fields[0]
    for other in fields[1:]:
        np.minimum(h, other, out=h)
    wall = _time.perf_counter() - t0
    counters = {
        "time_steps": p.steps,
        "trajectory_points": p.trajectory_points,
        "cells_updated": int(np.count_nonzero(h < p.initial_height)),
        "deposits": sum(c.get("deposits", 0) for c in ctrs),
    }
    return h, p, counters, wall


def locate(x, y, spacing, x_min, y_min, m, n):
    """surface_grid.py:78-89."""
    if not (math.isfinite(x) and math.isfinite(y)):
        raise OracleDomainError("non-finite")
    i = math.floor((x - x_min) / spacing + 0.5)
    j = math.floor((y - y_min) / spacing + 0.5)
    if 0 <= i <= m and 0 <= j <= n:
        return (i, j)
    return None


# --------------------------------------------------------------- roughness
MM_TO_UM = 1000.0


def areal_metrics(heights2d, initial_height, roi=None, uncut="raise", leveling="mean"):
    """roughness.py:76-135 with leveling='mean'. ``uncut='exclude'`` is the
    product's documented extension (statistics over machined cells only).
    Returns dict with Sa Sq Sp Sv Sz Ssk Sku cell_count (µm)."""
    mm, nn = heights2d.shape[0] - 1, heights2d.shape[1] - 1
    if roi is None:
        roi = (0, 0, mm, nn)
    i_lo, j_lo, i_hi, j_hi = roi
    if not (0 <= i_lo <= i_hi <= mm and 0 <= j_lo <= j_hi <= nn):
        raise OracleDomainError("roi outside grid")
    block = heights2d[i_lo:i_hi + 1, j_lo:j_hi + 1]
    cut = block < initial_height
    if uncut == "raise":
        if not cut.all():
            raise OracleDomainError("roi contains uncut cells")
        z = block * MM_TO_UM
    else:
        z = block[cut] * MM_TO_UM
        if z.size == 0:
            raise OracleDomainError("no machined cells in roi")
    if leveling == "plane":
        # roughness.py:108-113: least-squares plane over node offsets (i, j)
        if uncut != "raise":
            xi, yj = np.nonzero(cut)
        else:
            xi, yj = np.meshgrid(np.arange(block.shape[0]), np.arange(block.shape[1]), indexing="ij")
            xi, yj = xi.ravel(), yj.ravel()
        a = np.column_stack([xi, yj, np.ones(z.size)])
        coef, *_ = np.linalg.lstsq(a, z.ravel(), rcond=None)
        d = z.ravel() - a @ coef
    else:
        d = z - z.mean()
    sa = float(np.mean(np.abs(d)))
    sq = float(np.sqrt(np.mean(d * d)))
    sp = float(np.max(d))
    sv = float(-np.min(d))
    if sq == 0.0:
        ssk = sku = None
    else:
        ssk = float(np.mean(d ** 3) / sq ** 3)
        sku = float(np.mean(d ** 4) / sq ** 4)
    return {"Sa": sa, "Sq": sq, "Sp": sp, "Sv": sv, "Sz": sp + sv, "Ssk": ssk, "Sku": sku,
            "cell_count": int(z.size)}


def profile_roughness(heights_1d, initial_height, uncut="raise"):
    """roughness.py:183-188 (Ra = mean|z - mean z| in µm) plus Rz = Rp + Rv
    (the product's extension, mirroring Sz = Sp + Sv, roughness.py:118-132)."""
    h = np.asarray(heights_1d)
    cut = h < initial_height
    if uncut == "raise":
        if not cut.all():
            raise OracleDomainError("profile crosses uncut cells")
        z = h * MM_TO_UM
    else:
        z = h[cut] * MM_TO_UM
    if z.size < 2:
        raise OracleDomainError("line roughness needs at least 2 samples")
    d = z - z.mean()
    ra = float(np.mean(np.abs(d)))
    rz = float(np.max(d)) + float(-np.min(d))
    return {"Ra": ra, "Rz": rz, "n": int(z.size)}


# ------------------------------------------------------------------ dataset
def lhs_sample(ranges, count, seed):
    """dataset.py:91-105: per dimension rng.permutation(count), rng.random(count)."""
    if count < 1 or not ranges:
        raise OracleConfigError("bad lhs request")
    rng = np.random.default_rng(seed)
    out = np.empty((count, len(ranges)), dtype=np.float64)
    for d, (low, high) in enumerate(ranges):
        strata = rng.permutation(count)
        offsets = rng.random(count)
        unit = (strata + offsets) / count
        out[:, d] = low + (high - low) * unit
    return out


def default_cpu_workers():
    return os.cpu_count() or 1
