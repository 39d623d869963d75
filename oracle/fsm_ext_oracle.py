"""EXTENDED CPU ORACLE — TEST INFRASTRUCTURE ONLY.

NumPy statement of the product's extended FSM model (DESIGN.md §3
"Extended kinematics"): the reference FSM sweep (engine.py:215-313) plus the
BASELINE.json features the reference does not have — ball-end profile,
helix lag, tool-axis runout (offset rho at phase lambda), lead tilt,
sinusoidal radial vibration, per-flute Gaussian edge-radius noise and raster
passes with stepover. Only tests/, smoke() and bench.py's CPU-baseline leg may
import it; the product never does.

Parity status for the extensions: UNPINNED BY THE REFERENCE (the reference has
no such features). What is pinned:
  * with no kinematic extension active, ``ext_sweep`` dispatches to the
    reference restatement ``fsm_oracle`` (pinned bit-exact to the reference
    goldens), passes composing by elementwise min exactly as
    HeightField.merge_min would (surface_grid.py:131-134);
  * ``tests/test_host_cpu.py::test_ext_zero_formulation_is_reference_on_goldens``
    checks that the extended formulation with all extensions at zero gives
    the reference's heights bit-exactly on the golden configurations;
    ``test_ext_oracle_*`` in the same file check geometric properties of the
    extensions (ball-end raster scallop height, tilt re-levelling to z0,
    edge-noise standard deviation and correlation length).
The formulas below are the definition the CUDA kernel is checked against.
"""

from __future__ import annotations

import math
import time
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass

import numpy as np

from . import fsm_oracle as ref
from .fma import fma


def _get(ext, name, default=0.0):
    if ext is None:
        return default
    v = getattr(ext, name, default)
    return default if v is None else v


def kinematic_extensions_active(ext) -> bool:
    return bool(
        _get(ext, "force_extended", False)
        or _get(ext, "profile", "insert") != "insert"
        or _get(ext, "helix_angle_rad") != 0.0
        or _get(ext, "runout_offset_mm") != 0.0
        or _get(ext, "tilt_rad") != 0.0
        or _get(ext, "vib_amplitude_mm") != 0.0
        or _get(ext, "noise_sigma_mm") != 0.0
    )


def edge_noise(teeth, n, sigma, corr, ds, seed):
    """Gaussian-smoothed white noise along the edge, one row per flute.
    Kernel std g = corr/(2 ds) samples (autocorrelation exp(-x^2/4g^2) reaches
    1/e at x = corr); rescaled by 1/sqrt(sum k^2) so the stationary std is sigma."""
    rng = np.random.default_rng(seed)
    white = rng.standard_normal((teeth, n))
    g = corr / (2.0 * ds)
    if g < 0.5:
        return sigma * white
    w = int(math.ceil(4.0 * g))
    x = np.arange(-w, w + 1, dtype=np.float64)
    k = np.exp(-0.5 * (x / g) ** 2)
    norm = math.sqrt(float(np.sum(k * k)))
    out = np.empty((teeth, n))
    for t in range(teeth):
        out[t] = sigma * (np.convolve(white[t], k, mode="same") / norm)
    return out


@dataclass
class ExtPlan:
    m: int
    n: int
    spacing: float
    x_min: float
    y_min: float
    teeth: int
    points: int
    xt: np.ndarray      # (Z, N) tool-frame x (time invariant)
    yt: np.ndarray
    zt: np.ndarray
    zw: np.ndarray      # (Z, N) workpiece z when no tilt: zt + zoff
    base: list          # per tooth phase + 2pi(K-1)/Z
    dt: float
    t_start: float
    steps: int
    x0: float
    y0: float
    z0: float
    zoff: float
    feed_speed: float
    omega: float
    tilt_c: float
    tilt_s: float
    tilt: bool
    vib_amp: float
    vib_omega: float
    vib_phase: float
    pass_x0: list
    initial_height: float

    @property
    def trajectory_points(self):
        return self.steps * self.teeth * self.points * len(self.pass_x0)


def ext_rows(tool, k, profile):
    """kinematics.py:85-99 with the radial placement D/2 dropped for the
    ball-end profile (flutes meet at the tool axis)."""
    e = ref.edge_to_tool_rows(tool, k)
    if profile == "ball":
        runouts = tool.runouts_mm or ((0.0, 0.0),) * tool.tooth_count
        e[0][3] = 0.0 + (k - 1) * runouts[k - 1][0]
    return e


def ext_plan(cfg, ext) -> ExtPlan:
    tool, proc, grid = cfg.tool, cfg.process, cfg.grid
    r = tool.insert_radius_mm
    a_p = proc.depth_of_cut_mm
    if a_p > r:
        raise ref.OracleConfigError("depth of cut exceeds insert radius")
    profile = _get(ext, "profile", "insert")
    tau = _get(ext, "tilt_rad")
    z_n = tool.tooth_count
    if profile == "insert":
        half = ref.effective_half_length(r, a_p, proc.feed_per_tooth_mm, tool.radial_rake_rad)
        n = cfg.edge_point_count or ref.default_point_count(half, grid.spacing_mm)
        ex, ey, ez = ref.edge_arrays(r, half, n)
        sq = r - ez
        nx = ex / r
        nz = -sq / r
        arc = 2.0 * r * math.asin(min(1.0, half / r))
    elif profile == "ball":
        n = cfg.edge_point_count
        if n is None or n < 2:
            raise ref.OracleConfigError("ball profile needs edge_point_count >= 2")
        kmax = min(math.pi / 2.0, math.acos((r - a_p) / r) + abs(tau))
        kap = kmax * np.arange(n, dtype=np.float64) / (n - 1)
        kap[-1] = kmax
        nx = np.sin(kap)
        nz = -np.cos(kap)
        ex = r * nx
        ey = np.zeros(n)
        ez = r - r * np.cos(kap)
        arc = r * kmax
    else:
        raise ref.OracleConfigError(f"unknown profile {profile!r}")
    sigma = _get(ext, "noise_sigma_mm")
    if sigma != 0.0:
        delta = edge_noise(z_n, n, sigma, _get(ext, "noise_corr_mm"), arc / (n - 1),
                           int(_get(ext, "noise_seed", 0)))
    beta = _get(ext, "helix_angle_rad")
    rho = _get(ext, "runout_offset_mm")
    lam = _get(ext, "runout_phase_rad")
    if beta != 0.0:
        r_ref = _get(ext, "helix_ref_radius_mm", None)
        if r_ref is None:
            r_ref = tool.cutting_diameter_mm / 2.0 if profile == "insert" else r
        tanb_over_r = math.tan(beta) / r_ref

    x0, y0, z0 = proc.initial_position_mm
    if z0 is None:
        z0 = 0.0
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
        e = ext_rows(tool, k, profile)
        qx = ((e[0][0] * px + e[0][1] * py) + e[0][2] * pz) + e[0][3]
        qy = ((e[1][0] * px + e[1][1] * py) + e[1][2] * pz) + e[1][3]
        qz = ((e[2][0] * px + e[2][1] * py) + e[2][2] * pz) + e[2][3]
        if beta != 0.0:
            psi = pz * tanb_over_r
            cps = np.cos(psi)
            sps = np.sin(psi)
            qx, qy = cps * qx + sps * qy, (-sps) * qx + cps * qy
        if rho != 0.0:
            ang = lam + (2.0 * math.pi) * (k - 1) / z_n
            qx = qx + rho * math.cos(ang)
            qy = qy + rho * math.sin(ang)
        xt[k - 1], yt[k - 1], zt[k - 1] = qx, qy, qz

    tilt = tau != 0.0
    tc, ts = math.cos(tau), math.sin(tau)
    z_shift = 0.0
    if tilt:
        z_shift = -float(np.min(tc * zt - abs(ts) * np.sqrt(xt * xt + yt * yt)))
    zoff = z0 + z_shift
    zw = zt + zoff

    dt = ref.time_step(cfg)
    amp = _get(ext, "vib_amplitude_mm")
    if cfg.span_s is None:
        # reference auto-span margin (engine.py:158, D/2 + dL) widened by the
        # extensions' reach, so it reduces to the reference when they are zero
        if profile == "insert":
            margin = tool.cutting_diameter_mm / 2.0 + half
        else:
            margin = r * math.sin(kmax)
        margin = margin + (abs(rho) + abs(amp) + 5.0 * abs(sigma)
                           + abs(ts) * float(np.max(np.abs(zt))))
        y0 = grid.y_min_mm - margin
        t_start = 0.0
        y_max = grid.y_min_mm + grid.n * grid.spacing_mm
        t_end = (y_max + margin - y0) / proc.feed_speed_mm_s
    else:
        t_start, t_end = cfg.span_s
        if t_start < 0 or t_end <= t_start:
            raise ref.OracleConfigError("bad span")
        if y0 is None:
            raise ref.OracleConfigError("initial y required with explicit span")
    steps = int(math.floor((t_end - t_start) / dt)) + 1
    passes = int(_get(ext, "passes", 1))
    stepover = _get(ext, "stepover_mm")
    pass_x0 = [x0 + k * stepover for k in range(passes)]
    fv = _get(ext, "vib_frequency_hz")
    return ExtPlan(
        m=grid.m, n=grid.n, spacing=grid.spacing_mm, x_min=grid.x_min_mm, y_min=grid.y_min_mm,
        teeth=z_n, points=n, xt=xt, yt=yt, zt=zt, zw=zw,
        base=[ref.tooth_base(proc.phase_rad, k, z_n) for k in range(1, z_n + 1)],
        dt=dt, t_start=t_start, steps=steps, x0=x0, y0=y0, z0=z0, zoff=zoff,
        feed_speed=proc.feed_speed_mm_s, omega=proc.angular_velocity_rad_s,
        tilt_c=tc, tilt_s=ts, tilt=tilt, vib_amp=amp, vib_omega=2.0 * math.pi * fv,
        vib_phase=_get(ext, "vib_phase_rad"), pass_x0=pass_x0,
        initial_height=z0 + a_p,
    )


def _ext_range(p: ExtPlan, x0p, lo_step, hi_step, heights, counters):
    m, n, dd = p.m, p.n, p.spacing
    n1 = n + 1
    wx_lo = p.x_min - 1.5 * dd
    wx_hi = p.x_min + m * dd + 1.5 * dd
    wy_lo = p.y_min - 1.5 * dd
    wy_hi = p.y_min + n * dd + 1.5 * dd
    chunk = max(64, 2_000_000 // max(p.points, 1))
    deposits = 0
    s = lo_step
    while s < hi_step:
        e_s = min(s + chunk, hi_step)
        t = p.t_start + np.arange(s, e_s, dtype=np.float64) * p.dt
        ty = p.y0 + p.feed_speed * t
        if p.vib_amp != 0.0:
            xoff = x0p + p.vib_amp * np.sin(p.vib_omega * t + p.vib_phase)
        else:
            xoff = np.full(t.shape, x0p)
        for ki in range(p.teeth):
            xt, yt, zt = p.xt[ki], p.yt[ki], p.zt[ki]
            th = p.base[ki] - p.omega * t
            c = np.cos(th)
            sn = np.sin(th)
            ns = -sn
            # conservative row cull (never changes results)
            xl, xh, yl, yh = xt.min(), xt.max(), yt.min(), yt.max()
            ux_lo = np.minimum(c * xl, c * xh) + np.minimum(sn * yl, sn * yh)
            ux_hi = np.maximum(c * xl, c * xh) + np.maximum(sn * yl, sn * yh)
            vy_lo = np.minimum(ns * xl, ns * xh) + np.minimum(c * yl, c * yh)
            vy_hi = np.maximum(ns * xl, ns * xh) + np.maximum(c * yl, c * yh)
            if p.tilt:
                zl, zh = zt.min(), zt.max()
                a1, a2 = p.tilt_c * vy_lo, p.tilt_c * vy_hi
                b1, b2 = p.tilt_s * zl, p.tilt_s * zh
                vy_lo = np.minimum(a1, a2) - max(b1, b2)
                vy_hi = np.maximum(a1, a2) - min(b1, b2)
            keep = np.flatnonzero((ux_hi + xoff >= wx_lo) & (ux_lo + xoff <= wx_hi)
                                  & (vy_hi + ty >= wy_lo) & (vy_lo + ty <= wy_hi))
            if keep.size == 0:
                continue
            ck, sk, nk = c[keep][:, None], sn[keep][:, None], ns[keep][:, None]
            if p.tilt:
                # fused lead-tilt model: one rounding per fma
                u = fma(ck, xt, sk * yt)
                v = fma(ck, yt, -(sk * xt))
                xw = u + xoff[keep][:, None]
                yw = fma(p.tilt_c, v, -(p.tilt_s * zt)) + ty[keep][:, None]
                zz = fma(p.tilt_s, v, (p.tilt_c * zt + p.zoff) + 0.0)
            else:
                u = ck * xt + sk * yt
                v = nk * xt + ck * yt
                xw = u + xoff[keep][:, None]
                yw = v + ty[keep][:, None]
            gi = np.floor((xw - p.x_min) / dd + 0.5)
            gj = np.floor((yw - p.y_min) / dd + 0.5)
            ok = (gi >= 0.0) & (gi <= m) & (gj >= 0.0) & (gj <= n)
            cnt = int(np.count_nonzero(ok))
            if cnt:
                deposits += cnt
                flat = gi[ok].astype(np.int64) * n1 + gj[ok].astype(np.int64)
                if p.tilt:
                    zv = zz[ok]
                else:
                    zv = np.broadcast_to(p.zw[ki], xw.shape)[ok]
                np.minimum.at(heights, flat, zv)
        s = e_s
    counters["deposits"] = counters.get("deposits", 0) + deposits


def ext_sweep(cfg, ext=None, workers=1, step_limit=None, windows=None, pass_limit=None):
    """Extended sweep over all passes. Returns (heights, plan, counters, wall).
    Bounded CPU-baseline samples only: ``step_limit`` truncates every pass to
    its first steps; ``windows`` = [(lo, hi), ...] sweeps only those step
    ranges; ``pass_limit`` only the first passes (extended path only)."""
    passes = int(_get(ext, "passes", 1))
    if not kinematic_extensions_active(ext):
        base = ref.plan(cfg)
        stepover = _get(ext, "stepover_mm")
        x0 = base.x0
        h = None
        dep = 0
        wall = 0.0
        for k in range(passes):
            base.x0 = x0 + k * stepover
            if step_limit is not None:
                base.steps = min(base.steps, step_limit)
            hk, _, ck, wk = ref.sweep(cfg, workers=workers, plan_obj=base)
            dep += ck["deposits"]
            wall += wk
            h = hk if h is None else np.minimum(h, hk)
        base.x0 = x0
        counters = {"time_steps": base.steps, "trajectory_points": base.trajectory_points * passes,
                    "cells_updated": int(np.count_nonzero(h < base.initial_height)),
                    "deposits": dep}
        return h, base, counters, wall

    p = ext_plan(cfg, ext)
    steps = p.steps if step_limit is None else min(p.steps, step_limit)
    pass_x0 = p.pass_x0 if pass_limit is None else p.pass_x0[:pass_limit]
    if windows is None:
        windows = [(0, steps)]
    w = max(1, workers)
    tasks = []
    for x0p in pass_x0:
        for lo, hi in windows:
            lo, hi = max(0, lo), min(hi, steps)
            if hi <= lo:
                continue
            k = max(1, min(w, hi - lo))
            b = [lo + round(i * (hi - lo) / k) for i in range(k + 1)]
            tasks += [(x0p, b[i], b[i + 1]) for i in range(k) if b[i] < b[i + 1]]
    sampled = sum(hi - lo for _, lo, hi in tasks) // max(1, len(pass_x0))
    nf = min(w, len(tasks))
    fields = [np.full((p.m + 1) * (p.n + 1), p.initial_height) for _ in range(nf)]
    ctrs = [dict() for _ in range(nf)]
    t0 = time.perf_counter()

    def run(slot):
        for ti in range(slot, len(tasks), nf):
            x0p, lo, hi = tasks[ti]
            _ext_range(p, x0p, lo, hi, fields[slot], ctrs[slot])

    if nf == 1:
        run(0)
    else:
        with ThreadPoolExecutor(max_workers=nf) as pool:
            list(pool.map(run, range(nf)))
    h = fields[0]
    for other in fields[1:]:
        np.minimum(h, other, out=h)
    wall = time.perf_counter() - t0
    counters = {"time_steps": steps, "trajectory_points": sampled * p.teeth * p.points * len(pass_x0),
                "cells_updated": int(np.count_nonzero(h < p.initial_height)),
                "deposits": sum(c.get("deposits", 0) for c in ctrs)}
    return h, p, counters, wall
