"""Areal and profile roughness on the GPU — drop-in for millsurf.roughness.

Areal parameters (roughness.py:26-135): z in µm = h * 1000, deviations from
the arithmetic mean, Sa = mean|d|, Sq = sqrt(mean d^2), Sp = max d,
Sv = -min d, Sz = Sp + Sv, Ssk = mean d^3 / Sq^3, Sku = mean d^4 / Sq^4
(None on a flat region). Two deterministic device passes
(msurf_areal_pass1: sum/max/min/counts; msurf_areal_pass2: the four central
moments around the device-computed mean) and one 9-double D2H read.

Profiles (roughness.py:138-188): Ra = mean|z - mean z| (µm); the product
adds Rz = Rp + Rv over the same profile, and ``profile_roughness`` evaluates
many profiles (e.g. "every 64th row") in one launch.

``uncut='raise'`` (default) mirrors the reference: any uncut cell in the ROI
raises DomainError (roughness.py:86-89). ``uncut='exclude'`` is the product's
documented extension for fine grids where sparse uncut cells remain
(SURVEY.md §0 fact 7): statistics over machined cells only.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _native
from .errors import DomainError
from .grid import HeightField

MM_TO_UM = 1000.0


@dataclass(frozen=True)
class ArealMetrics:
    sa_um: float
    sq_um: float
    sp_um: float
    sv_um: float
    sz_um: float
    ssk: float | None
    sku: float | None
    cell_count: int

    def to_json_dict(self) -> dict:
        return {"Sa_um": self.sa_um, "Sq_um": self.sq_um, "Sp_um": self.sp_um, "Sv_um": self.sv_um,
                "Sz_um": self.sz_um, "Ssk": self.ssk, "Sku": self.sku, "cell_count": self.cell_count}

    def to_text(self) -> str:
        rows = [("Sa", f"{self.sa_um:.6f} um"), ("Sq", f"{self.sq_um:.6f} um"),
                ("Sp", f"{self.sp_um:.6f} um"), ("Sv", f"{self.sv_um:.6f} um"),
                ("Sz", f"{self.sz_um:.6f} um"),
                ("Ssk", "undefined" if self.ssk is None else f"{self.ssk:.6f}"),
                ("Sku", "undefined" if self.sku is None else f"{self.sku:.6f}"),
                ("cells", str(self.cell_count))]
        w = max(len(k) for k, _ in rows)
        return "\n".join(f"{k:<{w}}  {v}" for k, v in rows)


@dataclass(frozen=True)
class LineProfile:
    """Feed profiles run along Y (fixed i), pick-feed along X (fixed j)."""

    direction: str
    index: int
    positions_mm: np.ndarray
    heights_mm: np.ndarray
    spacing_mm: float


@dataclass(frozen=True)
class ProfileRoughness:
    index: int
    ra_um: float
    rz_um: float
    rp_um: float
    rv_um: float
    sample_count: int


def _check_roi(spec, roi):
    if roi is None:
        roi = (0, 0, spec.m, spec.n)
    i_lo, j_lo, i_hi, j_hi = (int(v) for v in roi)
    if not (0 <= i_lo <= i_hi <= spec.m and 0 <= j_lo <= j_hi <= spec.n):
        raise DomainError(f"roi {roi} outside grid [0, {spec.m}] x [0, {spec.n}] or empty")
    return i_lo, j_lo, i_hi, j_hi


def _metrics_from_moments(st1, st2) -> ArealMetrics:
    n = st1[3]
    mean = st1[5]  # device: double-double sum / n, rounded once
    sa = float(st2[0] / n)
    sq = float(np.sqrt(st2[1] / n))
    sp = float(st1[1] - mean)
    sv = float(-(st1[2] - mean))
    if sq == 0.0:
        ssk = sku = None
    else:
        ssk = float((st2[2] / n) / sq ** 3)
        sku = float((st2[3] / n) / sq ** 4)
    return ArealMetrics(sa_um=sa, sq_um=sq, sp_um=sp, sv_um=sv, sz_um=sp + sv, ssk=ssk, sku=sku,
                        cell_count=int(n))


def _scratch(torch, device, n_work: int, n_out: int | None = None):
    """Reduction scratch for ONE call: ``n_work`` surfaces of work partials
    (MSURF_WORK_DOUBLES each) followed by ``n_out`` x 16 outputs, from the
    caching allocator (stream-ordered reuse, so concurrent callers on any
    streams or threads never share a buffer; ~80 KB per surface)."""
    n_out = n_work if n_out is None else n_out
    return torch.empty(n_work * _native.WORK_DOUBLES + n_out * 16, dtype=torch.float64, device=device)


def _areal_enqueue(lib, h_dev, ld, n_surf, surf_stride, roi_box, sentinels_dev, exclude, work, out, sp,
                   allreduce=None):
    """Enqueue both areal passes of ``n_surf`` surfaces; ``out`` (>= 10 n_surf
    doubles) receives stats1 [n_surf, 6] then moments [n_surf, 4]."""
    i_lo, j_lo, rows, cols = roi_box
    st1 = out[: n_surf * 6]
    st2 = out[n_surf * 6: n_surf * 10]
    _native.check(lib.msurf_areal_pass1(h_dev.data_ptr(), ld, surf_stride, n_surf, i_lo, j_lo, rows,
                                        cols, sentinels_dev.data_ptr(), int(exclude), work,
                                        st1.data_ptr(), sp))
    if allreduce is not None:
        allreduce(st1.view(n_surf, 6), "stats1")
    _native.check(lib.msurf_areal_pass2(h_dev.data_ptr(), ld, surf_stride, n_surf, i_lo, j_lo, rows,
                                        cols, sentinels_dev.data_ptr(), int(exclude), st1.data_ptr(),
                                        work, st2.data_ptr(), sp))
    if allreduce is not None:
        allreduce(st2.view(n_surf, 4), "moments")


def _split_moments(both, n_surf):
    return both[: n_surf * 6].reshape(n_surf, 6), both[n_surf * 6: n_surf * 10].reshape(n_surf, 4)


def areal_moments_device(h_dev, ld, n_surf, surf_stride, roi_box, sentinels_dev, exclude,
                         allreduce=None):
    """Run both areal passes; returns (stats1 [n_surf,5], moments [n_surf,4])
    on the host. ``allreduce(tensor, op)`` (strip sharding) combines the
    partial first-pass stats (kind "stats1": columns sum, max, min, n, n_uncut,
    mean — the callee recomputes the mean) and second-pass moments (kind
    "moments": four sums) across ranks in place."""
    torch = _native.require_cuda()
    lib = _native.lib()
    sc = _scratch(torch, h_dev.device, n_surf)
    out = sc[n_surf * _native.WORK_DOUBLES:]
    _areal_enqueue(lib, h_dev, ld, n_surf, surf_stride, roi_box, sentinels_dev, exclude, sc.data_ptr(), out,
                   _native.stream_ptr(), allreduce)
    return _split_moments(_native.readback(out[: n_surf * 10]), n_surf)


def _sentinel_tensor(torch, values, device):
    return torch.tensor(np.asarray(values, dtype=np.float64), device=device)


def _field_sentinel(torch, field, device):
    """Device stock height of a field: the sweep's own copy when available
    (no H2D copy / host sync), else a fresh 1-element tensor."""
    s = getattr(field, "_dev_sentinel", None)
    if s is not None and s.device == device:
        return s
    return _sentinel_tensor(torch, [field.initial_height_mm], device)


def areal_metrics(field: HeightField, roi=None, leveling: str = "mean", uncut: str = "raise") -> ArealMetrics:
    """Areal parameters over the inclusive node range (i_lo, j_lo, i_hi, j_hi).
    ``leveling='plane'`` removes the least-squares plane z ~ a*i + b*j + c
    (roughness.py:108-113) before the statistics."""
    if leveling not in ("mean", "plane"):
        raise DomainError(f"unknown leveling mode {leveling!r}")
    if leveling == "plane":
        return _areal_plane(field, roi, uncut)
    if uncut not in ("raise", "exclude"):
        raise DomainError(f"uncut must be 'raise' or 'exclude', got {uncut!r}")
    i_lo, j_lo, i_hi, j_hi = _check_roi(field.spec, roi)
    torch = _native.require_cuda()
    h = field.device_heights()
    sent = _field_sentinel(torch, field, h.device)
    st1, st2 = areal_moments_device(h, field.spec.n + 1, 1, 0,
                                    (i_lo, j_lo, i_hi - i_lo + 1, j_hi - j_lo + 1), sent,
                                    uncut == "exclude")
    return _finish_areal(st1[0], st2[0], uncut)


def _areal_plane(field: HeightField, roi, uncut: str) -> ArealMetrics:
    """Plane leveling on the device: normal-equation sums (pass 1), a 3x3
    solve on the host, deviation moments from the plane (pass 2)."""
    if uncut not in ("raise", "exclude"):
        raise DomainError(f"uncut must be 'raise' or 'exclude', got {uncut!r}")
    i_lo, j_lo, i_hi, j_hi = _check_roi(field.spec, roi)
    torch = _native.require_cuda()
    lib = _native.lib()
    h = field.device_heights()
    sent = _field_sentinel(torch, field, h.device)
    sc = _scratch(torch, h.device, 1)
    work = sc.data_ptr()
    out = sc[_native.WORK_DOUBLES:]
    rows, cols = i_hi - i_lo + 1, j_hi - j_lo + 1
    ld = field.spec.n + 1
    ex = int(uncut == "exclude")
    sp = _native.stream_ptr()
    _native.check(lib.msurf_areal_plane_pass1(h.data_ptr(), ld, 0, 1, i_lo, j_lo, rows, cols, sent.data_ptr(),
                                              ex, work, out.data_ptr(), sp))
    s1 = _native.readback(out[:10])
    if uncut == "raise" and s1[9] > 0:
        raise DomainError("roughness over unmachined stock is undefined: roi contains uncut cells")
    n = s1[0]
    if n <= 0:
        raise DomainError("no machined cells in roi")
    ata = np.array([[s1[3], s1[5], s1[1]], [s1[5], s1[4], s1[2]], [s1[1], s1[2], n]])
    atz = np.array([s1[7], s1[8], s1[6]])
    coef = np.linalg.lstsq(ata, atz, rcond=None)[0]
    cdev = torch.tensor(coef, dtype=torch.float64, device=h.device)
    _native.check(lib.msurf_areal_plane_pass2(h.data_ptr(), ld, 0, 1, i_lo, j_lo, rows, cols, sent.data_ptr(),
                                              ex, cdev.data_ptr(), work, out.data_ptr(), sp))
    s2 = _native.readback(out[:6])
    sa = float(s2[0] / n)
    sq = float(np.sqrt(s2[1] / n))
    spk, svl = float(s2[4]), float(-s2[5])
    if sq == 0.0:
        ssk = sku = None
    else:
        ssk = float((s2[2] / n) / sq ** 3)
        sku = float((s2[3] / n) / sq ** 4)
    return ArealMetrics(sa_um=sa, sq_um=sq, sp_um=spk, sv_um=svl, sz_um=spk + svl, ssk=ssk, sku=sku,
                        cell_count=int(n))


def _finish_areal(st1, st2, uncut) -> ArealMetrics:
    if uncut == "raise" and st1[4] > 0:
        raise DomainError("roughness over unmachined stock is undefined: roi contains uncut cells")
    if st1[3] <= 0:
        raise DomainError("no machined cells in roi")
    return _metrics_from_moments(st1, st2)


def areal_metrics_batch(fields, roi=None, uncut: str = "raise"):
    """Areal metrics of many fields: each run of consecutive same-shape fields
    that sit at a constant stride in one device buffer (the output of one
    simulate_batch launch group) is reduced in two launches; every run's
    passes are enqueued first and all results come back in ONE device-to-host
    copy. Returns a list of ArealMetrics or DomainError instances (per-sample
    status, dataset.py:177-180)."""
    if not fields:
        return []
    if uncut not in ("raise", "exclude"):
        raise DomainError(f"uncut must be 'raise' or 'exclude', got {uncut!r}")
    torch = _native.require_cuda()
    lib = _native.lib()
    devs = [f.device_heights() for f in fields]
    runs, a = [], 0  # (a, b, stride in doubles)
    while a < len(fields):
        b = a + 1
        spec = fields[a].spec
        st = None
        if b < len(fields) and fields[b].spec == spec and devs[b].device == devs[a].device:
            st = devs[b].data_ptr() - devs[a].data_ptr()
            if st <= 0 or st % 8:
                st = None
        if st is not None:
            while (b < len(fields) and fields[b].spec == spec and devs[b].device == devs[a].device
                   and devs[b].data_ptr() == devs[a].data_ptr() + (b - a) * st):
                b += 1
        runs.append((a, b, (st or 0) // 8))
        a = b
    res = [None] * len(runs)  # per run: (stats1, moments) or a DomainError for the run's one field
    todo = {}
    for r, (a, b, stride) in enumerate(runs):
        try:
            box = _check_roi(fields[a].spec, roi)
        except DomainError as exc:
            if b - a > 1:
                raise
            res[r] = exc
            continue
        todo.setdefault(devs[a].device, []).append((r, box))
    for dev, rs in todo.items():
        n_work = max(runs[r][1] - runs[r][0] for r, _ in rs)
        n_out = sum(runs[r][1] - runs[r][0] for r, _ in rs)
        sc = _scratch(torch, dev, n_work, n_out)
        outs = sc[n_work * _native.WORK_DOUBLES:]
        sp = _native.stream_ptr()
        pos, slots = 0, []
        for r, (i_lo, j_lo, i_hi, j_hi) in rs:
            a, b, stride = runs[r]
            n = b - a
            ss = [getattr(f, "_dev_sentinel", None) for f in fields[a:b]]
            if (all(x is not None and x.device == dev for x in ss)
                    and all(x.data_ptr() == ss[0].data_ptr() + 8 * k for k, x in enumerate(ss))):
                # the batch's own contiguous device sentinels (simulate_batch): no H2D copy
                sent = ss[0].as_strided((n,), (1,))
            else:
                sent = _sentinel_tensor(torch, [f.initial_height_mm for f in fields[a:b]], dev)
            _areal_enqueue(lib, devs[a], fields[a].spec.n + 1, n, stride,
                           (i_lo, j_lo, i_hi - i_lo + 1, j_hi - j_lo + 1), sent, uncut == "exclude",
                           sc.data_ptr(), outs[pos * 10: (pos + n) * 10], sp)
            slots.append((r, pos, n))
            pos += n
        both = _native.readback(outs[: n_out * 10])  # one read-back for every run on this device
        for r, p0, n in slots:
            res[r] = _split_moments(both[p0 * 10: (p0 + n) * 10], n)
    out = []
    for (a, b, _), rr in zip(runs, res):
        if isinstance(rr, DomainError):
            out.append(rr)
            continue
        for x, y in zip(*rr):
            try:
                out.append(_finish_areal(x, y, uncut))
            except DomainError as exc:
                out.append(exc)
    return out


def extract_profile(field: HeightField, direction: str, index=None, roi=None) -> LineProfile:
    """Feed-direction column (fixed x) or pick-feed row (fixed y) (roughness.py:138-180)."""
    spec = field.spec
    i_lo, j_lo, i_hi, j_hi = _check_roi(spec, roi)
    if direction == "feed":
        idx = round(spec.m / 2) if index is None else index
        if not i_lo <= idx <= i_hi:
            raise DomainError(f"feed profile index {idx} outside roi columns {i_lo}..{i_hi}")
        start, length, step = idx * (spec.n + 1) + j_lo, j_hi - j_lo + 1, 1
        positions = spec.y_coords()[j_lo:j_hi + 1]
    elif direction == "pickfeed":
        idx = round(spec.n / 2) if index is None else index
        if not j_lo <= idx <= j_hi:
            raise DomainError(f"pick-feed profile index {idx} outside roi rows {j_lo}..{j_hi}")
        start, length, step = i_lo * (spec.n + 1) + idx, i_hi - i_lo + 1, spec.n + 1
        positions = spec.x_coords()[i_lo:i_hi + 1]
    else:
        raise DomainError(f"direction must be 'feed' or 'pickfeed', got {direction!r}")
    if field.on_device:
        h = field.device_heights()
        heights = h[start: start + (length - 1) * step + 1: step].cpu().numpy()
    else:
        heights = field.heights[start: start + (length - 1) * step + 1: step].copy()
    if np.any(heights >= field.initial_height_mm):
        raise DomainError(f"{direction} profile at index {idx} crosses uncut cells")
    return LineProfile(direction=direction, index=idx, positions_mm=positions.copy(),
                       heights_mm=heights, spacing_mm=spec.spacing_mm)


_STARTS = {}  # (device, stream, profile offsets) -> device int64 tensor


def _starts_device(torch, dev, starts):
    """Device copy of the profile offsets. Repeated calls with the same
    profile set (the usual every-64th-row query) on the same stream reuse it
    (stream order puts its upload before every later use); a new set goes
    through pinned memory as an asynchronous H2D (a pageable copy would block
    the host until the stream drains)."""
    a = np.asarray(starts, dtype=np.int64)
    key = (dev.index, _native.stream_ptr(), a.tobytes())
    t = _STARTS.get(key)
    if t is None:
        t = torch.from_numpy(a).pin_memory().to(dev, non_blocking=True)
        if len(_STARTS) >= 32:
            try:
                _STARTS.pop(next(iter(_STARTS)), None)
            except (StopIteration, RuntimeError):  # emptied / resized by another thread
                pass
        _STARTS[key] = t
    return t


def _profiles_device(h_dev, n_surf, surf_stride, starts, length, step, sentinels_dev, exclude,
                     stats_in=None):
    """One msurf_profiles launch; returns the [n_surf, n_prof, 8] rows on the host."""
    torch = _native.require_cuda()
    lib = _native.lib()
    dev = h_dev.device
    n_prof = len(starts)
    st = _starts_device(torch, dev, starts)
    out = torch.empty(n_surf * n_prof * 8, dtype=torch.float64, device=dev)
    _native.check(lib.msurf_profiles(h_dev.data_ptr(), surf_stride, n_surf, st.data_ptr(), n_prof,
                                     length, step, sentinels_dev.data_ptr(), int(exclude),
                                     stats_in.data_ptr() if stats_in is not None else None,
                                     out.data_ptr(), _native.stream_ptr()))
    return out


def _finish_profile(row, idx, uncut) -> ProfileRoughness:
    s, n, n_unc, zmax, zmin, sabs, mean = row[:7]
    if uncut == "raise" and n_unc > 0:
        raise DomainError(f"profile at index {idx} crosses uncut cells")
    if n < 2:
        raise DomainError("line roughness needs at least 2 samples")
    rp, rv = float(zmax - mean), float(-(zmin - mean))
    return ProfileRoughness(index=int(idx), ra_um=float(sabs / n), rz_um=rp + rv, rp_um=rp, rv_um=rv,
                            sample_count=int(n))


def _finish_profiles(rows, indices, uncut):
    """_finish_profile over all rows at once (same IEEE operations per row,
    same first error in profile order)."""
    n, n_unc = rows[:, 1], rows[:, 2]
    bad = (n < 2) | ((n_unc > 0) if uncut == "raise" else False)
    if bad.any():
        k = int(np.argmax(bad))
        return [_finish_profile(rows[k], indices[k], uncut)]  # raises the reference's error
    mean = rows[:, 6]
    rp = rows[:, 3] - mean
    rv = -(rows[:, 4] - mean)
    cols = zip(indices, (rows[:, 5] / n).tolist(), (rp + rv).tolist(), rp.tolist(), rv.tolist(),
               n.astype(np.int64).tolist())
    return [ProfileRoughness(int(i), ra, rz, p, v, c) for i, ra, rz, p, v, c in cols]


def profile_roughness(field: HeightField, indices=None, direction: str = "feed", every: int | None = None,
                      roi=None, uncut: str = "raise"):
    """Ra and Rz of many profiles in one launch. ``every=64`` takes every 64th
    feed profile (fixed x index i = 0, 64, 128, ...) inside the ROI."""
    spec = field.spec
    i_lo, j_lo, i_hi, j_hi = _check_roi(spec, roi)
    if direction == "feed":
        if indices is None:
            indices = list(range(i_lo, i_hi + 1, every)) if every else [round(spec.m / 2)]
        for idx in indices:
            if not i_lo <= idx <= i_hi:
                raise DomainError(f"feed profile index {idx} outside roi columns {i_lo}..{i_hi}")
        starts = [idx * (spec.n + 1) + j_lo for idx in indices]
        length, step = j_hi - j_lo + 1, 1
    elif direction == "pickfeed":
        if indices is None:
            indices = list(range(j_lo, j_hi + 1, every)) if every else [round(spec.n / 2)]
        for idx in indices:
            if not j_lo <= idx <= j_hi:
                raise DomainError(f"pick-feed profile index {idx} outside roi rows {j_lo}..{j_hi}")
        starts = [i_lo * (spec.n + 1) + idx for idx in indices]
        length, step = i_hi - i_lo + 1, spec.n + 1
    else:
        raise DomainError(f"direction must be 'feed' or 'pickfeed', got {direction!r}")
    torch = _native.require_cuda()
    h = field.device_heights()
    sent = _field_sentinel(torch, field, h.device)
    rows = _profiles_device(h, 1, 0, starts, length, step, sent, uncut == "exclude")
    rows = _native.readback(rows).reshape(len(indices), 8)
    return _finish_profiles(rows, indices, uncut)


def line_roughness(profile: LineProfile) -> float:
    """Ra of a profile in µm (roughness.py:183-188), reduced on the device."""
    if profile.heights_mm.size < 2:
        raise DomainError("line roughness needs at least 2 samples")
    torch = _native.require_cuda()
    h = torch.from_numpy(np.ascontiguousarray(profile.heights_mm, dtype=np.float64)).cuda()
    sent = _sentinel_tensor(torch, [np.inf], h.device)
    row = _native.readback(_profiles_device(h, 1, 0, [0], h.numel(), 1, sent, False))
    return float(row[5] / row[1])
