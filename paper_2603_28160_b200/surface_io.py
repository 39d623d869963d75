"""Surface files and exports — drop-in for millsurf/surface_io.py:1-146.

SRTF (surface_io.py:3-20): 48-byte little-endian header ``<4sIIIdddd`` =
magic "SRTF", version 1, m, n, spacing, x_min, y_min, sentinel, then the
(m+1)(n+1) fp64 heights row-major over (i, j). The fp64 payload is exactly
the device Z-map's bytes, so ``write_surface`` streams a field that lives in
HBM straight to disk: fixed-size chunks are copied D2H into two pinned
buffers on a side stream while the previous chunk is written (copy and file
write overlap), and the file appears under its final name only after an
atomic rename. ``read_surface`` validates magic, version and payload length
like the reference (SurfaceFormatError) and can place the heights on the GPU.

Graymap (surface_io.py:100-131) is computed on the device by two
libmsurf kernels (range reduction over the machined cells, then a
transposing quantiser that writes the big-endian 16-bit image), so only
2 bytes per node cross PCIe. The CSV view is text formatting and stays on the
host, byte-identical to the reference's ``f"{v:.6f}"`` rows.
"""

from __future__ import annotations

import json
import os
import struct
from pathlib import Path

import numpy as np

from . import _native
from .errors import DomainError, SurfaceFormatError
from .grid import GridSpec, HeightField
from .roughness import _check_roi, areal_metrics

__all__ = ["MAGIC", "VERSION", "GRAY_MID", "atomic_write_bytes", "write_surface", "read_surface",
           "write_heights_csv", "write_graymap", "graymap_pixels", "export_views"]

MAGIC = b"SRTF"
VERSION = 1
_HEADER = struct.Struct("<4sIIIdddd")
GRAY_MID = 32768
MM_TO_UM = 1000.0
STREAM_CHUNK_BYTES = 64 << 20


def _tmp_name(path: Path) -> Path:
    return path.with_name(path.name + ".tmp")


def atomic_write_bytes(path, payload: bytes) -> None:
    """Whole-file atomic write: temp name, then rename (surface_io.py:42-47)."""
    path = Path(path)
    tmp = _tmp_name(path)
    with open(tmp, "wb") as fh:
        fh.write(payload)
    os.replace(tmp, path)


def _header(field: HeightField) -> bytes:
    g = field.spec
    return _HEADER.pack(MAGIC, VERSION, g.m, g.n, g.spacing_mm, g.x_min_mm, g.y_min_mm, field.initial_height_mm)


def _stream_device_payload(fh, dev, chunk_bytes: int) -> None:
    """D2H of a contiguous fp64 device tensor in chunks, double-buffered in
    pinned memory: chunk k copies on a side stream while chunk k-1 is
    written to ``fh``."""
    import torch

    n = dev.numel()
    per = max(1, chunk_bytes // 8)
    bounds = [(lo, min(n, lo + per)) for lo in range(0, n, per)]
    bufs = [torch.empty(min(per, n), dtype=torch.float64, pin_memory=True) for _ in range(min(2, len(bounds)))]
    evs = [torch.cuda.Event() for _ in bufs]
    side = torch.cuda.Stream(device=dev.device)
    side.wait_stream(torch.cuda.current_stream(dev.device))  # after the field's producer

    def flush(k):
        evs[k % 2].synchronize()
        lo, hi = bounds[k]
        fh.write(memoryview(bufs[k % 2][: hi - lo].numpy()).cast("B"))

    for k, (lo, hi) in enumerate(bounds):
        with torch.cuda.stream(side):  # bufs[k % 2] was flushed at iteration k - 1
            bufs[k % 2][: hi - lo].copy_(dev[lo:hi], non_blocking=True)
            evs[k % 2].record(side)
        if k:
            flush(k - 1)
    if bounds:
        flush(len(bounds) - 1)


def write_surface(field: HeightField, path, *, chunk_bytes: int = STREAM_CHUNK_BYTES) -> None:
    """SRTF writer (surface_io.py:50-61). A device-resident field is streamed
    from HBM without materialising a host copy of the whole map."""
    path = Path(path)
    tmp = _tmp_name(path)
    with open(tmp, "wb") as fh:
        fh.write(_header(field))
        if field.on_device and field._pending is None:
            _stream_device_payload(fh, field.device_heights().reshape(-1), chunk_bytes)
        else:
            fh.write(field.heights.astype("<f8", copy=False).tobytes())
    os.replace(tmp, path)


def read_surface(path, *, device: bool = False) -> HeightField:
    """SRTF reader (surface_io.py:64-83): rejects bad magic, unknown versions
    and payloads whose length disagrees with the header. ``device=True``
    uploads the heights to the current GPU (the roughness kernels then run
    on them without another copy)."""
    blob = Path(path).read_bytes()
    if len(blob) < _HEADER.size:
        raise SurfaceFormatError(f"{path}: file shorter than the {_HEADER.size}-byte header")
    magic, version, m, n, spacing, x_min, y_min, sentinel = _HEADER.unpack_from(blob)
    if magic != MAGIC:
        raise SurfaceFormatError(f"{path}: bad magic {magic!r}, expected {MAGIC!r}")
    if version != VERSION:
        raise SurfaceFormatError(f"{path}: unsupported format version {version}")
    expected = (m + 1) * (n + 1) * 8
    payload = memoryview(blob)[_HEADER.size:]
    if len(payload) != expected:
        raise SurfaceFormatError(f"{path}: payload is {len(payload)} bytes, header promises {expected} "
                                 f"({m + 1}x{n + 1} float64)")
    heights = np.frombuffer(payload, dtype="<f8").astype(np.float64)
    spec = GridSpec(spacing_mm=spacing, x_min_mm=x_min, y_min_mm=y_min, m=m, n=n)
    if device:
        import torch

        dev = torch.from_numpy(heights).pin_memory().to("cuda", non_blocking=True)
        return HeightField(spec, sentinel, device=dev)
    return HeightField(spec, sentinel, heights)


def write_heights_csv(field: HeightField, path, roi=None) -> None:
    """Heights in um; header row = x coordinates (mm), then one row per y
    node across x (surface_io.py:86-97), byte-identical formatting."""
    g = field.spec
    i_lo, j_lo, i_hi, j_hi = _check_roi(g, roi)
    block = field.as_array()[i_lo: i_hi + 1, j_lo: j_hi + 1] * MM_TO_UM
    xs = g.x_coords()[i_lo: i_hi + 1]
    lines = [",".join(f"{x:.6f}" for x in xs)]
    lines.extend(",".join(f"{v:.6f}" for v in col) for col in block.T)
    atomic_write_bytes(path, ("\n".join(lines) + "\n").encode())


def graymap_pixels(field: HeightField, roi=None) -> np.ndarray:
    """The P5 image body on the device: (cols, rows) big-endian uint16
    (image row = y node), min-max normalised over the machined cells."""
    import torch

    lib = _native.lib()
    g = field.spec
    i_lo, j_lo, i_hi, j_hi = _check_roi(g, roi)
    rows, cols = i_hi - i_lo + 1, j_hi - j_lo + 1
    h = field.device_heights()
    dev = h.device
    sent = torch.tensor([field.initial_height_mm], dtype=torch.float64, device=dev)
    work = torch.empty(_native.WORK_DOUBLES + 3, dtype=torch.float64, device=dev)
    rng3 = work[_native.WORK_DOUBLES:]
    sp = _native.stream_ptr()
    _native.check(lib.msurf_graymap_range(h.data_ptr(), g.n + 1, i_lo, j_lo, rows, cols, sent.data_ptr(),
                                          work.data_ptr(), rng3.data_ptr(), sp))
    pix = torch.empty(rows * cols, dtype=torch.int16, device=dev)
    _native.check(lib.msurf_graymap_pixels(h.data_ptr(), g.n + 1, i_lo, j_lo, rows, cols, sent.data_ptr(),
                                           rng3.data_ptr(), pix.data_ptr(), sp))
    if int(rng3[2].item()) == 0:
        raise DomainError("graymap export needs at least one machined cell in the roi")
    out = torch.empty(pix.shape, dtype=torch.int16, pin_memory=True)
    out.copy_(pix)
    return out.numpy().view(">u2").reshape(cols, rows)


def write_graymap(field: HeightField, path, roi=None) -> None:
    """16-bit binary PGM (P5), uncut -> 0, flat machined -> mid-gray
    (surface_io.py:100-131); quantised on the GPU."""
    img = graymap_pixels(field, roi)
    header = f"P5\n{img.shape[1]} {img.shape[0]}\n65535\n".encode()
    atomic_write_bytes(path, header + img.tobytes())


def export_views(field: HeightField, out_dir, roi=None, basename: str = "surface") -> dict:
    """CSV grid, graymap and metrics JSON for a roi (surface_io.py:134-146)."""
    out_dir = Path(out_dir)
    out_dir.mkdir(parents=True, exist_ok=True)
    paths = {"csv": out_dir / f"{basename}.csv", "graymap": out_dir / f"{basename}.pgm",
             "metrics": out_dir / f"{basename}_metrics.json"}
    # device work first (graymap, metrics), then the host-side CSV text
    write_graymap(field, paths["graymap"], roi)
    metrics = areal_metrics(field, roi)
    atomic_write_bytes(paths["metrics"], (json.dumps(metrics.to_json_dict(), indent=2) + "\n").encode())
    write_heights_csv(field, paths["csv"], roi)
    return paths
