"""ctypes binding of libmsurf.so (include/msurf.h) and device plumbing.

PyTorch is used only for device memory, pinned staging buffers and the
current CUDA stream. Every compute step runs in libmsurf.so; if the library
or a CUDA device is missing the product raises NativeUnavailableError —
there is no CPU fallback.
"""

from __future__ import annotations

import ctypes
import os
import threading

import numpy as np

from .errors import MillsurfError, NativeUnavailableError

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("MSURF_LIB") or os.path.join(_HERE, "libmsurf.so")
ABI_VERSION = 7
NUM_CTRS = 5
SWEEP_DIAG = 0x100  # MSURF_SWEEP_DIAG: count deposits/atomics per point
SWEEP_TRACE = 0x200  # MSURF_SWEEP_TRACE: diagnostics + a trace of every RED.MIN (roofline only)
SWEEP_WIDE = 0x400  # MSURF_SWEEP_WIDE: eight-warp 64-step CTAs for a tilt by-value launch
RED_BLOCKS = 1024
WORK_DOUBLES = RED_BLOCKS * 10  # MSURF_WORK_DOUBLES: reduction scratch per surface

c_double, c_int64, c_int32, c_void_p = ctypes.c_double, ctypes.c_int64, ctypes.c_int32, ctypes.c_void_p


class MsurfJob(ctypes.Structure):
    """Mirror of msurf_job (include/msurf.h)."""

    _fields_ = [
        ("spacing", c_double), ("x_min", c_double), ("y_min", c_double),
        ("m", c_int64), ("n", c_int64), ("j_lo", c_int64), ("j_hi", c_int64), ("ld", c_int64),
        ("keys", c_void_p),
        ("t_start", c_double), ("dt", c_double), ("steps", c_int64),
        ("step_lo", c_int64), ("step_hi", c_int64),
        ("y0", c_double), ("feed_speed", c_double), ("omega", c_double),
        ("tooth_base", c_void_p), ("tooth_rows", c_void_p),
        ("pts", c_void_p), ("tooth_box", c_void_p), ("chunk_circ", c_void_p), ("chunk_f32", c_void_p),
        ("pass_x0", c_void_p),
        ("tilt_c", c_double), ("tilt_s", c_double), ("zoff", c_double),
        ("vib_amp", c_double), ("vib_omega", c_double), ("vib_phase", c_double),
        ("trig_table", c_void_p), ("vib_table", c_void_p),
        ("traj", c_void_p), ("min_index", c_void_p), ("counters", c_void_p), ("zcap", c_void_p),
        ("stage", c_void_p),
        ("teeth", c_int32), ("points", c_int32), ("passes", c_int32), ("tooth_lo", c_int32),
        ("tooth_n", c_int32), ("reserved0", c_int32),
    ]


# the same layout as a NumPy structured dtype: SweepBatch builds its descriptor
# tables as arrays of these rows (one np.array call per launch group)
JOB_DTYPE = np.dtype(MsurfJob)


class MsurfGeomIn(ctypes.Structure):
    """Mirror of msurf_geom_in (include/msurf.h)."""

    _fields_ = [
        ("mode", c_int32), ("teeth", c_int32), ("points", c_int32), ("profile", c_int32),
        ("radius", c_double), ("half", c_double), ("kmax", c_double), ("tan_beta_over_r", c_double),
        ("tilt_c", c_double), ("tilt_s", c_double), ("z0", c_double),
        ("rows", c_void_p), ("delta", c_void_p), ("runout_xy", c_void_p),
    ]


# the same layout as a NumPy structured dtype (planner fills B records at once)
GEOM_IN_DTYPE = np.dtype(MsurfGeomIn)

EXPORTS = {
    "msurf_abi_version": (ctypes.c_int, []),
    "msurf_zcap_tile": (ctypes.c_int, []),
    "msurf_last_error": (ctypes.c_char_p, []),
    "msurf_sizeof_job": (ctypes.c_int, []),
    "msurf_tile_steps": (ctypes.c_int, []),
    "msurf_fill_keys": (ctypes.c_int, [c_void_p, c_int64, c_int32, c_void_p, c_void_p]),
    "msurf_sweep": (ctypes.c_int, [c_void_p, c_int32, c_void_p, c_int64, c_int32, c_int32, c_void_p, c_void_p]),
    "msurf_sweep_job": (ctypes.c_int, [c_void_p, c_int32, c_int32, c_void_p]),
    "msurf_decode_strips": (ctypes.c_int, [c_void_p, c_void_p, c_int64, c_int64, c_int32, c_void_p, c_void_p,
                                           c_void_p, c_void_p]),
    "msurf_decode": (ctypes.c_int, [c_void_p, c_int64, c_int32, c_void_p, c_void_p, c_void_p]),
    "msurf_zcap_refresh": (ctypes.c_int, [c_void_p, c_int64, c_int64, c_int64, c_void_p, c_void_p, c_void_p,
                                          c_void_p]),
    "msurf_sweep_job_capped": (ctypes.c_int, [c_void_p, c_int32, c_int32, c_void_p, c_void_p]),
    "msurf_sweep_jobs_capped": (ctypes.c_int, [c_void_p, c_int32, c_int32, c_int32, c_void_p, c_int32, c_void_p,
                                               c_int64, c_int32, c_void_p]),
    "msurf_stage_bytes": (ctypes.c_int, [c_void_p, c_int32, ctypes.POINTER(c_int64)]),
    "msurf_anchor_stream": (c_void_p, [c_int32]),
    "msurf_stream_wait": (ctypes.c_int, [c_void_p, c_void_p]),
    "msurf_areal_pass1": (ctypes.c_int, [c_void_p, c_int64, c_int64, c_int32, c_int64, c_int64,
                                         c_int64, c_int64, c_void_p, c_int32, c_void_p, c_void_p,
                                         c_void_p]),
    "msurf_areal_pass2": (ctypes.c_int, [c_void_p, c_int64, c_int64, c_int32, c_int64, c_int64,
                                         c_int64, c_int64, c_void_p, c_int32, c_void_p, c_void_p,
                                         c_void_p, c_void_p]),
    "msurf_areal_plane_pass1": (ctypes.c_int, [c_void_p, c_int64, c_int64, c_int32, c_int64, c_int64,
                                               c_int64, c_int64, c_void_p, c_int32, c_void_p, c_void_p,
                                               c_void_p]),
    "msurf_areal_plane_pass2": (ctypes.c_int, [c_void_p, c_int64, c_int64, c_int32, c_int64, c_int64,
                                               c_int64, c_int64, c_void_p, c_int32, c_void_p, c_void_p,
                                               c_void_p, c_void_p]),
    "msurf_profiles": (ctypes.c_int, [c_void_p, c_int64, c_int32, c_void_p, c_int32, c_int64,
                                      c_int64, c_void_p, c_int32, c_void_p, c_void_p, c_void_p]),
    "msurf_graymap_range": (ctypes.c_int, [c_void_p, c_int64, c_int64, c_int64, c_int64, c_int64, c_void_p,
                                           c_void_p, c_void_p, c_void_p]),
    "msurf_graymap_pixels": (ctypes.c_int, [c_void_p, c_int64, c_int64, c_int64, c_int64, c_int64, c_void_p,
                                            c_void_p, c_void_p, c_void_p]),
    "msurf_microbench": (ctypes.c_int, [c_int32, ctypes.POINTER(c_double)]),
    "msurf_trace_arm": (ctypes.c_int, [c_void_p, c_int64, c_void_p, c_void_p]),
    "msurf_red_lines": (ctypes.c_int, [c_void_p, c_int64, c_void_p, c_void_p]),
    "msurf_red_sectors": (ctypes.c_int, [c_void_p, c_int64, c_void_p, c_void_p, c_void_p]),
    "msurf_host_alloc": (c_void_p, [c_int64]),
    "msurf_host_free": (ctypes.c_int, [c_void_p]),
    "msurf_readback": (ctypes.c_int, [c_void_p, c_void_p, c_int64, c_void_p]),
    "msurf_readback_sync": (ctypes.c_int, [c_void_p, c_void_p, c_int64, c_void_p]),
    "msurf_copy2d_d2h": (ctypes.c_int, [c_void_p, c_int64, c_void_p, c_int64, c_int64, c_int64, c_void_p]),
    "msurf_plan_geometry": (ctypes.c_int, [c_void_p, c_void_p, c_void_p, c_void_p, c_void_p]),
    "msurf_plan_geometry_many": (ctypes.c_int, [c_void_p, c_int32, c_void_p, c_void_p, c_void_p, c_void_p, c_int32]),
    "msurf_plan_finish_many": (ctypes.c_int, [c_void_p, c_int32, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p,
                                              c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_int32]),
    "msurf_plan_finish": (ctypes.c_int, [c_void_p, c_void_p, c_void_p, c_void_p, c_double, c_void_p, c_void_p,
                                         c_void_p, c_void_p, c_void_p, c_void_p, c_void_p]),
}

_lib = None
_lock = threading.Lock()


def load_library(path: str = LIB_PATH):
    """Load libmsurf.so and declare every exported symbol (no GPU needed)."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(path):
            raise NativeUnavailableError(
                f"{path} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`")
        lib = ctypes.CDLL(path)
        for name, (res, args) in EXPORTS.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        if lib.msurf_abi_version() != ABI_VERSION:
            raise NativeUnavailableError("libmsurf.so ABI version mismatch; rebuild")
        if lib.msurf_sizeof_job() != ctypes.sizeof(MsurfJob):
            raise NativeUnavailableError("msurf_job layout mismatch between header and binding")
        _lib = lib
        return lib


def lib():
    return _lib if _lib is not None else load_library()


def check(rc: int) -> None:
    if rc != 0:
        raise MillsurfError("libmsurf: " + lib().msurf_last_error().decode())


_torch_ok = None


def require_cuda():
    global _torch_ok
    if _torch_ok is not None:
        return _torch_ok
    import torch

    if not torch.cuda.is_available():
        raise NativeUnavailableError("no CUDA device: the FSM sweep runs only on the GPU")
    lib()
    _torch_ok = torch
    return torch


def _raw_stream_query():
    """The private raw current-stream query (~0.3 us instead of ~8 us for a
    torch.cuda.Stream object) when this torch build has it, else None."""
    import torch

    c = torch._C
    f, g = getattr(c, "_cuda_getCurrentRawStream", None), getattr(c, "_cuda_getDevice", None)
    if f is None or g is None:
        return None
    try:
        f(g())
    except Exception:  # renamed / changed signature in this build
        return None
    return lambda: f(g())


_RAW_STREAM = []


def stream_ptr(stream=None) -> int:
    """Raw cudaStream_t of ``stream`` or of the current device's current
    stream; falls back to the public torch.cuda.current_stream() when the
    private fast query is unavailable."""
    if stream is not None:
        return int(stream.cuda_stream)
    if not _RAW_STREAM:
        _RAW_STREAM.append(_raw_stream_query())
    q = _RAW_STREAM[0]
    if q is not None:
        return q()
    import torch

    return int(torch.cuda.current_stream().cuda_stream)


READBACK_MAX = 1 << 20  # bytes; larger results take a copy-engine D2H
_mailboxes = {}
_mailbox_lock = threading.Lock()


def readback(t) -> np.ndarray:
    """Host copy of a small device tensor (reduction results). The values are
    stored into mapped page-locked memory by a kernel on the current stream
    (msurf_readback), so the read does not queue behind a large D2H copy
    already in flight on the copy engine (the heights prefetch)."""
    import torch

    nbytes = t.numel() * t.element_size()
    if nbytes == 0 or nbytes > READBACK_MAX or nbytes % 8 or not t.is_contiguous() or t.device.type != "cuda":
        return t.cpu().numpy()
    dev = t.device.index if t.device.index is not None else torch.cuda.current_device()
    with _mailbox_lock:
        mb = _mailboxes.get(dev)
        if mb is None:
            ptr = lib().msurf_host_alloc(READBACK_MAX)
            if not ptr:
                raise NativeUnavailableError(f"msurf_host_alloc: {lib().msurf_last_error().decode()}")
            mb = _mailboxes[dev] = (np.frombuffer((ctypes.c_char * READBACK_MAX).from_address(ptr), dtype=np.uint8),
                                    ptr)
        box, ptr = mb
        # kernel + stream sync in one foreign call (ctypes drops the GIL meanwhile)
        check(lib().msurf_readback_sync(t.data_ptr(), ptr, nbytes, stream_ptr()))
        dt = _NP_DTYPES.get(t.dtype)
        if dt is None:
            dt = _NP_DTYPES[t.dtype] = np.dtype(str(t.dtype).replace("torch.", ""))
        return box[:nbytes].view(dt).copy().reshape(tuple(t.shape))


_NP_DTYPES = {}


class Arena:
    """Packs many small host arrays into one pinned staging buffer and one
    device buffer, so a sweep's inputs cross PCIe in a single H2D copy."""

    def __init__(self):
        self._parts = []
        self._direct = []  # (offset, page-locked torch tensor): DMA'd after the staged copy
        self.size = 0

    def add(self, arr, pinned=None) -> int:
        """Reserve room for ``arr``; ``pinned`` = a page-locked torch uint8
        tensor holding the same bytes: copied to HBM by DMA, not staged."""
        a = arr if isinstance(arr, np.ndarray) and arr.flags.c_contiguous else np.ascontiguousarray(arr)
        off = (self.size + 255) & ~255
        if pinned is not None and pinned.numel() == a.nbytes:
            self._direct.append((off, pinned))
            self._parts.append((off, None))
        else:
            self._parts.append((off, a))
        self.size = off + a.nbytes
        return off

    def reserve(self, nbytes: int) -> int:
        off = (self.size + 255) & ~255
        self._parts.append((off, None))
        self.size = off + nbytes
        return off

    def upload(self, device, fill_structs=None):
        """Allocate the device buffer, let ``fill_structs(base_ptr)`` return
        [(offset, bytes)] (descriptors holding device pointers), then copy
        everything with one cudaMemcpyAsync on the current stream."""
        import torch

        dev = torch.empty(max(self.size, 1), dtype=torch.uint8, device=device)
        base = dev.data_ptr()
        extra = fill_structs(base) if fill_structs else []
        # pinned staging from torch's caching host allocator: a block is reused
        # only after the copy that read it has completed (event recorded by the
        # non-blocking copy), so uploads of consecutive launch groups never wait
        stage = torch.empty(max(self.size, 1), dtype=torch.uint8, pin_memory=True)
        hp = stage.data_ptr()
        # ctypes.memmove drops the GIL while it copies (a planner thread keeps running)
        for off, a in self._parts:
            if a is not None and a.nbytes:
                ctypes.memmove(hp + off, a.ctypes.data, a.nbytes)
        for off, b in extra:
            b = b if isinstance(b, np.ndarray) else np.frombuffer(b, dtype=np.uint8)
            ctypes.memmove(hp + off, b.ctypes.data, b.nbytes)
        dev.copy_(stage, non_blocking=True)
        for off, t in self._direct:  # torch records the copies: the pinned blocks are not reused early
            dev[off: off + t.numel()].copy_(t, non_blocking=True)
        return dev
