import ctypes, sys
sys.path.insert(0, '.')
import torch
from paper_2603_28160_b200 import _native
torch.cuda.init()
lib = _native.lib()
r = ctypes.c_double(0.0)
for w, name in [(0, "DADD/DMUL ops/s"), (1, "DFMA/s"), (2, "RED.MIN.64 random 128MiB /s"), (3, "RED.MIN.64 random 32MiB /s"), (4, "RED.MIN.64 warp-run 32MiB /s")]:
    _native.check(lib.msurf_microbench(w, ctypes.byref(r)))
    print(f"MB {w} {name}: {r.value:.4g}")
