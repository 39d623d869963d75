import ctypes, sys
sys.path.insert(0,'.')
from paper_2603_28160_b200 import _native
import torch
torch.cuda.init()
lib=_native.lib(); r=ctypes.c_double()
for w in (0,3,4):
    _native.check(lib.msurf_microbench(w, ctypes.byref(r))); print(w, '%.4g'%r.value)
for L in range(1,33):
    _native.check(lib.msurf_microbench(32+L, ctypes.byref(r))); print('L',L,'%.4g instr/s  %.4g lines/s  %.4g lanes/s'%(r.value, r.value*L, r.value*(min(16,32) if L==1 else 32)))
