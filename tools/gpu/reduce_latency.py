"""Host latency of the small reduction calls on a resident config 2 field."""
import sys, time
sys.path.insert(0, '.')
import numpy as np
import torch
import paper_2603_28160_b200 as ms
from paper_2603_28160_b200 import configs, roughness, _native

cfg, ext, meta = configs.config2()
res = ms.simulate(cfg, ext)
f = res.field
f.device_heights()
torch.cuda.synchronize()


def T(fn, n=200):
    for _ in range(10):
        fn()
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(n):
        fn()
    return (time.perf_counter() - t) / n * 1e6


dev = torch.device("cuda", 0)
x = torch.zeros(160, dtype=torch.float64, device=dev)
starts = list(range(0, 1001, 64))
print("areal_metrics us", T(lambda: ms.areal_metrics(f, uncut="exclude")))
print("profile_roughness us", T(lambda: ms.profile_roughness(f, every=64, uncut="exclude")))
print("readback(160 doubles) us", T(lambda: _native.readback(x)))
print(".cpu() 160 doubles us", T(lambda: x.cpu().numpy()))
print("pin_memory+H2D starts us", T(lambda: torch.from_numpy(np.asarray(starts, dtype=np.int64)).pin_memory().to(dev, non_blocking=True)))
print("torch.tensor(starts, device) us", T(lambda: torch.tensor(starts, dtype=torch.int64, device=dev)))
print("empty launch-ish (x.zero_) us", T(lambda: x.zero_()))
sent = roughness._field_sentinel(torch, f, dev)
h = f.device_heights()
st = [i * 1002 for i in range(0, 1001, 64)]
print("_profiles_device only us", T(lambda: roughness._profiles_device(h, 1, 0, st, 1001, 1, sent, True)))
