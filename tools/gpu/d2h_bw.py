import torch, time
dev = torch.device("cuda", 0)
for mb in (8, 64, 512):
    n = mb << 20
    src = torch.empty(n, dtype=torch.uint8, device=dev)
    dst = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    for _ in range(2): dst.copy_(src, non_blocking=True); torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(5): dst.copy_(src, non_blocking=True)
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t) / 5
    # two streams concurrently, two halves
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    h = n // 2
    t = time.perf_counter()
    for _ in range(5):
        with torch.cuda.stream(s1): dst[:h].copy_(src[:h], non_blocking=True)
        with torch.cuda.stream(s2): dst[h:].copy_(src[h:], non_blocking=True)
    torch.cuda.synchronize()
    dt2 = (time.perf_counter() - t) / 5
    hs = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    t = time.perf_counter()
    for _ in range(5): src.copy_(hs, non_blocking=True)
    torch.cuda.synchronize()
    dt3 = (time.perf_counter() - t) / 5
    print(f"{mb} MB: D2H {n/dt/1e9:.1f} GB/s, D2H 2 streams {n/dt2/1e9:.1f} GB/s, H2D {n/dt3/1e9:.1f} GB/s")
