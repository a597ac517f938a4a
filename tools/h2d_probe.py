import torch, time
for mb in (32, 64, 256, 1024):
    n = mb * (1 << 20)
    hp = torch.empty(n, dtype=torch.uint8).pin_memory()
    dd = torch.empty(n, dtype=torch.uint8, device="cuda")
    dd.copy_(hp, non_blocking=True); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(4): dd.copy_(hp, non_blocking=True)
    e1.record(); torch.cuda.synchronize()
    print(mb, "MB", 4 * n / (e0.elapsed_time(e1) / 1e3) / 1e9, "GB/s")
    # two streams
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    d2 = torch.empty_like(dd); h2 = torch.empty(n, dtype=torch.uint8).pin_memory()
    torch.cuda.synchronize(); t = time.perf_counter()
    for _ in range(4):
        with torch.cuda.stream(s1): dd.copy_(hp, non_blocking=True)
        with torch.cuda.stream(s2): d2.copy_(h2, non_blocking=True)
    torch.cuda.synchronize(); print("  2 streams", 8 * n / (time.perf_counter() - t) / 1e9, "GB/s")
