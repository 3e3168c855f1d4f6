import torch, time
for mb in (2.4, 24, 240):
    n = int(mb * 1e6 / 8)
    h = torch.empty(n, dtype=torch.float64).pin_memory()
    d = torch.empty(n, dtype=torch.float64, device="cuda")
    for _ in range(3):
        d.copy_(h, non_blocking=True); torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(20):
        d.copy_(h, non_blocking=True); torch.cuda.synchronize()
    dt = (time.perf_counter() - t) / 20
    t = time.perf_counter()
    for _ in range(20):
        h.copy_(d, non_blocking=True); torch.cuda.synchronize()
    dt2 = (time.perf_counter() - t) / 20
    print(f"{mb} MB: H2D {dt*1e6:.0f} us ({mb/1e3/dt:.1f} GB/s), D2H {dt2*1e6:.0f} us ({mb/1e3/dt2:.1f} GB/s)")
