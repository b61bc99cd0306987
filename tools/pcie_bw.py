import torch, time
n = 67_000_000 // 4 * 4
h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
d = torch.empty(n, dtype=torch.uint8, device="cuda")
for direction in ("h2d", "d2h"):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(20):
        if direction == "h2d":
            d.copy_(h, non_blocking=True)
        else:
            h.copy_(d, non_blocking=True)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    print(direction, round(20 * n / dt / 1e9, 1), "GB/s")
