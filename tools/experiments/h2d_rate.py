import torch, time
for gb in (1, 4, 8):
    n = gb << 28
    h = torch.empty(n, dtype=torch.int32, pin_memory=True)
    d = torch.empty(n, dtype=torch.int32, device="cuda")
    d.copy_(h, non_blocking=True); torch.cuda.synchronize()
    t = time.time()
    for _ in range(3):
        d.copy_(h, non_blocking=True)
    torch.cuda.synchronize()
    dt = (time.time() - t) / 3
    print(f"H2D {gb} GB: {gb * 2**30 / dt / 1e9:.1f} GB/s", flush=True)
    t = time.time(); h.copy_(d, non_blocking=True); torch.cuda.synchronize(); dt = time.time() - t
    print(f"D2H {gb} GB: {gb * 2**30 / dt / 1e9:.1f} GB/s", flush=True)
    del h, d
