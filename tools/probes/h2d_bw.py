import torch, time
for gb in (1, 4):
    n = gb << 28
    h = torch.empty(n, dtype=torch.float32).pin_memory()
    d = torch.empty(n, dtype=torch.float32, device="cuda")
    d.copy_(h); torch.cuda.synchronize()
    t = time.perf_counter(); d.copy_(h, non_blocking=True); torch.cuda.synchronize(); dt = time.perf_counter() - t
    print(f"H2D {gb} GB: {gb*(1<<30)/dt/1e9:.1f} GB/s")
    t = time.perf_counter(); h.copy_(d, non_blocking=True); torch.cuda.synchronize(); dt = time.perf_counter() - t
    print(f"D2H {gb} GB: {gb*(1<<30)/dt/1e9:.1f} GB/s")
