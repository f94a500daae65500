import torch, time
n = 200_000_000 // 8
d = torch.empty(n, dtype=torch.float64, device="cuda")
h = torch.empty(n, dtype=torch.float64, pin_memory=True)
h.copy_(d); torch.cuda.synchronize()
for _ in range(3):
    t0 = time.perf_counter(); h.copy_(d, non_blocking=True); torch.cuda.synchronize(); t1 = time.perf_counter()
    d.copy_(h, non_blocking=True); torch.cuda.synchronize(); t2 = time.perf_counter()
    print(f"D2H {200/(t1-t0)/1e3:.1f} GB/s  H2D {200/(t2-t1)/1e3:.1f} GB/s")
