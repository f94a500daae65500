"""D2H / H2D bandwidth into pinned memory: one copy vs chunks on several streams."""
import time
import torch

n = 6 * 2054 * 2055
d = torch.randn(n, dtype=torch.float64, device="cuda")
h = torch.empty(n, dtype=torch.float64, pin_memory=True)
h.copy_(d.cpu())
for k in (1, 2, 4, 8):
    streams = [torch.cuda.Stream() for _ in range(k)]
    for rep in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        ch = (n + k - 1) // k
        for i, s in enumerate(streams):
            with torch.cuda.stream(s):
                h[i * ch:(i + 1) * ch].copy_(d[i * ch:(i + 1) * ch], non_blocking=True)
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        for i, s in enumerate(streams):
            with torch.cuda.stream(s):
                d[i * ch:(i + 1) * ch].copy_(h[i * ch:(i + 1) * ch], non_blocking=True)
        torch.cuda.synchronize()
        t2 = time.perf_counter()
    print(f"chunks {k}: D2H {n * 8 / (t1 - t0) / 1e9:.1f} GB/s  H2D {n * 8 / (t2 - t1) / 1e9:.1f} GB/s")
