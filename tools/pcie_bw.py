"""Host<->device copy bandwidth from page-locked memory (the e2e floor)."""
import time

import torch

for gb in (0.5, 2.0):
    n = int(gb * (1 << 30))
    h = torch.empty(n, dtype=torch.uint8).pin_memory()
    d = torch.empty(n, dtype=torch.uint8, device="cuda")
    for direction in ("h2d", "d2h"):
        best = 1e9
        for _ in range(5):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            if direction == "h2d":
                d.copy_(h, non_blocking=True)
            else:
                h.copy_(d, non_blocking=True)
            torch.cuda.synchronize()
            best = min(best, time.perf_counter() - t0)
        print(f"{direction} {gb:.1f} GiB: {n / best / 1e9:.1f} GB/s", flush=True)
