"""Host<->device copy bandwidth with pinned buffers (diagnostic for the e2e numbers)."""
import time

import torch

n = 32_000_000  # 256 MB of doubles
h = torch.empty(n, dtype=torch.float64).pin_memory()
d = torch.empty(n, dtype=torch.float64, device="cuda")
for name, f in (("h2d", lambda: d.copy_(h, non_blocking=True)), ("d2h", lambda: h.copy_(d, non_blocking=True))):
    f()
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(5):
        f()
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t) / 5
    print(f"{name}: {n * 8 / dt / 1e9:.1f} GB/s")
