"""Plain pinned D2H of a 1.08 GB buffer with 1, 2 and 4 concurrent streams (copy-engine parallelism).  GPU tool."""
import time
import torch
n = 1078 * 1024 * 1024 // 4
src = torch.empty(n, dtype=torch.int32, device="cuda")
dst = torch.empty(n, dtype=torch.int32, pin_memory=True)
for ns in (1, 2, 4, 1):
    streams = [torch.cuda.Stream() for _ in range(ns)]
    chunk = n // ns
    def go():
        for i, s in enumerate(streams):
            with torch.cuda.stream(s):
                dst[i * chunk:(i + 1) * chunk].copy_(src[i * chunk:(i + 1) * chunk], non_blocking=True)
        torch.cuda.synchronize()
    go(); go()
    t = time.perf_counter()
    for _ in range(5):
        go()
    dt = (time.perf_counter() - t) / 5
    print(f"{ns} streams: {dt * 1e3:.2f} ms  {n * 4 / dt / 1e9:.1f} GB/s")
