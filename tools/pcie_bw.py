"""Host<->device copy bandwidth from pinned memory with 1..4 concurrent
streams (one copy engine each), 8 GB D2H / 0.4 GB H2D like bench.py's e2e."""
import time

import torch

GB = 1 << 30
src = torch.empty(8 * GB // 4, dtype=torch.float32, device="cuda")
dst = torch.empty(8 * GB // 4, dtype=torch.float32).pin_memory()
hsrc = torch.empty(GB // 4, dtype=torch.float32).pin_memory()
ddst = torch.empty(GB // 4, dtype=torch.float32, device="cuda")
for ns in (1, 2, 3, 4, 8):
    streams = [torch.cuda.Stream() for _ in range(ns)]
    n = src.numel()
    for rep in range(2):
        torch.cuda.synchronize()
        t = time.perf_counter()
        for i, s in enumerate(streams):
            a, b = n * i // ns, n * (i + 1) // ns
            with torch.cuda.stream(s):
                dst[a:b].copy_(src[a:b], non_blocking=True)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t
    print(f"D2H {ns} streams: {8 / dt:.1f} GiB/s", flush=True)
    m = hsrc.numel()
    torch.cuda.synchronize()
    t = time.perf_counter()
    for i, s in enumerate(streams):
        a, b = m * i // ns, m * (i + 1) // ns
        with torch.cuda.stream(s):
            ddst[a:b].copy_(hsrc[a:b], non_blocking=True)
    torch.cuda.synchronize()
    print(f"H2D {ns} streams: {1 / (time.perf_counter() - t):.1f} GiB/s", flush=True)
