"""Host->device bandwidth of a 34.4 GB pinned buffer (the C4 matrix) with 1, 2
and 4 concurrent streams / copy engines (e2e floor of bench.py)."""
import time

import torch

n = 34359738368 // 8
h = torch.empty(n, dtype=torch.float64, pin_memory=True)
d = torch.empty(n, dtype=torch.float64, device="cuda")
for ns in (1, 2, 4, 1):
    s = [torch.cuda.Stream() for _ in range(ns)]
    best = 0.0
    for it in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        q = n // ns
        for i in range(ns):
            with torch.cuda.stream(s[i]):
                d[i * q:(i + 1) * q].copy_(h[i * q:(i + 1) * q], non_blocking=True)
        torch.cuda.synchronize()
        best = max(best, 34.36 / (time.perf_counter() - t0))
    print(f"h2d {ns} stream(s): {best:.2f} GB/s", flush=True)
# chunked on one stream in 4096-column pieces of a 65536-row matrix (the upload pipeline's granularity)
for chunk_cols in (1024, 4096, 8192):
    q = 65536 * chunk_cols
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for i in range(0, n, q):
        d[i:i + q].copy_(h[i:i + q], non_blocking=True)
    torch.cuda.synchronize()
    print(f"h2d chunks of {chunk_cols} columns: {34.36 / (time.perf_counter() - t0):.2f} GB/s", flush=True)
