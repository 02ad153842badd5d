import torch, time
n = 34359738368 // 8
h = torch.empty(n, dtype=torch.float64, pin_memory=True)
d = torch.empty(n, dtype=torch.float64, device="cuda")
for it in range(3):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    d.copy_(h, non_blocking=True); torch.cuda.synchronize()
    t = time.perf_counter() - t0
    print("h2d GB/s", 34.36 / t)
s = [torch.cuda.Stream() for _ in range(4)]
for it in range(2):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    q = n // 4
    for i in range(4):
        with torch.cuda.stream(s[i]):
            d[i*q:(i+1)*q].copy_(h[i*q:(i+1)*q], non_blocking=True)
    torch.cuda.synchronize()
    print("h2d 4 streams GB/s", 34.36 / (time.perf_counter() - t0))
