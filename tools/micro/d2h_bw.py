import torch, time
n = 1920*1080*3
d = torch.empty(n, dtype=torch.float32, device='cuda')
h = [torch.empty(n, dtype=torch.float32, pin_memory=True) for _ in range(4)]
torch.cuda.synchronize()
for rep in range(2):
    t0 = time.perf_counter()
    for i in range(200):
        h[i % 4].copy_(d, non_blocking=True)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    print(f"D2H {200*n*4/dt/1e9:.1f} GB/s, {dt/200*1e6:.0f} us per 24.9 MB frame")
s2 = torch.cuda.Stream()
for rep in range(2):
    t0 = time.perf_counter()
    with torch.cuda.stream(s2):
        for i in range(100):
            h[i % 4].copy_(d, non_blocking=True)
    for i in range(100):
        h[(i+2) % 4].copy_(d, non_blocking=True)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    print(f"2 streams D2H {200*n*4/dt/1e9:.1f} GB/s")
