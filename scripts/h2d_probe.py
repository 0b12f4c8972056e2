import torch, time, platform, os
print(platform.machine(), os.cpu_count())
n = 80 * 2**20
h = torch.empty(n, dtype=torch.uint8).pin_memory(); d = torch.empty(n, dtype=torch.uint8, device="cuda")
h.fill_(7)
for name, fn in [("h2d", lambda: d.copy_(h, non_blocking=True)), ("d2h", lambda: h.copy_(d, non_blocking=True))]:
    fn(); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(20): fn()
    torch.cuda.synchronize(); t = (time.perf_counter() - t0) / 20
    print(name, round(n / t / 1e9, 1), "GB/s")
g = torch.cuda.CUDAGraph()
s = torch.cuda.Stream()
d.zero_(); torch.cuda.synchronize()
with torch.cuda.graph(g):
    d.copy_(h, non_blocking=True)
g.replay(); torch.cuda.synchronize()
print("graph copy ok:", bool((d == 7).all()))
h[:10] = 3; g.replay(); torch.cuda.synchronize(); print("graph sees host update:", int(d[0]))
