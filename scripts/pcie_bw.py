import torch, time
n = 147_456_000  # 16 images of 1920x1200 fp32 bytes
h = torch.empty(n // 4, dtype=torch.float32).pin_memory()
d = torch.empty(n // 4, dtype=torch.float32, device="cuda")
s = torch.cuda.Stream()
for name, src, dst in [("h2d", h, d), ("d2h", d, h)]:
    for _ in range(3):
        dst.copy_(src, non_blocking=True)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        dst.copy_(src, non_blocking=True)
    e1.record(); torch.cuda.synchronize()
    print(name, n * 10 / (e0.elapsed_time(e1) * 1e-3) / 1e9, "GB/s")
# concurrent both directions
h2 = torch.empty(n // 4, dtype=torch.float32).pin_memory(); d2 = torch.empty(n // 4, dtype=torch.float32, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
torch.cuda.synchronize(); t0 = time.perf_counter()
for _ in range(10):
    with torch.cuda.stream(s1): d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
torch.cuda.synchronize(); dt = time.perf_counter() - t0
print("both", n * 10 / dt / 1e9, "GB/s each")
