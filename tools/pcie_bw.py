import torch, time
n = 65 * 1024 * 1024
h = torch.empty(n, dtype=torch.uint8).pin_memory()
d = torch.empty(n, dtype=torch.uint8, device="cuda")
for _ in range(3): d.copy_(h, non_blocking=True)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(10): d.copy_(h, non_blocking=True)
b.record(); torch.cuda.synchronize()
print("H2D %.1f GB/s" % (10 * n / (a.elapsed_time(b) * 1e-3) / 1e9))
h2 = torch.empty(n // 8, dtype=torch.uint8).pin_memory()
s = torch.cuda.Stream()
with torch.cuda.stream(s):
    a.record()
    for _ in range(8): d[: n // 8].copy_(h2, non_blocking=True)
    b.record()
torch.cuda.synchronize()
print("H2D 8MB chunks %.1f GB/s" % (n / (a.elapsed_time(b) * 1e-3) / 1e9))
