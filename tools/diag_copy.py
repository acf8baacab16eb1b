import torch, time
dev = torch.device("cuda", 0)
h = torch.empty(64 << 20, dtype=torch.float32).pin_memory()
d = torch.empty_like(h, device=dev)
s1 = torch.cuda.Stream(); s2 = torch.cuda.Stream()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda.synchronize()
e0.record(s1)
with torch.cuda.stream(s1):
    d.copy_(h, non_blocking=True)
e1.record(s1)
torch.cuda.synchronize()
print("H2D 256MB ms", e0.elapsed_time(e1), "GB/s", 256e6 / (e0.elapsed_time(e1) * 1e6))
a = torch.randn(8192, 8192, device=dev)
torch.cuda.synchronize()
t = time.perf_counter()
with torch.cuda.stream(s2):
    for _ in range(20): a @ a
torch.cuda.synchronize(); tc = time.perf_counter() - t
t = time.perf_counter()
with torch.cuda.stream(s2):
    for _ in range(20): a @ a
with torch.cuda.stream(s1):
    d.copy_(h, non_blocking=True)
torch.cuda.synchronize(); tb = time.perf_counter() - t
print("compute alone", tc * 1e3, "compute + concurrent copy", tb * 1e3)
