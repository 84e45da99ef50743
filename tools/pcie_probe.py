import torch, time
n = 1 << 28
a = torch.empty(n, dtype=torch.int64).pin_memory()
b = torch.empty(n, dtype=torch.int64).pin_memory()
da = torch.empty(n, dtype=torch.int64, device="cuda")
db = torch.empty(n, dtype=torch.int64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
for _ in range(2):
    da.copy_(a, non_blocking=True); torch.cuda.synchronize()
t = time.perf_counter(); da.copy_(a, non_blocking=True); torch.cuda.synchronize(); h2d = time.perf_counter() - t
t = time.perf_counter(); b.copy_(db, non_blocking=True); torch.cuda.synchronize(); d2h = time.perf_counter() - t
t = time.perf_counter()
with torch.cuda.stream(s1): da.copy_(a, non_blocking=True)
with torch.cuda.stream(s2): b.copy_(db, non_blocking=True)
torch.cuda.synchronize(); both = time.perf_counter() - t
print(f"H2D {8*n/h2d/1e9:.1f} GB/s ({h2d*1e3:.1f} ms)  D2H {8*n/d2h/1e9:.1f} GB/s ({d2h*1e3:.1f} ms)  concurrent {both*1e3:.1f} ms")
