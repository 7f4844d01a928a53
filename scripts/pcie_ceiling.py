"""PCIe copy ceiling for the e2e figure: 1.2 GB H2D and 0.4 GB D2H (one
100M-query config-3 step) from pinned memory, alone and concurrently."""
import torch, time
n = 300_000_000  # 1.2 GB of f32
h = torch.empty(n, dtype=torch.float32).pin_memory()
d = torch.empty(n, dtype=torch.float32, device="cuda")
ho = torch.empty(n // 3, dtype=torch.float32).pin_memory()
do = torch.empty(n // 3, dtype=torch.float32, device="cuda")
for _ in range(2):
    d.copy_(h, non_blocking=True); torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); d.copy_(h, non_blocking=True); e1.record(); torch.cuda.synchronize()
print("H2D GB/s", 1.2e9 / (e0.elapsed_time(e1) / 1e3) / 1e9)
e0.record(); ho.copy_(do, non_blocking=True); e1.record(); torch.cuda.synchronize()
print("D2H GB/s", 0.4e9 / (e0.elapsed_time(e1) / 1e3) / 1e9)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
torch.cuda.synchronize(); t0 = time.perf_counter()
with torch.cuda.stream(s1): d.copy_(h, non_blocking=True)
with torch.cuda.stream(s2): ho.copy_(do, non_blocking=True)
torch.cuda.synchronize(); dt = time.perf_counter() - t0
print("concurrent 1.2 GB H2D + 0.4 GB D2H: ms", dt * 1e3, " -> casts/s equiv", 100e6 / dt / 1e9, "G")
