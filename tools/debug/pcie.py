import torch, time
n = 806_400_000 // 2
h = torch.empty(n, dtype=torch.bfloat16).pin_memory()
d = torch.empty(n, dtype=torch.bfloat16, device="cuda")
for _ in range(2):
    d.copy_(h, non_blocking=True)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); d.copy_(h, non_blocking=True); e1.record(); torch.cuda.synchronize()
print("H2D 806MB ms", e0.elapsed_time(e1), "GB/s", 806.4 / e0.elapsed_time(e1))
o = torch.empty(n // 3, dtype=torch.bfloat16).pin_memory()
e0.record(); o.copy_(d[: n // 3], non_blocking=True); e1.record(); torch.cuda.synchronize()
print("D2H 269MB ms", e0.elapsed_time(e1))
t0 = time.perf_counter(); x = torch.empty(n // 3, dtype=torch.bfloat16, pin_memory=True); t1 = time.perf_counter()
print("pinned alloc 269MB s", t1 - t0)
t0 = time.perf_counter(); x2 = torch.empty(n // 3, dtype=torch.bfloat16, pin_memory=True); t1 = time.perf_counter()
print("pinned alloc again s", t1 - t0)
del x; x3 = torch.empty(n // 3, dtype=torch.bfloat16, pin_memory=True); t2 = time.perf_counter()
print("after free s", t2 - t1)
