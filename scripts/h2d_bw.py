"""Pinned host -> device copy bandwidth on this box (debug aid for bench e2e)."""
import torch
n = 468268800 // 4
h = torch.empty(n, dtype=torch.float32).pin_memory()
d = torch.empty(n, dtype=torch.float32, device="cuda")
s = torch.cuda.Stream()
for label, chunks in (("one copy", 1), ("4 copies", 4)):
    for _ in range(2):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(s):
            e0.record(s)
            step = n // chunks
            for c in range(chunks):
                d[c * step:(c + 1) * step].copy_(h[c * step:(c + 1) * step], non_blocking=True)
            e1.record(s)
        e1.synchronize()
    ms = e0.elapsed_time(e1)
    print(f"{label}: {ms:.2f} ms  {n * 4 / ms / 1e6:.1f} GB/s")
dh = torch.empty(n, dtype=torch.float32).pin_memory()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); dh.copy_(d, non_blocking=True); e1.record(); e1.synchronize()
print(f"D2H pinned: {n * 4 / e0.elapsed_time(e1) / 1e6:.1f} GB/s")
