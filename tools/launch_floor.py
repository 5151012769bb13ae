"""Event-timed floor for a trivial kernel on this GPU (context for the c1 latency
config): python tools/launch_floor.py"""
import torch

x = torch.zeros(1024, device="cuda")
flush = torch.ones(128 << 20, dtype=torch.int32, device="cuda")
ts = []
for i in range(60):
    flush.sum()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    x.add_(1.0)
    e1.record()
    torch.cuda.synchronize()
    if i >= 10:
        ts.append(e0.elapsed_time(e1) * 1e3)
ts.sort()
print(f"trivial kernel, event-timed after an L2 flush: median {ts[len(ts) // 2]:.2f} us, min {ts[0]:.2f} us")
