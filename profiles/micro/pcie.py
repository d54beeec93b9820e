"""Pinned host <-> device copy bandwidth for the host drop-in's 4.2 MB fp64 feature batch."""
import torch

n = 512 * 1024  # D x B fp64
h = torch.empty(n, dtype=torch.float64, pin_memory=True)
d = torch.empty(n, dtype=torch.float64, device="cuda")
s = torch.cuda.Stream()
for name, fn in [("H2D", lambda: d.copy_(h, non_blocking=True)), ("D2H", lambda: h.copy_(d, non_blocking=True))]:
    with torch.cuda.stream(s):
        for _ in range(5):
            fn()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(50):
            fn()
        e1.record()
    s.synchronize()
    ms = e0.elapsed_time(e1) / 50
    print(f"{name}: {ms * 1e3:.1f} us per 4.19 MB = {n * 8 / ms / 1e6:.1f} GB/s")
