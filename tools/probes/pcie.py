"""Pinned host<->device copy bandwidth on this box: H2D alone, D2H alone, both
concurrently (the ceiling of bench.py's e2e leg)."""
import torch
n = 1 << 30
h1 = torch.empty(n, dtype=torch.uint8, pin_memory=True)
h2 = torch.empty(n, dtype=torch.uint8, pin_memory=True)
d1 = torch.empty(n, dtype=torch.uint8, device="cuda")
d2 = torch.empty(n, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def timed(fn, reps=5):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / 1e3 / reps
def h2d():
    with torch.cuda.stream(s1): d1.copy_(h1, non_blocking=True)
    torch.cuda.current_stream().wait_stream(s1)
def d2h():
    with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
    torch.cuda.current_stream().wait_stream(s2)
def both():
    with torch.cuda.stream(s1): d1.copy_(h1, non_blocking=True)
    with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
    torch.cuda.current_stream().wait_stream(s1); torch.cuda.current_stream().wait_stream(s2)
t = timed(h2d); print(f"H2D pinned: {n / t / 1e9:.1f} GB/s")
t = timed(d2h); print(f"D2H pinned: {n / t / 1e9:.1f} GB/s")
t = timed(both); print(f"H2D+D2H concurrent: {n / t / 1e9:.1f} GB/s each direction")
