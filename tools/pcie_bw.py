"""PCIe ceiling for the host-buffer path: pinned H2D, D2H, and both at once."""
import torch

n = 1 << 28  # 2 GiB of float64 per buffer
h1 = torch.empty(n, dtype=torch.float64, pin_memory=True)
h2 = torch.empty(n, dtype=torch.float64, pin_memory=True)
d1 = torch.empty(n, dtype=torch.float64, device="cuda")
d2 = torch.empty(n, dtype=torch.float64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
gb = n * 8 / 1e9


def timed(fn, reps=3):
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        torch.cuda.synchronize()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) / 1e3)
    return best


t = timed(lambda: d1.copy_(h1, non_blocking=True))
print(f"H2D {gb / t:.1f} GB/s")
t = timed(lambda: h2.copy_(d2, non_blocking=True))
print(f"D2H {gb / t:.1f} GB/s")


def both():
    with torch.cuda.stream(s1):
        d1.copy_(h1, non_blocking=True)
    with torch.cuda.stream(s2):
        h2.copy_(d2, non_blocking=True)


t = timed(both)
print(f"H2D+D2H concurrent: {gb / t:.1f} GB/s each direction")
