"""Pinned host <-> device copy bandwidth (one direction, and both at once on
two streams) for 512 MB, CUDA events; the bound on bench.py's e2e step."""
import torch

n = 128 * 1024 * 1024  # floats = 512 MB
h = torch.empty(n, pin_memory=True)
h2 = torch.empty(n, pin_memory=True)
d = torch.empty(n, device="cuda")
d2 = torch.empty(n, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def t(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def both():
    c = torch.cuda.current_stream()
    s1.wait_stream(c)
    s2.wait_stream(c)
    with torch.cuda.stream(s1):
        d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2):
        h2.copy_(d2, non_blocking=True)
    c.wait_stream(s1)
    c.wait_stream(s2)


a = t(lambda: d.copy_(h, non_blocking=True))
b = t(lambda: h2.copy_(d2, non_blocking=True))
c = t(both)
gb = n * 4 / 1e9
print(f"h2d {gb / a * 1e3:.1f} GB/s ({a:.2f} ms / 512 MB)  d2h {gb / b * 1e3:.1f} GB/s ({b:.2f} ms)  "
      f"duplex {c:.2f} ms for 512 MB each way")
