"""Pinned host <-> device copy rates for the C2 e2e payload sizes (the ceiling of bench.py's
e2e leg): H2D alone, D2H alone, both at once on two streams."""
import torch

N = 16384 * 26 * 64 * 4  # the gradient / pooled tensor, bytes
h_in = torch.empty(N, dtype=torch.uint8).pin_memory()
h_out = torch.empty(N, dtype=torch.uint8).pin_memory()
d_in = torch.empty(N, dtype=torch.uint8, device="cuda")
d_out = torch.empty(N, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn, it=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(it):
        fn()
    torch.cuda.current_stream().wait_stream(s1)
    torch.cuda.current_stream().wait_stream(s2)
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / it


def h2d():
    with torch.cuda.stream(s1):
        d_in.copy_(h_in, non_blocking=True)


def d2h():
    with torch.cuda.stream(s2):
        h_out.copy_(d_out, non_blocking=True)


def both():
    h2d()
    d2h()


for name, fn in [("h2d", h2d), ("d2h", d2h), ("both", both)]:
    ms = timed(fn)
    print(f"{name:5s} {ms:.3f} ms  {N / ms / 1e6:.1f} GB/s per direction")
