"""PCIe copy rates of this box: pinned H2D alone, D2H alone, both at once
(two streams), in GB/s -- the ceiling of the e2e (host-buffer) numbers."""
import time
import torch

n = 256 << 20
h1 = torch.empty(n, dtype=torch.uint8).pin_memory()
h2 = torch.empty(n, dtype=torch.uint8).pin_memory()
d1 = torch.empty(n, dtype=torch.uint8, device="cuda")
d2 = torch.empty(n, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn, reps=5):
    fn(); torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t) / reps


def h2d():
    with torch.cuda.stream(s1):
        d1.copy_(h1, non_blocking=True)


def d2h():
    with torch.cuda.stream(s2):
        h2.copy_(d2, non_blocking=True)


def both():
    h2d(); d2h()


for name, fn, b in (("h2d", h2d, n), ("d2h", d2h, n), ("both", both, 2 * n)):
    print(f"{name}: {b / timed(fn) / 1e9:.1f} GB/s")
