"""PCIe bound of the C2 e2e call: pinned H2D / D2H of one 32-RHS block (7.68 MB), alone and concurrent."""
import time

import torch

nbytes = 30000 * 32 * 8
h_in = torch.empty(nbytes // 8, dtype=torch.float64).pin_memory()
h_out = torch.empty_like(h_in).pin_memory()
d_in = torch.empty(nbytes // 8, dtype=torch.float64, device="cuda")
d_out = torch.empty_like(d_in)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timeit(fn, reps=50):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    ts.sort()
    return ts[len(ts) // 2] * 1e6


def h2d():
    with torch.cuda.stream(s1):
        d_in.copy_(h_in, non_blocking=True)


def d2h():
    with torch.cuda.stream(s2):
        h_out.copy_(d_out, non_blocking=True)


def both():
    h2d()
    d2h()


for name, fn in (("h2d", h2d), ("d2h", d2h), ("both_concurrent", both)):
    us = timeit(fn)
    print(f"{name}: {us:.1f} us  ({nbytes / us / 1e3:.1f} GB/s per direction)")
