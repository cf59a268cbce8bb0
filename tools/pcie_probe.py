#!/usr/bin/env python
"""PCIe ceiling for bench.py's e2e leg (run under gpurun): pinned 4 GiB
host <-> device copies, H2D alone, D2H alone and both at once on two streams
(the shape of dsfft_execute_host's pipeline).  Prints GB/s per direction."""
import time

import torch

n = 4 << 30
h_in = torch.empty(n, dtype=torch.uint8, pin_memory=True)
h_out = torch.empty(n, dtype=torch.uint8, pin_memory=True)
d_in = torch.empty(n, dtype=torch.uint8, device="cuda")
d_out = torch.empty(n, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t) / reps


def h2d():
    with torch.cuda.stream(s1):
        d_in.copy_(h_in, non_blocking=True)


def d2h():
    with torch.cuda.stream(s2):
        h_out.copy_(d_out, non_blocking=True)


def both():
    h2d()
    d2h()


for name, fn in (("H2D alone", h2d), ("D2H alone", d2h), ("H2D + D2H concurrently", both)):
    dt = timed(fn)
    print(f"{name}: {n / dt / 1e9:.1f} GB/s per direction ({dt * 1e3:.1f} ms for 4 GiB)")
