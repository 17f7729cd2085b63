"""Bidirectional pinned-host copy bandwidth at the bench's volume (8.56 GB each way)
with an idle GPU and while one-call solves run back to back on another stream:
what the pipelined e2e path can reach.

    python tools/pcie_busy.py
"""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1912_03565_b200 import _native, workloads as wl  # noqa: E402
from paper_1912_03565_b200.tridiag import device_coefficients  # noqa: E402

dev = torch.device("cuda", 0)
w = wl.workload(4)
n = w.n
plan = _native.get_plan(n, n, n, dev)
device_coefficients(plan, w.scheme, w.profile, w.grid)
F = wl.device_rhs(w, dev)
U = torch.empty_like(F)
work = plan.workspace(0)
h1 = torch.empty(F.shape, dtype=torch.float64, pin_memory=True)
h2 = torch.empty(F.shape, dtype=torch.float64, pin_memory=True)
d1, d2 = torch.empty_like(F), torch.empty_like(F)
s1, s2, s3 = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()
nbytes = F.numel() * 8


def copies(reps, busy):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        with torch.cuda.stream(s1):
            d1.copy_(h1, non_blocking=True)
        with torch.cuda.stream(s2):
            h2.copy_(d2, non_blocking=True)
        if busy:
            with torch.cuda.stream(s3):
                for _ in range(busy):
                    _native.check(plan.lib.hfb_solve(plan.handle, _native.ptr(F), _native.ptr(U),
                                                     _native.ptr(work),
                                                     _native.current_stream(dev)), "solve")
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps


copies(1, 1)
for busy in (0, 1, 4, 9):
    t = copies(4, busy)
    print(f"{busy} solves per copy pair: {t * 1e3:.1f} ms per 8.56 GB each way -> "
          f"{nbytes / 1e9 / t:.1f} GB/s per direction")
