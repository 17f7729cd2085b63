"""Pinned-host copy bandwidth: H2D alone, D2H alone, both at once (separate streams).

    python tools/pcie.py [--gb 4]
"""
import argparse
import time

import torch

ap = argparse.ArgumentParser()
ap.add_argument("--gb", type=float, default=4.0)
a = ap.parse_args()
n = int(a.gb * 2**30 / 8)
h1 = torch.empty(n, dtype=torch.float64).pin_memory()
h2 = torch.empty(n, dtype=torch.float64).pin_memory()
d1 = torch.empty(n, dtype=torch.float64, device="cuda")
d2 = torch.empty(n, dtype=torch.float64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def run(h2d, d2h):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    if h2d:
        with torch.cuda.stream(s1):
            d1.copy_(h1, non_blocking=True)
    if d2h:
        with torch.cuda.stream(s2):
            h2.copy_(d2, non_blocking=True)
    torch.cuda.synchronize()
    return time.perf_counter() - t0


run(True, True)
for name, args in (("h2d", (True, False)), ("d2h", (False, True)), ("both", (True, True))):
    t = min(run(*args) for _ in range(3))
    gbs = a.gb * 2**30 / 1e9 / t
    print(f"{name}: {t * 1e3:.1f} ms for {a.gb} GiB each way -> {gbs:.1f} GB/s per direction")
