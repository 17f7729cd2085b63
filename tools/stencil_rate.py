"""HBM rate of the compact RHS operator (K1, hfb_rhs_fourth) at n^3.

    python tools/stencil_rate.py [--n 1023]
"""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1912_03565_b200 import _native, workloads as wl  # noqa: E402
from paper_1912_03565_b200.tridiag import device_coefficients  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=1023)
ap.add_argument("--reps", type=int, default=5)
a = ap.parse_args()
n = a.n
dev = torch.device("cuda", 0)
P = _native.ptr
w = wl.workload(4, n)
plan = _native.get_plan(n, n, n, dev)
device_coefficients(plan, w.scheme, w.profile, w.grid)
lib = plan.lib
f = torch.rand((n + 2, n + 2, n + 2), dtype=torch.float64, device=dev)
F = torch.empty((n, n, n), dtype=torch.float64, device=dev)
st = plan.stream()


def timed(fn, nbytes, name):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(a.reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / a.reps
    print(f"{name}: {ms:.3f} ms, {nbytes / ms / 1e6:.0f} GB/s (algorithmic {nbytes / 1e9:.2f} GB)")


ref = None
for v in (0, 16, 32, 64):
    lib.hfb_set_tuning(20, v)
    timed(lambda: _native.check(lib.hfb_rhs_fourth(plan.handle, P(f), P(F), 1e-6, st), "rhs4"),
          8 * ((n + 2) ** 3 + n ** 3), f"rhs_fourth (K1), tuning 20 = {v}")
    if ref is None:
        ref = F.clone()
    else:
        assert torch.equal(F, ref), v
lib.hfb_set_tuning(20, 32)

# the 27-point apply (fold mode 1 and plain mode 0), all 27 terms
ext = f
rhs = torch.rand((n, n, n), dtype=torch.float64, device=dev)
refs = {}
# (key 20, key 24, key 25): gathers, marching, streamed (levels per CTA, rows per warp)
VARIANTS = [(0, 0, 4, 0), (32, 0, 4, 0), (32, 64, 4, 0), (32, 64, 2, 0), (32, 32, 4, 1),
            (32, 64, 4, 1), (32, 128, 4, 1)]
for v20, v24, v25, v27 in VARIANTS:
    lib.hfb_set_tuning(20, v20)
    lib.hfb_set_tuning(24, v24)
    lib.hfb_set_tuning(25, v25)
    lib.hfb_set_tuning(27, v27)
    for mode in (0, 1):
        timed(lambda: _native.check(lib.hfb_apply27(plan.handle, P(ext), P(rhs), P(F), 0x7FFFFFF,
                                                    mode, st), "apply27"),
              8 * ((n + 2) ** 3 + (2 if mode else 1) * n ** 3),
              f"apply27 mode {mode}, tuning 20/24/25/27 = {v20}/{v24}/{v25}/{v27}")
        if mode not in refs:
            refs[mode] = F.clone()
        else:
            assert torch.equal(F, refs[mode]), (mode, v20, v24, v25, v27)
lib.hfb_set_tuning(20, 32)
lib.hfb_set_tuning(24, 32)
lib.hfb_set_tuning(25, 4)
print("apply27 bitwise equal across variants")

# the residual sum of squares (zero boundary, interior u)
u = torch.rand((n, n, n), dtype=torch.float64, device=dev)
npart = int(lib.hfb_residual_partials(plan.handle))
part = torch.empty(npart, dtype=torch.float64, device=dev)
vals = {}
for v20, v24, v25, v27 in VARIANTS:
    lib.hfb_set_tuning(20, v20)
    lib.hfb_set_tuning(24, v24)
    lib.hfb_set_tuning(25, v25)
    lib.hfb_set_tuning(27, v27)
    timed(lambda: _native.check(lib.hfb_residual_sq(plan.handle, P(u), P(rhs), P(part), 0x7FFFFFF,
                                                    st), "residual"),
          8 * 2 * n ** 3, f"residual_sq, tuning 20/24/25/27 = {v20}/{v24}/{v25}/{v27}")
    vals[(v20, v24, v25, v27)] = float(part.sum())
lib.hfb_set_tuning(20, 32)
lib.hfb_set_tuning(24, 32)
lib.hfb_set_tuning(25, 4)
lib.hfb_set_tuning(27, 1)
print("residual sums", vals)
r0 = list(vals.values())[0]
assert all(abs(x - r0) <= 1e-12 * abs(r0) for x in vals.values()), vals
