"""Per-launch stage times of the lean (one-volume) one-call solve at n_x = n_y = n,
n_z planes (default 2047 x 2047 x 64): the 2047^3 schedule on a slice that ncu can
replay.

    python tools/lean_probe.py [--n 2047] [--nz 64]
"""
import argparse
import ctypes
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1912_03565_b200 as hb  # noqa: E402
from paper_1912_03565_b200 import _native  # noqa: E402
from paper_1912_03565_b200.tridiag import device_coefficients  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=2047)
ap.add_argument("--nz", type=int, default=64)
ap.add_argument("--reps", type=int, default=5)
a = ap.parse_args()
dev = torch.device("cuda", 0)
g = hb.make_grid(hb.Domain(0, 1, 0, 1, 0, 1), a.n, a.n, a.nz)
plan = _native.get_plan(a.n, a.n, a.nz, dev)
device_coefficients(plan, hb.SchemeKind.FOURTH_ORDER, hb.constant_profile(-1.0, g), g)
plan.set_workspace_mode(1)
F = torch.rand((a.nz, a.n, a.n), dtype=torch.float64, device=dev)
work = plan.workspace(0)
lib, P = plan.lib, _native.ptr
for _ in range(2):
    _native.check(lib.hfb_solve(plan.handle, P(F), P(F), P(work), plan.stream()), "solve")
torch.cuda.synchronize()
_native.check(lib.hfb_stage_timing(plan.handle, a.reps), "stage_timing")
for _ in range(a.reps):
    _native.check(lib.hfb_solve(plan.handle, P(F), P(F), P(work), plan.stream()), "solve")
torch.cuda.synchronize()
buf = (ctypes.c_float * (5 * a.reps))()
k = ctypes.c_int(0)
_native.check(lib.hfb_stage_times(plan.handle, buf, ctypes.byref(k)), "stage_times")
ms = [sum(buf[5 * r + i] for r in range(k.value)) / k.value for i in range(5)]
print("lean stages ms:", " ".join(f"{v:.3f}" for v in ms))
