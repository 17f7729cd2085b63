"""One (or a few) full solves of a BASELINE config on cuda:0 — for ncu launch lists.

    python tools/one_solve.py [--cfg 4] [--reps 1]
"""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1912_03565_b200 import _native, workloads as wl  # noqa: E402
from paper_1912_03565_b200.tridiag import device_coefficients  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--cfg", type=int, default=4)
ap.add_argument("--n", type=int, default=None)
ap.add_argument("--reps", type=int, default=1)
a = ap.parse_args()
dev = torch.device("cuda", 0)
w = wl.workload(a.cfg, a.n)
n = w.n
plan = _native.get_plan(n, n, n, dev)
device_coefficients(plan, w.scheme, w.profile, w.grid)
F = wl.device_rhs(w, dev)
U = torch.empty_like(F)
work = plan.workspace(0)
for _ in range(a.reps):
    _native.check(plan.lib.hfb_solve(plan.handle, _native.ptr(F), _native.ptr(U),
                                     _native.ptr(work), plan.stream()), "solve")
plan.fetch_status()
torch.cuda.synchronize()
print("ok", float(U.abs().max()))
