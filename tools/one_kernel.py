"""Run one stage kernel on a small slab (for ncu captures).

    python tools/one_kernel.py {x|y|t|solve} [--n 1023] [--nz 8]
"""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1912_03565_b200 import _native, workloads as wl  # noqa: E402
from paper_1912_03565_b200.tridiag import device_coefficients  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("stage")
ap.add_argument("--n", type=int, default=1023)
ap.add_argument("--nz", type=int, default=8)
ap.add_argument("--reps", type=int, default=2)
a = ap.parse_args()
dev = torch.device("cuda", 0)
n, nz = a.n, a.nz
w = wl.workload(4, n)
plan = _native.get_plan(n, n, nz, dev)
g = w.grid.__class__(w.grid.domain, n, n, nz, w.grid.h_x, w.grid.h_y, w.grid.h_z)
prof = w.profile.__class__(k2=w.profile.k2[:nz + 2], k2_z=w.profile.k2_z[:nz + 2],
                           k2_zz=w.profile.k2_zz[:nz + 2], gamma=w.profile.gamma)
device_coefficients(plan, w.scheme, prof, g)
lib, h, st, P = plan.lib, plan.handle, plan.stream(), _native.ptr
F = torch.rand((nz, n, n), device=dev, dtype=torch.float64)
cpw = torch.empty_like(F)
work = plan.workspace(0)
fn = {"x": lambda: lib.hfb_transform_lines_x(h, P(F), 0, n, P(None), st),
      "y": lambda: lib.hfb_transform_lines_y(h, P(F), 0, n, P(None), st),
      "t": lambda: lib.hfb_solve_slab(h, P(F), n, 0, P(cpw), st),
      "stack": lambda: lib.hfb_transform_stack(h, P(F), 0, nz, P(work), st),
      "solve": lambda: lib.hfb_solve(h, P(F), P(F), P(work), st)}[a.stage]
for _ in range(a.reps):
    assert fn() == 0
torch.cuda.synchronize()
print("ok")
