"""Per-kernel timing of the solve stages with CUDA events (diagnostic tool).

    python tools/stage_times.py [--n 1023] [--reps 3]
"""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1912_03565_b200 import _native, workloads as wl  # noqa: E402
from paper_1912_03565_b200.tridiag import device_coefficients  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=1023)
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--cfg", type=int, default=4)
a = ap.parse_args()
dev = torch.device("cuda", 0)
w = wl.workload(a.cfg, a.n)
n = a.n
plan = _native.get_plan(n, n, n, dev)
device_coefficients(plan, w.scheme, w.profile, w.grid)
lib, h, st = plan.lib, plan.handle, plan.stream()
F = wl.device_rhs(w, dev)
U = torch.empty_like(F)
cpw = torch.empty_like(F)
work = plan.workspace(0)
P = _native.ptr
stages = {
    "dst_x (all rows)": lambda: lib.hfb_transform_lines_x(h, P(F), 0, n, P(None), st),
    "dst_y (all cols)": lambda: lib.hfb_transform_lines_y(h, P(F), 0, n, P(None), st),
    "thomas (all modes)": lambda: lib.hfb_solve_slab(h, P(F), n, 0, P(cpw), st),
    "stack (x^T + y^T)": lambda: lib.hfb_transform_stack(h, P(F), 0, n, P(work), st),    "full solve": lambda: lib.hfb_solve(h, P(F), P(U), P(work), st),
}
pts = n ** 3
for name, fn in stages.items():
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(a.reps):
        rc = fn()
        assert rc == 0, rc
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / a.reps
    print(f"{name:22s} {ms:9.3f} ms  {pts / ms / 1e6:10.3e} pts/s  "
          f"{16 * pts / ms / 1e6:8.1f} GB/s at 16 B/pt")

if os.environ.get("HFB_SWEEP"):
    for E in (16, 32):
        for NF in (0, 1, 2, 4):
            lib.hfb_set_tuning(0, E)
            lib.hfb_set_tuning(1, NF)
            for name in ("dst_x (all rows)", "stack (x^T + y^T)"):
                fn = stages[name]
                fn()
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                for _ in range(a.reps):
                    fn()
                e1.record()
                torch.cuda.synchronize()
                print(f"E={E} NF={NF} {name:20s} {e0.elapsed_time(e1) / a.reps:8.3f} ms")
