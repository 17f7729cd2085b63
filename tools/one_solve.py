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
ap.add_argument("--tune", default="", help="key=value,... passed to hfb_set_tuning")
ap.add_argument("--time", action="store_true", help="print the mean solve time (CUDA events)")
ap.add_argument("--stages", action="store_true", help="also print the mean per-launch times")
a = ap.parse_args()
dev = torch.device("cuda", 0)
w = wl.workload(a.cfg, a.n)
n = w.n
plan = _native.get_plan(n, n, n, dev)
device_coefficients(plan, w.scheme, w.profile, w.grid)
F = wl.device_rhs(w, dev)
U = F if a.cfg == 5 else torch.empty_like(F)  # 2047^3 only fits in place
work = plan.workspace(0)
for kv in filter(None, a.tune.split(",")):
    k, v = kv.split("=")
    plan.lib.hfb_set_tuning(int(k), int(v))


def solve():
    _native.check(plan.lib.hfb_solve(plan.handle, _native.ptr(F), _native.ptr(U),
                                     _native.ptr(work), plan.stream()), "solve")


if a.time:
    solve()
    torch.cuda.synchronize()
    if a.stages:
        import ctypes
        _native.check(plan.lib.hfb_stage_timing(plan.handle, a.reps), "stage_timing")
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(a.reps):
        solve()
    e1.record()
    torch.cuda.synchronize()
    print(f"tune={a.tune} n={n} ms/solve={e0.elapsed_time(e1) / a.reps:.3f}")
    if a.stages:
        buf = (ctypes.c_float * (5 * a.reps))()
        k = ctypes.c_int(0)
        _native.check(plan.lib.hfb_stage_times(plan.handle, buf, ctypes.byref(k)), "stage_times")
        ms = [sum(buf[5 * r + i] for r in range(k.value)) / k.value for i in range(5)]
        print("  stages ms: " + " ".join(f"{v:.3f}" for v in ms))
        plan.lib.hfb_stage_timing(plan.handle, 0)
else:
    for _ in range(a.reps):
        solve()
plan.fetch_status()
torch.cuda.synchronize()
print("ok", max(float(U.max()), -float(U.min())))
