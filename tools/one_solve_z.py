"""Complex k(z) one-call solves (hfb_solve_z) on cuda:0:
mean time and per-launch stage times.

    python tools/one_solve_z.py [--n 511] [--reps 5]
"""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1912_03565_b200 as hb  # noqa: E402
from paper_1912_03565_b200 import _native  # noqa: E402
from paper_1912_03565_b200.tridiag import device_coefficients  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=511)
ap.add_argument("--reps", type=int, default=5)
ap.add_argument("--tune", default="")
a = ap.parse_args()
n = a.n
dev = torch.device("cuda", 0)
g = hb.make_grid(hb.Domain(0, 1, 0, 1, 0, 1), n, n, n)
z = np.linspace(0.0, 1.0, n + 2)
k2 = (40.0 + 8.0j) * (1 + 0.3 * np.sin(2 * np.pi * z)) ** 2
prof = hb.CoefficientProfile(k2=k2, k2_z=np.gradient(k2, z), k2_zz=np.zeros_like(k2))
plan = _native.get_plan(n, n, n, dev)
device_coefficients(plan, hb.SchemeKind.SIXTH_ORDER, prof, g)
for kv in filter(None, a.tune.split(",")):
    k, v = kv.split("=")
    plan.lib.hfb_set_tuning(int(k), int(v))
rng = np.random.default_rng(5)
tr = torch.from_numpy(rng.standard_normal((n, n, n))).to(dev)
ti = torch.from_numpy(rng.standard_normal((n, n, n))).to(dev)
ur, ui = torch.empty_like(tr), torch.empty_like(ti)
work = plan.workspace(3)
P = _native.ptr


def solve():
    _native.check(plan.lib.hfb_solve_z(plan.handle, P(tr), P(ti), P(ur), P(ui), P(work),
                                       plan.stream()), "solve_z")


solve()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(a.reps):
    solve()
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / a.reps
print(f"complex solve n={n} tune={a.tune}: {ms:.3f} ms, {n ** 3 / (ms * 1e-3):.3e} pts/s")
