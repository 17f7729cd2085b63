"""End-to-end time of the drop-in API on host arrays: solve_discrete(Field3D(F), zero
boundary) for the cfg4 workload, F float64 and complex128 (the reference's dtype),
including every host<->device copy; prints pts/s and the PhaseTimings.

    python tools/dropin_e2e.py [--cfg 4] [--reps 3]
"""
import argparse
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1912_03565_b200 as hb  # noqa: E402
from paper_1912_03565_b200 import workloads as wl  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--cfg", type=int, default=4)
ap.add_argument("--reps", type=int, default=3)
a = ap.parse_args()
w = wl.workload(a.cfg)
F = wl.host_rhs(w)
out = {}
for name, arr in (("float64", F), ("complex128", F.astype(complex))):
    hb.solve_discrete(hb.Field3D(arr[:8].copy()), hb.BoundaryData.zero(), w.scheme,
                      hb.CoefficientProfile(k2=w.profile.k2[:10], k2_z=w.profile.k2_z[:10],
                                            k2_zz=w.profile.k2_zz[:10], gamma=w.profile.gamma),
                      hb.make_grid(hb.Domain(0, 1, 0, 1, 0, 9 / (w.n + 1)), w.n, w.n, 8))
    ts = []
    for _ in range(a.reps):
        t0 = time.perf_counter()
        u, t = hb.solve_discrete(hb.Field3D(arr), hb.BoundaryData.zero(), w.scheme, w.profile,
                                 w.grid)
        ts.append(time.perf_counter() - t0)
        assert u.values.dtype == arr.dtype
        del u
    best = min(ts)
    out[name] = {"s": best, "pts_per_s": w.n ** 3 / best,
                 "phases": {k: getattr(t, k) for k in ("setup_s", "transform_s", "exchange_s",
                                                       "tridiag_s", "total_s")}}
    del arr
print(json.dumps(out))
