"""Bitwise fingerprint of one-call solves under the library HFB_LIBRARY names
(same-box comparison of two builds: the hashes must agree when a change is
meant to leave the arithmetic alone).

    HFB_LIBRARY=path/to/lib.so python tools/bits.py [cfg ...]
"""
import hashlib
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1912_03565_b200 import _native, workloads as wl  # noqa: E402
from paper_1912_03565_b200.tridiag import device_coefficients  # noqa: E402

dev = torch.device("cuda", 0)
for kv in filter(None, os.environ.get("HFB_TUNE", "").split(",")):  # e.g. HFB_TUNE=32=0
    k, v = kv.split("=")
    _native.load_library().hfb_set_tuning(int(k), int(v))
for spec in (sys.argv[1:] or ["1", "2", "3", "4"]):
    cfg, _, n = spec.partition(":")
    w = wl.workload(int(cfg), int(n) if n else None)
    plan = _native.get_plan(w.n, w.n, w.n, dev)
    device_coefficients(plan, w.scheme, w.profile, w.grid)
    F = wl.device_rhs(w, dev)
    for lean in (0, 1):
        _native.check(plan.lib.hfb_plan_set_workspace_mode(plan.handle, lean), "mode")
        U = torch.empty_like(F)
        work = plan.workspace(0)
        hs = []
        for rep in range(2):  # the second solve reads the plan's cached cp checkpoints (key 32)
            U.zero_()
            _native.check(plan.lib.hfb_solve(plan.handle, _native.ptr(F), _native.ptr(U),
                                             _native.ptr(work), plan.stream()), "solve")
            torch.cuda.synchronize()
            hs.append(hashlib.sha256(U.cpu().numpy().tobytes()).hexdigest()[:16])
        assert hs[0] == hs[1], hs
        print(f"cfg{cfg} n={w.n} lean={lean} sha256={hs[0]}")
        del U, work
    del F, plan
    _native._plans.clear()
    torch.cuda.empty_cache()
