"""Dense DST-I products: FP64 tensor cores (DMMA, tuning key 16 = 1) against the
CUDA-core GEMM (key 16 = 0), the whole-plane DMMA 2D DST (key 18, N <= 64), and
the FFT engine for power-of-two N + 1 (the dense path forced by key 17). Times hfb_transform_stack over a stack of
N x N planes (~256 MB) and checks every variant against the FFT / first result.

    python tools/dense_bench.py [--n 31 63 100 125 250 500]
"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1912_03565_b200 import _native  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, nargs="+", default=[15, 31, 40, 63, 100, 127, 250])
ap.add_argument("--reps", type=int, default=5)
a = ap.parse_args()
dev = torch.device("cuda", 0)
lib = _native.load_library()
P = _native.ptr
res = []
for n in a.n:
    nz = max(1, (32 << 20) // (n * n))
    plan = _native.get_plan(n, n, nz, dev)
    x = torch.randn((nz, n, n), dtype=torch.float64, device=dev)
    work = plan.workspace(1)
    pow2 = (n + 1) & n == 0
    variants = ([("fft", {17: 0, 18: 0})] if pow2 else []) + \
        ([("dmma2d", {17: 0, 18: n})] if n <= 64 else []) + \
        [("dense_dmma", {16: 1, 17: n, 18: 0}), ("dense_cuda_core", {16: 0, 17: n, 18: 0})]
    out = {}
    row = {"n": n, "planes": nz}
    for name, knobs in variants:
        for k, v in knobs.items():
            lib.hfb_set_tuning(k, v)
        y = x.clone()
        _native.check(lib.hfb_transform_stack(plan.handle, P(y), 0, nz, P(work), plan.stream()), name)
        torch.cuda.synchronize()
        out[name] = y.clone()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(a.reps):
            _native.check(lib.hfb_transform_stack(plan.handle, P(y), 0, nz, P(work),
                                                  plan.stream()), name)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / a.reps
        row[name + "_ms"] = ms
        row[name + "_gpts"] = nz * n * n / ms / 1e6
    lib.hfb_set_tuning(16, 1)
    lib.hfb_set_tuning(17, 0)
    lib.hfb_set_tuning(18, 0)
    ref = out[variants[0][0]]
    for name, _ in variants[1:]:
        row[name + "_maxrel"] = float((out[name] - ref).abs().max() / ref.abs().max())
    res.append(row)
    print(json.dumps(row), flush=True)
