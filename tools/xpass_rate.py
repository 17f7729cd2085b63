"""Throughput of the x-pass (ROW mode DST engine) for different line lengths
at a fixed total volume: separates per-line-pair group barriers (T = M/16
threads: 1 warp at M = 512, 2 at 1024, 4 at 2048) from the FFT's log M work.

    python tools/xpass_rate.py
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1912_03565_b200 import _native  # noqa: E402

total = 1 << 30  # doubles
for nx in (255, 511, 1023, 2047):
    ny = 1023
    nz = max(1, total // (nx * ny))
    t = torch.rand((nz, ny, nx), dtype=torch.float64, device="cuda")
    plan = _native.get_plan(nx, ny, nz, t.device)
    work = plan.workspace(1)
    f = lambda: plan.lib.hfb_transform_lines_x(plan.handle, _native.ptr(t), 0, ny,
                                               _native.ptr(work), plan.stream())
    f()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        f()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    pts = nx * ny * nz
    m = (nx + 1).bit_length() - 1
    print(f"M={nx + 1:5d} threads/pair={(nx + 1) // 16:4d} ms={ms:.3f} "
          f"Gpts/s={pts / ms / 1e6:.1f} ns/(pt*log2M)={ms * 1e6 / (pts * m):.4f}")
    del t, work
    torch.cuda.empty_cache()
