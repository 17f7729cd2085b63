"""Forward 2D DST (x ROW pass + y tensor-box pass, hfb_forward_modes) on chunks
of c planes: per-point time when a chunk's source, scratch and output stay in
L2, against the full-volume rate. Diagnostic for an L2-resident x -> y schedule.

    python tools/chunk_rate.py [--n 1023] [--chunks 1,2,4,8]
"""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1912_03565_b200 import _native  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=1023)
ap.add_argument("--chunks", default="1,2,4,8,16")
a = ap.parse_args()
n = a.n
dev = torch.device("cuda", 0)


def rate(c, reps, distinct):
    """ms per plane for `reps` forward_modes calls on c-plane chunks; `distinct`
    chunks cycle through different memory (distinct * c planes in all)."""
    plan = _native.get_plan(n, n, c, dev)
    ld = plan.lib.hfb_modes_ld(plan.handle)
    src = torch.rand((distinct, c, n, n), dtype=torch.float64, device=dev)
    modes = torch.empty((distinct, c, n, ld), dtype=torch.float64, device=dev)
    work = plan.workspace(5)
    st = plan.stream()
    f = lambda i: plan.lib.hfb_forward_modes(plan.handle, _native.ptr(src[i]),
                                             _native.ptr(modes[i]), _native.ptr(work), st)
    for i in range(distinct):
        assert f(i) == 0
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for r in range(reps):
        f(r % distinct)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    del src, modes, work
    torch.cuda.empty_cache()
    return ms / c


full = rate(64, 6, 8)  # 512 planes cycled: HBM-streamed
print(f"streamed (64-plane calls over 512 planes): {full * 1e3:.1f} us/plane "
      f"-> {full * n:.2f} ms per {n} planes")
for c in (int(x) for x in a.chunks.split(",")):
    hot = rate(c, max(8, 256 // c), 1)
    print(f"c={c:3d}  same chunk (L2-hot): {hot * 1e3:.1f} us/plane -> {hot * n:.2f} ms")
