"""Pinned-host copy bandwidth with the copies split over several streams per
direction (chunked), alone and bidirectional (diagnostic).

    python tools/pcie2.py [--gb 4] [--streams 1,2,4] [--chunk-mb 256]
"""
import argparse
import time

import torch

ap = argparse.ArgumentParser()
ap.add_argument("--gb", type=float, default=4.0)
ap.add_argument("--streams", default="1,2,4")
ap.add_argument("--chunk-mb", type=int, default=256)
a = ap.parse_args()
n = int(a.gb * 2**30 / 8)
h1 = torch.empty(n, dtype=torch.float64).pin_memory()
h2 = torch.empty(n, dtype=torch.float64).pin_memory()
d1 = torch.empty(n, dtype=torch.float64, device="cuda")
d2 = torch.empty(n, dtype=torch.float64, device="cuda")
ch = a.chunk_mb * 2**20 // 8


def run(h2d, d2h, ss_in, ss_out):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for i, o in enumerate(range(0, n, ch)):
        if h2d:
            with torch.cuda.stream(ss_in[i % len(ss_in)]):
                d1[o:o + ch].copy_(h1[o:o + ch], non_blocking=True)
        if d2h:
            with torch.cuda.stream(ss_out[i % len(ss_out)]):
                h2[o:o + ch].copy_(d2[o:o + ch], non_blocking=True)
    torch.cuda.synchronize()
    return time.perf_counter() - t0


for k in (int(x) for x in a.streams.split(",")):
    si = [torch.cuda.Stream() for _ in range(k)]
    so = [torch.cuda.Stream() for _ in range(k)]
    run(True, True, si, so)
    for name, args in (("h2d", (True, False)), ("d2h", (False, True)), ("both", (True, True))):
        t = min(run(*args, si, so) for _ in range(3))
        print(f"streams/dir={k} {name}: {a.gb * 2**30 / 1e9 / t:.1f} GB/s per direction")
