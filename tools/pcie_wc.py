"""Pinned-host copy bandwidth with the H2D source in WRITE-COMBINED pinned memory
(cudaHostAllocWriteCombined) against ordinary pinned memory: H2D alone and H2D +
D2H at once (raw cudaMemcpyAsync on two streams).

    python tools/pcie_wc.py [--gb 4]
"""
import argparse
import ctypes
import time

import torch

ap = argparse.ArgumentParser()
ap.add_argument("--gb", type=float, default=4.0)
a = ap.parse_args()
nbytes = int(a.gb * 2**30)
rt = ctypes.CDLL("libcudart.so.12")
torch.cuda.init()
d1 = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
d2 = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
vp = ctypes.c_void_p


def host_alloc(flags):
    p = vp()
    rc = rt.cudaHostAlloc(ctypes.byref(p), ctypes.c_size_t(nbytes), ctypes.c_uint(flags))
    assert rc == 0, rc
    ctypes.memset(p, 1, nbytes)
    return p


def run(src, dst, h2d, d2h):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    if h2d:
        rc = rt.cudaMemcpyAsync(vp(d1.data_ptr()), src, ctypes.c_size_t(nbytes), 1, vp(s1.cuda_stream))
        assert rc == 0
    if d2h:
        rc = rt.cudaMemcpyAsync(dst, vp(d2.data_ptr()), ctypes.c_size_t(nbytes), 2, vp(s2.cuda_stream))
        assert rc == 0
    torch.cuda.synchronize()
    return time.perf_counter() - t0


out = host_alloc(0)
for name, flags in (("pinned", 0), ("write-combined", 4), ("portable+mapped", 3)):
    src = host_alloc(flags)
    run(src, out, True, True)
    for what, args in (("h2d", (True, False)), ("d2h", (False, True)), ("both", (True, True))):
        t = min(run(src, out, *args) for _ in range(3))
        print(f"{name:16s} {what}: {t * 1e3:.1f} ms for {a.gb} GiB each way -> "
              f"{nbytes / 1e9 / t:.1f} GB/s per direction")
    rt.cudaFreeHost(src)
