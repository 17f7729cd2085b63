"""Per-rank GPU time of the transpose-free distributed solve
(distributed.solve_partitioned_carry), measured on ONE GPU by running one
rank's stages, plus the pipeline bubble of the carries. A projection for P
GPUs, not a multi-GPU measurement.

The timed rank sits in the middle of the z-order (it has both neighbours).
Every rank's sweeps run, one after another on this GPU (forward in rank order,
backward in reverse), so each carry is published before the launch that
reads it and nothing waits on a concurrent kernel; only the middle rank's
launches are timed. Projection:

  T(P) = dst + zfwd + zbwd + idst + (P - 1) (zfwd + zbwd) / waves + carry_nvl

waves = ceil(blocks / resident CTAs): rank p + 1 starts its first wave of
blocks when rank p finishes its first wave, so every boundary costs one wave
per direction; carry_nvl = the 24 B per mode per boundary at 900 GB/s.

    python tools/carry_estimate.py --cfg 4 --parts 2 4 8
"""
import argparse
import json
import math
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1912_03565_b200 as hb  # noqa: E402
from paper_1912_03565_b200 import _native, distributed as hd, workloads as wl  # noqa: E402
from paper_1912_03565_b200.tridiag import device_coefficients  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--cfg", type=int, default=4)
ap.add_argument("--parts", type=int, nargs="+", default=[2, 4, 8])
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--resident", type=int, default=4, help="carry-kernel CTAs per SM at occupancy")
ap.add_argument("--tune", default="", help="key=value,... passed to hfb_set_tuning (key 12: CTA cap)")
a = ap.parse_args()
tune = dict(map(int, kv.split("=")) for kv in filter(None, a.tune.split(",")))
for k, v in tune.items():
    _native.load_library().hfb_set_tuning(k, v)
if tune.get(12, 0) > 0:
    a.resident = min(a.resident, tune[12])
w = wl.workload(a.cfg)
g = w.grid
n_pts = g.n_x * g.n_y * g.n_z
dev = torch.device("cuda", 0)
P_ = _native.ptr
zplan = _native.get_plan(g.n_x, g.n_y, g.n_z, dev)
device_coefficients(zplan, w.scheme, w.profile, g)
lib, st = zplan.lib, zplan.stream()
ld = int(lib.hfb_modes_ld(zplan.handle))
size, nblk = hd.carry_layout(zplan, ld)
sms = torch.cuda.get_device_properties(dev).multi_processor_count
waves = math.ceil(nblk / (sms * a.resident))
res = []
for P in a.parts:
    ex = hb.make_exchange_plan(g, P)
    zr = ex.partition.z_ranges
    r = P // 2 if P > 1 else 0  # a middle rank (both neighbours)
    z0, z1 = zr[r]
    kpz = z1 - z0
    tplan = _native.get_plan(g.n_x, g.n_y, kpz, dev)
    F = torch.rand((kpz, g.n_y, g.n_x), dtype=torch.float64, device=dev)
    # every rank's slab of mode rows (the untimed ranks hold random modes)
    modes = [torch.rand((q1 - q0) * g.n_x * ld, dtype=torch.float64, device=dev) for q0, q1 in zr]
    cps = [torch.empty(((q1 - q0) + 7) // 8 * g.n_x * ld, dtype=torch.float64, device=dev)
           for q0, q1 in zr]
    regions = [torch.zeros(size, dtype=torch.float64, device=dev) for _ in zr]
    out = torch.empty((kpz, g.n_y, g.n_x), dtype=torch.float64, device=dev)
    work = tplan.workspace(5)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(6)]

    def sweep(q, d, epoch):
        peer = (q + 1 if q + 1 < P else None) if d == 0 else (q - 1 if q > 0 else None)
        _native.check(lib.hfb_zsolve_carry(zplan.handle, d, P_(modes[q]), ld, zr[q][0],
                                           zr[q][1] - zr[q][0], P_(cps[q]), P_(regions[q]),
                                           P_(regions[peer]) if peer is not None else None,
                                           epoch, st), f"sweep {q} {d}")

    best = None
    for rep in range(a.reps):
        epoch = rep + 1
        for q in range(P):  # forward sweeps in rank order: every carry-in is published
            if q == r:
                ev[0].record()
                _native.check(lib.hfb_forward_modes(tplan.handle, P_(F), P_(modes[r]), P_(work),
                                                    st), "forward_modes")
                ev[1].record()
                sweep(q, 0, epoch)
                ev[2].record()
            else:
                sweep(q, 0, epoch)
        for q in reversed(range(P)):  # backward sweeps in reverse order
            if q == r:
                ev[3].record()
                sweep(q, 1, epoch)
                ev[4].record()
                _native.check(lib.hfb_inverse_modes(tplan.handle, P_(modes[r]), P_(out), st),
                              "inverse_modes")
                ev[5].record()
            else:
                sweep(q, 1, epoch)
        torch.cuda.synchronize()
        t = [ev[0].elapsed_time(ev[1]), ev[1].elapsed_time(ev[2]), ev[3].elapsed_time(ev[4]),
             ev[4].elapsed_time(ev[5])]
        best = t if best is None or sum(t) < sum(best) else best
    code = hd.carry_status_code(zplan)
    assert code == 0, f"a carry was missing in the estimate (code {code})"
    del modes, cps, regions
    dst, zf, zb, idst = best
    bubble = (P - 1) * (zf + zb) / waves if P > 1 else 0.0
    carry_ms = (24 * g.n_x * g.n_y / 900e9 * 1e3) if P > 1 else 0.0
    total = dst + zf + zb + idst + bubble + carry_ms
    res.append({"parts": P, "rank": r, "levels": kpz, "forward_dst_ms": dst, "zsolve_fwd_ms": zf,
                "zsolve_bwd_ms": zb, "inverse_dst_ms": idst, "waves": waves,
                "bubble_ms": bubble, "carry_nvlink_ms": carry_ms, "projected_ms": total,
                "projected_pts_per_s": n_pts / (total / 1e3)})
print(json.dumps({"cfg": a.cfg, "tune": a.tune, "blocks": nblk, "resident_per_sm": a.resident,
                  "projection": res}, indent=1))
