"""CUDA-graph replay vs plain launches of the one-call solve for the small configs.

    python tools/graph_probe.py
"""
import sys, torch
sys.path.insert(0, '/root/repo')
from paper_1912_03565_b200 import _native, workloads as wl
from paper_1912_03565_b200.tridiag import device_coefficients
dev = torch.device('cuda', 0)
for cfg in (1, 2, 3):
    w = wl.workload(cfg); n = w.n
    plan = _native.get_plan(n, n, n, dev)
    device_coefficients(plan, w.scheme, w.profile, w.grid)
    F = wl.device_rhs(w, dev); U = torch.empty_like(F); work = plan.workspace(0)
    P = _native.ptr
    s = torch.cuda.Stream()
    def solve(st):
        _native.check(plan.lib.hfb_solve(plan.handle, P(F), P(U), P(work), st), 'solve')
    with torch.cuda.stream(s):
        for _ in range(3): solve(s.cuda_stream)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    R = 200 if cfg < 3 else 20
    with torch.cuda.stream(s):
        e0.record(s)
        for _ in range(R): solve(s.cuda_stream)
        e1.record(s)
    torch.cuda.synchronize(); t_plain = e0.elapsed_time(e1) / R
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        solve(s.cuda_stream)
    torch.cuda.synchronize()
    ref = U.clone()
    with torch.cuda.stream(s):
        e0.record(s)
        for _ in range(R): g.replay()
        e1.record(s)
    torch.cuda.synchronize(); t_graph = e0.elapsed_time(e1) / R
    print(f"cfg{cfg} n={n}: plain {t_plain*1e3:.1f} us/solve, graph {t_graph*1e3:.1f} us/solve, same={torch.equal(ref, U)}")
