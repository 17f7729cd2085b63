#!/usr/bin/env python
"""Benchmark: grid points solved per second (fp64) for BASELINE config 4 on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--cfg C]

A step is one full direct solve (forward 2D DST-I -> per-mode Thomas along z ->
inverse 2D DST-I) of the config's seeded synthetic RHS. N=1: the whole grid
on one GPU; N>1 (torchrun, one rank per GPU): z-slabs, NCCL all-to-all to
y-slabs for the z-solves and back (the reference's Partitioned geometry),
strong scaling of the same grid. Rank 0 prints ONE JSON line.

`value` times device-resident data with CUDA events (inputs, 8.6 GB, are far
larger than L2). `e2e` goes through the C-ABI host-buffer entry
(hfb_solve_host: pinned H2D, solve, D2H). `cpu_baseline` times the stock
reference the same way (one sample).
`--impl reference` times the UNMODIFIED reference (helmfft, installed into
oracle/_ref by oracle/build_ref.sh) on the host cores: stock solve_discrete
with SharedWorkers on a bounded z-slab sample of the same workload.
"""

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "grid points solved/sec (fp64) at 1/2/4/8 B200; % of HBM/NVLink roofline"
ALG_BYTES_PER_PT = 48  # 3 stages x (8 B read + 8 B write)
# Per launch of the one-call solve: every kernel reads and writes the volume
# once (8 B + 8 B per point) — its algorithmic minimum as a separate launch.
STAGE_ALG_BYTES = 16
STAGES_FAST = ["dstE x rows F->S1", "dstE y columns S1->S2 (tensor boxes)",
               "thomas_tma z-solve S2", "dstE inverse y rows S2", "dstE inverse x columns S2->U"]
STAGES_WAVE = ["dstE x rows F->S1", "dstE y columns + forward elimination S1->S2 x', CP cp",
               "(z-solve fused into the y-passes)",
               "back substitution + dstE inverse y rows S2 (planes descending)",
               "dstE inverse x columns S2->U"]
# bytes each launch must move in the wavefront-fused schedule: the y-pass reads
# the x-pass output and writes x' and cp; the inverse y-pass reads both back
STAGE_BYTES_WAVE = [16, 24, 0, 24, 16]
STAGES_LEAN = ["dstE x rows->columns F->S", "dstE y rows S", "thomas_tma z-solve S",
               "dstE inverse y rows S", "dstE inverse x columns S->U"]
FALLBACK_HBM = 6650.0


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--cfg", type=int, default=4)
    ap.add_argument("--e2e-steps", type=int, default=20,
                    help="steps of the end-to-end loop (the pipelined host path amortises its "
                         "fill and drain, one unoverlapped copy each way, over them)")
    ap.add_argument("--cpu-planes", type=int, default=None,
                    help="z-planes of the oracle CPU sample (default: all n for the "
                         "cpu_baseline, n/4 per step for --impl reference)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-dropin", action="store_true",
                    help="skip the drop-in API's end-to-end timing on host arrays")
    ap.add_argument("--partitioned-path", action="store_true",
                    help="use the multi-GPU (partitioned) path even at N = 1")
    ap.add_argument("--exchange", default="alltoall", choices=["carry", "alltoall"],
                    help="multi-GPU z-solve: the reference's slab<->pencil all-to-all over "
                         "NCCL (default: plain NCCL collectives) or the transpose-free carries "
                         "through CUDA-IPC peer memory (its protocol is verified live on one "
                         "GPU; cross-GPU runs unmeasured)")
    ap.add_argument("--launch-check", action="store_true",
                    help="CPU test of the launcher: every rank joins a gloo group and rank 0 "
                         "prints the world size seen by an all-reduce")
    return ap.parse_args()


def host_ram_bytes():
    try:
        return os.sysconf("SC_PAGE_SIZE") * os.sysconf("SC_PHYS_PAGES")
    except (ValueError, OSError):
        return 64 << 30


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as fh:
            d = json.load(fh)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return FALLBACK_HBM, "fallback (B200_PROFILING.md)"


def workload_config(w, n_gpus, exchange="alltoall"):
    multi = ("zslab{}+peer_carry" if exchange == "carry" else "zslab{}+nccl_alltoall").format(n_gpus)
    return {"workload": f"cfg{w.cfg}: {WORKLOAD_TEXT[w.cfg]}", "n": w.n,
            "points": w.n ** 3, "scheme": getattr(w.scheme, "value", "table"),
            "rhs": w.rhs_kind, "seed": w.seed,
            "parallelism": "single" if n_gpus == 1 else multi,
            "l2_flush": f"inputs {w.n ** 3 * 8 / 1e9:.1f} GB >> 126 MB L2 (no flush needed)"}


WORKLOAD_TEXT = {
    1: "4th-order Helmholtz 31^3, k=10(1+0.5 sin pi z)",
    2: "6th-order Helmholtz 127^3, k=10(1+0.5 sin pi z)",
    3: "6th-order Helmholtz 511^3, k=40(1+0.3 sin 2 pi z), F~N(0,1)",
    4: "4th-order conv-diff 1023^3, -lap u + 1.5 u_z (gamma=-1.5), F~U[-1,1]",
    5: "general 27-pt table 2047^3, seeded rows, centre=1.5 sum|off|, F~N(0,1)",
}


class ClockSampler:
    """nvidia-smi clocks/throttle sampling during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.path = tempfile.mktemp(prefix="clocks_", suffix=".csv")

    def start(self):
        try:
            self.fh = open(self.path, "w")
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"], stdout=self.fh,
                stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return None
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.fh.close()
        sm, mx, reasons = [], [], set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for line in open(self.path):
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                mx.append(float(parts[2]))
            except ValueError:
                continue
            for name, flag in zip(names, parts[5:9]):
                if flag.lower() == "active":
                    reasons.add(name)
        os.unlink(self.path)
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx),
                "samples": len(sm), "reasons": sorted(reasons)}


def dist_setup(n_gpus, force=False):
    import torch
    import torch.distributed as dist
    if force and "RANK" not in os.environ:  # a one-rank group for --partitioned-path
        import socket
        with socket.socket() as sk:
            sk.bind(("127.0.0.1", 0))
            port = sk.getsockname()[1]
        os.environ.update(RANK="0", LOCAL_RANK="0", WORLD_SIZE="1", MASTER_ADDR="127.0.0.1",
                          MASTER_PORT=str(port))
    if n_gpus > 1 or "RANK" in os.environ:
        # NCCL's INFO lines (communicator init: rank / nranks) go to stderr: main()
        # points fd 1 at stderr until the one JSON line
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        if not dist.is_initialized():
            local = int(os.environ.get("LOCAL_RANK", 0))
            torch.cuda.set_device(local)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        return dist.get_rank(), dist.get_world_size(), int(os.environ.get("LOCAL_RANK", 0))
    return 0, 1, 0


def oracle_baseline(w, planes, workers):
    """Oracle port on the first `planes` z-planes (full n x n planes) of the workload."""
    from oracle import helm_oracle as orc
    from paper_1912_03565_b200 import stencil as st
    import paper_1912_03565_b200 as hb
    g = hb.make_grid(hb.Domain(0, 1, 0, 1, 0, (planes + 1) / (w.n + 1)), w.n, w.n, planes)
    if isinstance(w.scheme, hb.StencilTable):
        T = tuple(t[:planes] for t in (w.scheme.A, w.scheme.B, w.scheme.C, w.scheme.D))
    else:
        prof = w.profile
        k = lambda a: np.real(np.asarray(a))[:planes + 2]
        T = orc.weight_table(w.scheme.value, k(prof.k2), k(prof.k2_z), k(prof.k2_zz),
                             complex(prof.gamma).real, (g.h_x, g.h_y, g.h_z), planes)
    cx, cy = orc.mode_cosines(w.n, w.n)
    from paper_1912_03565_b200 import workloads as wl
    F = wl.host_rhs(w, planes=planes)
    orc.solve(F[:2], tuple(t[:2] for t in T), cx, cy, workers=workers)  # warm the FFT plans
    t0 = time.perf_counter()
    orc.solve(F, T, cx, cy, workers=workers)
    dt = time.perf_counter() - t0
    del st
    return planes * w.n * w.n / dt, dt


def reference_sample(w, planes, workers):
    """The UNMODIFIED reference (oracle/_ref, installed by oracle/build_ref.sh) on
    the first `planes` z-levels of the workload (full n x n planes, same step h,
    the same seeded host F as complex128): stock helmfft.solve_discrete with
    SharedWorkers(min(workers, planes)) (Sequential() for workers = 1), the call
    BASELINE.md §2 names. Returns (pts/s by total_s, pts/s by transform +
    exchange + tridiag, PhaseTimings) or None without the reference."""
    from oracle import ref_bridge as rb
    hf = rb.load()
    if hf is None:
        return None
    F, sch, prof, g = rb.reference_case(hf, w, planes)
    _, t = rb.solve_reference(hf, F, sch, prof, g, workers)
    pts = planes * w.n * w.n
    return pts / t.total_s, pts / (t.transform_s + t.exchange_s + t.tridiag_s), t


def default_ref_planes(w):
    # about 64 Mi points per sample: a few seconds of the reference on 8-32 cores
    return max(2, min(w.n, (64 << 20) // (w.n * w.n)))


def run_reference(args):
    """CPU reference arm: the stock reference (kind "reference"), each step one
    bounded sample of the workload; the oracle port when the reference is not
    installed (kind "port")."""
    if args.gpus > 1 or "RANK" in os.environ:
        if int(os.environ.get("RANK", 0)) != 0:
            return
    from paper_1912_03565_b200 import workloads as wl
    w = wl.workload(args.cfg)
    cores = os.cpu_count() or 1
    planes = args.cpu_planes or default_ref_planes(w)
    kind = "reference"
    if reference_sample(w, 2, cores) is None:  # warms the FFT plans too
        kind = "port"
    vals, stage_vals, parts = [], [], []
    if kind == "reference":
        for _ in range(args.warmup):
            reference_sample(w, max(2, planes // 4), cores)
        for _ in range(args.steps):
            v, vs, t = reference_sample(w, planes, cores)
            vals.append(v)
            stage_vals.append(vs)
            parts.append(t)
        seq_planes = max(2, planes // 8)
        seq = reference_sample(w, seq_planes, 1)
        port_v, _ = oracle_baseline(w, planes, cores)
        tmed = parts[len(parts) // 2]
        sample = (f"stock helmfft.solve_discrete (oracle/_ref) with SharedWorkers({min(cores, planes)}) "
                  f"on the first {planes} of {w.n} z-planes (full {w.n}x{w.n} planes, same h, "
                  f"same seeded F as complex128) per step; value = points / PhaseTimings.total_s")
        extra = {"stages_value": statistics.median(stage_vals),
                 "stages_definition": "points / (transform_s + exchange_s + tridiag_s)",
                 "phase_timings_s": {"setup": tmed.setup_s, "transform": tmed.transform_s,
                                     "exchange": tmed.exchange_s, "tridiag": tmed.tridiag_s,
                                     "total": tmed.total_s},
                 "sequential": {"value": seq[0], "stages_value": seq[1], "cores": 1,
                                "sample": f"Sequential() on the first {seq_planes} z-planes"},
                 "port": {"value": port_v, "cores": cores,
                          "sample": f"oracle port (numpy/scipy, batched DUCC0) on the same "
                                    f"{planes} planes"}}
    else:
        for _ in range(args.warmup):
            oracle_baseline(w, max(2, planes // 4), cores)
        for _ in range(args.steps):
            vals.append(oracle_baseline(w, planes, cores)[0])
        sample = (f"{planes} of {w.n} z-planes (full {w.n}x{w.n} planes) per step, "
                  f"oracle port numpy/scipy DUCC0, {cores} threads (reference not installed)")
        extra = {}
    value = statistics.median(vals)
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "pts/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": planes * w.n * w.n / value * 1e3,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic", "config": workload_config(w, args.gpus),
            "cpu_baseline": {"value": value, "unit": "pts/s", "cores": cores, "kind": kind,
                             "sample": sample, **extra},
            "e2e": {"value": value, "unit": "pts/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    emit(line)


def dropin_e2e(w, hb, F_dev):
    """The drop-in API end to end on host arrays, as a reference user calls it:
    solve_discrete(Field3D(F), BoundaryData.zero(), scheme, profile, grid) with F
    a float64 and a complex128 (the reference's dtype) numpy array — upload,
    fold, solve, download included (best of 2 calls after one warm-up)."""
    Fh = F_dev.cpu().numpy()
    out = {}
    for name, arr in (("float64", Fh), ("complex128", None)):
        if arr is None:
            arr = Fh.astype(np.complex128)
        ts = []
        for _ in range(3):
            t0 = time.perf_counter()
            u, _ = hb.solve_discrete(hb.Field3D(arr), hb.BoundaryData.zero(), w.scheme,
                                     w.profile, w.grid)
            ts.append(time.perf_counter() - t0)
            del u
        best = min(ts[1:])
        out[name] = {"value": w.n ** 3 / best, "unit": "pts/s", "s_per_call": best,
                     "h2d_bytes": w.n ** 3 * 8, "d2h_bytes": arr.nbytes}
        del arr
    out["path"] = ("paper_1912_03565_b200.solve_discrete on numpy arrays (pipelined pinned "
                   "staging, device fold), one blocking call per step")
    return out


def run_ours(args):
    import ctypes
    import torch
    import torch.distributed as dist

    import paper_1912_03565_b200 as hb
    from paper_1912_03565_b200 import _native, workloads as wl
    from paper_1912_03565_b200.tridiag import device_coefficients

    rank, world, local = dist_setup(args.gpus, force=args.partitioned_path)
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    w = wl.workload(args.cfg)
    n = w.n
    lib = _native.load_library()
    # --partitioned-path: run the multi-GPU code path even on one rank (checks
    # the NCCL collectives and per-rank stages on a one-GPU box)
    multi = world > 1 or args.partitioned_path

    def barrier():
        if multi:
            dist.barrier(device_ids=[local])

    if not multi:
        plan = _native.get_plan(n, n, n, dev)
        device_coefficients(plan, w.scheme, w.profile, w.grid)
        F = wl.device_rhs(w, dev)
        # 2047^3 (137 GB in + out) only fits in place
        U = F if args.cfg == 5 else torch.empty_like(F)
        work = plan.workspace(0)
        st = plan.stream()

        def step():
            _native.check(lib.hfb_solve(plan.handle, _native.ptr(F), _native.ptr(U),
                                        _native.ptr(work), st), "solve")
    else:
        from paper_1912_03565_b200 import distributed as hd
        ex = hb.make_exchange_plan(w.grid, world)
        z0, z1 = ex.partition.z_ranges[rank]
        # this rank's planes of the one-GPU volume (same values at every N)
        F = wl.device_rhs(w, dev, planes=z1 - z0, z0=z0)

        solve_part = (hd.solve_partitioned_carry if args.exchange == "carry"
                      else hd.solve_partitioned)
        check_part = hd.check_status_carry if args.exchange == "carry" else hd.check_status

        def step():
            # pivot (and carry) agreement once after the timed loop (it synchronises the host)
            solve_part(F, w.scheme, w.profile, w.grid, check=False)

    for _ in range(max(3, args.warmup)):
        step()
    if not multi:
        plan.fetch_status()
    torch.cuda.synchronize(dev)
    sampler = ClockSampler(local)
    sampler.start()
    time.sleep(0.3)
    if not multi:  # per-launch CUDA events on the solve's stream, inside the timed region
        _native.check(lib.hfb_stage_timing(plan.handle, args.steps), "stage_timing")
    l0 = lib.hfb_launch_count()
    barrier()
    torch.cuda.synchronize(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.steps):
        step()
    e1.record()
    torch.cuda.synchronize(dev)
    barrier()
    launches = int(lib.hfb_launch_count() - l0)
    clocks = sampler.stop()
    if multi:
        check_part(w.grid, None, dev)
    stage_ms = None
    if not multi:
        buf = (ctypes.c_float * (5 * args.steps))()
        nslots = ctypes.c_int(0)
        _native.check(lib.hfb_stage_times(plan.handle, buf, ctypes.byref(nslots)), "stage_times")
        _native.check(lib.hfb_stage_timing(plan.handle, 0), "stage_timing")
        k = nslots.value
        stage_ms = [sum(buf[5 * r + i] for r in range(k)) / k for i in range(5)]
    ms = e0.elapsed_time(e1) / args.steps
    validate = None
    if not multi and U is not F:
        # the bench checks its own output: relative residual of the 27-point
        # system for the last timed solve (hfb_residual_sq on the device)
        res = hb.residual_l2(U, F, w.scheme, w.profile, w.grid)
        validate = {"rel_residual": res / float(torch.linalg.vector_norm(F).item()),
                    "definition": "||A U - F|| / ||F|| after the timed steps (device "
                                  "27-point residual, tests/test_gpu_parity_r2.py pins it)"}
    if multi:
        t = torch.tensor([ms], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    points = n ** 3
    value = points / (ms / 1e3)

    # ---- end to end through the C-ABI host-buffer entry (pinned H2D + solve + D2H)
    e2e = None
    if not args.no_e2e:
        vol_bytes = F.numel() * 8
        # the pipelined path keeps three device volumes and four pinned host volumes;
        # 2047^3 (68.6 GB a volume) only fits the blocking in-place call
        pipelined = 4 * vol_bytes < 0.6 * host_ram_bytes() and args.cfg != 5
        if not multi and not pipelined:
            hin = torch.empty(F.shape, dtype=torch.float64, pin_memory=True)
            hin.copy_(F)
            nbytes = vol_bytes
            del F, U
            torch.cuda.empty_cache()
            status = _native.HfbStatus()
            t0 = time.perf_counter()
            nblock = max(1, min(args.e2e_steps, 8))  # seconds each at 2047^3
            for _ in range(nblock):
                _native.check(lib.hfb_solve_host(plan.handle, _native.ptr(hin), _native.ptr(hin),
                                                 _native.ptr(work), st, ctypes.byref(status)),
                              "e2e")
            e2e_s = sync_s = (time.perf_counter() - t0) / nblock
            del hin
        elif not multi:
            # two pinned (input, output) pairs, as a caller streaming right-hand sides
            hins = [torch.empty(F.shape, dtype=torch.float64, pin_memory=True) for _ in range(2)]
            houts = [torch.empty(F.shape, dtype=torch.float64, pin_memory=True) for _ in range(2)]
            for h in hins:
                h.copy_(F)
            status = _native.HfbStatus()
            # latency of one synchronous call (H2D + solve + D2H)
            _native.check(lib.hfb_solve_host(plan.handle, _native.ptr(hins[0]),
                                             _native.ptr(houts[0]), _native.ptr(work), st,
                                             ctypes.byref(status)), "e2e")
            t0 = time.perf_counter()
            _native.check(lib.hfb_solve_host(plan.handle, _native.ptr(hins[0]),
                                             _native.ptr(houts[0]), _native.ptr(work), st,
                                             ctypes.byref(status)), "e2e")
            sync_s = time.perf_counter() - t0
            # throughput of pipelined calls (H2D of step k+1 and D2H of step k-1
            # overlap the solve of step k); every step still copies its input in
            # and its result out
            _native.check(lib.hfb_solve_host_async(plan.handle, _native.ptr(hins[0]),
                                                   _native.ptr(houts[0]), _native.ptr(work),
                                                   st), "e2e")
            _native.check(lib.hfb_host_sync(plan.handle, ctypes.byref(status)), "e2e")
            t0 = time.perf_counter()
            for k in range(args.e2e_steps):
                _native.check(lib.hfb_solve_host_async(plan.handle, _native.ptr(hins[k % 2]),
                                                       _native.ptr(houts[k % 2]),
                                                       _native.ptr(work), st), "e2e")
            _native.check(lib.hfb_host_sync(plan.handle, ctypes.byref(status)), "e2e")
            e2e_s = (time.perf_counter() - t0) / args.e2e_steps
            nbytes = F.numel() * 8
            del hins, houts
        else:
            from paper_1912_03565_b200 import distributed as hd
            hin = F.cpu().pin_memory()
            hout = torch.empty_like(hin).pin_memory()
            steps = max(1, min(args.e2e_steps, 4))
            barrier()
            t0 = time.perf_counter()
            for _ in range(steps):
                d = hin.to(dev, non_blocking=True)
                u = solve_part(d, w.scheme, w.profile, w.grid)
                hout.copy_(u, non_blocking=True)
                torch.cuda.synchronize(dev)
            barrier()
            e2e_s = (time.perf_counter() - t0) / steps
            tt = torch.tensor([e2e_s], device=dev, dtype=torch.float64)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            e2e_s = float(tt.item())
            nbytes = points * 8  # every rank copies its slab: the whole volume per step
        e2e = {"value": points / e2e_s, "unit": "pts/s", "h2d_bytes_per_step": nbytes,
               "d2h_bytes_per_step": nbytes, "ms_per_step": e2e_s * 1e3,
               "path": f"pinned H2D + {solve_part.__name__} + pinned D2H per rank" if multi
               else ("C-ABI hfb_solve_host_async, pinned host buffers, "
                     f"{args.e2e_steps} pipelined steps + hfb_host_sync") if pipelined
               else "C-ABI hfb_solve_host, one pinned host volume in place (blocking)"}
        if not multi:
            e2e["sync_ms_per_step"] = sync_s * 1e3  # one blocking hfb_solve_host call
        if not multi and args.cfg != 5 and not args.no_dropin:
            e2e["dropin"] = dropin_e2e(w, hb, F)

    if rank != 0:
        if multi:
            dist.destroy_process_group()
        return

    peak, peak_src = peaks()
    pipe_achieved = ALG_BYTES_PER_PT * points / (ms / 1e3) / 1e9 / (world if multi else 1)
    traffic_tab = {}
    prof_path = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(prof_path):
        try:
            traffic_tab = json.load(open(prof_path)).get(f"cfg{args.cfg}", {})
        except Exception:
            traffic_tab = {}
    pipeline = {"alg_bytes_per_point": ALG_BYTES_PER_PT, "achieved_GBs": pipe_achieved,
                "frac": pipe_achieved / peak,
                "definition": "SURVEY.md 8(d): 3 stages x (8 B read + 8 B write) per point "
                              "over the whole step"}
    if stage_ms is not None:
        lean = bool(getattr(plan, "lean", False))
        wave = stage_ms[2] <= 1e-3 < stage_ms[1]
        names = STAGES_WAVE if wave else STAGES_LEAN if lean else STAGES_FAST
        nbytes = STAGE_BYTES_WAVE if wave else [STAGE_ALG_BYTES] * 5
        stages = [{"kernel": nm, "ms": t, "alg_bytes_per_point": b,
                   "achieved_GBs": b * points / (t / 1e3) / 1e9 if t > 1e-3 else 0.0,
                   "traffic_bytes": traffic_tab.get(nm)}
                  for nm, t, b in zip(names, stage_ms, nbytes)]
        dom = max(stages, key=lambda e: e["ms"])
        roofline = {"bound": "hbm", "achieved": dom["achieved_GBs"], "peak": peak, "unit": "GB/s",
                    "frac": dom["achieved_GBs"] / peak, "traffic": dom["traffic_bytes"],
                    "kernel": dom["kernel"], "kernel_ms": dom["ms"],
                    "alg_bytes_per_launch": dom["alg_bytes_per_point"] * points,
                    "share_of_step": dom["ms"] / ms, "peak_source": peak_src,
                    "stages": stages, "pipeline": pipeline}
    else:
        roofline = {"bound": "hbm", "achieved": pipe_achieved, "peak": peak, "unit": "GB/s",
                    "frac": pipe_achieved / peak, "traffic": None,
                    "kernel": "whole solve pipeline (all launches of one step, max over ranks)",
                    "peak_source": peak_src, "pipeline": pipeline}
    cpu = None
    if not args.no_cpu and not multi:
        cores = os.cpu_count() or 1
        planes = args.cpu_planes or default_ref_planes(w)
        t0 = time.perf_counter()
        ref = reference_sample(w, planes, cores)
        if ref is not None:
            cpu = {"value": ref[0], "unit": "pts/s", "cores": cores, "kind": "reference",
                   "sample": f"stock helmfft.solve_discrete (oracle/_ref), SharedWorkers("
                             f"{min(cores, planes)}), first {planes} of {n} z-planes (full "
                             f"{n}x{n} planes), {time.perf_counter() - t0:.1f} s; value = "
                             f"points / total_s", "stages_value": ref[1]}
        else:
            v, dt = oracle_baseline(w, planes, cores)
            cpu = {"value": v, "unit": "pts/s", "cores": cores, "kind": "port",
                   "sample": f"{planes} of {n} z-planes (full {n}x{n} planes), "
                             f"{dt:.1f} s, numpy/scipy oracle"}
    line = {"metric": METRIC, "value": value, "unit": "pts/s", "n_gpus": world,
            "steps": args.steps, "warmup": max(3, args.warmup), "ms_per_step": ms,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic (seeded, generated on device)",
            "config": workload_config(w, world, args.exchange), "roofline": roofline, "cpu_baseline": cpu,
            "e2e": e2e, "gpu_launches": launches, "clocks": clocks, "check": validate,
            "device": torch.cuda.get_device_name(dev)}
    emit(line)
    if dist.is_initialized():
        dist.destroy_process_group()


_STDOUT_FD = None


def emit(line):
    """Print the one JSON result line on the real stdout. Everything else that
    reaches file descriptor 1 during the run (library banners such as NCCL's
    version line) was redirected to stderr by main()."""
    sys.stdout.flush()
    if _STDOUT_FD is not None:
        os.write(_STDOUT_FD, (json.dumps(line) + "\n").encode())
    else:
        print(json.dumps(line), flush=True)


def self_launch(args):
    """`python bench.py --gpus N` with N > 1 outside a launcher: start N local
    ranks under torch.distributed.run (one process per GPU, rendezvous on
    127.0.0.1) with the same arguments; rank 0's JSON line passes through on
    stdout, everything else (NCCL INFO included) on stderr. Returns the exit code."""
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1",
           f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    env = dict(os.environ, BENCH_SELF_LAUNCHED="1")
    env.setdefault("OMP_NUM_THREADS", "1")
    return subprocess.call(cmd, env=env)


def launch_check(args):
    import torch
    import torch.distributed as dist
    dist.init_process_group("gloo")
    t = torch.ones(1)
    dist.all_reduce(t)
    if dist.get_rank() == 0:
        emit({"launch_check": True, "world": dist.get_world_size(), "sum": int(t.item()),
              "n_gpus": args.gpus, "self_launched": os.environ.get("BENCH_SELF_LAUNCHED") == "1"})
    dist.destroy_process_group()


def main():
    global _STDOUT_FD
    args = parse()
    if args.gpus > 1 and "RANK" not in os.environ and "LOCAL_RANK" not in os.environ:
        sys.exit(self_launch(args))
    sys.stdout.flush()
    _STDOUT_FD = os.dup(1)
    os.dup2(2, 1)  # stdout -> stderr until the result line
    if args.launch_check:
        launch_check(args)
    elif args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
