"""Three-stage direct solve on B200: the drop-in for helmfft.solver.

Same entry points and arguments as the reference (solver.py:38-422):
``solve_discrete(rhs, boundary, scheme, profile, grid, config)``,
``solve_direct(problem, config)``, ``solve_with_timings(problem, config)``,
the mode dataclasses, ``plan_partition`` and the exchange plans.

Every mode runs on the GPU — there is no CPU path:

- ``Sequential()`` / ``SharedWorkers(w)`` / ``Device()``: the single-GPU
  pipeline (forward 2D DST-I -> per-mode Thomas -> inverse 2D DST-I) of the
  sm_100a library in one call (hfb_solve); its phase timings split the
  device time into transform_s (the four DST launches) and tridiag_s (the
  z-solve) from the library's per-launch CUDA events, as the reference
  reports them. ``Device(staged=True)`` runs the three stages as separate
  calls. Host
  worker counts are validated like the reference and otherwise irrelevant:
  parallelism is the GPU's.
- ``Partitioned(p, t)``: the reference's slab <-> pencil geometry on one
  device: part p transforms its z-slab, the blocks (kpz(p), kpy(q), n_x)
  are redistributed by a device copy, part q solves its y-slab with mode
  offset y0(q), and the blocks go back. Every part runs the same per-line
  arithmetic, so the answer equals the single-device one bit for bit.
  The multi-GPU version (one process per GPU, NCCL all-to-all) is
  ``distributed.solve_partitioned``.

Phase timings come from CUDA events on the solve's stream.
"""

import ctypes
import threading
import time
from dataclasses import dataclass, field
from typing import Callable, Optional, Union

import numpy as np

from . import _device as dv
from ._native import check, get_plan, ptr
from .assembly import BoundaryData, Field3D, build_rhs, fold_device_parts, fold_dirichlet
from .errors import InvalidPartitionError
from .grid import CoefficientProfile, Grid3D
from .spectral import make_plan
from .stencil import scheme_key
from .transport import STAGE_FORWARD, STAGE_INVERSE, InProcessMesh  # noqa: F401
from .tridiag import device_coefficients

PER_PLANE = "per-plane"
PER_LINE_BATCH = "per-line-batch"


@dataclass(frozen=True)
class Sequential:
    pass


@dataclass(frozen=True)
class SharedWorkers:
    workers: int


@dataclass(frozen=True)
class Partitioned:
    parts: int
    workers_per_part: int = 1


@dataclass(frozen=True)
class Device:
    """Explicit single-GPU mode. ``staged=True`` runs the three stages as
    separate library calls (per-stage timings); the default is the whole
    pipeline in one call."""

    staged: bool = False


Mode = Union[Sequential, SharedWorkers, Partitioned, Device]


@dataclass(frozen=True)
class SolverConfig:
    mode: Mode = field(default_factory=Sequential)
    transform_parallelism: str = PER_PLANE
    # factory(n_parts) -> list of transports, one per part (the reference's plugin
    # hook, solver.py:65-66): Partitioned mode then routes its blocks through
    # them (_solve_transport); None = the device moves the blocks itself
    transport_factory: Optional[Callable] = None


@dataclass(frozen=True)
class PhaseTimings:
    setup_s: float = 0.0
    transform_s: float = 0.0
    exchange_s: float = 0.0
    tridiag_s: float = 0.0
    total_s: float = 0.0


def plan_partition(extent: int, parts: int):
    """Contiguous half-open ranges, sizes differing by at most one, larger first (solver.py:78-93)."""
    if parts < 1 or parts > extent:
        raise InvalidPartitionError(f"cannot split {extent} indices into {parts} parts")
    size, extra = divmod(extent, parts)
    bounds = np.cumsum([0] + [size + (p < extra) for p in range(parts)])
    return [(int(a), int(b)) for a, b in zip(bounds[:-1], bounds[1:])]


@dataclass(frozen=True)
class PartitionPlan:
    """Per-part z-ranges (transforms) and y-ranges (tridiagonal stage) (solver.py:96-112)."""

    z_ranges: tuple
    y_ranges: tuple

    @property
    def n_parts(self):
        return len(self.z_ranges)


def make_partition_plan(grid: Grid3D, parts: int) -> PartitionPlan:
    return PartitionPlan(tuple(plan_partition(grid.n_z, parts)),
                         tuple(plan_partition(grid.n_y, parts)))


@dataclass(frozen=True)
class ExchangePlan:
    """Geometry of the z-slab <-> y-slab redistribution (solver.py:115-143)."""

    n_x: int
    n_y: int
    n_z: int
    partition: PartitionPlan

    @property
    def n_parts(self):
        return self.partition.n_parts

    def block_extents(self, sender: int, receiver: int):
        """(ext_x, ext_y, ext_z) of the forward block sender -> receiver."""
        z0, z1 = self.partition.z_ranges[sender]
        y0, y1 = self.partition.y_ranges[receiver]
        return (self.n_x, y1 - y0, z1 - z0)

    def total_volume(self):
        return sum(int(np.prod(self.block_extents(p, q)))
                   for p in range(self.n_parts) for q in range(self.n_parts))


def make_exchange_plan(grid: Grid3D, parts: int) -> ExchangePlan:
    return ExchangePlan(grid.n_x, grid.n_y, grid.n_z, make_partition_plan(grid, parts))


def exchange_forward(plan: ExchangePlan, transport, part: int, z_slab):
    """z-slab (kpz, n_y, n_x) -> y-slab (n_z, kpy, n_x) through a transport (solver.py:146-174).

    Host-array contract of the reference, blocks sent in ascending
    destination order; the device pipelines use device copies / NCCL instead.
    """
    zr, yr = plan.partition.z_ranges, plan.partition.y_ranges
    (z0, z1), (y0, y1) = zr[part], yr[part]
    if tuple(z_slab.shape) != (z1 - z0, plan.n_y, plan.n_x):
        raise ValueError(f"z-slab shape {tuple(z_slab.shape)} != {(z1 - z0, plan.n_y, plan.n_x)}")
    y_slab = np.empty((plan.n_z, y1 - y0, plan.n_x), dtype=z_slab.dtype)
    for q, (qy0, qy1) in enumerate(yr):
        if q == part:
            y_slab[z0:z1] = z_slab[:, y0:y1, :]
        else:
            transport.send(q, STAGE_FORWARD, np.ascontiguousarray(z_slab[:, qy0:qy1, :]))
    for q, (qz0, qz1) in enumerate(zr):
        if q != part:
            y_slab[qz0:qz1] = transport.receive(q, STAGE_FORWARD, plan.block_extents(q, part))
    return y_slab


def exchange_inverse(plan: ExchangePlan, transport, part: int, y_slab):
    """Inverse of exchange_forward (solver.py:177-201)."""
    zr, yr = plan.partition.z_ranges, plan.partition.y_ranges
    (z0, z1), (y0, y1) = zr[part], yr[part]
    if tuple(y_slab.shape) != (plan.n_z, y1 - y0, plan.n_x):
        raise ValueError(f"y-slab shape {tuple(y_slab.shape)} != {(plan.n_z, y1 - y0, plan.n_x)}")
    z_slab = np.empty((z1 - z0, plan.n_y, plan.n_x), dtype=y_slab.dtype)
    for q, (qz0, qz1) in enumerate(zr):
        if q == part:
            z_slab[:, y0:y1, :] = y_slab[z0:z1]
        else:
            transport.send(q, STAGE_INVERSE, np.ascontiguousarray(y_slab[qz0:qz1]))
    for q, (qy0, qy1) in enumerate(yr):
        if q != part:
            ext_x, _, ext_z = plan.block_extents(part, q)
            z_slab[:, qy0:qy1, :] = transport.receive(q, STAGE_INVERSE,
                                                      (ext_x, qy1 - qy0, ext_z))
    return z_slab


def _coerce_config(config):
    """Accept the reference's own SolverConfig / mode objects (helmfft.solver) as
    well as this package's: callers written against the reference (its harness,
    its tests) pass those. Matched by class name and fields."""
    if isinstance(config, SolverConfig) and isinstance(
            config.mode, (Sequential, SharedWorkers, Partitioned, Device)):
        return config
    mode = getattr(config, "mode", None)
    kind = type(mode).__name__
    if kind == "Sequential":
        mode = Sequential()
    elif kind == "SharedWorkers":
        mode = SharedWorkers(mode.workers)
    elif kind == "Partitioned":
        mode = Partitioned(mode.parts, getattr(mode, "workers_per_part", 1))
    elif kind == "Device":
        mode = Device(getattr(mode, "staged", False))
    else:
        raise ValueError(f"unknown mode {mode!r}")
    return SolverConfig(mode=mode,
                        transform_parallelism=getattr(config, "transform_parallelism", PER_PLANE),
                        transport_factory=getattr(config, "transport_factory", None))


def _validate_config(config: SolverConfig, grid: Grid3D):
    """Worker / part bounds exactly as the reference enforces them (solver.py:204-238)."""
    if config.transform_parallelism not in (PER_PLANE, PER_LINE_BATCH):
        raise ValueError(f"unknown transform parallelism {config.transform_parallelism!r}")
    mode = config.mode
    per_plane = config.transform_parallelism == PER_PLANE
    if isinstance(mode, (Sequential, Device)):
        return
    if isinstance(mode, SharedWorkers):
        w = mode.workers
        if w < 1:
            raise ValueError(f"worker count must be >= 1, got {w}")
        if per_plane and w > grid.n_z:
            raise InvalidPartitionError(f"{w} workers need {w} planes, grid has {grid.n_z}")
        if not per_plane and (w > grid.n_x or w > grid.n_y):
            raise InvalidPartitionError(f"{w} workers exceed line counts ({grid.n_x}, {grid.n_y})")
        return
    if isinstance(mode, Partitioned):
        p, t = mode.parts, mode.workers_per_part
        if p < 1 or t < 1:
            raise ValueError("part and worker counts must be >= 1")
        if p > grid.n_z or p > grid.n_y:
            raise InvalidPartitionError(f"{p} parts exceed slab extents ({grid.n_z}, {grid.n_y})")
        if per_plane and t > grid.n_z // p:
            raise InvalidPartitionError(
                f"{t} workers per part need as many local planes; smallest slab has "
                f"{grid.n_z // p}")
        if not per_plane and (t > grid.n_x or t > grid.n_y):
            raise InvalidPartitionError(
                f"{t} workers per part exceed line counts ({grid.n_x}, {grid.n_y})")
        return
    raise ValueError(f"unknown mode {mode!r}")


class _EventClock:
    """CUDA-event stopwatch on the current stream: marks, then seconds between them."""

    def __init__(self, torch, device):
        self.torch, self.device = torch, device
        self.marks = {}

    def mark(self, name):
        ev = self.torch.cuda.Event(enable_timing=True)
        ev.record(self.torch.cuda.current_stream(self.device))
        self.marks[name] = ev

    def seconds(self, a, b):
        self.marks[b].synchronize()
        return self.marks[a].elapsed_time(self.marks[b]) / 1e3


def _solve_part_device(plan, t, grid, config, clock, part_idx):
    """Run one real part in place on the device according to the mode."""
    torch = dv._torch()
    mode = config.mode
    lib, h = plan.lib, plan.handle
    st = plan.stream()
    n_z, n_y, n_x = grid.shape
    tag = f"{part_idx}"
    if isinstance(mode, Partitioned):
        # the multi-GPU per-rank stages, parts exchanging by device copies
        from .distributed import solve_partitioned_local
        res = solve_partitioned_local(t, None, None, grid, mode.parts, clock)
        if res is not None:
            u, phases = res
            t.copy_(u)
            return phases
        ex = make_exchange_plan(grid, mode.parts)
        work_t = plan.workspace(1)
        clock.mark("t0" + tag)
        for z0, z1 in ex.partition.z_ranges:
            check(lib.hfb_transform_stack(h, ptr(t), z0, z1, ptr(work_t), st), "transform")
        clock.mark("t1" + tag)
        y_slabs = [t[:, y0:y1, :].contiguous() for y0, y1 in ex.partition.y_ranges]
        clock.mark("t2" + tag)
        for (y0, y1), slab in zip(ex.partition.y_ranges, y_slabs):
            cpw = torch.empty_like(slab)
            check(lib.hfb_solve_slab(h, ptr(slab), y1 - y0, y0, ptr(cpw), st), "solve_slab")
        clock.mark("t3" + tag)
        for (y0, y1), slab in zip(ex.partition.y_ranges, y_slabs):
            t[:, y0:y1, :] = slab
        clock.mark("t4" + tag)
        for z0, z1 in ex.partition.z_ranges:
            check(lib.hfb_transform_stack(h, ptr(t), z0, z1, ptr(work_t), st), "transform")
        clock.mark("t5" + tag)
        return (clock.seconds("t0" + tag, "t1" + tag) + clock.seconds("t4" + tag, "t5" + tag),
                clock.seconds("t1" + tag, "t2" + tag) + clock.seconds("t3" + tag, "t4" + tag),
                clock.seconds("t2" + tag, "t3" + tag))
    staged = isinstance(mode, Device) and mode.staged
    if staged:
        work_t = plan.workspace(1)
        cpw = torch.empty_like(t)
        clock.mark("t0" + tag)
        check(lib.hfb_transform_stack(h, ptr(t), 0, n_z, ptr(work_t), st), "transform")
        clock.mark("t1" + tag)
        check(lib.hfb_solve_slab(h, ptr(t), n_y, 0, ptr(cpw), st), "solve_slab")
        clock.mark("t2" + tag)
        check(lib.hfb_transform_stack(h, ptr(t), 0, n_z, ptr(work_t), st), "transform")
        clock.mark("t3" + tag)
        return (clock.seconds("t0" + tag, "t1" + tag) + clock.seconds("t2" + tag, "t3" + tag),
                0.0, clock.seconds("t1" + tag, "t2" + tag))
    work = plan.workspace(0)
    with _StageSplit(plan) as split:
        check(lib.hfb_solve(h, ptr(t), ptr(t), ptr(work), st), "solve")
    return split.phases


class _StageSplit:
    """Phase split of one one-call solve (hfb_solve / hfb_solve_z) from the
    library's per-launch CUDA events (hfb_stage_timing): transform_s = the
    forward and inverse 2D DST launches, tridiag_s = the z-solve — the
    reference's PhaseTimings breakdown (solver.py:310-316)."""

    def __init__(self, plan):
        self.plan = plan
        self.phases = (0.0, 0.0, 0.0)

    def __enter__(self):
        check(self.plan.lib.hfb_stage_timing(self.plan.handle, 1), "stage_timing")
        return self

    def __exit__(self, exc_type, *exc):
        lib, h = self.plan.lib, self.plan.handle
        try:
            if exc_type is None:
                ms = (ctypes.c_float * 5)()
                nslots = ctypes.c_int(0)
                check(lib.hfb_stage_times(h, ms, ctypes.byref(nslots)), "stage_times")
                if nslots.value != 1:
                    raise RuntimeError("the solve recorded no stage events")
                if ms[2] <= 1e-3 < ms[1]:
                    # wavefront-fused schedule: the z-solve sweeps ride in the two
                    # y-pass launches (forward elimination / back substitution)
                    self.phases = ((ms[0] + ms[4]) / 1e3, 0.0, (ms[1] + ms[3]) / 1e3)
                else:
                    self.phases = ((ms[0] + ms[1] + ms[3] + ms[4]) / 1e3, 0.0, ms[2] / 1e3)
        finally:
            lib.hfb_stage_timing(h, 0)
        return False


def _solve_z_device(plan, tr, ti, grid, config, clock):
    """Complex-coefficient solve (complex k(z)) of the (re, im) pair in place."""
    torch = dv._torch()
    mode = config.mode
    lib, h = plan.lib, plan.handle
    st = plan.stream()
    n_z, n_y, n_x = grid.shape

    def transform(z0=0, z1=n_z):
        work_t = plan.workspace(1)
        for t in (tr, ti):
            check(lib.hfb_transform_stack(h, ptr(t), z0, z1, ptr(work_t), st), "transform")

    if isinstance(mode, Partitioned) or (isinstance(mode, Device) and mode.staged):
        parts = mode.parts if isinstance(mode, Partitioned) else 1
        ex = make_exchange_plan(grid, parts)
        clock.mark("z0")
        for z0, z1 in ex.partition.z_ranges:
            transform(z0, z1)
        clock.mark("z1")
        slabs = [(tr[:, y0:y1, :].contiguous(), ti[:, y0:y1, :].contiguous())
                 for y0, y1 in ex.partition.y_ranges]
        clock.mark("z2")
        for (y0, y1), (sr, si) in zip(ex.partition.y_ranges, slabs):
            cpw = torch.empty((2,) + tuple(sr.shape), dtype=torch.float64, device=sr.device)
            check(lib.hfb_solve_slab_z(h, ptr(sr), ptr(si), y1 - y0, y0, ptr(cpw), st),
                  "solve_slab_z")
        clock.mark("z3")
        for (y0, y1), (sr, si) in zip(ex.partition.y_ranges, slabs):
            tr[:, y0:y1, :] = sr
            ti[:, y0:y1, :] = si
        clock.mark("z4")
        for z0, z1 in ex.partition.z_ranges:
            transform(z0, z1)
        clock.mark("z5")
        return (clock.seconds("z0", "z1") + clock.seconds("z4", "z5"),
                clock.seconds("z1", "z2") + clock.seconds("z3", "z4"),
                clock.seconds("z2", "z3"))
    work = plan.workspace(3)
    with _StageSplit(plan) as split:
        check(lib.hfb_solve_z(h, ptr(tr), ptr(ti), ptr(tr), ptr(ti), ptr(work), st), "solve_z")
    return split.phases


def _solve_transport(plan, parts, grid, config):
    """Partitioned(p, t) with a caller-supplied ``transport_factory``: the
    reference's part-thread structure (solver.py:319-399) with its blocks routed
    through the caller's transports (its plugin hook, solver.py:323-327).

    One host thread per part, barrier-separated stages like the reference:
    the part transforms its z-slab on the device, downloads it, sends and
    receives the (kpz, kpy(q), n_x) blocks through ``transports[part]``
    (exchange_forward, ascending destination order), uploads its y-slab and
    runs the per-mode z-solves there with mode offset y0, and the mirror image
    back. A transport failure raises the transport's own exception (e.g.
    ExchangeError) exactly as the reference propagates it. The blocks hold the
    reference's dtype: complex128 when the field or the table is complex.
    Device calls are serialised by a lock (one device, one workspace); every
    arithmetic step is the same kernel as the in-device Partitioned mode."""
    torch = dv._torch()
    mode = config.mode
    nparts = mode.parts
    lib, h = plan.lib, plan.handle
    ex = make_exchange_plan(grid, nparts)
    transports = config.transport_factory(nparts)
    work_t = plan.workspace(1)
    dev_lock = threading.Lock()
    barrier = threading.Barrier(nparts)
    cplx = len(parts) == 2
    times = [None] * nparts
    errors = []

    def dev_call(fn):
        with dev_lock:
            with torch.cuda.device(plan.device):
                out = fn(plan.stream())
                torch.cuda.current_stream(plan.device).synchronize()
                return out

    def transform(z0, z1):
        def go(st):
            for t in parts:
                check(lib.hfb_transform_stack(h, ptr(t), z0, z1, ptr(work_t), st), "transform")
        dev_call(go)

    def host_slab(z0, z1):
        hs = [t[z0:z1].cpu().numpy() for t in parts]
        return hs[0] + 1j * hs[1] if cplx else hs[0]

    def run_part(part):
        try:
            tr = exs = tri = 0.0
            z0, z1 = ex.partition.z_ranges[part]
            y0, y1 = ex.partition.y_ranges[part]
            barrier.wait()
            t0 = time.perf_counter()
            transform(z0, z1)
            local = dev_call(lambda st: host_slab(z0, z1))
            tr += time.perf_counter() - t0
            barrier.wait()
            t0 = time.perf_counter()
            y_slab = exchange_forward(ex, transports[part], part, local)
            exs += time.perf_counter() - t0
            barrier.wait()
            t0 = time.perf_counter()

            def solve(st):
                re = dv.upload(np.ascontiguousarray(y_slab.real if cplx else y_slab), plan.device)
                if cplx:
                    im = dv.upload(np.ascontiguousarray(y_slab.imag), plan.device)
                    cpw = torch.empty((2,) + tuple(re.shape), dtype=torch.float64,
                                      device=plan.device)
                    if plan.complex_coef:
                        check(lib.hfb_solve_slab_z(h, ptr(re), ptr(im), y1 - y0, y0, ptr(cpw),
                                                   st), "solve_slab_z")
                    else:
                        for t in (re, im):
                            check(lib.hfb_solve_slab(h, ptr(t), y1 - y0, y0, ptr(cpw), st),
                                  "solve_slab")
                    return re.cpu().numpy() + 1j * im.cpu().numpy()
                cpw = torch.empty_like(re)
                check(lib.hfb_solve_slab(h, ptr(re), y1 - y0, y0, ptr(cpw), st), "solve_slab")
                return re.cpu().numpy()

            y_slab = dev_call(solve)
            tri += time.perf_counter() - t0
            barrier.wait()
            t0 = time.perf_counter()
            local = exchange_inverse(ex, transports[part], part, y_slab)
            exs += time.perf_counter() - t0
            barrier.wait()
            t0 = time.perf_counter()

            def put_back(st):
                for k, t in enumerate(parts):
                    src = (local.imag if k else local.real) if cplx else local
                    t[z0:z1].copy_(torch.from_numpy(np.ascontiguousarray(src)))

            dev_call(put_back)
            transform(z0, z1)
            tr += time.perf_counter() - t0
            times[part] = (tr, exs, tri)
        except BaseException as exc:  # propagate to the caller, release the peers
            errors.append(exc)
            barrier.abort()

    threads = [threading.Thread(target=run_part, args=(q,)) for q in range(nparts)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    for tp in transports:
        tp.close()
    if errors:
        for exc in errors:  # the root cause rather than broken-barrier fallout
            if not isinstance(exc, threading.BrokenBarrierError):
                raise exc
        raise errors[0]
    return tuple(max(t[i] for t in times) for i in range(3))


def solve_discrete(rhs: Field3D, boundary: BoundaryData, scheme, profile: CoefficientProfile,
                   grid: Grid3D, config: SolverConfig = SolverConfig()):
    """Solve the 27-point system for a prebuilt (unfolded) right-hand side (solver.py:278-399).

    Returns (Field3D, PhaseTimings). The caller's rhs is never modified.
    A numpy rhs gives a numpy solution; a CUDA tensor rhs stays on its device.
    """
    torch = dv._torch()
    t_start = time.perf_counter()
    config = _coerce_config(config)
    _validate_config(config, grid)
    make_plan(grid.n_x, grid.n_y)
    scheme_key(scheme)
    values = dv.unwrap(rhs)
    if tuple(values.shape) != grid.shape:
        raise ValueError(f"rhs shape {tuple(values.shape)} != grid {grid.shape}")
    on_device = dv.is_tensor(values)
    device = values.device if on_device else torch.device("cuda", torch.cuda.current_device())
    plan = get_plan(grid.n_x, grid.n_y, grid.n_z, device)
    with plan.lock:
        device_coefficients(plan, scheme, profile, grid)
        if on_device:
            # float64 or complex128 CUDA tensors: private real parts (the caller's
            # field is never modified), then the fold on the device
            parts = fold_device_parts(dv.device_parts(values, copy=True), boundary, scheme,
                                      profile, grid, device)
        else:
            # host arrays: pipelined pinned upload of the caller's array (never
            # modified), then the Dirichlet fold on the device (assembly.py:258-274)
            parts = fold_device_parts(dv.upload_parts(values, device), boundary, scheme,
                                      profile, grid, device)
        # the fold may have switched the plan's coefficients back and forth
        device_coefficients(plan, scheme, profile, grid)
        torch.cuda.current_stream(device).synchronize()
        setup_s = time.perf_counter() - t_start
        clock = _EventClock(torch, device)
        transform_s = exchange_s = tridiag_s = 0.0
        if isinstance(config.mode, Partitioned) and config.transport_factory is not None:
            if plan.complex_coef:
                while len(parts) < 2:
                    parts.append(torch.zeros_like(parts[0]))
            transform_s, exchange_s, tridiag_s = _solve_transport(plan, parts, grid, config)
        elif plan.complex_coef:
            while len(parts) < 2:
                parts.append(torch.zeros_like(parts[0]))
            transform_s, exchange_s, tridiag_s = _solve_z_device(plan, parts[0], parts[1],
                                                                 grid, config, clock)
        else:
            for k, t in enumerate(parts):
                tr, ex, tri = _solve_part_device(plan, t, grid, config, clock, k)
                transform_s += tr
                exchange_s += ex
                tridiag_s += tri
        plan.fetch_status()
    if on_device:
        out = Field3D(dv.join_device(parts, values))
    else:
        out = Field3D(dv.download_parts(parts, values))
    timings = PhaseTimings(setup_s=setup_s, transform_s=transform_s, exchange_s=exchange_s,
                           tridiag_s=tridiag_s, total_s=time.perf_counter() - t_start)
    return out, timings


def solve_direct(problem, config: SolverConfig = SolverConfig()) -> Field3D:
    """Build the scheme RHS for a problem and solve it (solver.py:402-405)."""
    solution, _ = solve_with_timings(problem, config)
    return solution


def solve_with_timings(problem, config: SolverConfig = SolverConfig()):
    """solve_direct plus the phase breakdown; RHS time counts as setup (solver.py:408-422)."""
    t0 = time.perf_counter()
    rhs = build_rhs(problem.scheme, problem.source, problem.profile, problem.grid)
    rhs_s = time.perf_counter() - t0
    solution, t = solve_discrete(rhs, problem.boundary, problem.scheme, problem.profile,
                                 problem.grid, config)
    return solution, PhaseTimings(setup_s=t.setup_s + rhs_s, transform_s=t.transform_s,
                                  exchange_s=t.exchange_s, tridiag_s=t.tridiag_s,
                                  total_s=t.total_s + rhs_s)
