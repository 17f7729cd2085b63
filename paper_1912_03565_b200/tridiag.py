"""Per-mode tridiagonal systems along z, solved on the device (kernel (c)).

Drop-in for the reference's helmfft.tridiag (tridiag.py:1-167). After the
2D sine transform each mode pair (n, m) obeys an n_z x n_z tridiagonal
system whose row l couples levels l-1, l, l+1 through that row's plane
eigenvalues. The batched sweep (csrc/thomas.cu) gives every mode its own
thread and generates the eigenvalues from the 12 per-row weights, so
nothing per-plane is materialised.
"""

from dataclasses import dataclass

import numpy as np

from . import _device as dv
from ._native import check, get_plan, load_library, ptr
from .errors import SingularSystemError
from .grid import CoefficientProfile, Grid3D
from .stencil import (coefficient_table, coefficients_for, eigenvalue, is_complex_table,
                      mode_cosines, pack_table, pack_table_z, pivot_threshold)

PIVOT_RTOL = 1e-14


@dataclass(frozen=True)
class SpectralSystem:
    """Bands of one mode's system, rows l = 1..n_z (tridiag.py:25-39)."""

    n: int
    m: int
    sub: np.ndarray
    diag: np.ndarray
    sup: np.ndarray


def assemble_system(n: int, m: int, scheme, profile: CoefficientProfile,
                    grid: Grid3D) -> SpectralSystem:
    """Bands of mode (n, m), 1-based (tridiag.py:42-56). O(n_z) host work."""
    n_z = grid.n_z
    bands = np.zeros((3, n_z), dtype=complex)
    for l in range(1, n_z + 1):
        row = coefficients_for(scheme, profile, grid, l)
        for k, off in enumerate((-1, 0, 1)):
            if (off == -1 and l == 1) or (off == 1 and l == n_z):
                continue
            bands[k, l - 1] = eigenvalue(row, off, n, m, grid)
    return SpectralSystem(n=n, m=m, sub=bands[0], diag=bands[1], sup=bands[2])


def solve_system(system: SpectralSystem, rhs) -> np.ndarray:
    """Thomas elimination for one explicit system, on the device (tridiag.py:59-90)."""
    torch = dv._torch()
    n_z = len(system.diag)
    rhs = np.asarray(rhs, dtype=complex)
    if rhs.shape != (n_z,):
        raise ValueError(f"rhs length {rhs.shape} != system size {n_z}")
    bands = [np.asarray(b, dtype=complex) for b in (system.sub, system.diag, system.sup)]
    scale = max(float(np.abs(b).max()) for b in bands)
    if scale == 0.0:
        raise SingularSystemError("all-zero system", n=system.n, m=system.m)
    cplx = any(np.any(b.imag) for b in bands) or bool(np.any(rhs.imag))
    dev = torch.device("cuda", torch.cuda.current_device())

    def put(a):
        a = np.ascontiguousarray(a if cplx else a.real)
        if cplx:
            a = a.view(np.float64)
        return dv.upload(a, dev)

    sub, diag, sup, x = (put(a) for a in (*bands, rhs))
    cpw = torch.empty_like(x)
    thr = torch.tensor([PIVOT_RTOL * scale], dtype=torch.float64, device=dev)
    err = torch.full((1,), -1, dtype=torch.int64, device=dev)
    lib = load_library()
    stream = dv._torch().cuda.current_stream(dev).cuda_stream
    check(lib.hfb_solve_bands(ptr(sub), ptr(diag), ptr(sup), ptr(x), ptr(cpw), n_z, 1,
                              int(cplx), ptr(thr), ptr(err), stream), "solve_bands")
    bad = int(err.cpu().item())
    if bad != -1:
        row = bad % n_z
        raise SingularSystemError(f"vanishing pivot at row {row + 1}", n=system.n, m=system.m)
    out = dv.download(x)
    return out.view(np.complex128).copy() if cplx else out.astype(complex)


def device_coefficients(plan, scheme, profile, grid):
    """Upload the row table + cosines of (scheme, profile, grid) to a DevicePlan
    (a complex table — complex k(z) — as real and imaginary parts)."""
    table = coefficient_table(scheme, profile, grid)
    cx, cy = mode_cosines(grid)
    thr = pivot_threshold(table, PIVOT_RTOL)
    if is_complex_table(table):
        re, im = pack_table_z(table)
        key = (re.tobytes(), im.tobytes(), grid.n_x, grid.n_y, thr)
        plan.set_coefficients_z(re, im, cx, cy, thr, key=key)
    else:
        packed = pack_table(table)
        key = (packed.tobytes(), grid.n_x, grid.n_y, thr)
        plan.set_coefficients(packed, cx, cy, thr, key=key)
    return table


def _slab_device(t, scheme, profile, grid, m_start):
    n_z, m_count, n_x = t.shape
    plan = get_plan(grid.n_x, grid.n_y, grid.n_z, t.device)
    with plan.lock:
        device_coefficients(plan, scheme, profile, grid)
        if plan.complex_coef:
            raise NotImplementedError("complex k(z) needs complex values: pass a complex "
                                      "numpy slab")
        torch = dv._torch()
        work = torch.empty((n_z, m_count, n_x), dtype=torch.float64, device=t.device)
        check(plan.lib.hfb_solve_slab(plan.handle, ptr(t), m_count, m_start, ptr(work),
                                      plan.stream()), "solve_slab")
        plan.fetch_status()


def _slab_device_z(tr, ti, scheme, profile, grid, m_start):
    n_z, m_count, n_x = tr.shape
    plan = get_plan(grid.n_x, grid.n_y, grid.n_z, tr.device)
    with plan.lock:
        device_coefficients(plan, scheme, profile, grid)
        torch = dv._torch()
        work = torch.empty((2, n_z, m_count, n_x), dtype=torch.float64, device=tr.device)
        check(plan.lib.hfb_solve_slab_z(plan.handle, ptr(tr), ptr(ti), m_count, m_start,
                                        ptr(work), plan.stream()), "solve_slab_z")
        plan.fetch_status()


def solve_slab(values, scheme, profile: CoefficientProfile, grid: Grid3D,
               m_start: int = 0) -> None:
    """Sweep a (n_z, M, n_x) slab in place; local row j is mode m_start + j (tridiag.py:112-123)."""
    if values.shape[1] == 0:
        return
    if tuple(values.shape) != (grid.n_z, values.shape[1], grid.n_x):
        raise ValueError(f"slab shape {tuple(values.shape)} does not match the grid")
    complex_table = is_complex_table(coefficient_table(scheme, profile, grid))
    if dv.is_tensor(values):
        parts = dv.device_parts(values)
        if complex_table:
            if len(parts) < 2:
                raise TypeError("complex k(z) needs a complex slab")
            _slab_device_z(parts[0], parts[1], scheme, profile, grid, m_start)
        else:
            for t in parts:
                _slab_device(t, scheme, profile, grid, m_start)
        dv.store_device(values, parts)
        return
    torch = dv._torch()
    dev = torch.device("cuda", torch.cuda.current_device())
    if complex_table:
        if not np.iscomplexobj(values):
            raise TypeError("complex k(z) needs a complex slab")
        tr = dv.upload(np.ascontiguousarray(values.real), dev)
        ti = dv.upload(np.ascontiguousarray(values.imag), dev)
        _slab_device_z(tr, ti, scheme, profile, grid, m_start)
        values.real[...] = dv.download(tr)
        values.imag[...] = dv.download(ti)
        return
    parts = []
    for part in dv.real_parts(values):
        t = dv.upload(part, dev)
        _slab_device(t, scheme, profile, grid, m_start)
        parts.append(dv.download(t))
    dv.write_back(values, parts)


def solve_all(transformed_rhs, scheme, profile: CoefficientProfile, grid: Grid3D,
              pencil_range=None) -> None:
    """Solve the systems of an m-range [start, stop) in place (tridiag.py:93-109)."""
    values = dv.unwrap(transformed_rhs)
    n_z, n_y, n_x = values.shape
    start, stop = (0, n_y) if pencil_range is None else pencil_range
    if not 0 <= start <= stop <= n_y:
        raise IndexError(f"pencil range ({start}, {stop}) outside 0..{n_y}")
    if start == stop:
        return
    if dv.is_tensor(values):
        dv.device_parts(values[:1, :1, :1])  # CUDA float64 / complex128 check
        sub = values[:, start:stop, :].contiguous()
        solve_slab(sub, scheme, profile, grid, m_start=start)
        values[:, start:stop, :] = sub
        return
    sub = np.ascontiguousarray(values[:, start:stop, :])
    solve_slab(sub, scheme, profile, grid, m_start=start)
    values[:, start:stop, :] = sub
