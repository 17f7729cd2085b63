"""Orthonormal 2D type-I sine transform on the device (kernels (b)/(d)).

Drop-in for the reference's helmfft.spectral (spectral.py:20-111): the 1D
kernel S[n, i] = sqrt(2/(N+1)) sin(pi n i/(N+1)) is symmetric and
orthogonal, so forward and inverse are the same map. The 2D transform is
the x-pass then the y-pass, as in the reference.

Every transform runs in the sm_100a library (csrc/dst.cu): an FFT-based
DST-I when N+1 is a power of two, a dense DST-I product otherwise.
``dst2d_reference`` keeps the reference's dense cross-check on the device.
"""

import threading
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from . import _device as dv
from ._native import check, get_plan, ptr

_PLAN_LOCK = threading.Lock()


@dataclass(frozen=True)
class TransformPlan:
    """Extents of (n_y, n_x) planes; immutable and shareable (spectral.py:23-43)."""

    n_x: int
    n_y: int
    _dense: dict = field(default_factory=dict, repr=False, compare=False)

    def dense_kernel(self, n: int) -> np.ndarray:
        """Dense orthonormal DST-I matrix of size n (for cross-checks)."""
        with _PLAN_LOCK:
            if n not in self._dense:
                idx = np.arange(1, n + 1)
                r = np.outer(idx, idx) % (2 * (n + 1))
                self._dense[n] = np.sqrt(2.0 / (n + 1)) * np.sin(np.pi * r / (n + 1))
            return self._dense[n]


def make_plan(n_x: int, n_y: int) -> TransformPlan:
    if n_x < 1 or n_y < 1:
        raise ValueError(f"plan extents must be >= 1, got ({n_x}, {n_y})")
    with _PLAN_LOCK:
        return TransformPlan(n_x=n_x, n_y=n_y)


def _lines_x(t, nz, ny, nx, y0=0, y1=None):
    """x-pass over rows [y0, y1) of every plane of a (nz, ny, nx) device tensor, in place."""
    plan = get_plan(nx, ny, nz, t.device)
    y1 = ny if y1 is None else y1
    with plan.lock:
        work = plan.workspace(1)
        check(plan.lib.hfb_transform_lines_x(plan.handle, ptr(t), y0, y1, ptr(work),
                                             plan.stream()), "transform_lines_x")


def _lines_y(t, nz, ny, nx, x0=0, x1=None):
    plan = get_plan(nx, ny, nz, t.device)
    x1 = nx if x1 is None else x1
    with plan.lock:
        work = plan.workspace(1)
        check(plan.lib.hfb_transform_lines_y(plan.handle, ptr(t), x0, x1, ptr(work),
                                             plan.stream()), "transform_lines_y")


def _stack(t, z0, z1):
    nz, ny, nx = t.shape
    plan = get_plan(nx, ny, nz, t.device)
    with plan.lock:
        work = plan.workspace(1)
        check(plan.lib.hfb_transform_stack(plan.handle, ptr(t), z0, z1, ptr(work),
                                           plan.stream()), "transform_stack")


def _apply_host(values, fn, device=None):
    """Run fn on device copies of each real part of a host array; return the parts."""
    torch = dv._torch()
    device = device or torch.device("cuda", torch.cuda.current_device())
    out = []
    for part in dv.real_parts(values):
        t = dv.upload(part, device)
        fn(t)
        out.append(dv.download(t))
    return out


def dst_lines(values, axis: int):
    """Orthonormal DST-I along one axis (the 1D pass); returns a new array.

    Supports the last axis (contiguous lines) and the second-to-last axis
    (strided columns), which covers every use in the reference.
    """
    if dv.is_tensor(values):
        parts = dv.device_parts(values, copy=True)
        for t in parts:
            _dst_lines_tensor(t, axis)
        return dv.join_device(parts, values)
    arr = np.asarray(values)
    parts = _apply_host(arr, lambda t: _dst_lines_tensor(t, axis))
    return dv.join_parts(parts, arr)


def _dst_lines_tensor(t, axis):
    nd = t.dim()
    ax = axis % nd
    if nd == 1:
        _lines_x(t.view(1, 1, -1), 1, 1, t.shape[0])
        return
    shape3 = (int(np.prod(t.shape[:-2])) if nd > 2 else 1, t.shape[-2], t.shape[-1])
    v = t.view(shape3)
    if ax == nd - 1:
        _lines_x(v, *shape3)
    elif ax == nd - 2:
        _lines_y(v, *shape3)
    else:
        raise NotImplementedError("device DST along the z axis is not part of the path")


def dst2d(plan: TransformPlan, plane):
    """2D orthonormal sine transform of one (n_y, n_x) plane (spectral.py:59-63)."""
    shape = tuple(plane.shape)
    if shape != (plan.n_y, plan.n_x):
        raise ValueError(f"plane shape {shape} != plan ({plan.n_y}, {plan.n_x})")
    if dv.is_tensor(plane):
        parts = dv.device_parts(plane, copy=True)
        for t in parts:
            _stack(t.view(1, plan.n_y, plan.n_x), 0, 1)
        return dv.join_device(parts, plane)
    arr = np.asarray(plane)
    parts = _apply_host(arr.reshape(1, plan.n_y, plan.n_x), lambda t: _stack(t, 0, 1))
    return dv.join_parts([p.reshape(shape) for p in parts], arr)


def dst2d_reference(plan: TransformPlan, plane):
    """Dense S_y @ plane @ S_x, the independent cross-check (spectral.py:66-72), on the device."""
    torch = dv._torch()
    shape = tuple(plane.shape)
    if shape != (plan.n_y, plan.n_x):
        raise ValueError(f"plane shape {shape} != plan ({plan.n_y}, {plan.n_x})")
    dev = plane.device if dv.is_tensor(plane) else torch.device("cuda", torch.cuda.current_device())
    sx = torch.from_numpy(plan.dense_kernel(plan.n_x)).to(dev)
    sy = torch.from_numpy(plan.dense_kernel(plan.n_y)).to(dev)
    if dv.is_tensor(plane):
        return dv.join_device([sy @ p @ sx for p in dv.device_parts(plane)], plane)
    arr = np.asarray(plane)
    parts = [dv.download(sy @ dv.upload(p, dev) @ sx) for p in dv.real_parts(arr)]
    return dv.join_parts(parts, arr)


def transform_stack(plan: TransformPlan, field3d, plane_range: Optional[tuple] = None) -> None:
    """Transform z-planes [start, stop) of a field in place (spectral.py:75-91)."""
    values = dv.unwrap(field3d)
    if tuple(values.shape[1:]) != (plan.n_y, plan.n_x):
        raise ValueError(f"plane shape {tuple(values.shape[1:])} != plan ({plan.n_y}, {plan.n_x})")
    n_z = values.shape[0]
    start, stop = (0, n_z) if plane_range is None else plane_range
    if not 0 <= start <= stop <= n_z:
        raise IndexError(f"plane range ({start}, {stop}) outside 0..{n_z}")
    if start == stop:
        return
    if dv.is_tensor(values):
        dv.apply_inplace(values, lambda t: _stack(t, start, stop))
        return
    sub = values[start:stop]
    parts = _apply_host(sub, lambda t: _stack(t, 0, stop - start))
    dv.write_back(sub, parts)


def transform_lines_x(field3d, y_range: tuple) -> None:
    """x-pass on every plane, rows [start, stop) only, in place (spectral.py:94-101)."""
    values = dv.unwrap(field3d)
    start, stop = y_range
    if start == stop:
        return
    nz, ny, nx = values.shape
    if dv.is_tensor(values):
        dv.apply_inplace(values, lambda t: _lines_x(t, nz, ny, nx, start, stop))
        return
    parts = _apply_host(values, lambda t: _lines_x(t, nz, ny, nx, start, stop))
    dv.write_back(values, parts)


def transform_lines_y(field3d, x_range: tuple) -> None:
    """y-pass on every plane, columns [start, stop) only, in place (spectral.py:104-111)."""
    values = dv.unwrap(field3d)
    start, stop = x_range
    if start == stop:
        return
    nz, ny, nx = values.shape
    if dv.is_tensor(values):
        dv.apply_inplace(values, lambda t: _lines_y(t, nz, ny, nx, start, stop))
        return
    parts = _apply_host(values, lambda t: _lines_y(t, nz, ny, nx, start, stop))
    dv.write_back(values, parts)
