"""Fields, right-hand sides, Dirichlet folding and the 27-point operator.

Drop-in for the reference's helmfft.assembly (assembly.py:1-289). Analytic
callables are sampled on the host (they are Python functions, exactly as in
the reference); every arithmetic operator on N^3 data runs on the device:

- ``build_rhs``: the fourth-order 7-point RHS operator (kernel (a)) and the
  pointwise 2nd/6th/cd4 combinations;
- ``fold_dirichlet`` / ``apply_stencil`` / ``residual_l2``: the 27-point
  operator with the reference's term order and zero-weight skipping.

Fields hold numpy arrays (the reference's type; real float64 is kept real,
complex stays complex) or torch CUDA float64 tensors (device-resident
pipelines; results stay on the device).
"""

import ctypes
from dataclasses import dataclass
from typing import Callable, Optional

import numpy as np

from . import _device as dv
from ._native import check, get_plan, ptr
from .errors import UnsupportedSchemeError
from .grid import CoefficientProfile, Grid3D
from .stencil import scheme_key, term_mask


class Field3D:
    """Scalar field on the interior nodes, shape (n_z, n_y, n_x), x fastest.

    Row index of node (i, j, l) (1-based) is (i-1) + n_x (j-1) + n_x n_y (l-1)
    (assembly.py:28-58).
    """

    def __init__(self, values):
        if dv.is_tensor(values):
            if values.dim() != 3:
                raise ValueError(f"Field3D needs a 3D array, got ndim={values.dim()}")
            self.values = values
            return
        arr = np.asarray(values)
        if not (np.iscomplexobj(arr) or arr.dtype == np.float64):
            arr = arr.astype(np.float64)
        if arr.ndim != 3:
            raise ValueError(f"Field3D needs a 3D array, got ndim={arr.ndim}")
        self.values = arr

    def __repr__(self):
        return f"Field3D(shape={tuple(self.values.shape)}, dtype={self.values.dtype})"

    @classmethod
    def zeros(cls, grid: Grid3D) -> "Field3D":
        return cls(np.zeros(grid.shape, dtype=np.float64))

    @property
    def extents(self):
        n_z, n_y, n_x = self.values.shape
        return (n_x, n_y, n_z)

    @property
    def on_device(self):
        return dv.is_tensor(self.values)

    def copy(self) -> "Field3D":
        return Field3D(self.values.clone() if self.on_device else self.values.copy())

    def ravel(self):
        return self.values.reshape(-1)

    def numpy(self):
        return dv.download(self.values) if self.on_device else self.values


class BoundaryData:
    """Dirichlet values on the closed-box boundary lattice (assembly.py:61-112)."""

    def __init__(self, fn: Optional[Callable] = None, array=None, known_zero: bool = False):
        if (fn is None) == (array is None):
            raise ValueError("provide exactly one of fn or array")
        self._fn = fn
        self._array = None if array is None else np.asarray(array)
        self.known_zero = known_zero

    @classmethod
    def zero(cls) -> "BoundaryData":
        def nothing(x, y, z):
            return np.zeros(np.broadcast(x, y, z).shape)
        return cls(fn=nothing, known_zero=True)

    @classmethod
    def from_function(cls, fn) -> "BoundaryData":
        return cls(fn=fn)

    @classmethod
    def from_array(cls, array) -> "BoundaryData":
        return cls(array=array)

    def closed_box(self, grid: Grid3D) -> np.ndarray:
        """(n_z+2, n_y+2, n_x+2) with boundary values set and a zero interior."""
        shape = (grid.n_z + 2, grid.n_y + 2, grid.n_x + 2)
        if self._array is not None:
            if self._array.shape != shape:
                raise ValueError(f"boundary array shape {self._array.shape} != closed box {shape}")
            box = np.array(self._array, dtype=complex)
            box[1:-1, 1:-1, 1:-1] = 0.0
            return box
        box = np.zeros(shape, dtype=complex)
        xs, ys, zs = (grid.x_nodes(closed=True), grid.y_nodes(closed=True),
                      grid.z_nodes(closed=True))
        # faces in the reference's order; shared edges/corners get equal values
        for zi in (0, -1):
            box[zi, :, :] = self._fn(xs[None, :], ys[:, None], zs[zi])
        for yi in (0, -1):
            box[:, yi, :] = self._fn(xs[None, :], ys[yi], zs[:, None])
        for xi in (0, -1):
            box[:, :, xi] = self._fn(xs[xi], ys[None, :], zs[:, None])
        return box


@dataclass
class SourceSpec:
    """Source f and the analytic derivatives the RHS of each scheme needs (assembly.py:115-146)."""

    f: Callable
    f_z: Optional[Callable] = None
    f_xx: Optional[Callable] = None
    f_yy: Optional[Callable] = None
    f_zz: Optional[Callable] = None
    lap_f: Optional[Callable] = None
    d4_f: Optional[Callable] = None
    f_xxyy: Optional[Callable] = None
    f_xxzz: Optional[Callable] = None
    f_yyzz: Optional[Callable] = None

    @classmethod
    def zero(cls) -> "SourceSpec":
        def nothing(x, y, z):
            return np.zeros(np.broadcast(x, y, z).shape)
        return cls(*([nothing] * 10))

    def require(self, names):
        missing = [n for n in names if getattr(self, n) is None]
        if missing:
            raise ValueError(f"source is missing required derivatives: {missing}")


def _sample(fn, grid, closed=False):
    x = grid.x_nodes(closed=closed)[None, None, :]
    y = grid.y_nodes(closed=closed)[None, :, None]
    z = grid.z_nodes(closed=closed)[:, None, None]
    shape = tuple(s + (2 if closed else 0) for s in grid.shape)
    return np.broadcast_to(np.asarray(fn(x, y, z)), shape)


def _device_of(device):
    torch = dv._torch()
    if device is None:
        return torch.device("cuda", torch.cuda.current_device())
    return torch.device(device)


def _split_all(arrays):
    """Real parts of several sampled fields, aligned: list over parts of lists over fields."""
    cplx = any(np.iscomplexobj(a) and np.any(np.imag(a)) for a in arrays)
    re = [np.ascontiguousarray(np.real(a), dtype=np.float64) for a in arrays]
    if not cplx:
        return [re]
    return [re, [np.ascontiguousarray(np.imag(a), dtype=np.float64) for a in arrays]]


def _real_profile(arr, what):
    arr = np.asarray(arr)
    if np.iscomplexobj(arr) and np.any(arr.imag):
        raise NotImplementedError(f"complex {what} is not supported by the fp64-real kernels yet")
    return np.ascontiguousarray(np.real(arr), dtype=np.float64)


def build_rhs(scheme, source: SourceSpec, profile: CoefficientProfile, grid: Grid3D,
              device=None, keep_on_device=False) -> Field3D:
    """Scheme right-hand side F on the interior nodes (assembly.py:162-226).

    Sampling is host work; the operator/combination runs on the device.
    Returns a host Field3D unless keep_on_device.
    """
    torch = dv._torch()
    dev = _device_of(device)
    key = scheme_key(scheme)
    plan = get_plan(grid.n_x, grid.n_y, grid.n_z, dev)
    hz2 = grid.h_z**2
    if key == "4":
        fields = [_sample(source.f, grid, closed=True)]
    elif key == "2":
        fields = [_sample(source.f, grid)]
    elif key == "6":
        if not grid.uniform:
            raise UnsupportedSchemeError("sixth-order RHS needs a uniform grid step")
        source.require(["f_z", "lap_f", "d4_f", "f_xxyy", "f_xxzz", "f_yyzz"])
        names = ["f", "lap_f", "d4_f", "f_xxyy", "f_xxzz", "f_yyzz", "f_z"]
        fields = [_sample(getattr(source, n), grid) for n in names]
    elif key == "cd4":
        source.require(["f_z", "f_xx", "f_yy", "f_zz"])
        names = ["f", "f_xx", "f_yy", "f_z", "f_zz"]
        fields = [_sample(getattr(source, n), grid) for n in names]
    else:
        raise ValueError(f"build_rhs has no formula for scheme {scheme!r}")
    def _imag(a):
        a = np.asarray(a)
        return np.iscomplexobj(a) and bool(np.any(a.imag))

    zk = key == "6" and (_imag(profile.k2) or _imag(profile.k2_z))
    zg = key == "cd4" and complex(profile.gamma).imag != 0
    if zk or zg:
        # complex coefficients: one complex combination (both parts at once)
        with plan.lock:
            st = plan.stream()
            up = lambda a: dv.upload(np.ascontiguousarray(a, dtype=np.float64), dev)
            re = [up(np.real(a)) for a in fields]
            im = [up(np.imag(a)) if np.iscomplexobj(a) else torch.zeros_like(re[0])
                  for a in fields]
            pr = (ctypes.c_void_p * 7)(*[t.data_ptr() for t in re])
            pi = (ctypes.c_void_p * 7)(*[t.data_ptr() for t in im])
            outr = torch.empty(grid.shape, dtype=torch.float64, device=dev)
            outi = torch.empty_like(outr)
            if zk:
                k = [np.asarray(profile.k2, complex)[1:-1], np.asarray(profile.k2_z, complex)[1:-1]]
                kt = [up(k[0].real), up(k[0].imag), up(k[1].real), up(k[1].imag)]
                check(plan.lib.hfb_rhs_sixth_z(plan.handle, pr, pi, *[ptr(t) for t in kt], hz2,
                                               ptr(outr), ptr(outi), st), "rhs_sixth_z")
            else:
                g = complex(profile.gamma)
                check(plan.lib.hfb_rhs_convdiff_z(plan.handle, pr, pi, grid.h_x**2, grid.h_y**2,
                                                  hz2, g.real, g.imag, ptr(outr), ptr(outi), st),
                      "rhs_convdiff_z")
            outs = [outr, outi]
    else:
        outs = None
    if outs is not None:
        if keep_on_device:
            return Field3D(dv.join_device(outs, outs[0]))
        return Field3D(dv.download(outs[0]) + 1j * dv.download(outs[1]))
    outs = []
    with plan.lock:
        for part in _split_all(fields):
            ins = [dv.upload(a, dev) for a in part]
            out = torch.empty(grid.shape, dtype=torch.float64, device=dev)
            st = plan.stream()
            if key == "4":
                check(plan.lib.hfb_rhs_fourth(plan.handle, ptr(ins[0]), ptr(out), hz2, st),
                      "rhs_fourth")
            elif key == "2":
                check(plan.lib.hfb_rhs_second(plan.handle, ptr(ins[0]), ptr(out), hz2, st),
                      "rhs_second")
            elif key == "6":
                k2 = dv.upload(_real_profile(np.asarray(profile.k2)[1:-1], "k^2"), dev)
                k2z = dv.upload(_real_profile(np.asarray(profile.k2_z)[1:-1], "(k^2)_z"), dev)
                check(plan.lib.hfb_rhs_sixth(plan.handle, *[ptr(t) for t in ins], ptr(k2),
                                             ptr(k2z), hz2, ptr(out), st), "rhs_sixth")
            else:
                gamma = complex(profile.gamma)
                check(plan.lib.hfb_rhs_convdiff(plan.handle, *[ptr(t) for t in ins],
                                                grid.h_x**2, grid.h_y**2, hz2, gamma.real,
                                                ptr(out), st), "rhs_convdiff")
            outs.append(out)
    if keep_on_device:
        return Field3D(dv.join_device(outs, outs[0]))
    parts = [dv.download(o) for o in outs]
    return Field3D(parts[0] if len(parts) == 1 else parts[0] + 1j * parts[1])


def _with_coefficients(plan, scheme, profile, grid):
    from .tridiag import device_coefficients
    return device_coefficients(plan, scheme, profile, grid)


def _apply_parts(ext_parts, rhs_parts, scheme, profile, grid, mode, device):
    """mode 0: A ext; mode 1: rhs - A ext; per real part (real table) or on the
    (re, im) pair (complex table, complex k(z)); returns device tensors."""
    torch = dv._torch()
    plan = get_plan(grid.n_x, grid.n_y, grid.n_z, device)
    outs = []
    zeros = lambda like_shape: torch.zeros(like_shape, dtype=torch.float64, device=device)
    with plan.lock:
        table = _with_coefficients(plan, scheme, profile, grid)
        mask = term_mask(table)
        if plan.complex_coef:
            ext = list(ext_parts) + [torch.zeros_like(ext_parts[0])] * (2 - len(ext_parts))
            rhs = [None, None]
            if mode == 1:
                rhs = list(rhs_parts) + [zeros(grid.shape)] * (2 - len(rhs_parts))
            outs = [torch.empty(grid.shape, dtype=torch.float64, device=device) for _ in range(2)]
            check(plan.lib.hfb_apply27_z(plan.handle, ptr(ext[0]), ptr(ext[1]), ptr(rhs[0]),
                                         ptr(rhs[1]), ptr(outs[0]), ptr(outs[1]), mask, mode,
                                         plan.stream()), "apply27_z")
            return outs
        for k in range(max(len(ext_parts), len(rhs_parts) if rhs_parts else 0)):
            ext = ext_parts[k] if k < len(ext_parts) else torch.zeros_like(ext_parts[0])
            rhs = None
            if mode == 1:
                rhs = rhs_parts[k] if k < len(rhs_parts) else zeros(grid.shape)
            out = torch.empty(grid.shape, dtype=torch.float64, device=device)
            check(plan.lib.hfb_apply27(plan.handle, ptr(ext), ptr(rhs), ptr(out), mask, mode,
                                       plan.stream()), "apply27")
            outs.append(out)
    return outs


def _parts_of(values, device):
    if dv.is_tensor(values):
        return dv.device_parts(values)
    return dv.upload_parts(values, device)


def _result(outs, like):
    if dv.is_tensor(like):
        return Field3D(dv.join_device(outs, like))
    return Field3D(dv.download_parts(outs, like))


def apply_stencil(u: Field3D, boundary: BoundaryData, scheme, profile: CoefficientProfile,
                  grid: Grid3D) -> Field3D:
    """Matrix-free A u including boundary contributions (assembly.py:247-255)."""
    values = dv.unwrap(u)
    if tuple(values.shape) != grid.shape:
        raise ValueError(f"field shape {tuple(values.shape)} != grid {grid.shape}")
    device = values.device if dv.is_tensor(values) else _device_of(None)
    box = boundary.closed_box(grid)
    interior = dv.download(values) if dv.is_tensor(values) else values
    box[1:-1, 1:-1, 1:-1] = interior
    outs = _apply_parts(_parts_of(box, device), None, scheme, profile, grid, 0, device)
    return _result(outs, values)


def fold_dirichlet(rhs: Field3D, boundary: BoundaryData, scheme, profile: CoefficientProfile,
                   grid: Grid3D) -> Field3D:
    """Move the boundary values to the right-hand side; returns a copy (assembly.py:258-274)."""
    values = dv.unwrap(rhs)
    if tuple(values.shape) != grid.shape:
        raise ValueError(f"rhs shape {tuple(values.shape)} != grid {grid.shape}")
    if boundary.known_zero:
        return Field3D(values.clone() if dv.is_tensor(values) else values.copy())
    box = boundary.closed_box(grid)
    if not np.any(box):
        return Field3D(values.clone() if dv.is_tensor(values) else values.copy())
    device = values.device if dv.is_tensor(values) else _device_of(None)
    ext_parts = _parts_of(box, device)
    rhs_parts = _parts_of(values, device)
    outs = _apply_parts(ext_parts, rhs_parts, scheme, profile, grid, 1, device)
    return _result(outs, values)


def fold_device_parts(rhs_parts, boundary: BoundaryData, scheme, profile: CoefficientProfile,
                      grid: Grid3D, device):
    """fold_dirichlet on right-hand sides already on the device ([re] or [re, im]
    float64 tensors; the result may gain an imaginary part from complex boundary
    data). A zero boundary returns the parts themselves."""
    if boundary.known_zero:
        return list(rhs_parts)
    box = boundary.closed_box(grid)
    if not np.any(box):
        return list(rhs_parts)
    return _apply_parts(_parts_of(box, device), list(rhs_parts), scheme, profile, grid, 1,
                        device)


def residual_l2(u: Field3D, rhs_folded: Field3D, scheme, profile: CoefficientProfile,
                grid: Grid3D) -> float:
    """||A u - F||_2 with homogeneous boundary values (assembly.py:277-289)."""
    torch = dv._torch()
    uv, fv = dv.unwrap(u), dv.unwrap(rhs_folded)
    if tuple(uv.shape) != tuple(fv.shape):
        raise ValueError(f"extent mismatch: {tuple(uv.shape)} vs {tuple(fv.shape)}")
    device = uv.device if dv.is_tensor(uv) else _device_of(None)
    u_parts, f_parts = _parts_of(uv, device), _parts_of(fv, device)
    plan = get_plan(grid.n_x, grid.n_y, grid.n_z, device)
    total = 0.0
    with plan.lock:
        table = _with_coefficients(plan, scheme, profile, grid)
        mask = term_mask(table)
        npart = int(plan.lib.hfb_residual_partials(plan.handle))
        if plan.complex_coef:
            u2 = list(u_parts) + [torch.zeros_like(u_parts[0])] * (2 - len(u_parts))
            f2 = list(f_parts) + [torch.zeros_like(f_parts[0])] * (2 - len(f_parts))
            partial = torch.empty(npart, dtype=torch.float64, device=device)
            check(plan.lib.hfb_residual_sq_z(plan.handle, ptr(u2[0]), ptr(u2[1]), ptr(f2[0]),
                                             ptr(f2[1]), ptr(partial), mask, plan.stream()),
                  "residual_z")
            return float(np.sqrt(float(partial.sum().item())))
        for k in range(max(len(u_parts), len(f_parts))):
            uk = u_parts[k] if k < len(u_parts) else torch.zeros_like(u_parts[0])
            fk = f_parts[k] if k < len(f_parts) else torch.zeros_like(f_parts[0])
            partial = torch.empty(npart, dtype=torch.float64, device=device)
            check(plan.lib.hfb_residual_sq(plan.handle, ptr(uk), ptr(fk), ptr(partial), mask,
                                           plan.stream()), "residual")
            total += float(partial.sum().item())
    return float(np.sqrt(total))
