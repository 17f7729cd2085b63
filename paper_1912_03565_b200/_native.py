"""ctypes binding of the sm_100a C-ABI (include/helmfft_b200.h).

This is the only place the package touches the native library. PyTorch owns
every device buffer (``torch.empty(..., device="cuda")``); the library
borrows raw pointers and enqueues on the caller's current torch stream.
There is no CPU fallback: a missing library or device raises
NativeUnavailableError.
"""

import ctypes
import os
import threading

import numpy as np

from .errors import (ExchangeError, InvalidPartitionError, NativeUnavailableError,
                     SingularSystemError)

LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "_lib",
                        "libhelmfft_b200.so")

HFB_OK = 0
HFB_ERR_ARGUMENT = 1
HFB_ERR_RANGE = 2
HFB_ERR_SINGULAR = 3
HFB_ERR_PARTITION = 4
HFB_ERR_EXCHANGE = 5
HFB_ERR_CUDA = 6
HFB_ERR_NO_COEFFICIENTS = 7

OP_SOLVE, OP_TRANSFORM, OP_SLAB = 0, 1, 2


class HfbStatus(ctypes.Structure):
    _fields_ = [("code", ctypes.c_int), ("l", ctypes.c_int64), ("m", ctypes.c_int64),
                ("n", ctypes.c_int64), ("sender", ctypes.c_int), ("receiver", ctypes.c_int),
                ("msg", ctypes.c_char * 256)]


_vp, _i, _d, _u32 = ctypes.c_void_p, ctypes.c_int, ctypes.c_double, ctypes.c_uint32
_ip = ctypes.POINTER(ctypes.c_int)

# name -> (restype, argtypes); the exported surface of include/helmfft_b200.h
SIGNATURES = {
    "hfb_version": (ctypes.c_char_p, []),
    "hfb_strerror": (ctypes.c_char_p, [_i]),
    "hfb_launch_count": (ctypes.c_uint64, []),
    "hfb_set_tuning": (None, [_i, _i]),
    "hfb_plan_set_workspace_mode": (_i, [_vp, _i]),
    "hfb_plan_trim": (_i, [_vp]),
    "hfb_stage_timing": (_i, [_vp, _i]),
    "hfb_modes_ld": (_i, [_vp]),
    "hfb_rhs_sixth_z": (_i, [_vp, _vp, _vp, _vp, _vp, _vp, _vp, ctypes.c_double, _vp, _vp,
                             _vp]),
    "hfb_rhs_convdiff_z": (_i, [_vp, _vp, _vp] + [ctypes.c_double] * 5 + [_vp, _vp, _vp]),
    "hfb_forward_modes": (_i, [_vp, _vp, _vp, _vp, _vp]),
    "hfb_inverse_modes": (_i, [_vp, _vp, _vp, _vp]),
    "hfb_solve_modes": (_i, [_vp, _vp, _i, _i, _i, _vp, _vp]),
    "hfb_solve_modes_perm": (_i, [_vp, _vp, _i, _i, _i, _ip, _vp, _vp]),
    "hfb_pack_modes": (_i, [_vp, _vp, _vp, _ip, _i, _vp]),
    "hfb_unpack_modes": (_i, [_vp, _vp, _vp, _ip, _i, _vp]),
    "hfb_forward_blocks": (_i, [_vp, _vp, _vp, _vp, _ip, _i, _vp]),
    "hfb_inverse_blocks": (_i, [_vp, _vp, _vp, _vp, _ip, _i, _vp]),
    "hfb_solve_host_async": (_i, [_vp, _vp, _vp, _vp, _vp]),
    "hfb_host_sync": (_i, [_vp, _vp]),
    "hfb_plan_set_coefficients_z": (_i, [_vp, _vp, _vp, _vp, _vp, ctypes.c_double]),
    "hfb_solve_z": (_i, [_vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    "hfb_solve_slab_z": (_i, [_vp, _vp, _vp, _i, _i, _vp, _vp]),
    "hfb_apply27_z": (_i, [_vp, _vp, _vp, _vp, _vp, _vp, _vp, ctypes.c_uint32, _i, _vp]),
    "hfb_residual_sq_z": (_i, [_vp, _vp, _vp, _vp, _vp, _vp, ctypes.c_uint32, _vp]),
    "hfb_stage_times": (_i, [_vp, _vp, _vp]),
    "hfb_plan_create": (_i, [_i, _i, _i, _i, ctypes.POINTER(_vp)]),
    "hfb_plan_destroy": (_i, [_vp]),
    "hfb_plan_set_coefficients": (_i, [_vp, _vp, _vp, _vp, _d]),
    "hfb_workspace_bytes": (ctypes.c_size_t, [_vp, _i]),
    "hfb_transform_stack": (_i, [_vp, _vp, _i, _i, _vp, _vp]),
    "hfb_transform_lines_x": (_i, [_vp, _vp, _i, _i, _vp, _vp]),
    "hfb_transform_lines_y": (_i, [_vp, _vp, _i, _i, _vp, _vp]),
    "hfb_solve_slab": (_i, [_vp, _vp, _i, _i, _vp, _vp]),
    "hfb_solve_bands": (_i, [_vp, _vp, _vp, _vp, _vp, _i, _i, _i, _vp, _vp, _vp]),
    "hfb_solve": (_i, [_vp, _vp, _vp, _vp, _vp]),
    "hfb_solve_host": (_i, [_vp, _vp, _vp, _vp, _vp, ctypes.POINTER(HfbStatus)]),
    "hfb_status_fetch": (_i, [_vp, _vp, ctypes.POINTER(HfbStatus)]),
    "hfb_rhs_fourth": (_i, [_vp, _vp, _vp, _d, _vp]),
    "hfb_rhs_second": (_i, [_vp, _vp, _vp, _d, _vp]),
    "hfb_rhs_sixth": (_i, [_vp] + [_vp] * 9 + [_d, _vp, _vp]),
    "hfb_rhs_convdiff": (_i, [_vp] + [_vp] * 5 + [_d, _d, _d, _d, _vp, _vp]),
    "hfb_apply27": (_i, [_vp, _vp, _vp, _vp, _u32, _i, _vp]),
    "hfb_residual_partials": (_i, [_vp]),
    "hfb_residual_sq": (_i, [_vp, _vp, _vp, _vp, _u32, _vp]),
    "hfb_pack_yblocks": (_i, [_vp, _vp, _vp, _i, _ip, _i, _vp]),
    "hfb_carry_layout": (_i, [_vp, _i, ctypes.POINTER(ctypes.c_longlong), _ip]),
    "hfb_zsolve_carry": (_i, [_vp, _i, _vp, _i, _i, _i, _vp, _vp, _vp, _u32, _vp]),
    "hfb_carry_check": (_i, [_vp, _vp, _ip]),
    "hfb_zsolve_carry_vranks": (_i, [_vp, _i, _i, _vp, _i, _ip, _ip, _vp, _vp, _u32, _vp]),
    "hfb_carry_layout_z": (_i, [_vp, _i, ctypes.POINTER(ctypes.c_longlong), _ip]),
    "hfb_zsolve_carry_z": (_i, [_vp, _i, _vp, _vp, _i, _i, _i, _vp, _vp, _vp, _u32, _vp]),
    "hfb_ipc_handle": (_i, [_vp, _vp, ctypes.POINTER(ctypes.c_longlong)]),
    "hfb_ipc_open": (_i, [_vp, ctypes.c_longlong, ctypes.POINTER(_vp)]),
    "hfb_ipc_close": (_i, [_vp, ctypes.c_longlong]),
    "hfb_unpack_yblocks": (_i, [_vp, _vp, _vp, _i, _ip, _i, _vp]),
}

_lib = None
_lock = threading.Lock()


def load_library(path=None):
    """Load (once) and type the C-ABI library; raises NativeUnavailableError.
    HFB_LIBRARY overrides the in-tree path (A/B builds of the same ABI)."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        path = path or os.environ.get("HFB_LIBRARY") or LIB_PATH
        if not os.path.exists(path):
            raise NativeUnavailableError(
                f"{path} is missing: build it with `make` (or __graft_entry__.build())")
        try:
            lib = ctypes.CDLL(path)
        except OSError as exc:
            raise NativeUnavailableError(f"cannot load {path}: {exc}") from exc
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
        return lib


def exported_symbols(path=LIB_PATH):
    """Names of SIGNATURES that the built library actually exports (no CUDA call)."""
    lib = ctypes.CDLL(path)
    return [n for n in SIGNATURES if hasattr(lib, n)]


def _torch():
    import torch
    if not torch.cuda.is_available():
        raise NativeUnavailableError("no CUDA device visible; the solver has no CPU path")
    return torch


def check(code, what=""):
    """Map an hfb_code to the reference exception classes."""
    if code == HFB_OK:
        return
    lib = load_library()
    text = lib.hfb_strerror(code).decode()
    msg = f"{what}: {text}" if what else text
    if code == HFB_ERR_ARGUMENT:
        raise ValueError(msg)
    if code == HFB_ERR_RANGE:
        raise IndexError(msg)
    if code == HFB_ERR_PARTITION:
        raise InvalidPartitionError(msg)
    if code == HFB_ERR_EXCHANGE:
        raise ExchangeError(msg)
    if code == HFB_ERR_SINGULAR:
        raise SingularSystemError(msg)
    raise RuntimeError(msg)


def ptr(t):
    return ctypes.c_void_p(t.data_ptr()) if t is not None else ctypes.c_void_p(0)


def current_stream(device):
    torch = _torch()
    return ctypes.c_void_p(torch.cuda.current_stream(device).cuda_stream)


class DevicePlan:
    """Owns one hfb_plan (extents + transform tables + coefficient table)."""

    def __init__(self, n_x, n_y, n_z, device):
        torch = _torch()
        self.lib = load_library()
        self.device = torch.device(device)
        index = self.device.index if self.device.index is not None else torch.cuda.current_device()
        self.device = torch.device("cuda", index)
        self.extents = (n_x, n_y, n_z)
        handle = ctypes.c_void_p()
        with torch.cuda.device(index):
            check(self.lib.hfb_plan_create(n_x, n_y, n_z, index, ctypes.byref(handle)),
                  "plan_create")
        self.handle = handle
        self._coef_key = None
        self.lean = False  # one-call solve workspace layout (hfb_plan_set_workspace_mode)
        self.complex_coef = False  # the uploaded table is complex (complex k(z))
        self.lock = threading.RLock()

    def __del__(self):
        lib, h = getattr(self, "lib", None), getattr(self, "handle", None)
        if lib is not None and h:
            try:
                lib.hfb_plan_destroy(h)
            except Exception:
                pass

    def set_coefficients(self, packed, cx, cy, threshold, key=None):
        """Upload a packed table (see stencil.pack_table) unless `key` matches the last one."""
        if key is not None and key == self._coef_key:
            return
        packed = np.ascontiguousarray(packed, dtype=np.float64)
        cx = np.ascontiguousarray(cx, dtype=np.float64)
        cy = np.ascontiguousarray(cy, dtype=np.float64)
        check(self.lib.hfb_plan_set_coefficients(
            self.handle, packed.ctypes.data_as(_vp), cx.ctypes.data_as(_vp),
            cy.ctypes.data_as(_vp), float(threshold)), "set_coefficients")
        self._coef_key = key
        self.complex_coef = False

    def set_coefficients_z(self, packed_re, packed_im, cx, cy, threshold, key=None):
        """Complex table (complex k(z)): real and imaginary parts, pack_table layout."""
        if key is not None and key == self._coef_key:
            return
        re = np.ascontiguousarray(packed_re, dtype=np.float64)
        im = np.ascontiguousarray(packed_im, dtype=np.float64)
        cx = np.ascontiguousarray(cx, dtype=np.float64)
        cy = np.ascontiguousarray(cy, dtype=np.float64)
        check(self.lib.hfb_plan_set_coefficients_z(
            self.handle, re.ctypes.data_as(_vp), im.ctypes.data_as(_vp), cx.ctypes.data_as(_vp),
            cy.ctypes.data_as(_vp), float(threshold)), "set_coefficients_z")
        self._coef_key = key
        self.complex_coef = True

    def workspace(self, op):
        """Device workspace for op (see hfb_workspace_bytes). For the one-call
        solve (op 0) the fast two-volume layout is tried first; when it does
        not fit, the plan switches to the lean one-volume layout."""
        torch = _torch()
        nbytes = int(self.lib.hfb_workspace_bytes(self.handle, op))
        if nbytes == 0:
            return None
        try:
            return torch.empty(nbytes, dtype=torch.uint8, device=self.device)
        except torch.OutOfMemoryError:
            trim_plans()  # the other cached plans' own device memory (checkpoint caches)
            torch.cuda.empty_cache()
            try:
                return torch.empty(nbytes, dtype=torch.uint8, device=self.device)
            except torch.OutOfMemoryError:
                if op not in (0, 3):
                    raise
        torch.cuda.empty_cache()
        self.set_workspace_mode(True)
        nbytes = int(self.lib.hfb_workspace_bytes(self.handle, op))
        return torch.empty(nbytes, dtype=torch.uint8, device=self.device)

    def set_workspace_mode(self, lean):
        check(self.lib.hfb_plan_set_workspace_mode(self.handle, int(lean)), "set_workspace_mode")
        self.lean = bool(lean)

    def stream(self):
        return current_stream(self.device)

    def fetch_status(self):
        """Synchronise and raise SingularSystemError for a latched pivot failure."""
        st = HfbStatus()
        code = self.lib.hfb_status_fetch(self.handle, self.stream(), ctypes.byref(st))
        if code == HFB_ERR_SINGULAR:
            raise SingularSystemError(st.msg.decode(), n=int(st.n), m=int(st.m))
        check(code, "status")


_plans = {}
_plans_lock = threading.Lock()


def trim_plans():
    """hfb_plan_trim on every cached plan: frees the memory the plans allocated
    themselves (the z-solve's cached checkpoints); the next solve rebuilds it."""
    with _plans_lock:
        plans = list(_plans.values())
    for plan in plans:
        plan.lib.hfb_plan_trim(plan.handle)


def get_plan(n_x, n_y, n_z, device=None) -> DevicePlan:
    """Cached plan per (extents, device)."""
    torch = _torch()
    dev = torch.device("cuda", torch.cuda.current_device()) if device is None \
        else torch.device(device)
    if dev.index is None:
        dev = torch.device("cuda", torch.cuda.current_device())
    key = (n_x, n_y, n_z, dev.index)
    with _plans_lock:
        plan = _plans.get(key)
        if plan is None:
            plan = DevicePlan(n_x, n_y, n_z, dev)
            _plans[key] = plan
        return plan
