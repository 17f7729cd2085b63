"""Host <-> device array plumbing for the operator modules.

Operators accept numpy arrays (the reference's type: complex128, usually
with zero imaginary part) or torch CUDA float64 tensors. Device kernels are
fp64-real; a complex array with a non-zero imaginary part is handled as two
real solves (the operators are real and linear, so real and imaginary parts
never mix when the coefficients are real).
"""

import threading
import warnings

import numpy as np

from ._native import NativeUnavailableError, _torch


def is_tensor(x):
    try:
        import torch
    except ImportError:  # pragma: no cover
        return False
    return isinstance(x, torch.Tensor)


def unwrap(field):
    """Field3D-like (anything with .values) or raw array / tensor -> raw array.
    (A torch tensor has a .values() method of its own: it is returned as is.)"""
    if is_tensor(field) or isinstance(field, np.ndarray):
        return field
    return field.values if hasattr(field, "values") else field


def real_parts(arr):
    """Split a host array into its real parts: [re] or [re, im] (float64, C order)."""
    a = np.asarray(arr)
    if np.iscomplexobj(a):
        re = np.ascontiguousarray(a.real, dtype=np.float64)
        if np.any(a.imag):
            return [re, np.ascontiguousarray(a.imag, dtype=np.float64)]
        return [re]
    return [np.ascontiguousarray(a, dtype=np.float64)]


def upload(host, device):
    """float64 host array -> contiguous float64 device tensor."""
    torch = _torch()
    arr = np.ascontiguousarray(host, dtype=np.float64)
    if not arr.flags.writeable:
        arr = arr.copy()
    t = torch.from_numpy(arr)
    return t.to(device=device, non_blocking=False)


def download(t):
    return t.detach().cpu().numpy()


def device_tensor(x, device=None):
    """Validate a torch tensor for the kernels: CUDA float64 contiguous."""
    torch = _torch()
    if x.dtype != torch.float64:
        raise TypeError(f"device fields must be float64, got {x.dtype}")
    if not x.is_cuda:
        raise NativeUnavailableError("device fields must live on a CUDA device")
    return x.contiguous()


def device_parts(x, copy=False):
    """CUDA tensor -> its real parts for the kernels: [re] for float64, [re, im]
    for complex128 (torch stores complex interleaved; the kernels take split
    planes, so the two parts are new contiguous tensors). copy=True also gives
    a float64 tensor a private copy (operators that must not touch the caller's
    field)."""
    torch = _torch()
    if not x.is_cuda:
        raise NativeUnavailableError("device fields must live on a CUDA device")
    if x.dtype == torch.complex128:
        return [x.real.contiguous(), x.imag.contiguous()]
    if x.dtype != torch.float64:
        raise TypeError(f"device fields must be float64 or complex128, got {x.dtype}")
    t = x.contiguous()
    return [t.clone() if copy and t.data_ptr() == x.data_ptr() else t]


def join_device(parts, like):
    """Inverse of device_parts: complex128 when the caller's field is complex or
    the result gained an imaginary part (complex k(z), complex boundary data)."""
    torch = _torch()
    if like.dtype == torch.complex128 or len(parts) > 1:
        im = parts[1] if len(parts) > 1 else torch.zeros_like(parts[0])
        return torch.complex(parts[0], im)
    return parts[0]


def store_device(dst, parts):
    """Write real parts back into the caller's CUDA tensor (in-place operators)."""
    torch = _torch()
    if dst.dtype == torch.complex128:
        dst.real.copy_(parts[0])
        if len(parts) > 1:
            dst.imag.copy_(parts[1])
        else:
            dst.imag.zero_()
    elif parts[0].data_ptr() != dst.data_ptr() or not dst.is_contiguous():
        dst.copy_(parts[0])


def apply_inplace(x, fn):
    """Run an in-place real operator on every real part of the CUDA tensor x and
    store the results in x (also for non-contiguous views, whose kernel input is
    a contiguous copy)."""
    parts = device_parts(x)
    for p in parts:
        fn(p)
    store_device(x, parts)


def join_parts(parts, like):
    """Inverse of real_parts: rebuild an array of the caller's dtype."""
    if len(parts) == 1:
        re = parts[0]
        return re.astype(complex) if np.iscomplexobj(like) else re
    return parts[0] + 1j * parts[1]


def write_back(dst, parts):
    """Store results into the caller's host array in place."""
    if np.iscomplexobj(dst):
        dst.real[...] = parts[0]
        dst.imag[...] = parts[1] if len(parts) > 1 else 0.0
    else:
        dst[...] = parts[0]


# ------------------------------------------------- pipelined host <-> device copies
# Host arrays travel through two reusable pinned staging buffers per device on a
# dedicated copy stream: the (multi-threaded) host copy of chunk k overlaps the
# DMA of chunk k - 1 (or k + 1 on the way back), so a solve_discrete on numpy
# arrays moves at close to the PCIe rate instead of a pageable synchronous copy.
# Strided host views (the real / imaginary part of a complex128 array) are
# gathered / scattered by the host copy itself: no temporary host arrays.
_CHUNK = 8 << 20  # doubles per staging buffer (64 MB)
_staging = {}
_staging_lock = threading.Lock()


class _Staging:
    def __init__(self, device, n):
        torch = _torch()
        self.device = device
        self.n = n
        self.bufs = [torch.empty(n, dtype=torch.float64, pin_memory=True) for _ in range(2)]
        self.stream = torch.cuda.Stream(device)
        self.events = [torch.cuda.Event() for _ in range(2)]
        self.lock = threading.Lock()


def _stage(device, plane):
    torch = _torch()
    dev = torch.device(device)
    key = dev.index if dev.index is not None else torch.cuda.current_device()
    need = max(_CHUNK, plane)
    with _staging_lock:
        st = _staging.get(key)
        if st is None or st.n < need:
            st = _staging[key] = _Staging(torch.device("cuda", key), need)
        return st


def _chunks(shape, n):
    rows = shape[0] if shape else 1
    plane = int(np.prod(shape[1:])) if len(shape) > 1 else 1
    step = max(1, n // max(plane, 1))
    for a in range(0, rows, step):
        yield a, min(rows, a + step)


def _host_tensor(view):
    torch = _torch()
    with warnings.catch_warnings():  # read-only inputs are only read
        warnings.simplefilter("ignore")
        return torch.from_numpy(view)


def h2d(src, dst):
    """Copy the float64 host view `src` (any positive strides) into the
    contiguous device tensor `dst` of the same shape."""
    torch = _torch()
    src = np.asarray(src)
    if src.ndim == 0 or src.size == 0:
        dst.copy_(_host_tensor(np.ascontiguousarray(src)))
        return
    plane = src.size // src.shape[0]
    st = _stage(dst.device, plane)
    with st.lock:
        cur = torch.cuda.current_stream(dst.device)
        st.stream.wait_stream(cur)
        for k, (a, b) in enumerate(_chunks(src.shape, st.n)):
            i = k & 1
            st.events[i].synchronize()  # the DMA that last read buffer i is done
            hb = st.bufs[i][:(b - a) * plane].view((b - a,) + src.shape[1:])
            hb.copy_(_host_tensor(src[a:b]))
            with torch.cuda.stream(st.stream):
                dst[a:b].copy_(hb, non_blocking=True)
                st.events[i].record(st.stream)
        cur.wait_stream(st.stream)
        for e in st.events:
            e.synchronize()  # the buffers are free for the next caller


def d2h(src, dst):
    """Copy the contiguous device tensor `src` into the writeable float64 host
    view `dst` (any positive strides) of the same shape; synchronous."""
    torch = _torch()
    if dst.ndim == 0 or dst.size == 0:
        dst[...] = src.cpu().numpy()
        return
    plane = dst.size // dst.shape[0]
    st = _stage(src.device, plane)
    with st.lock:
        st.stream.wait_stream(torch.cuda.current_stream(src.device))
        pending = None
        for k, (a, b) in enumerate(_chunks(dst.shape, st.n)):
            i = k & 1
            hb = st.bufs[i][:(b - a) * plane].view((b - a,) + dst.shape[1:])
            with torch.cuda.stream(st.stream):
                hb.copy_(src[a:b], non_blocking=True)
                st.events[i].record(st.stream)
            if pending is not None:
                j, pa, pb, phb = pending
                st.events[j].synchronize()
                _host_tensor(dst[pa:pb]).copy_(phb)
            pending = (i, a, b, hb)
        j, pa, pb, phb = pending
        st.events[j].synchronize()
        _host_tensor(dst[pa:pb]).copy_(phb)


def _any_nonzero(view):
    torch = _torch()
    for a, b in _chunks(view.shape, _CHUNK):
        if bool(_host_tensor(view[a:b]).ne(0).any()):
            return True
    return False


def upload_parts(arr, device):
    """Host array -> [re] or [re, im] contiguous float64 device tensors (the
    imaginary part only when it is not zero), by pipelined pinned copies."""
    torch = _torch()
    a = np.asarray(arr)
    if np.iscomplexobj(a):
        if a.dtype != np.complex128:
            a = a.astype(np.complex128)
        views = [a.real]
        if _any_nonzero(a.imag):
            views.append(a.imag)
    else:
        views = [a if a.dtype == np.float64 else a.astype(np.float64)]
    out = []
    for v in views:
        t = torch.empty(v.shape, dtype=torch.float64, device=device)
        h2d(v, t)
        out.append(t)
    return out


def download_parts(parts, like):
    """[re] or [re, im] device tensors -> a new host array: complex128 when `like`
    is complex or there is an imaginary part, else float64."""
    torch = _torch()
    cplx = len(parts) > 1 or np.iscomplexobj(like)
    shape = tuple(parts[0].shape)
    if not cplx:
        out = np.empty(shape, dtype=np.float64)
        d2h(parts[0], out)
        return out
    out = np.empty(shape, dtype=np.complex128)
    d2h(parts[0], out.real)
    if len(parts) > 1:
        d2h(parts[1], out.imag)
    else:
        _host_tensor(out.imag).zero_()
    return out
