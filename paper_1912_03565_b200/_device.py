"""Host <-> device array plumbing for the operator modules.

Operators accept numpy arrays (the reference's type: complex128, usually
with zero imaginary part) or torch CUDA float64 tensors. Device kernels are
fp64-real; a complex array with a non-zero imaginary part is handled as two
real solves (the operators are real and linear, so real and imaginary parts
never mix when the coefficients are real).
"""

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
