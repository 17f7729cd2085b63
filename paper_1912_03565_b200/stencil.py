"""Row weights of the 27-point compact schemes and the plane-operator spectrum.

Host-side and O(n_z): the weights depend on z only, so the per-row table is
12 numbers per level. It is built here (vectorised over levels) and uploaded
once per solve; the Thomas kernels generate every eigenvalue from it on the
fly. Formulas follow the reference helmfft.stencil (stencil.py:70-161);
the arithmetic is arranged so that, for a real profile, every weight equals
the real part of the reference's complex value bit for bit.

Layout of a level's weights (stencil.py:36-58): four values a, b, c, d per
level offset k in {0, 1, 2} = {l-1, l, l+1}; a multiplies the 4 corners
(i+-1, j+-1), b the 2 x-neighbours, c the 2 y-neighbours, d the centre.

Beyond the reference's four schemes, :class:`StencilTable` carries an
arbitrary per-row weight table of the same admissible class (z-dependent
only, symmetric in +-x and +-y) — the paper's general 27-diagonal family
(PAPER.md:149-155), BASELINE config 5.
"""

import enum
from dataclasses import dataclass

import numpy as np

from .errors import UnsupportedSchemeError
from .grid import CoefficientProfile, Grid3D


class SchemeKind(enum.Enum):
    """Same members and values as the reference (stencil.py:29-33)."""

    SECOND_ORDER = "2"
    FOURTH_ORDER = "4"
    SIXTH_ORDER = "6"
    CONVECTION_DIFFUSION_4 = "cd4"


_KNOWN = {"2", "4", "6", "cd4"}


def scheme_key(scheme) -> str:
    """Scheme identity as a string; accepts this package's SchemeKind, the
    reference's SchemeKind (same .value), a StencilTable, or the raw value."""
    if isinstance(scheme, StencilTable):
        return "table"
    value = getattr(scheme, "value", scheme)
    if value not in _KNOWN:
        raise ValueError(f"unknown scheme {scheme!r}")
    return value


@dataclass(frozen=True)
class StencilCoefficients:
    """One row's weights at levels (l-1, l, l+1) (stencil.py:36-58)."""

    a: np.ndarray
    b: np.ndarray
    c: np.ndarray
    d: np.ndarray
    r_zx: float
    r_zy: float

    def level(self, offset):
        k = offset + 1
        return self.a[k], self.b[k], self.c[k], self.d[k]

    def row_sum(self):
        return complex(np.sum(4 * self.a + 2 * self.b + 2 * self.c + self.d))


class StencilTable:
    """An explicit per-row weight table of the admissible 27-point class.

    A, B, C, D: arrays of shape (n_z, 3); column k is level offset k - 1.
    Used as the ``scheme`` argument wherever a SchemeKind is accepted.
    """

    value = "table"

    def __init__(self, A, B, C, D):
        arrs = [np.asarray(t) for t in (A, B, C, D)]
        shapes = {t.shape for t in arrs}
        if len(shapes) != 1 or len(arrs[0].shape) != 2 or arrs[0].shape[1] != 3:
            raise ValueError(f"table arrays must share a (n_z, 3) shape, got {shapes}")
        self.A, self.B, self.C, self.D = arrs

    @property
    def n_z(self):
        return self.A.shape[0]

    def __repr__(self):
        return f"StencilTable(n_z={self.n_z})"


def _ratios(grid):
    return grid.h_z**2 / grid.h_x**2, grid.h_z**2 / grid.h_y**2


def _qdiv(x, c):
    """Division of a profile-dependent term by a constant, written as numpy's
    complex128 / real evaluates it in the reference: x * (1/c)."""
    return x * (1.0 / c)


def _levels(profile, n_z):
    """Profile samples at levels l-1, l, l+1 for rows l = 1..n_z."""
    k2 = np.asarray(profile.k2)
    if len(k2) != n_z + 2:
        raise ValueError(f"profile has {len(k2)} levels, grid needs {n_z + 2}")
    return k2[:-2], k2[1:-1], k2[2:]


def _dtype(profile):
    parts = (profile.k2, profile.k2_z, profile.k2_zz, profile.gamma)
    return complex if any(np.iscomplexobj(p) and np.any(np.imag(p)) for p in parts) else float


def _as(profile_arr, dtype):
    arr = np.asarray(profile_arr)
    return arr.real.astype(float) if dtype is float else arr.astype(complex)


def _table_second(profile, grid, dt):
    n = grid.n_z
    r_zx, r_zy = _ratios(grid)
    k2c = _as(_levels(profile, n)[1], dt)
    A, B, C, D = (np.zeros((n, 3), dtype=dt) for _ in range(4))
    B[:, 1] = r_zx
    C[:, 1] = r_zy
    D[:, 0] = D[:, 2] = 1.0
    D[:, 1] = -2.0 * (r_zx + r_zy + 1.0) + grid.h_z**2 * k2c
    return A, B, C, D


def _table_fourth(profile, grid, dt):
    n = grid.n_z
    r_zx, r_zy = _ratios(grid)
    hz2 = grid.h_z**2
    k2m, k2c, k2p = (_as(v, dt) for v in _levels(profile, n))
    A, B, C, D = (np.zeros((n, 3), dtype=dt) for _ in range(4))
    off_b, off_c = (1.0 + r_zx) / 12.0, (1.0 + r_zy) / 12.0
    B[:, 0] = B[:, 2] = off_b
    C[:, 0] = C[:, 2] = off_c
    base = 2.0 / 3.0 - (r_zx + r_zy) / 6.0
    q = _qdiv
    D[:, 0] = base + q(hz2 * k2m, 12.0)
    D[:, 2] = base + q(hz2 * k2p, 12.0)
    A[:, 1] = (r_zx + r_zy) / 12.0
    B[:, 1] = q(4.0 * r_zx - r_zy - 1.0 + q(hz2 * k2c, 2.0), 6.0)
    C[:, 1] = q(4.0 * r_zy - r_zx - 1.0 + q(hz2 * k2c, 2.0), 6.0)
    D[:, 1] = -4.0 * (1.0 + r_zx + r_zy) / 3.0 + q(hz2 * k2c, 2.0)
    return A, B, C, D


def _table_sixth(profile, grid, dt):
    if not grid.uniform:
        raise UnsupportedSchemeError(
            f"sixth-order scheme needs h_x = h_y = h_z, got ({grid.h_x}, {grid.h_y}, {grid.h_z})")
    n = grid.n_z
    h = grid.h_z
    h2, h3, h4 = h**2, h**3, h**4
    k2m, k2c, k2p = (_as(v, dt) for v in _levels(profile, n))
    k2z = _as(np.asarray(profile.k2_z)[1:-1], dt)
    k2zz = _as(np.asarray(profile.k2_zz)[1:-1], dt)
    A, B, C, D = (np.zeros((n, 3), dtype=dt) for _ in range(4))
    q = _qdiv
    A[:, 0] = A[:, 2] = 1.0 / 30.0
    lower = 1.0 / 10.0 + q(h2 * k2m, 90.0) - q(h3 * k2z, 120.0)
    upper = 1.0 / 10.0 + q(h2 * k2p, 90.0) + q(h3 * k2z, 120.0)
    B[:, 0] = C[:, 0] = lower
    B[:, 2] = C[:, 2] = upper
    tilt = q(h3 * k2z, 20.0)
    D[:, 0] = 7.0 / 15.0 - q(h2 * k2m, 90.0) - tilt * (1.0 / 3.0 + q(h2 * k2m, 6.0))
    D[:, 2] = 7.0 / 15.0 - q(h2 * k2p, 90.0) + tilt * (1.0 / 3.0 + q(h2 * k2p, 6.0))
    A[:, 1] = 1.0 / 10.0 + q(h2 * k2c, 90.0)
    B[:, 1] = C[:, 1] = 7.0 / 15.0 - q(h2 * k2c, 90.0)
    D[:, 1] = (-64.0 / 15.0 + q(14.0 * h2 * k2c, 15.0) - q(h4 * (k2c * k2c), 20.0)
               + q(h4 * k2zz, 20.0))
    return A, B, C, D


def _table_convdiff(profile, grid, dt):
    if np.asarray(profile.k2).any():
        raise ValueError("convection-diffusion weights expect a zero k^2 profile")
    A, B, C, D = _table_fourth(profile, grid, dt)
    r_zx, r_zy = _ratios(grid)
    gamma = profile.gamma
    g = (gamma.real if dt is float else complex(gamma)) * grid.h_z
    down, up = 1.0 - g / 2.0, 1.0 + g / 2.0
    B[:, 0] *= down
    B[:, 2] *= up
    C[:, 0] *= down
    C[:, 2] *= up
    D[:, 0] = D[:, 0] - (g / 12.0) * (4.0 - r_zx - r_zy - g)
    D[:, 2] = D[:, 2] + (g / 12.0) * (4.0 - r_zx - r_zy + g)
    D[:, 1] = D[:, 1] - g**2 / 6.0
    return A, B, C, D


_TABLES = {
    "2": _table_second,
    "4": _table_fourth,
    "6": _table_sixth,
    "cd4": _table_convdiff,
}


def coefficient_table(scheme, profile: CoefficientProfile, grid: Grid3D):
    """(A, B, C, D), each (n_z, 3): row l-1 holds level l's weights (stencil.py:177-195).

    Real float64 arrays when the profile is real (the only case the device
    kernels take), complex otherwise.
    """
    if isinstance(scheme, StencilTable):
        if scheme.n_z != grid.n_z:
            raise ValueError(f"table has {scheme.n_z} rows, grid has n_z = {grid.n_z}")
        return scheme.A, scheme.B, scheme.C, scheme.D
    key = scheme_key(scheme)
    return _TABLES[key](profile, grid, _dtype(profile))


def _row(scheme, profile, grid, l):
    if not 1 <= l <= grid.n_z:
        raise IndexError(f"row level {l} outside 1..{grid.n_z}")
    A, B, C, D = coefficient_table(scheme, profile, grid)
    r_zx, r_zy = _ratios(grid)
    if scheme_key(scheme) == "6":
        r_zx = r_zy = 1.0
    return StencilCoefficients(*(np.asarray(t[l - 1], dtype=complex) for t in (A, B, C, D)),
                               r_zx, r_zy)


def coefficients_second(profile, grid, l):
    return _row(SchemeKind.SECOND_ORDER, profile, grid, l)


def coefficients_fourth(profile, grid, l):
    return _row(SchemeKind.FOURTH_ORDER, profile, grid, l)


def coefficients_sixth(profile, grid, l):
    return _row(SchemeKind.SIXTH_ORDER, profile, grid, l)


def coefficients_convdiff(profile, grid, l):
    return _row(SchemeKind.CONVECTION_DIFFUSION_4, profile, grid, l)


def coefficients_for(scheme, profile, grid, l) -> StencilCoefficients:
    return _row(scheme, profile, grid, l)


def mode_cosines(grid: Grid3D):
    """cos(pi n/(n_x+1)), n = 1..n_x, and cos(pi m/(n_y+1)), m = 1..n_y (stencil.py:219-223)."""
    cx = np.cos(np.pi * np.arange(1, grid.n_x + 1) / (grid.n_x + 1))
    cy = np.cos(np.pi * np.arange(1, grid.n_y + 1) / (grid.n_y + 1))
    return cx, cy


def eigenvalue(coeffs: StencilCoefficients, level_offset: int, n: int, m: int,
               grid: Grid3D) -> complex:
    """Plane-operator eigenvalue 4a cx cy + 2b cx + 2c cy + d of mode (n, m) (stencil.py:198-216)."""
    if not 1 <= n <= grid.n_x:
        raise IndexError(f"mode n={n} outside 1..{grid.n_x}")
    if not 1 <= m <= grid.n_y:
        raise IndexError(f"mode m={m} outside 1..{grid.n_y}")
    a, b, c, d = coeffs.level(level_offset)
    cx = np.cos(np.pi * n / (grid.n_x + 1))
    cy = np.cos(np.pi * m / (grid.n_y + 1))
    return 4.0 * a * cx * cy + 2.0 * b * cx + 2.0 * c * cy + d


def eigenvalue_plane(a, b, c, d, cx, cy):
    """Eigenvalues of one level's operator for all (m, n): shape (len(cy), len(cx)) (stencil.py:226-234)."""
    cy = np.asarray(cy)[:, None]
    cx = np.asarray(cx)[None, :]
    return 4.0 * a * (cy * cx) + 2.0 * b * cx + 2.0 * c * cy + d


def pivot_threshold(table, rtol=1e-14):
    """PIVOT_RTOL * max |weight| over the whole table (tridiag.py:22, 136-137)."""
    return rtol * max(float(np.abs(t).max()) for t in table)


def is_complex_table(table) -> bool:
    """True when some weight has a non-zero imaginary part (complex k(z))."""
    return any(np.iscomplexobj(t) and np.any(np.imag(t)) for t in table)


def pack_table(table) -> np.ndarray:
    """(A, B, C, D) -> the C-ABI layout table[l*12 + k*4 + {a,b,c,d}] (float64).
    Complex tables go through pack_table_z."""
    A, B, C, D = (np.asarray(t) for t in table)
    if is_complex_table((A, B, C, D)):
        raise ValueError("complex table: use pack_table_z")
    packed = np.stack([np.real(t).astype(np.float64) for t in (A, B, C, D)], axis=-1)
    return np.ascontiguousarray(packed.reshape(-1))


def pack_table_z(table):
    """Complex (A, B, C, D) -> (real parts, imaginary parts), each in the
    pack_table layout (hfb_plan_set_coefficients_z)."""
    A, B, C, D = (np.asarray(t, dtype=complex) for t in table)
    re = np.stack([t.real for t in (A, B, C, D)], axis=-1)
    im = np.stack([t.imag for t in (A, B, C, D)], axis=-1)
    return (np.ascontiguousarray(re.reshape(-1), dtype=np.float64),
            np.ascontiguousarray(im.reshape(-1), dtype=np.float64))


def term_mask(table) -> int:
    """27-bit mask of the (level offset, plane offset) terms whose weight column
    is not identically zero, in the reference's accumulation order
    (assembly.py:20-25, 236-243)."""
    A, B, C, D = (np.asarray(t) for t in table)
    names = (A, A, A, A, B, B, C, C, D)
    mask = 0
    for k in range(3):
        for o, w in enumerate(names):
            if np.any(w[:, k]):
                mask |= 1 << (k * 9 + o)
    return mask
