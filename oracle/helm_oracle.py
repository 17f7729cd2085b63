"""CPU oracle for the B200 solve path — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
--impl reference legs may import this module. The product package
(paper_1912_03565_b200) never imports it and has no CPU path.

A numpy restatement of the reference helmfft's algorithm for the hot path,
each function citing the reference lines it follows. The DST-I runs in
scipy.fft.dst(type=1, norm="ortho") — the same third-party kernel the
reference calls (spectral.py:56; scipy >= 1.10 per pyproject.toml:10-13,
1.18.1 here, DUCC0 backend) — and ``dense_dst_matrix`` restates the
reference's independent dense cross-check (spectral.py:66-72,
oracle.py:106-114).

Parity of this restatement is pinned against vectors produced by the real
reference (tests/golden/make_golden.py, run in the build container where
/root/reference exists) and against the reference's own known-answer tests
(test_spectral.py:37-52, test_tridiag.py:24-46).
"""

import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import scipy.fft

PIVOT_RTOL = 1e-14  # tridiag.py:22


class OracleSingular(ArithmeticError):
    def __init__(self, msg, n, m, l):
        super().__init__(msg)
        self.n, self.m, self.l = n, m, l


# --------------------------------------------------------------- weights
def _cdiv(x, c):
    """numpy's complex128 / real: x * (1/c) (ufunc loop: scl = 1/c, re*scl)."""
    return x * (1.0 / c)


def row_weights(scheme, k2, k2_z, k2_zz, gamma, h, l):
    """(a, b, c, d) at offsets (l-1, l, l+1) for row level l (1-based),
    restating stencil.py:70-161 one row at a time. h = (h_x, h_y, h_z);
    k2, k2_z, k2_zz hold the n_z + 2 closed-grid samples (real, or complex for
    complex k(z))."""
    hx, hy, hz = h
    r_zx, r_zy = hz**2 / hx**2, hz**2 / hy**2
    # complex k^2 (complex k(z)): the same formulas in complex128
    dt = complex if any(np.iscomplexobj(v) and np.any(np.imag(v)) for v in (k2, k2_z, k2_zz)) \
        else float
    a, b, c, d = (np.zeros(3, dtype=dt) for _ in range(4))
    if scheme == "2":  # stencil.py:70-82
        b[1], c[1] = r_zx, r_zy
        d[0] = d[2] = 1.0
        d[1] = -2.0 * (r_zx + r_zy + 1.0) + hz**2 * k2[l]
        return a, b, c, d
    # The reference computes in complex128; numpy divides a complex numerator by a
    # real constant as x * (1/c) (reciprocal, then product), so those divisions
    # are written as q(x, c) below; real / real stays a true division.
    q = _cdiv
    if scheme in ("4", "cd4"):  # stencil.py:85-104
        hz2 = hz**2
        b[0] = b[2] = (1.0 + r_zx) / 12.0
        c[0] = c[2] = (1.0 + r_zy) / 12.0
        d[0] = 2.0 / 3.0 - (r_zx + r_zy) / 6.0 + q(hz2 * k2[l - 1], 12.0)
        d[2] = 2.0 / 3.0 - (r_zx + r_zy) / 6.0 + q(hz2 * k2[l + 1], 12.0)
        a[1] = (r_zx + r_zy) / 12.0
        b[1] = q(4.0 * r_zx - r_zy - 1.0 + q(hz2 * k2[l], 2.0), 6.0)
        c[1] = q(4.0 * r_zy - r_zx - 1.0 + q(hz2 * k2[l], 2.0), 6.0)
        d[1] = -4.0 * (1.0 + r_zx + r_zy) / 3.0 + q(hz2 * k2[l], 2.0)
        if scheme == "cd4":  # stencil.py:136-161 (Python complex: true divisions)
            if np.any(k2):
                raise ValueError("convection-diffusion needs k^2 = 0")
            g = gamma * hz
            b[0] *= 1.0 - g / 2.0
            b[2] *= 1.0 + g / 2.0
            c[0] *= 1.0 - g / 2.0
            c[2] *= 1.0 + g / 2.0
            d[0] = d[0] - (g / 12.0) * (4.0 - r_zx - r_zy - g)
            d[2] = d[2] + (g / 12.0) * (4.0 - r_zx - r_zy + g)
            d[1] = d[1] - g**2 / 6.0
        return a, b, c, d
    if scheme == "6":  # stencil.py:107-133
        if not (hx == hy == hz):
            raise ValueError("sixth order needs a uniform grid")
        s2, s3, s4 = hz**2, hz**3, hz**4
        km, kc, kp, kz, kzz = k2[l - 1], k2[l], k2[l + 1], k2_z[l], k2_zz[l]
        a[0] = a[2] = 1.0 / 30.0
        b[0] = c[0] = 1.0 / 10.0 + q(s2 * km, 90.0) - q(s3 * kz, 120.0)
        b[2] = c[2] = 1.0 / 10.0 + q(s2 * kp, 90.0) + q(s3 * kz, 120.0)
        d[0] = 7.0 / 15.0 - q(s2 * km, 90.0) - q(s3 * kz, 20.0) * (1.0 / 3.0 + q(s2 * km, 6.0))
        d[2] = 7.0 / 15.0 - q(s2 * kp, 90.0) + q(s3 * kz, 20.0) * (1.0 / 3.0 + q(s2 * kp, 6.0))
        a[1] = 1.0 / 10.0 + q(s2 * kc, 90.0)
        b[1] = c[1] = 7.0 / 15.0 - q(s2 * kc, 90.0)
        d[1] = (-64.0 / 15.0 + q(14.0 * s2 * kc, 15.0) - q(s4 * (kc * kc), 20.0)
                + q(s4 * kzz, 20.0))
        return a, b, c, d
    raise ValueError(f"unknown scheme {scheme!r}")


def weight_table(scheme, k2, k2_z, k2_zz, gamma, h, n_z):
    """(A, B, C, D) arrays (n_z, 3), row l-1 = level l (stencil.py:177-195)."""
    rows = [row_weights(scheme, k2, k2_z, k2_zz, gamma, h, l) for l in range(1, n_z + 1)]
    return tuple(np.array([r[i] for r in rows]) for i in range(4))


def mode_cosines(n_x, n_y):
    """stencil.py:219-223."""
    cx = np.cos(np.pi * np.arange(1, n_x + 1) / (n_x + 1))
    cy = np.cos(np.pi * np.arange(1, n_y + 1) / (n_y + 1))
    return cx, cy


# ------------------------------------------------------------- transforms
def dst_stack(values, workers=1):
    """Orthonormal 2D DST-I of every z-plane, x-pass then y-pass (spectral.py:75-91).
    Returns a new array. workers == 1 goes plane by plane exactly like the
    reference; workers > 1 batches the whole stack (threaded DUCC0)."""
    if workers <= 1:
        out = np.empty_like(values)
        for l in range(values.shape[0]):
            plane = scipy.fft.dst(values[l], type=1, norm="ortho", axis=1)
            out[l] = scipy.fft.dst(plane, type=1, norm="ortho", axis=0)
        return out
    out = scipy.fft.dst(values, type=1, norm="ortho", axis=-1, workers=workers)
    return scipy.fft.dst(out, type=1, norm="ortho", axis=-2, workers=workers)


def dense_dst_matrix(n):
    """S[a, b] = sqrt(2/(n+1)) sin(pi a b/(n+1)), 1-based (spectral.py:35-43, oracle.py:106-109)."""
    idx = np.arange(1, n + 1)
    return np.sqrt(2.0 / (n + 1)) * np.sin(np.pi * (np.outer(idx, idx) % (2 * (n + 1))) / (n + 1))


def dst_stack_dense(values):
    """Same map through the dense matrices (spectral.py:66-72)."""
    sx, sy = dense_dst_matrix(values.shape[-1]), dense_dst_matrix(values.shape[-2])
    return np.einsum("mj,zji,in->zmn", sy, values, sx, optimize=True)


# ----------------------------------------------------------------- Thomas
def thomas_sweep(w, table, cx, cy, m_offset=0):
    """Vectorised Thomas over every (m, n) line of a (n_z, M, n_x) slab, in place
    (tridiag.py:126-167), with the pivot screen of tridiag.py:136-151."""
    A, B, C, D = table
    n_z = w.shape[0]
    thr = PIVOT_RTOL * max(float(np.abs(t).max()) for t in table)
    cyc, cxr = cy[:, None], cx[None, :]

    def lam(l, k):  # stencil.py:226-234
        return 4.0 * A[l, k] * (cyc * cxr) + 2.0 * B[l, k] * cxr + 2.0 * C[l, k] * cyc + D[l, k]

    def screen(den, l):
        bad = np.abs(den) < thr
        if bad.any():
            mi, ni = np.argwhere(bad)[0]
            raise OracleSingular(f"vanishing pivot at row {l + 1}", int(ni + 1),
                                 int(m_offset + mi + 1), l + 1)

    # numpy's complex division (the reference's arithmetic) multiplies by the
    # reciprocal of a real denominator; r = 1/den reproduces it for real data
    cp = np.empty_like(w)
    den = lam(0, 1)
    screen(den, 0)
    r = 1.0 / den
    cp[0] = lam(0, 2) * r
    w[0] = w[0] * r
    for l in range(1, n_z):
        lo = lam(l, 0)
        den = lam(l, 1) - lo * cp[l - 1]
        screen(den, l)
        r = 1.0 / den
        if l < n_z - 1:
            cp[l] = lam(l, 2) * r
        w[l] = (w[l] - lo * w[l - 1]) * r
    for l in range(n_z - 2, -1, -1):
        w[l] -= cp[l] * w[l + 1]
    return w


def solve_line(sub, diag, sup, rhs):
    """Single explicit tridiagonal system (tridiag.py:59-90)."""
    n = len(diag)
    scale = max(np.abs(sub).max(), np.abs(diag).max(), np.abs(sup).max())
    cp = np.zeros(n, dtype=np.result_type(diag, rhs))
    x = np.array(rhs, dtype=cp.dtype)
    for l in range(n):
        den = diag[0] if l == 0 else diag[l] - sub[l] * cp[l - 1]
        if abs(den) < PIVOT_RTOL * scale:
            raise OracleSingular(f"vanishing pivot at row {l + 1}", None, None, l + 1)
        if l < n - 1:
            cp[l] = sup[l] / den
        x[l] = (x[l] if l == 0 else x[l] - sub[l] * x[l - 1]) / den
    for l in range(n - 2, -1, -1):
        x[l] -= cp[l] * x[l + 1]
    return x


# -------------------------------------------------------- full pipeline
def solve(F, table, cx, cy, workers=1):
    """Homogeneous-Dirichlet solve: DST -> Thomas -> DST (solver.py:293-317 with
    the fold a copy, assembly.py:268-269). F is (n_z, n_y, n_x); returns U
    (complex when F or the table is complex: complex k(z))."""
    cplx = np.iscomplexobj(F) or any(np.iscomplexobj(t) and np.any(np.imag(t)) for t in table)
    w = dst_stack(np.array(F, dtype=complex if cplx else np.float64), workers)
    if workers <= 1:
        thomas_sweep(w, table, cx, cy)
    else:
        n_y = w.shape[1]
        cuts = np.linspace(0, n_y, min(workers, n_y) + 1).astype(int)

        def run(i):
            sub = np.ascontiguousarray(w[:, cuts[i]:cuts[i + 1], :])
            thomas_sweep(sub, table, cx, cy[cuts[i]:cuts[i + 1]], int(cuts[i]))
            w[:, cuts[i]:cuts[i + 1], :] = sub

        with ThreadPoolExecutor(max_workers=len(cuts) - 1) as ex:
            list(ex.map(run, range(len(cuts) - 1)))
    return dst_stack(w, workers)


# --------------------------------------------------------------- operators
_PLANE_TERMS = (((-1, -1), 0), ((1, -1), 0), ((-1, 1), 0), ((1, 1), 0),
                ((-1, 0), 1), ((1, 0), 1), ((0, -1), 2), ((0, 1), 2), ((0, 0), 3))


def accumulate27(ext, table):
    """27-point operator on a closed box (assembly.py:20-25, 229-244), same term
    order and zero-column skipping. Returns the interior result."""
    n_z, n_y, n_x = (s - 2 for s in ext.shape)
    out = np.zeros((n_z, n_y, n_x), dtype=np.result_type(ext, *table))
    for dl in (-1, 0, 1):
        k = dl + 1
        for (di, dj), wi in _PLANE_TERMS:
            w = table[wi][:, k]
            if not np.any(w):
                continue
            blk = ext[1 + dl:1 + dl + n_z, 1 + dj:1 + dj + n_y, 1 + di:1 + di + n_x]
            out += w[:, None, None] * blk
    return out


def rhs_fourth(f_closed, h_z):
    """F = h_z^2 (f/2 + (1/12) sum of the 6 face neighbours) (assembly.py:183-193)."""
    fc = f_closed
    core = fc[1:-1, 1:-1, 1:-1]
    nb = (fc[1:-1, 1:-1, :-2] + fc[1:-1, 1:-1, 2:] + fc[1:-1, :-2, 1:-1]
          + fc[1:-1, 2:, 1:-1] + fc[:-2, 1:-1, 1:-1] + fc[2:, 1:-1, 1:-1])
    return h_z**2 * (0.5 * core + _cdiv(nb, 12.0))  # complex / 12.0 in the reference


def rhs_sixth(f, lap, d4, fxxyy, fxxzz, fyyzz, fz, k2_int, k2z_int, h):
    """assembly.py:195-213 with sampled fields; k2_int = k2[1:-1]."""
    h2 = h**2
    h4 = h2 * h2
    mixed = fxxyy + fxxzz + fyyzz
    r = h2 * (f + (h2 / 12.0) * lap + (h4 / 360.0) * d4 + (h4 / 90.0) * mixed)
    r = r - (h4 / 20.0) * k2_int[:, None, None] * f
    r = r + (h2 * h4 / 60.0) * k2z_int[:, None, None] * fz
    return r


def residual_l2(U, F, table):
    """||A U - F||_2 with a zero boundary (assembly.py:277-289)."""
    ext = np.zeros(tuple(s + 2 for s in U.shape))
    ext[1:-1, 1:-1, 1:-1] = U
    return float(np.linalg.norm((accumulate27(ext, table) - F).ravel()))


def default_workers():
    return max(1, os.cpu_count() or 1)


