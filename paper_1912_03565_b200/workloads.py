"""The five BASELINE.json configurations as seeded synthetic workloads.

Not part of the solve path: shared by the tests, ``bench.py`` and
``__graft_entry__.smoke``. No public benchmark suite is involved; inputs
are seeded synthetic fields with BASELINE.json's shapes and distributions
(SURVEY.md §8(d)). Seeds are recorded here and in DESIGN.md.

cfg1  4th order Helmholtz, unit cube, N=31,   k = 10(1 + 0.5 sin pi z)
cfg2  6th order Helmholtz, unit cube, N=127,  same k
cfg3  6th order Helmholtz, unit cube, N=511,  k = 40(1 + 0.3 sin 2 pi z), F ~ N(0,1)
cfg4  4th order conv-diff, unit cube, N=1023, -lap u + 1.5 u_z (gamma = -1.5), F ~ U[-1,1]
      (b_x, b_y cannot be represented by the paper's class; z-projection)
cfg5  general admissible 27-point table, N=2047, per-row weights ~ N(0,1) from seed 50,
      centre = 1.5 x sum |off-diagonal|, F ~ N(0,1)
"""

import math
from dataclasses import dataclass

import numpy as np

from .grid import CoefficientProfile, Domain, make_grid
from .stencil import SchemeKind, StencilTable

PI = math.pi
SEEDS = {1: 1, 2: 2, 3: 3, 4: 4, 5: 5}
TABLE_SEED = 50
SIZES = {1: 31, 2: 127, 3: 511, 4: 1023, 5: 2047}


@dataclass
class Workload:
    cfg: int
    n: int
    scheme: object
    grid: object
    profile: CoefficientProfile
    rhs_kind: str   # "uniform" | "normal" | "manufactured"
    seed: int


def unit_grid(n):
    return make_grid(Domain(0.0, 1.0, 0.0, 1.0, 0.0, 1.0), n, n, n)


# k^2 = 100 (1 + 0.5 sin pi z)^2 = 100 (1.125 + sin pi z - 0.125 cos 2 pi z)
def _k2_a(z):
    return 100.0 * (1.0 + 0.5 * np.sin(PI * z)) ** 2


def _k2_a_derivs(z, order):
    s1, c1, s2, c2 = np.sin(PI * z), np.cos(PI * z), np.sin(2 * PI * z), np.cos(2 * PI * z)
    table = {
        0: 112.5 + 100.0 * s1 - 12.5 * c2,
        1: 100.0 * PI * c1 + 25.0 * PI * s2,
        2: -100.0 * PI**2 * s1 + 50.0 * PI**2 * c2,
        3: -100.0 * PI**3 * c1 - 100.0 * PI**3 * s2,
        4: 100.0 * PI**4 * s1 - 200.0 * PI**4 * c2,
    }
    return table[order]


def profile_a(grid):
    z = grid.z_nodes(closed=True)
    return CoefficientProfile(k2=_k2_a(z).astype(complex),
                              k2_z=_k2_a_derivs(z, 1).astype(complex),
                              k2_zz=_k2_a_derivs(z, 2).astype(complex))


def profile_b(grid):
    """k = 40 (1 + 0.3 sin 2 pi z)."""
    z = grid.z_nodes(closed=True)
    s, c = np.sin(2 * PI * z), np.cos(2 * PI * z)
    k2 = 1600.0 * (1.0 + 0.3 * s) ** 2
    k2_z = 1920.0 * PI * (1.0 + 0.3 * s) * c
    k2_zz = 1920.0 * PI**2 * (0.6 * c**2 - 2.0 * (1.0 + 0.3 * s) * s)
    return CoefficientProfile(k2=k2.astype(complex), k2_z=k2_z.astype(complex),
                              k2_zz=k2_zz.astype(complex))


def general_table(n_z, seed=TABLE_SEED):
    """cfg5 weights: a, b, c (n_z, 3) and d at offsets -1/+1 ~ N(0,1); the centre
    d[:, 1] = 1.5 (4 sum|a| + 2 sum|b| + 2 sum|c| + |d_-1| + |d_+1|)."""
    rng = np.random.default_rng(seed)
    A = rng.standard_normal((n_z, 3))
    B = rng.standard_normal((n_z, 3))
    C = rng.standard_normal((n_z, 3))
    D = np.zeros((n_z, 3))
    D[:, 0] = rng.standard_normal(n_z)
    D[:, 2] = rng.standard_normal(n_z)
    off = (4.0 * np.abs(A).sum(1) + 2.0 * np.abs(B).sum(1) + 2.0 * np.abs(C).sum(1)
           + np.abs(D[:, 0]) + np.abs(D[:, 2]))
    D[:, 1] = 1.5 * off
    return StencilTable(A, B, C, D)


def workload(cfg, n=None):
    n = SIZES[cfg] if n is None else n
    grid = unit_grid(n)
    seed = SEEDS[cfg]
    if cfg == 1:
        return Workload(1, n, SchemeKind.FOURTH_ORDER, grid, profile_a(grid), "uniform", seed)
    if cfg == 2:
        return Workload(2, n, SchemeKind.SIXTH_ORDER, grid, profile_a(grid), "uniform", seed)
    if cfg == 3:
        return Workload(3, n, SchemeKind.SIXTH_ORDER, grid, profile_b(grid), "normal", seed)
    if cfg == 4:
        zeros = np.zeros(n + 2, dtype=complex)
        prof = CoefficientProfile(k2=zeros, k2_z=zeros.copy(), k2_zz=zeros.copy(), gamma=-1.5)
        return Workload(4, n, SchemeKind.CONVECTION_DIFFUSION_4, grid, prof, "uniform", seed)
    if cfg == 5:
        zeros = np.zeros(n + 2, dtype=complex)
        prof = CoefficientProfile(k2=zeros, k2_z=zeros.copy(), k2_zz=zeros.copy())
        return Workload(5, n, general_table(n), grid, prof, "normal", seed)
    raise ValueError(f"unknown config {cfg}")


def host_rhs(w: Workload, planes=None):
    """Seeded discrete F (float64, (n_z, n_y, n_x)) on the host; `planes` limits n_z
    (a bounded sample for CPU baselines; the first planes of the same stream)."""
    nz = w.n if planes is None else planes
    rng = np.random.default_rng(w.seed)
    shape = (nz, w.n, w.n)
    if w.rhs_kind == "normal":
        return rng.standard_normal(shape)
    return rng.uniform(-1.0, 1.0, shape)


RHS_CHUNK = 8  # device_rhs draws planes in seeded chunks of this many planes


def device_rhs(w: Workload, device, planes=None, z0=0):
    """Seeded F generated directly on the device (large configs; torch Philox).

    Planes [z0, z0 + planes) of the workload's volume (all n by default). The
    volume is drawn in chunks of RHS_CHUNK planes, chunk c from its own
    generator seeded (seed, c), so any z-slab (one rank's part of a
    multi-GPU run) equals the same planes of the one-GPU volume bit for bit."""
    import torch
    nz = w.n - z0 if planes is None else planes
    out = torch.empty((nz, w.n, w.n), device=device, dtype=torch.float64)
    g = torch.Generator(device=device)
    c = z0 // RHS_CHUNK
    while c * RHS_CHUNK < z0 + nz:
        a, b = c * RHS_CHUNK, min((c + 1) * RHS_CHUNK, w.n)
        g.manual_seed(w.seed * 1_000_003 + c)
        shape = (b - a, w.n, w.n)
        if w.rhs_kind == "normal":
            blk = torch.randn(shape, generator=g, device=device, dtype=torch.float64)
        else:
            blk = torch.rand(shape, generator=g, device=device, dtype=torch.float64)
            blk.mul_(2.0).sub_(1.0)
        lo, hi = max(a, z0), min(b, z0 + nz)
        out[lo - z0:hi - z0].copy_(blk[lo - a:hi - a])
        del blk
        c += 1
    return out


# --------------------------------------------- manufactured solution (cfg1/2)
# u = sin(pi x) sin(2 pi y) sin(3 pi z); lap u = -14 pi^2 u; f = (k^2 - 14 pi^2) u.
def _g(z, order):
    """d^order/dz^order of g(z) = (k^2(z) - 14 pi^2) sin(3 pi z)."""
    K = [_k2_a_derivs(z, k) - (14.0 * PI**2 if k == 0 else 0.0) for k in range(5)]
    w = 3.0 * PI
    S = [np.sin(w * z), w * np.cos(w * z), -w**2 * np.sin(w * z), -w**3 * np.cos(w * z),
         w**4 * np.sin(w * z)]
    binom = [math.comb(order, k) for k in range(order + 1)]
    return sum(binom[k] * K[k] * S[order - k] for k in range(order + 1))


def manufactured_u(x, y, z):
    return np.sin(PI * x) * np.sin(2 * PI * y) * np.sin(3 * PI * z)


def manufactured_source():
    """SourceSpec-compatible callables for f = (k^2 - 14 pi^2) u (cfg1/cfg2 RHS-A)."""
    from .assembly import SourceSpec

    def xy(x, y):
        return np.sin(PI * x) * np.sin(2 * PI * y)

    def f(x, y, z):
        return xy(x, y) * _g(z, 0)

    def f_z(x, y, z):
        return xy(x, y) * _g(z, 1)

    def f_zz(x, y, z):
        return xy(x, y) * _g(z, 2)

    def f_xx(x, y, z):
        return -PI**2 * f(x, y, z)

    def f_yy(x, y, z):
        return -4.0 * PI**2 * f(x, y, z)

    def lap_f(x, y, z):
        return -5.0 * PI**2 * f(x, y, z) + f_zz(x, y, z)

    def d4_f(x, y, z):
        return 17.0 * PI**4 * f(x, y, z) + xy(x, y) * _g(z, 4)

    def f_xxyy(x, y, z):
        return 4.0 * PI**4 * f(x, y, z)

    def f_xxzz(x, y, z):
        return -PI**2 * f_zz(x, y, z)

    def f_yyzz(x, y, z):
        return -4.0 * PI**2 * f_zz(x, y, z)

    return SourceSpec(f=f, f_z=f_z, f_xx=f_xx, f_yy=f_yy, f_zz=f_zz, lap_f=lap_f, d4_f=d4_f,
                      f_xxyy=f_xxyy, f_xxzz=f_xxzz, f_yyzz=f_yyzz)
