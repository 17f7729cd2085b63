"""Inputs of the round-2 golden cases (tests/golden/make_golden_r2.py), rebuilt
bit-identically on any box: seeded numpy streams and the workloads' tables.

Each case returns (F, T, (n_x, n_y, n_z), scheme, profile, grid):
F the host right-hand side, T the oracle's (A, B, C, D) weight table, and
scheme / profile / grid the package objects for the device path.
"""
import numpy as np

import paper_1912_03565_b200 as hb
from oracle import helm_oracle as orc
from paper_1912_03565_b200 import workloads as wl


def slab_grid(n, planes):
    """The full n^3 grid's first `planes` levels: same step h = 1/(n+1)."""
    return hb.make_grid(hb.Domain(0.0, 1.0, 0.0, 1.0, 0.0, (planes + 1) / (n + 1)), n, n, planes)


def zero_profile(n_z, gamma=0.0):
    z = np.zeros(n_z + 2, complex)
    return hb.CoefficientProfile(k2=z, k2_z=z.copy(), k2_zz=z.copy(), gamma=gamma)


def _cd4_table(g, gamma):
    z = np.zeros(g.n_z + 2)
    return orc.weight_table("cd4", z, z, z, gamma, (g.h_x, g.h_y, g.h_z), g.n_z)


def case(name):
    if name in ("gen63", "gen127"):
        n = int(name[3:])
        tab = wl.general_table(n)
        g = hb.make_grid(hb.Domain(0, 1, 0, 1, 0, 1), n, n, n)
        F = np.random.default_rng(500 + n).standard_normal((n, n, n))
        return F, (tab.A, tab.B, tab.C, tab.D), (n, n, n), tab, zero_profile(n), g
    if name == "cfg5s":
        w = wl.workload(5)
        P = 16
        T = tuple(t[:P] for t in (w.scheme.A, w.scheme.B, w.scheme.C, w.scheme.D))
        g = slab_grid(2047, P)
        return (wl.host_rhs(w, planes=P), T, (2047, 2047, P), hb.StencilTable(*T),
                zero_profile(P), g)
    if name == "cfg4s":
        w = wl.workload(4)
        P = 8
        g = slab_grid(1023, P)
        return (wl.host_rhs(w, planes=P), _cd4_table(g, -1.5), (1023, 1023, P),
                hb.SchemeKind.CONVECTION_DIFFUSION_4, zero_profile(P, -1.5), g)
    if name == "cd4n127":
        g = hb.make_grid(hb.Domain(0, 1, 0, 1, 0, 1), 127, 127, 127)
        F = np.random.default_rng(41).uniform(-1.0, 1.0, (127, 127, 127))
        return (F, _cd4_table(g, -1.5), (127, 127, 127), hb.SchemeKind.CONVECTION_DIFFUSION_4,
                zero_profile(127, -1.5), g)
    raise KeyError(name)


SUMMARY = {"gen127": (63, 8), "cfg5s": (7, 16), "cfg4s": (3, 8), "cd4n127": (63, 8)}


def summary_errors(name, U, golden):
    """Relative L2 errors of U's summaries (plane, subsample, norm) against the
    reference's (make_golden_r2.summaries)."""
    plane, sub = SUMMARY[name]
    p = U[plane][::sub, ::sub] if U.shape[1] > 256 else U[plane]
    s = U[:, ::sub, ::sub]
    rel = lambda a, b: float(np.linalg.norm(a - b) / np.linalg.norm(b))
    nrm = golden[f"{name}_norms"][0]
    return (rel(p, golden[f"{name}_plane"]), rel(s, golden[f"{name}_sub"]),
            abs(np.linalg.norm(U) - nrm) / nrm)
