"""Bridge to the UNMODIFIED reference (`helmfft`) — TEST / BASELINE INFRASTRUCTURE ONLY.

Imports the stock reference package from oracle/_ref (installed by
oracle/build_ref.sh; it travels to the GPU box) or, in the build container,
from /root/reference/pkg/src. Only tests/ and bench.py's CPU reference legs use
this module; the product package never imports it.

``reference_case(w, planes)`` turns one of the package's workloads into the
reference's own objects: the first `planes` z-levels of the workload's grid
(same step h), the same seeded host F, and the scheme. BASELINE cfg5's general
admissible table has no public reference API; it enters through the
reference's ``stencil._BUILDERS`` hook (stencil.py:164-174),
which ``table_scheme`` swaps in for the duration of a ``with`` block.
"""

import contextlib
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
_CANDIDATES = (os.path.join(HERE, "_ref"), "/root/reference/pkg/src")


def load():
    """The stock reference module, or None when neither location has it."""
    try:
        import helmfft  # noqa: F401
        return sys.modules["helmfft"]
    except ImportError:
        pass
    for cand in _CANDIDATES:
        if os.path.isfile(os.path.join(cand, "helmfft", "solver.py")):
            sys.path.insert(0, cand)
            import helmfft
            return helmfft
    return None


@contextlib.contextmanager
def table_scheme(hf, table):
    """Swap stencil._BUILDERS[SECOND_ORDER] for an explicit per-row table; yields
    the SchemeKind that now selects it."""
    from helmfft import stencil as ref_stencil
    A, B, C, D = (np.asarray(t) for t in table)

    def build(profile, grid, l):
        return ref_stencil.StencilCoefficients(
            A[l - 1].astype(complex), B[l - 1].astype(complex), C[l - 1].astype(complex),
            D[l - 1].astype(complex), 1.0, 1.0)

    saved = ref_stencil._BUILDERS[hf.SchemeKind.SECOND_ORDER]
    ref_stencil._BUILDERS[hf.SchemeKind.SECOND_ORDER] = build
    try:
        yield hf.SchemeKind.SECOND_ORDER
    finally:
        ref_stencil._BUILDERS[hf.SchemeKind.SECOND_ORDER] = saved


def reference_case(hf, w, planes):
    """(F complex128, scheme or table, profile, grid) of the reference for the
    first `planes` levels of workload `w` (a package workloads.Workload)."""
    n = w.n
    g = hf.make_grid(hf.Domain(0.0, 1.0, 0.0, 1.0, 0.0, (planes + 1) / (n + 1)), n, n, planes)
    prof = w.profile
    k = lambda a: np.asarray(a, complex)[:planes + 2]
    # a slab's closed levels are the full profile's first planes + 2
    rprof = hf.CoefficientProfile(k2=k(prof.k2), k2_z=k(prof.k2_z), k2_zz=k(prof.k2_zz),
                                  gamma=complex(prof.gamma))
    scheme = getattr(w.scheme, "value", "table")
    if scheme == "table":
        sch = tuple(np.asarray(t)[:planes] for t in (w.scheme.A, w.scheme.B, w.scheme.C,
                                                      w.scheme.D))
    else:
        sch = {"2": hf.SchemeKind.SECOND_ORDER, "4": hf.SchemeKind.FOURTH_ORDER,
               "6": hf.SchemeKind.SIXTH_ORDER,
               "cd4": hf.SchemeKind.CONVECTION_DIFFUSION_4}[scheme]
    from paper_1912_03565_b200 import workloads as wl
    F = wl.host_rhs(w, planes=planes).astype(complex)
    return F, sch, rprof, g


def solve_reference(hf, F, sch, prof, grid, workers):
    """Stock hf.solve_discrete on the case; returns (U complex128, PhaseTimings).
    workers <= 1 runs Sequential(), else SharedWorkers(min(workers, n_z))."""
    mode = hf.Sequential() if workers <= 1 else hf.SharedWorkers(min(workers, grid.n_z))
    cfg = hf.SolverConfig(mode=mode)
    if isinstance(sch, tuple):
        with table_scheme(hf, sch) as kind:
            u, t = hf.solve_discrete(hf.Field3D(F), hf.BoundaryData.zero(), kind, prof, grid, cfg)
    else:
        u, t = hf.solve_discrete(hf.Field3D(F), hf.BoundaryData.zero(), sch, prof, grid, cfg)
    return u.values, t
