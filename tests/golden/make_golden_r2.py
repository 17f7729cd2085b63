"""Round-2 golden fixtures from the REAL reference (helmfft) — build container only.

Run:  python tests/golden/make_golden_r2.py
(imports the unmodified reference from /root/reference/pkg/src, or from
oracle/_ref when that is where it was installed; writes
tests/golden/golden_r2.npz, which travels to the GPU box.)

These pin the configurations BASELINE.json times, at sizes the reference
finishes here in seconds:

* ``gen63_*``  — the cfg5 class (general admissible 27-point table, seed-50
  rows, centre = 1.5 x sum|off-diagonal|) at 63^3, full solution; and at
  127^3, summaries (one plane, a stride-8 subsample, norms);
* ``cfg5s_*``  — the cfg5 workload itself on its first 16 z-planes:
  2047 x 2047 planes, the first 16 rows of the cfg5 table, F = the first 16
  planes of the cfg5 N(0,1) stream (workloads.host_rhs(w5, planes=16));
  summaries of U;
* ``cfg4s_*``  — the cfg4 workload (cd4, gamma = -1.5) on its first 8 z-planes
  of 1023 x 1023 (same step h = 1/1024), F = the first 8 planes of the cfg4
  U[-1, 1] stream; summaries of U;
* ``cd4n127_*`` — cd4 gamma = -1.5 at 127^3 (cfg4's scheme on a full cube),
  uniform F from default_rng(41); summaries.

The general table enters the reference through its ``stencil._BUILDERS`` hook
(stencil.py:164-174), the only way the reference accepts an arbitrary
admissible table.
"""

import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.abspath(os.path.join(HERE, "..", ".."))
for cand in ("/root/reference/pkg/src", os.path.join(ROOT, "oracle", "_ref")):
    if os.path.isdir(os.path.join(cand, "helmfft")):
        sys.path.insert(0, cand)
        break
sys.path.insert(0, ROOT)

import helmfft as hf  # noqa: E402
from helmfft import stencil as ref_stencil  # noqa: E402

from paper_1912_03565_b200 import workloads as wl  # noqa: E402


class TableBuilder:
    """Swaps stencil._BUILDERS[SECOND_ORDER] for an explicit per-row table."""

    def __init__(self, table):
        self.table = table
        self.saved = None

    def __enter__(self):
        A, B, C, D = self.table

        def build(profile, grid, l):
            return ref_stencil.StencilCoefficients(
                A[l - 1].astype(complex), B[l - 1].astype(complex), C[l - 1].astype(complex),
                D[l - 1].astype(complex), 1.0, 1.0)

        self.saved = ref_stencil._BUILDERS[hf.SchemeKind.SECOND_ORDER]
        ref_stencil._BUILDERS[hf.SchemeKind.SECOND_ORDER] = build
        return hf.SchemeKind.SECOND_ORDER

    def __exit__(self, *exc):
        ref_stencil._BUILDERS[hf.SchemeKind.SECOND_ORDER] = self.saved


def solve_ref(F, scheme, prof, grid, workers=8):
    cfg = hf.SolverConfig(mode=hf.SharedWorkers(min(workers, grid.n_z)))
    u, _ = hf.solve_discrete(hf.Field3D(F.astype(complex)), hf.BoundaryData.zero(), scheme, prof,
                             grid, cfg)
    assert np.abs(u.values.imag).max() == 0.0
    return u.values.real.copy()


def summaries(prefix, U, out, plane, sub):
    out[f"{prefix}_plane"] = U[plane][::sub, ::sub] if U.shape[1] > 256 else U[plane]
    out[f"{prefix}_sub"] = U[:, ::sub, ::sub]
    out[f"{prefix}_norms"] = np.array([np.linalg.norm(U), np.abs(U).max(), U.sum()])


def slab_grid(n, planes):
    """The full n^3 grid's first `planes` levels: same step h = 1/(n+1)."""
    return hf.make_grid(hf.Domain(0.0, 1.0, 0.0, 1.0, 0.0, (planes + 1) / (n + 1)), n, n, planes)


def main():
    out = {}
    t0 = time.time()
    # ---- cfg5 class at 63^3 (full) and 127^3 (summaries)
    for n in (63, 127):
        tab = wl.general_table(n)
        T = (tab.A, tab.B, tab.C, tab.D)
        g = hf.make_grid(hf.Domain(0, 1, 0, 1, 0, 1), n, n, n)
        F = np.random.default_rng(500 + n).standard_normal((n, n, n))
        with TableBuilder(T) as sch:
            U = solve_ref(F, sch, hf.constant_profile(0.0, g), g)
        if n == 63:
            out["gen63_U"] = U
        else:
            summaries("gen127", U, out, 63, 8)
    # ---- cfg5 workload, first 16 planes of 2047^2
    w5 = wl.workload(5)
    P5 = 16
    T5 = tuple(t[:P5] for t in (w5.scheme.A, w5.scheme.B, w5.scheme.C, w5.scheme.D))
    g5 = slab_grid(2047, P5)
    F5 = wl.host_rhs(w5, planes=P5)
    with TableBuilder(T5) as sch:
        U5 = solve_ref(F5, sch, hf.constant_profile(0.0, g5), g5)
    del F5
    summaries("cfg5s", U5, out, 7, 16)
    del U5
    # ---- cfg4 workload, first 8 planes of 1023^2
    w4 = wl.workload(4)
    P4 = 8
    g4 = slab_grid(1023, P4)
    F4 = wl.host_rhs(w4, planes=P4)
    U4 = solve_ref(F4, hf.SchemeKind.CONVECTION_DIFFUSION_4,
                   hf.constant_profile(0.0, g4, gamma=-1.5), g4)
    summaries("cfg4s", U4, out, 3, 8)
    del U4, F4
    # ---- cd4 at 127^3 (cfg4's scheme on a full cube)
    g = hf.make_grid(hf.Domain(0, 1, 0, 1, 0, 1), 127, 127, 127)
    F = np.random.default_rng(41).uniform(-1.0, 1.0, (127, 127, 127))
    U = solve_ref(F, hf.SchemeKind.CONVECTION_DIFFUSION_4,
                  hf.constant_profile(0.0, g, gamma=-1.5), g)
    summaries("cd4n127", U, out, 63, 8)

    path = os.path.join(HERE, "golden_r2.npz")
    np.savez_compressed(path, **out)
    print(f"wrote {path}: {os.path.getsize(path) / 1e6:.2f} MB, {len(out)} arrays, "
          f"{time.time() - t0:.0f} s")


if __name__ == "__main__":
    main()
