"""Generate the golden fixtures from the REAL reference (helmfft) — build container only.

Run:  PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py
(/root/reference exists only in the build container; the committed .npz
files travel to the GPU box and pin both the oracle and the CUDA path.)

Every array here is produced by the reference's public API on seeded inputs
(numpy default_rng) that tests regenerate bit-identically; for BASELINE
config 5 the general weight table enters through the reference's
``stencil._BUILDERS`` hook, since the reference has no
public API for an arbitrary admissible table.
"""

import math
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REF)
sys.path.insert(0, os.path.abspath(os.path.join(HERE, "..", "..")))

import helmfft as hf  # noqa: E402
from helmfft import stencil as ref_stencil  # noqa: E402
from helmfft.spectral import dst_lines  # noqa: E402

from paper_1912_03565_b200 import workloads as wl  # noqa: E402


def ref_grid(n, domain=(0.0, 1.0, 0.0, 1.0, 0.0, 1.0), nxyz=None):
    nx, ny, nz = nxyz or (n, n, n)
    return hf.make_grid(hf.Domain(*domain), nx, ny, nz)


def ref_profile(prof):
    return hf.CoefficientProfile(k2=np.asarray(prof.k2, complex), k2_z=np.asarray(prof.k2_z, complex),
                                 k2_zz=np.asarray(prof.k2_zz, complex), gamma=complex(prof.gamma))


def ref_scheme(key):
    return {"2": hf.SchemeKind.SECOND_ORDER, "4": hf.SchemeKind.FOURTH_ORDER,
            "6": hf.SchemeKind.SIXTH_ORDER, "cd4": hf.SchemeKind.CONVECTION_DIFFUSION_4}[key]


def table_of(scheme, prof, grid):
    return np.stack([t.real for t in hf.coefficient_table(scheme, prof, grid)])


def solve_ref(F, scheme, prof, grid):
    u, _ = hf.solve_discrete(hf.Field3D(F.astype(complex)), hf.BoundaryData.zero(), scheme, prof,
                             grid)
    assert np.abs(u.values.imag).max() == 0.0
    return u.values.real.copy()


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


def main():
    out = {}
    # ---- coefficient tables for every scheme (pin the host table builders)
    g31 = ref_grid(31)
    pa = ref_profile(wl.profile_a(wl.unit_grid(31)))
    for key in ("2", "4", "6"):
        out[f"table_{key}_cfg1prof"] = table_of(ref_scheme(key), pa, g31)
    pcd = hf.constant_profile(0.0, g31, gamma=-1.5)
    out["table_cd4_g-1.5"] = table_of(hf.SchemeKind.CONVECTION_DIFFUSION_4, pcd, g31)
    pcd100 = hf.constant_profile(0.0, g31, gamma=-100.0)
    out["table_cd4_g-100"] = table_of(hf.SchemeKind.CONVECTION_DIFFUSION_4, pcd100, g31)
    ganiso = ref_grid(0, (0.0, math.pi, 0.0, 2.0, 0.0, 1.0), (9, 7, 6))
    paniso = hf.constant_profile(2.0, ganiso)
    for key in ("2", "4"):
        out[f"table_{key}_aniso"] = table_of(ref_scheme(key), paniso, ganiso)
    cx, cy = ref_stencil.mode_cosines(g31)
    out["cx31"], out["cy31"] = cx, cy
    pb = ref_profile(wl.profile_b(wl.unit_grid(63)))
    out["table_6_cfg3prof_n63"] = table_of(hf.SchemeKind.SIXTH_ORDER, pb, ref_grid(63))

    # ---- known answers of the DST (test_spectral.py:37-52)
    out["dst_basis3"] = dst_lines(np.array([1.0, 0.0, 0.0]), axis=0).real
    rng = np.random.default_rng(7)
    for n in (1, 2, 3, 7, 15, 31, 63, 125, 127):
        plane = rng.standard_normal((n, n))
        out[f"dst2d_in_{n}"] = plane
        out[f"dst2d_out_{n}"] = hf.dst2d(hf.make_plan(n, n), plane.astype(complex)).real

    # ---- cfg1, RHS-B (uniform F, solve only)
    w1 = wl.workload(1)
    F1 = wl.host_rhs(w1)
    out["cfg1_F_sum"] = np.array([F1.sum(), np.abs(F1).sum()])
    out["cfg1_U"] = solve_ref(F1, hf.SchemeKind.FOURTH_ORDER, pa, g31)

    # ---- cfg1, RHS-A (manufactured, through the 4th-order RHS operator)
    src = wl.manufactured_source()
    ref_src = hf.SourceSpec(**{k: getattr(src, k) for k in
                               ("f", "f_z", "f_xx", "f_yy", "f_zz", "lap_f", "d4_f",
                                "f_xxyy", "f_xxzz", "f_yyzz")})
    FA = hf.build_rhs(hf.SchemeKind.FOURTH_ORDER, ref_src, pa, g31).values.real
    out["cfg1A_F"] = FA
    UA = solve_ref(FA, hf.SchemeKind.FOURTH_ORDER, pa, g31)
    out["cfg1A_U"] = UA

    # ---- convergence studies (errors vs the analytic u) for 4th and 6th order
    conv = []
    for key in ("4", "6"):
        for n in (31, 63, 127):
            g = ref_grid(n)
            p = ref_profile(wl.profile_a(wl.unit_grid(n)))
            F = hf.build_rhs(ref_scheme(key), ref_src, p, g)
            u, _ = hf.solve_discrete(F, hf.BoundaryData.zero(), ref_scheme(key), p, g)
            x = g.x_nodes()[None, None, :]
            y = g.y_nodes()[None, :, None]
            z = g.z_nodes()[:, None, None]
            exact = wl.manufactured_u(x, y, z)
            diff = u.values.real - exact
            conv.append([float(key), n, np.abs(diff).max(),
                         np.linalg.norm(diff) / np.linalg.norm(exact)])
            if key == "6" and n == 31:
                out["cfg2A_n31_F"] = F.values.real
                out["cfg2A_n31_U"] = u.values.real
    out["convergence"] = np.array(conv)

    # ---- cfg2 full size (127^3, 6th order, uniform F): summaries only
    w2 = wl.workload(2)
    F2 = wl.host_rhs(w2)
    U2 = solve_ref(F2, hf.SchemeKind.SIXTH_ORDER, ref_profile(w2.profile), ref_grid(127))
    out["cfg2_U_plane63"] = U2[63]
    out["cfg2_U_sub8"] = U2[::8, ::8, ::8]
    out["cfg2_U_norms"] = np.array([np.linalg.norm(U2), np.abs(U2).max(), U2.sum()])

    # ---- cd4 (cfg4 scheme) small, and the general table (cfg5 class) small
    g15 = ref_grid(15)
    F15 = np.random.default_rng(11).uniform(-1, 1, (15, 15, 15))
    out["cd4_n15_F"] = F15
    out["cd4_n15_U"] = solve_ref(F15, hf.SchemeKind.CONVECTION_DIFFUSION_4,
                                 hf.constant_profile(0.0, g15, gamma=-1.5), g15)
    tab = wl.general_table(15)
    T = (tab.A, tab.B, tab.C, tab.D)
    out["gen_n15_table"] = np.stack(T)
    F15b = np.random.default_rng(12).standard_normal((15, 15, 15))
    out["gen_n15_F"] = F15b
    with TableBuilder(T) as sch:
        out["gen_n15_U"] = solve_ref(F15b, sch, hf.constant_profile(0.0, g15), g15)
    # anisotropic, non power-of-two extents (dense DST path), 4th order
    Fan = np.random.default_rng(13).standard_normal((6, 7, 9))
    out["aniso_F"] = Fan
    out["aniso_U"] = solve_ref(Fan, hf.SchemeKind.FOURTH_ORDER, paniso, ganiso)

    # ---- resonance: second order, k^2 tuned so mode (n=2, m=3) is singular at row 1
    gr = ref_grid(0, (0.0, math.pi, 0.0, math.pi, 0.0, math.pi), (5, 6, 4))
    r_zx, r_zy = gr.h_z**2 / gr.h_x**2, gr.h_z**2 / gr.h_y**2
    cxr, cyr = ref_stencil.mode_cosines(gr)
    k2 = (2.0 * (r_zx + r_zy + 1.0) - 2.0 * r_zx * cxr[1] - 2.0 * r_zy * cyr[2]) / gr.h_z**2
    try:
        solve_ref(np.ones((4, 6, 5)), hf.SchemeKind.SECOND_ORDER, hf.constant_profile(k2, gr), gr)
        raise AssertionError("expected a singular system")
    except hf.SingularSystemError as exc:
        out["resonance"] = np.array([k2, exc.n, exc.m])

    # ---- complex k(z): complex profiles, complex fields
    def zsolve(F, bnd, scheme, prof, grid):
        b = hf.BoundaryData.zero() if bnd is None else hf.BoundaryData.from_array(bnd)
        u, _ = hf.solve_discrete(hf.Field3D(np.asarray(F, complex)), b, scheme, prof, grid)
        return u.values.copy()

    zlev = np.linspace(0.0, 1.0, 33)
    k2z4 = 100.0 * (1 + 0.5 * np.sin(np.pi * zlev)) ** 2 * (1 + 0.3j)
    pz4 = hf.CoefficientProfile(k2=k2z4, k2_z=np.zeros(33, complex), k2_zz=np.zeros(33, complex))
    rz = np.random.default_rng(101)
    Fz4 = rz.standard_normal((31, 31, 31)) + 1j * rz.standard_normal((31, 31, 31))
    out["z4_k2"] = k2z4  # F regenerates from default_rng(101) in the tests
    out["z4_table"] = np.stack(hf.coefficient_table(hf.SchemeKind.FOURTH_ORDER, pz4, g31))
    out["z4_U"] = zsolve(Fz4, None, hf.SchemeKind.FOURTH_ORDER, pz4, g31)

    s = 1 + 0.3 * np.sin(2 * np.pi * zlev)
    sz = 0.6 * np.pi * np.cos(2 * np.pi * zlev)
    szz = -1.2 * np.pi ** 2 * np.sin(2 * np.pi * zlev)
    c6 = 1600.0 * (1 + 0.2j)
    pz6 = hf.CoefficientProfile(k2=c6 * s ** 2, k2_z=c6 * 2 * s * sz,
                                k2_zz=c6 * 2 * (sz ** 2 + s * szz))
    rz = np.random.default_rng(102)
    Fz6 = rz.standard_normal((31, 31, 31)) + 1j * rz.standard_normal((31, 31, 31))
    out["z6_k2"], out["z6_k2z"], out["z6_k2zz"] = pz6.k2, pz6.k2_z, pz6.k2_zz
    # F regenerates from default_rng(102) in the tests
    out["z6_U"] = zsolve(Fz6, None, hf.SchemeKind.SIXTH_ORDER, pz6, g31)

    # non-cubic, power-of-two line lengths, complex Dirichlet data, real F
    gzb = ref_grid(0, (0.0, 1.0, 0.0, 2.0, 0.0, 0.5), (15, 31, 9))
    rz = np.random.default_rng(103)
    k2b = 30.0 * (rz.standard_normal(11) + 1j * rz.standard_normal(11))
    pzb = hf.CoefficientProfile(k2=k2b, k2_z=np.zeros(11, complex), k2_zz=np.zeros(11, complex))
    Fzb = rz.standard_normal((9, 31, 15))
    Bzb = rz.standard_normal((11, 33, 17)) + 1j * rz.standard_normal((11, 33, 17))
    out["zb_k2"], out["zb_F"], out["zb_B"] = k2b, Fzb, Bzb
    out["zb_U"] = zsolve(Fzb, Bzb, hf.SchemeKind.SECOND_ORDER, pzb, gzb)

    # generic (non-power-of-two) sizes, every scheme but cd4: random complex
    # profiles, fields and boundary (the reference's dense-oracle criterion,
    # test_acceptance.py:161-186)
    gd = ref_grid(0, (0.0, math.pi, 0.0, math.pi, 0.0, math.pi), (6, 6, 6))
    rz = np.random.default_rng(104)
    for key in ("2", "4", "6"):
        prof = hf.CoefficientProfile(k2=rz.standard_normal(8) + 1j * rz.standard_normal(8),
                                     k2_z=rz.standard_normal(8) + 0j,
                                     k2_zz=rz.standard_normal(8) + 0j)
        F = rz.standard_normal((6, 6, 6)) + 1j * rz.standard_normal((6, 6, 6))
        B = rz.standard_normal((8, 8, 8)) + 1j * rz.standard_normal((8, 8, 8))
        out[f"zd{key}_k2"], out[f"zd{key}_k2z"], out[f"zd{key}_k2zz"] = \
            prof.k2, prof.k2_z, prof.k2_zz
        out[f"zd{key}_F"], out[f"zd{key}_B"] = F, B
        out[f"zd{key}_U"] = zsolve(F, B, ref_scheme(key), prof, gd)

    # complex right-hand sides: 6th order with a complex profile, cd4 with a
    # complex gamma (assembly.py:195-224 in complex arithmetic) — F and the solve
    zr_src = ref_src
    out["zr6_F"] = hf.build_rhs(hf.SchemeKind.SIXTH_ORDER, zr_src, pz6, g31).values
    out["zr6_U"] = zsolve(out["zr6_F"], None, hf.SchemeKind.SIXTH_ORDER, pz6, g31)
    pcdz = hf.constant_profile(0.0, g15, gamma=-1.5 + 0.5j)
    out["zrcd_F"] = hf.build_rhs(hf.SchemeKind.CONVECTION_DIFFUSION_4, zr_src, pcdz, g15).values
    out["zrcd_U"] = zsolve(out["zrcd_F"], None, hf.SchemeKind.CONVECTION_DIFFUSION_4, pcdz, g15)

    path = os.path.join(HERE, "golden.npz")
    np.savez_compressed(path, **out)
    print(f"wrote {path}: {os.path.getsize(path) / 1e6:.2f} MB, {len(out)} arrays")


if __name__ == "__main__":
    main()
