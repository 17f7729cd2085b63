"""Parity of the sm_100a path against the oracle and the reference's goldens.

All tests call through the C-ABI (ctypes) on cuda:0. Tolerances: the north
star's 1e-10 relative L2 is the bar; the measured noise floor is ~1e-14, so
tighter tolerances are asserted where the arithmetic allows (stated inline).
"""
import math

import numpy as np
import pytest

import paper_1912_03565_b200 as hb
from oracle import helm_oracle as orc
from paper_1912_03565_b200 import workloads as wl

pytestmark = pytest.mark.gpu
PI = math.pi
TOL = 1e-10  # north_star: relative L2 vs the reference CPU solver
# Golden comparisons: different (but equally accurate) DST/Thomas rounding,
# amplified by the conditioning of each system: measured ~1e-13 for the
# well-conditioned configs, ~1e-11 for the near-resonant 6th-order cfg3.
PARITY = 1e-11


def rel_l2(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / np.linalg.norm(b))


def oracle_table(scheme_key, prof, g):
    return orc.weight_table(scheme_key, np.real(prof.k2), np.real(prof.k2_z),
                            np.real(prof.k2_zz), complex(prof.gamma).real,
                            (g.h_x, g.h_y, g.h_z), g.n_z)


# ---------------------------------------------------------------- DST-I
@pytest.mark.parametrize("n", [1, 2, 3, 7, 15, 31, 63, 125, 127])
def test_dst2d_matches_reference_goldens(golden, cuda, n):
    out = hb.dst2d(hb.make_plan(n, n), golden[f"dst2d_in_{n}"])
    assert np.abs(out - golden[f"dst2d_out_{n}"]).max() < 1e-13 * max(1, np.abs(out).max())


@pytest.mark.parametrize("nx,ny,nz", [(255, 255, 3), (511, 127, 2), (1023, 1023, 1),
                                      (2047, 31, 2), (31, 2047, 1), (9, 7, 6), (64, 33, 4)])
def test_transform_stack_vs_scipy(cuda, nx, ny, nz):
    rng = np.random.default_rng(nx + ny + nz)
    data = rng.standard_normal((nz, ny, nx))
    f = hb.Field3D(data.copy())
    hb.transform_stack(hb.make_plan(nx, ny), f)
    ref = orc.dst_stack(data, workers=4)
    assert np.abs(f.values - ref).max() < 1e-13 * np.abs(ref).max()


def test_basis_vector_and_single_mode(cuda):
    out = hb.dst_lines(np.array([1.0, 0.0, 0.0]), axis=0)
    assert np.allclose(out, [0.5, 1 / math.sqrt(2), 0.5], atol=1e-15)
    n_x, n_y, n0, m0 = 8, 6, 3, 2
    i, j = np.arange(1, n_x + 1), np.arange(1, n_y + 1)
    plane = np.sin(PI * m0 * j / (n_y + 1))[:, None] * np.sin(PI * n0 * i / (n_x + 1))[None, :]
    out = hb.dst2d(hb.make_plan(n_x, n_y), plane)
    expect = np.zeros_like(out)
    expect[m0 - 1, n0 - 1] = math.sqrt((n_x + 1) * (n_y + 1)) / 2.0
    assert np.abs(out - expect).max() < 1e-12


@pytest.mark.parametrize("n", [1, 2, 3, 4, 5, 7, 8, 9, 31, 125, 127, 511])
def test_involution_and_norm(cuda, n):
    rng = np.random.default_rng(n)
    plane = rng.standard_normal((n, n))
    plan = hb.make_plan(n, n)
    once = hb.dst2d(plan, plane)
    twice = hb.dst2d(plan, once)
    assert np.abs(twice - plane).max() <= 1e-13 * np.abs(plane).max()
    assert np.linalg.norm(once) == pytest.approx(np.linalg.norm(plane), rel=1e-13)


def test_dense_reference_path(cuda):
    rng = np.random.default_rng(3)
    plane = rng.standard_normal((32, 64))
    plan = hb.make_plan(64, 32)
    assert np.abs(hb.dst2d(plan, plane) - hb.dst2d_reference(plan, plane)).max() < 1e-12


def test_transform_disjoint_halves_bitwise(cuda):
    rng = np.random.default_rng(9)
    data = rng.standard_normal((8, 6, 7))
    full, halves = hb.Field3D(data.copy()), hb.Field3D(data.copy())
    plan = hb.make_plan(7, 6)
    hb.transform_stack(plan, full)
    hb.transform_stack(plan, halves, (0, 3))
    hb.transform_stack(plan, halves, (3, 8))
    assert np.array_equal(full.values, halves.values)
    data = rng.standard_normal((8, 63, 127))
    full, halves = hb.Field3D(data.copy()), hb.Field3D(data.copy())
    plan = hb.make_plan(127, 63)
    hb.transform_stack(plan, full)
    hb.transform_stack(plan, halves, (0, 3))
    hb.transform_stack(plan, halves, (3, 8))
    assert np.array_equal(full.values, halves.values)


def test_transform_ranges_validated(cuda):
    f = hb.Field3D(np.zeros((4, 3, 3)))
    with pytest.raises(IndexError):
        hb.transform_stack(hb.make_plan(3, 3), f, (0, 5))
    data = np.random.default_rng(2).standard_normal((3, 4, 4))
    f = hb.Field3D(data.copy())
    hb.transform_stack(hb.make_plan(4, 4), f, (1, 1))
    assert np.array_equal(f.values, data)


def test_line_batches_match_planes(cuda):
    rng = np.random.default_rng(5)
    data = rng.standard_normal((5, 63, 31))
    a, b = data.copy(), data.copy()
    hb.transform_stack(hb.make_plan(31, 63), a)
    hb.transform_lines_x(b, (0, 40))
    hb.transform_lines_x(b, (40, 63))
    hb.transform_lines_y(b, (0, 17))
    hb.transform_lines_y(b, (17, 31))
    assert np.abs(a - b).max() < 1e-13 * np.abs(a).max()


# ---------------------------------------------------------------- Thomas
def test_solve_system_known_answers(cuda):
    sys_ = hb.SpectralSystem(1, 1, np.array([0, -1, -1.0]), np.array([2, 2, 2.0]),
                             np.array([-1, -1, 0.0]))
    assert np.allclose(hb.solve_system(sys_, np.array([1.0, 0, 0])), [0.75, 0.5, 0.25],
                       atol=1e-15)
    rng = np.random.default_rng(11)
    n = 50
    diag = 4.0 + rng.standard_normal(n) + 1j * rng.standard_normal(n)
    sub = rng.standard_normal(n) * 0.5 + 0.3j
    sup = rng.standard_normal(n) * 0.5 - 0.2j
    sub[0] = sup[-1] = 0
    rhs = rng.standard_normal(n) + 1j * rng.standard_normal(n)
    x = hb.solve_system(hb.SpectralSystem(1, 1, sub, diag, sup), rhs)
    A = np.diag(diag) + np.diag(sub[1:], -1) + np.diag(sup[:-1], 1)
    expect = np.linalg.solve(A, rhs)
    assert np.abs(x - expect).max() < 1e-12 * np.abs(expect).max()
    with pytest.raises(hb.SingularSystemError):
        hb.solve_system(hb.SpectralSystem(1, 1, np.array([0, 1.0]), np.array([0, 1.0]),
                                          np.array([1.0, 0])), np.array([1.0, 1.0]))


@pytest.mark.parametrize("key,scheme", [("2", hb.SchemeKind.SECOND_ORDER),
                                        ("4", hb.SchemeKind.FOURTH_ORDER),
                                        ("6", hb.SchemeKind.SIXTH_ORDER)])
def test_solve_all_vs_oracle_sweep(cuda, key, scheme):
    g = wl.unit_grid(31)
    prof = wl.profile_a(g)
    data = orc.dst_stack(np.random.default_rng(23).standard_normal(g.shape))
    dev = data.copy()
    hb.solve_all(dev, scheme, prof, g)
    ref = orc.thomas_sweep(data.copy(), oracle_table(key, prof, g), *orc.mode_cosines(31, 31))
    # FMA-contracted eigenvalues vs numpy's separate products: ~1e-14 noise
    assert rel_l2(dev, ref) < 1e-13


def test_solve_all_disjoint_ranges_bitwise(cuda):
    g = hb.make_grid(hb.Domain(0, PI, 0, PI, 0, PI), 5, 6, 4)
    prof = hb.constant_profile(3.0, g)
    data = np.random.default_rng(17).standard_normal(g.shape)
    full, split = data.copy(), data.copy()
    hb.solve_all(full, hb.SchemeKind.FOURTH_ORDER, prof, g)
    hb.solve_all(split, hb.SchemeKind.FOURTH_ORDER, prof, g, (0, 2))
    hb.solve_all(split, hb.SchemeKind.FOURTH_ORDER, prof, g, (2, 6))
    assert np.array_equal(full, split)


def test_resonance_reports_reference_mode(golden, cuda):
    k2, n, m = golden["resonance"]
    g = hb.make_grid(hb.Domain(0, PI, 0, PI, 0, PI), 5, 6, 4)
    with pytest.raises(hb.SingularSystemError) as err:
        hb.solve_discrete(hb.Field3D(np.ones(g.shape)), hb.BoundaryData.zero(),
                          hb.SchemeKind.SECOND_ORDER, hb.constant_profile(k2, g), g)
    assert (err.value.n, err.value.m) == (int(n), int(m))
    g1 = hb.make_grid(hb.Domain(0, PI, 0, PI, 0, PI), 1, 1, 1)
    with pytest.raises(hb.SingularSystemError) as err:
        hb.solve_discrete(hb.Field3D(np.ones(g1.shape)), hb.BoundaryData.zero(),
                          hb.SchemeKind.SECOND_ORDER, hb.constant_profile(6.0 / g1.h_z**2, g1), g1)
    assert (err.value.n, err.value.m) == (1, 1)


# ---------------------------------------------------------- full solves
def solve(F, scheme, prof, g, config=None):
    u, t = hb.solve_discrete(hb.Field3D(F), hb.BoundaryData.zero(), scheme, prof, g,
                             config or hb.SolverConfig())
    return u.values, t


def test_cfg1_uniform_rhs(golden, cuda):
    w = wl.workload(1)
    u, t = solve(wl.host_rhs(w), w.scheme, w.profile, w.grid)
    assert rel_l2(u, golden["cfg1_U"]) < PARITY
    assert t.total_s >= t.transform_s + t.tridiag_s


def test_cfg1_manufactured_through_rhs_operator(golden, cuda):
    w = wl.workload(1)
    F = hb.build_rhs(w.scheme, wl.manufactured_source(), w.profile, w.grid)
    g = w.grid
    x = g.x_nodes(closed=True)[None, None, :]
    y = g.y_nodes(closed=True)[None, :, None]
    z = g.z_nodes(closed=True)[:, None, None]
    f_closed = np.broadcast_to(wl.manufactured_source().f(x, y, z), (33, 33, 33))
    assert np.array_equal(F.values, orc.rhs_fourth(f_closed, g.h_z))  # K1 bit-exact
    assert np.abs(F.values - golden["cfg1A_F"]).max() <= 1e-15 * np.abs(golden["cfg1A_F"]).max()
    u, _ = solve(F.values, w.scheme, w.profile, w.grid)
    assert rel_l2(u, golden["cfg1A_U"]) < PARITY


def test_cfg2_full_size_against_reference_summaries(golden, cuda):
    w = wl.workload(2)
    u, _ = solve(wl.host_rhs(w), w.scheme, w.profile, w.grid)
    assert rel_l2(u[63], golden["cfg2_U_plane63"]) < PARITY
    assert rel_l2(u[::8, ::8, ::8], golden["cfg2_U_sub8"]) < PARITY
    nrm, mx, sm = golden["cfg2_U_norms"]
    assert abs(np.linalg.norm(u) - nrm) < PARITY * nrm


def test_cfg2_sixth_order_rhs_and_solve(golden, cuda):
    g = wl.unit_grid(31)
    prof = wl.profile_a(g)
    F = hb.build_rhs(hb.SchemeKind.SIXTH_ORDER, wl.manufactured_source(), prof, g)
    assert np.abs(F.values - golden["cfg2A_n31_F"]).max() <= 1e-14 * np.abs(F.values).max()
    u, _ = solve(F.values, hb.SchemeKind.SIXTH_ORDER, prof, g)
    assert rel_l2(u, golden["cfg2A_n31_U"]) < PARITY


def test_convergence_orders(golden, cuda):
    """4th/6th-order rates on the manufactured solution (31^3 / 63^3 / 127^3)."""
    rows = golden["convergence"]
    src = wl.manufactured_source()
    for key, scheme in (("4", hb.SchemeKind.FOURTH_ORDER), ("6", hb.SchemeKind.SIXTH_ORDER)):
        errs = []
        for n in (31, 63, 127):
            g = wl.unit_grid(n)
            prof = wl.profile_a(g)
            F = hb.build_rhs(scheme, src, prof, g)
            u, _ = solve(F.values, scheme, prof, g)
            x = g.x_nodes()[None, None, :]
            y = g.y_nodes()[None, :, None]
            z = g.z_nodes()[:, None, None]
            exact = wl.manufactured_u(x, y, z)
            errs.append(np.abs(u - exact).max())
            ref = rows[(rows[:, 0] == float(key)) & (rows[:, 1] == n)][0]
            assert errs[-1] == pytest.approx(ref[2], rel=1e-6)
        orders = [math.log(errs[i] / errs[i + 1]) / math.log(2 * (n1 + 1) / (2 * (n0 + 1)))
                  for i, (n0, n1) in enumerate(((31, 63), (63, 127)))]
        lo, hi = (3.7, 4.3) if key == "4" else (5.6, 6.4)
        assert all(lo <= o <= hi for o in orders), orders


def test_cd4_and_general_table(golden, cuda):
    g = wl.unit_grid(15)
    u, _ = solve(golden["cd4_n15_F"], hb.SchemeKind.CONVECTION_DIFFUSION_4,
                 hb.constant_profile(0.0, g, gamma=-1.5), g)
    assert rel_l2(u, golden["cd4_n15_U"]) < PARITY
    T = golden["gen_n15_table"]
    u, _ = solve(golden["gen_n15_F"], hb.StencilTable(*T), hb.constant_profile(0.0, g), g)
    assert rel_l2(u, golden["gen_n15_U"]) < PARITY


def test_anisotropic_dense_path(golden, cuda):
    g = hb.make_grid(hb.Domain(0, PI, 0, 2.0, 0, 1.0), 9, 7, 6)
    u, _ = solve(golden["aniso_F"], hb.SchemeKind.FOURTH_ORDER, hb.constant_profile(2.0, g), g)
    assert rel_l2(u, golden["aniso_U"]) < PARITY


@pytest.mark.parametrize("cfg,planes", [(1, 31), (2, 127), (3, 511), (4, 64)])
def test_large_configs_vs_oracle(cuda, cfg, planes):
    """cfg1, cfg2 and cfg3 at full size with their seeded RHS; cfg4 on a 64-plane
    slab of the full 1023^2 planes here (its full 1023^3 is in
    test_gpu_parity_r2.py)."""
    w = wl.workload(cfg)
    # a slab keeps the full grid's step h = 1/(n+1): z-extent (planes + 1) h
    g = w.grid if planes == w.n else hb.make_grid(
        hb.Domain(0, 1, 0, 1, 0, (planes + 1) / (w.n + 1)), w.n, w.n, planes)
    prof = w.profile if planes == w.n else hb.CoefficientProfile(
        k2=np.zeros(planes + 2, complex), k2_z=np.zeros(planes + 2, complex),
        k2_zz=np.zeros(planes + 2, complex), gamma=w.profile.gamma)
    F = wl.host_rhs(w, planes=planes)
    u, _ = solve(F, w.scheme, prof, g)
    key = w.scheme.value
    ref = orc.solve(F, oracle_table(key, prof, g), *orc.mode_cosines(g.n_x, g.n_y), workers=8)
    err = rel_l2(u, ref)
    print(f"cfg{cfg} rel L2 vs oracle: {err:.3e}")
    assert err < TOL


def test_partitioned_and_shared_modes_bitwise(cuda):
    g = hb.make_grid(hb.Domain(0, PI, 0, 2.0, 0, 1.0), 15, 31, 12)
    prof = hb.constant_profile(5.0, g)
    F = np.random.default_rng(59).standard_normal(g.shape)
    # staged = the reference's stage order (x-then-y transform both ways); the
    # Partitioned mode runs the multi-GPU per-rank stages (mode-row blocks, the
    # one-call kernels), bit-identical to the one-call solve
    ref, _ = solve(F, hb.SchemeKind.FOURTH_ORDER, prof, g,
                   hb.SolverConfig(mode=hb.Device(staged=True)))
    one, _ = solve(F, hb.SchemeKind.FOURTH_ORDER, prof, g)
    for cfg in (hb.SolverConfig(), hb.SolverConfig(mode=hb.SharedWorkers(2)),
                hb.SolverConfig(mode=hb.Partitioned(1)), hb.SolverConfig(mode=hb.Partitioned(3)),
                hb.SolverConfig(mode=hb.Partitioned(4, 2)), hb.SolverConfig(mode=hb.Device())):
        u, t = solve(F, hb.SchemeKind.FOURTH_ORDER, prof, g, cfg)
        assert np.abs(u - ref).max() <= 1e-13 * np.abs(ref).max(), cfg
        if isinstance(cfg.mode, hb.Partitioned):
            assert np.array_equal(u, one)
            assert t.exchange_s > 0.0


def test_repeat_runs_bitwise_and_input_untouched(cuda):
    w = wl.workload(1)
    F = wl.host_rhs(w)
    keep = F.copy()
    u1, _ = solve(F, w.scheme, w.profile, w.grid)
    u2, _ = solve(F, w.scheme, w.profile, w.grid)
    assert np.array_equal(u1, u2) and np.array_equal(F, keep)


def test_linearity_and_complex_rhs(cuda):
    w = wl.workload(1)
    rng = np.random.default_rng(29)
    f1, f2 = rng.standard_normal(w.grid.shape), rng.standard_normal(w.grid.shape)
    u1, _ = solve(f1, w.scheme, w.profile, w.grid)
    u2, _ = solve(f2, w.scheme, w.profile, w.grid)
    uc, _ = solve(f1 + 1j * f2, w.scheme, w.profile, w.grid)
    assert np.abs(uc.real - u1).max() <= 1e-15 * np.abs(u1).max() * 10
    assert np.abs(uc.imag - u2).max() <= 1e-15 * np.abs(u2).max() * 10
    ul, _ = solve(0.7 * f1 - 1.3 * f2, w.scheme, w.profile, w.grid)
    assert np.abs(ul - (0.7 * u1 - 1.3 * u2)).max() < 1e-12 * np.abs(ul).max()


def test_zero_rhs_and_device_tensors(cuda):
    import torch
    w = wl.workload(1)
    u, _ = solve(np.zeros(w.grid.shape), w.scheme, w.profile, w.grid)
    assert not np.any(u)
    F = wl.host_rhs(w)
    t = torch.from_numpy(F).to(cuda)
    ut, _ = hb.solve_discrete(hb.Field3D(t), hb.BoundaryData.zero(), w.scheme, w.profile, w.grid)
    assert ut.values.is_cuda
    u, _ = solve(F, w.scheme, w.profile, w.grid)
    assert np.array_equal(ut.values.cpu().numpy(), u)


# ---------------------------------------------------- 27-point operator
def test_apply_fold_residual_vs_oracle(cuda):
    g = hb.make_grid(hb.Domain(0, PI, 0, 2.0, 0, 1.0), 9, 7, 6)
    prof = hb.constant_profile(2.0, g)
    rng = np.random.default_rng(43)
    box = rng.standard_normal((8, 9, 11))
    T = oracle_table("4", prof, g)
    bnd = hb.BoundaryData.from_array(box)
    ext = bnd.closed_box(g).real
    rhs = rng.standard_normal(g.shape)
    folded = hb.fold_dirichlet(hb.Field3D(rhs), bnd, hb.SchemeKind.FOURTH_ORDER, prof, g)
    assert np.array_equal(folded.values, rhs - orc.accumulate27(ext, T))  # bit-exact
    u = rng.standard_normal(g.shape)
    au = hb.apply_stencil(hb.Field3D(u), hb.BoundaryData.zero(), hb.SchemeKind.FOURTH_ORDER,
                          prof, g)
    e2 = np.zeros((8, 9, 11))
    e2[1:-1, 1:-1, 1:-1] = u
    assert np.array_equal(au.values, orc.accumulate27(e2, T))
    r = hb.residual_l2(hb.Field3D(u), hb.Field3D(rhs), hb.SchemeKind.FOURTH_ORDER, prof, g)
    assert r == pytest.approx(orc.residual_l2(u, rhs, T), rel=1e-12)


def test_nonzero_boundary_solve_vs_dense(cuda):
    """solve with folded Dirichlet data reproduces the dense 27-diagonal LU (test_solver.py:160-171)."""
    g = hb.make_grid(hb.Domain(0, PI, 0, PI, 0, PI), 6, 6, 6)
    prof = hb.constant_profile(2.0, g)
    rng = np.random.default_rng(41)
    F = rng.standard_normal(g.shape)
    box = rng.standard_normal((8, 8, 8))
    u, _ = hb.solve_discrete(hb.Field3D(F), hb.BoundaryData.from_array(box),
                             hb.SchemeKind.FOURTH_ORDER, prof, g)
    T = oracle_table("4", prof, g)
    n = 216
    A = np.zeros((n, n))
    for c in range(n):
        e = np.zeros(n)
        e[c] = 1.0
        ext = np.zeros((8, 8, 8))
        ext[1:-1, 1:-1, 1:-1] = e.reshape(6, 6, 6)
        A[:, c] = orc.accumulate27(ext, T).ravel()
    ext = np.array(box)
    ext[1:-1, 1:-1, 1:-1] = 0
    rhs = F - orc.accumulate27(ext, T)
    expect = np.linalg.solve(A, rhs.ravel()).reshape(6, 6, 6)
    assert np.abs(u.values - expect).max() < 1e-12 * np.abs(expect).max()


def test_cfg3_residual_at_full_size(cuda):
    """Size-independent property at 511^3: ||A U - F|| / ||F|| at roundoff."""
    import torch
    w = wl.workload(3)
    F = wl.device_rhs(w, cuda)
    u, _ = hb.solve_discrete(hb.Field3D(F), hb.BoundaryData.zero(), w.scheme, w.profile, w.grid)
    r = hb.residual_l2(u, hb.Field3D(F), w.scheme, w.profile, w.grid)
    # roundoff floor eps * ||A|| ||U|| / ||F||; ||U|| >> ||F|| near resonance
    assert r / float(torch.linalg.norm(F)) < 1e-11


# ------------------------------------------------- engine tuning variants
@pytest.fixture
def tuning():
    lib = hb._native.load_library()
    yield lib.hfb_set_tuning
    lib.hfb_set_tuning(0, 16)
    lib.hfb_set_tuning(1, 0)
    lib.hfb_set_tuning(2, 2)
    lib.hfb_set_tuning(3, 0)
    lib.hfb_set_tuning(4, 1)
    lib.hfb_set_tuning(5, 0)
    lib.hfb_set_tuning(6, 0)
    lib.hfb_set_tuning(9, 0)
    lib.hfb_set_tuning(10, 0)
    lib.hfb_set_tuning(13, 1)
    lib.hfb_set_tuning(14, 1)
    lib.hfb_set_tuning(29, 2)


@pytest.mark.parametrize("knobs", [((0, 32),), ((0, 32), (1, 2)), ((0, 32), (1, 1)), ((1, 1),),
                                   ((2, 0),), ((2, 3),), ((3, 1),), ((3, 3),), ((4, 0),),
                                   ((0, 32), (4, 0)), ((5, 0),), ((0, 32), (5, 1)),
                                   ((6, 1),), ((6, 1), (7, 1), (8, 2)), ((9, 1),),
                                   ((14, 0),), ((14, 0), (13, 0)), ((1, 1), (14, 1)),
                                   ((29, 0),), ((29, 1),),
                                   ((10, 2),)])
def test_tuning_variants_match_oracle(cuda, tuning, knobs):
    """Performance knobs change the FFT factorisation or the CTA shape, never
    the result beyond rounding: transforms (row, transposed-store and
    tensor-box column paths) and one-call solves against the oracle."""
    for k, v in knobs:
        tuning(k, v)
    rng = np.random.default_rng(7)
    for nx, ny, nz in [(255, 255, 3), (63, 127, 5), (1023, 63, 2), (31, 4095, 1)]:
        data = rng.standard_normal((nz, ny, nx))
        f = hb.Field3D(data.copy())
        hb.transform_stack(hb.make_plan(nx, ny), f)
        ref = orc.dst_stack(data, workers=4)
        assert np.abs(f.values - ref).max() < 1e-13 * np.abs(ref).max()
    w = wl.workload(1)
    F = wl.host_rhs(w)
    u, _ = solve(F, w.scheme, w.profile, w.grid)
    ref = orc.solve(F, oracle_table(w.scheme.value, w.profile, w.grid),
                    *orc.mode_cosines(w.grid.n_x, w.grid.n_y))
    assert rel_l2(u, ref) < PARITY


@pytest.mark.parametrize("shape", [(31, 31, 31), (127, 63, 33), (255, 15, 9), (2047, 15, 4),
                                   (2047, 31, 3)])
def test_lean_workspace_bitwise_equal_fast(cuda, shape):
    """The lean one-volume workspace (transposing x-pass stores) and the fast
    two-volume one (row/tensor-box passes) run the same per-line arithmetic."""
    import torch
    nx, ny, nz = shape
    g = hb.make_grid(hb.Domain(0, 1, 0, 1, 0, 1), nx, ny, nz)
    prof = hb.constant_profile(3.0, g)
    F = torch.from_numpy(np.random.default_rng(nx).standard_normal((nz, ny, nx))).cuda()
    plan = hb._native.get_plan(nx, ny, nz, F.device)
    hb.tridiag.device_coefficients(plan, hb.SchemeKind.FOURTH_ORDER, prof, g)
    outs = []
    for lean in (0, 1):
        plan.set_workspace_mode(lean)
        U = torch.empty_like(F)
        work = plan.workspace(0)
        hb._native.check(plan.lib.hfb_solve(plan.handle, hb._native.ptr(F), hb._native.ptr(U),
                                            hb._native.ptr(work), plan.stream()), "solve")
        plan.fetch_status()
        outs.append(U.cpu().numpy())
    plan.set_workspace_mode(0)
    assert np.array_equal(outs[0], outs[1])
    ref = orc.solve(F.cpu().numpy(), oracle_table("4", prof, g), *orc.mode_cosines(nx, ny))
    # the 2047-wide shapes are very anisotropic (h_z / h_x ~ 400): conditioning
    # amplifies rounding to ~1.5e-11, inside the north star's 1e-10
    assert rel_l2(outs[0], ref) < (PARITY if nx < 2047 else TOL)


# ------------------------------------------------------ complex k(z) (f1)
ZSCHEME = {"2": hb.SchemeKind.SECOND_ORDER, "4": hb.SchemeKind.FOURTH_ORDER,
           "6": hb.SchemeKind.SIXTH_ORDER}
ZCASES = [("z4", "4"), ("z6", "6"), ("zb", "2"), ("zd2", "2"), ("zd4", "4"), ("zd6", "6")]


def z_inputs(golden, name):
    from _zcases import z_case, z_grid
    dom, (nx, ny, nz) = z_grid(name)
    g = hb.make_grid(hb.Domain(*dom), nx, ny, nz)
    k2 = golden[f"{name}_k2"]
    prof = hb.CoefficientProfile(k2=k2, k2_z=golden.get(f"{name}_k2z", np.zeros_like(k2)),
                                 k2_zz=golden.get(f"{name}_k2zz", np.zeros_like(k2)))
    key = dict(ZCASES)[name]
    F, B, T, cs = z_case(golden, name, key)
    bnd = hb.BoundaryData.zero() if B is None else hb.BoundaryData.from_array(B)
    return g, prof, ZSCHEME[key], F, bnd


@pytest.mark.parametrize("name", [c for c, _ in ZCASES])
def test_complex_k_solves_vs_reference(golden, cuda, name):
    """Complex k(z) through solve_discrete: complex tables, complex z-solve
    (fused power-of-two path and the generic dense-DST path), complex fold."""
    g, prof, scheme, F, bnd = z_inputs(golden, name)
    u, _ = hb.solve_discrete(hb.Field3D(F), bnd, scheme, prof, g)
    assert np.iscomplexobj(u.values)
    assert rel_l2(u.values, golden[f"{name}_U"]) < PARITY


@pytest.mark.parametrize("mode", ["staged", "partitioned"])
def test_complex_k_modes_agree(golden, cuda, mode):
    g, prof, scheme, F, bnd = z_inputs(golden, "z4")
    cfg = hb.SolverConfig(mode=hb.Device(staged=True) if mode == "staged"
                          else hb.Partitioned(parts=3))
    u, _ = hb.solve_discrete(hb.Field3D(F), bnd, scheme, prof, g, cfg)
    assert rel_l2(u.values, golden["z4_U"]) < PARITY
    if mode == "partitioned":
        us, _ = hb.solve_discrete(hb.Field3D(F), bnd, scheme, prof, g,
                                  hb.SolverConfig(mode=hb.Device(staged=True)))
        assert np.array_equal(u.values, us.values)


def test_complex_k_residual_fold_and_guards(golden, cuda):
    g, prof, scheme, F, bnd = z_inputs(golden, "zb")
    Ff = hb.fold_dirichlet(hb.Field3D(F), bnd, scheme, prof, g)
    u, _ = hb.solve_discrete(hb.Field3D(F), bnd, scheme, prof, g)
    res = hb.residual_l2(u, Ff, scheme, prof, g)
    assert res < 1e-11 * np.linalg.norm(Ff.values)
    # A u (with the boundary) reproduces the unfolded rhs
    Au = hb.apply_stencil(u, bnd, scheme, prof, g)
    assert rel_l2(Au.values, F) < 1e-12
    # the real entry points refuse a complex table
    plan = hb._native.get_plan(g.n_x, g.n_y, g.n_z, hb._native._torch().device("cuda", 0))
    hb.tridiag.device_coefficients(plan, scheme, prof, g)
    assert plan.complex_coef
    import torch
    t = torch.zeros(g.shape, dtype=torch.float64, device="cuda")
    work = plan.workspace(0)
    assert plan.lib.hfb_solve(plan.handle, hb._native.ptr(t), hb._native.ptr(t),
                              hb._native.ptr(work), plan.stream()) == 1


@pytest.mark.parametrize("n", [255, 511])
def test_complex_k_large_vs_oracle(cuda, n):
    """Fused complex z-solve at 255^3 / 511^3 (64-plane slab) against the oracle."""
    planes = 64
    g = hb.make_grid(hb.Domain(0, 1, 0, 1, 0, (planes + 1) / (n + 1)), n, n, planes)
    z = np.linspace(0, (planes + 1) / (n + 1), planes + 2)
    prof = hb.CoefficientProfile(k2=(200.0 + 50.0j) * (1 + 0.3 * np.sin(6 * z)),
                                 k2_z=np.zeros(planes + 2, complex),
                                 k2_zz=np.zeros(planes + 2, complex))
    rng = np.random.default_rng(n)
    F = rng.standard_normal((planes, n, n)) + 1j * rng.standard_normal((planes, n, n))
    u, _ = hb.solve_discrete(hb.Field3D(F), hb.BoundaryData.zero(), hb.SchemeKind.FOURTH_ORDER,
                             prof, g)
    T = orc.weight_table("4", prof.k2, prof.k2_z, prof.k2_zz, 0.0, (g.h_x, g.h_y, g.h_z), planes)
    ref = orc.solve(F, T, *orc.mode_cosines(n, n), workers=8)
    assert rel_l2(u.values, ref) < TOL


def test_pipelined_host_solves_match_blocking(cuda):
    """hfb_solve_host_async: several right-hand sides in flight (three device
    volumes in rotation, copy streams) give exactly the blocking hfb_solve_host
    results."""
    import ctypes
    import torch
    w = wl.workload(1)
    n = w.n
    plan = hb._native.get_plan(n, n, n, torch.device("cuda", 0))
    hb.tridiag.device_coefficients(plan, w.scheme, w.profile, w.grid)
    work = plan.workspace(0)
    st = plan.stream()
    rng = np.random.default_rng(5)
    ins = [torch.from_numpy(rng.standard_normal((n, n, n))).pin_memory() for _ in range(5)]
    outs = [torch.empty_like(x).pin_memory() for x in ins]
    ref = [torch.empty_like(x).pin_memory() for x in ins]
    status = hb._native.HfbStatus()
    lib, ptr = plan.lib, hb._native.ptr
    for x, r in zip(ins, ref):
        hb._native.check(lib.hfb_solve_host(plan.handle, ptr(x), ptr(r), ptr(work), st,
                                            ctypes.byref(status)), "host")
    for x, o in zip(ins, outs):
        hb._native.check(lib.hfb_solve_host_async(plan.handle, ptr(x), ptr(o), ptr(work), st),
                         "async")
    hb._native.check(lib.hfb_host_sync(plan.handle, ctypes.byref(status)), "sync")
    for o, r in zip(outs, ref):
        assert torch.equal(o, r)
    T = oracle_table(w.scheme.value, w.profile, w.grid)
    assert rel_l2(outs[3].numpy(), orc.solve(ins[3].numpy(), T, *orc.mode_cosines(n, n))) < 1e-12


@pytest.mark.parametrize("shape", [(63, 63, 40), (255, 127, 17), (127, 255, 9)])
def test_fused_forward_sweep_bitwise(cuda, tuning, shape):
    """The y-pass with the forward Thomas sweep fused in (YF) + backward-only
    z-solve reproduces the unfused pipeline bit for bit (same arithmetic, same
    checkpoints), including a pivot latch on the same mode."""
    import torch
    nx, ny, nz = shape
    g = hb.make_grid(hb.Domain(0, 1, 0, 1, 0, 1), nx, ny, nz)
    prof = hb.constant_profile(5.0, g)
    F = torch.from_numpy(np.random.default_rng(nz).standard_normal((nz, ny, nx))).cuda()
    plan = hb._native.get_plan(nx, ny, nz, F.device)
    hb.tridiag.device_coefficients(plan, hb.SchemeKind.FOURTH_ORDER, prof, g)
    outs = []
    for fuse in (1, 0):
        tuning(5, fuse)
        U = torch.empty_like(F)
        work = plan.workspace(0)
        hb._native.check(plan.lib.hfb_solve(plan.handle, hb._native.ptr(F), hb._native.ptr(U),
                                            hb._native.ptr(work), plan.stream()), "solve")
        plan.fetch_status()
        outs.append(U.cpu().numpy())
    assert np.array_equal(outs[0], outs[1])


# ------------------------------------------------- multi-GPU path (row e)
def _emulated_partitioned(F, scheme, prof, g, parts):
    """Drive distributed.solve_partitioned's per-rank stages for `parts` ranks
    in one process, the all-to-alls emulated by slicing/concatenating the
    send buffers (no collective, no kernel waits on another)."""
    import torch
    from paper_1912_03565_b200 import distributed as hd
    ex = hb.make_exchange_plan(g, parts)
    sends, modes = [], []
    for r, (z0, z1) in enumerate(ex.partition.z_ranges):
        s, m = hd.forward_to_blocks(F[z0:z1].contiguous(), g, ex, r)
        sends.append(s)
        modes.append(m)
    splits = [hd.mode_split_sizes(ex, r)[0] for r in range(parts)]  # send splits per rank

    def chunk(buf, sizes, q):
        off = sum(sizes[:q])
        return buf[off:off + sizes[q]]

    recvs = [torch.cat([chunk(sends[p], splits[p], q) for p in range(parts)])
             for q in range(parts)]
    for r in range(parts):
        hd.solve_received(recvs[r], scheme, prof, g, ex, r)
        assert tuple(hd.mode_split_sizes(ex, r)[1]) == tuple(
            splits[p][r] for p in range(parts))
    rsplits = [hd.mode_split_sizes(ex, r)[1] for r in range(parts)]
    backs = [torch.cat([chunk(recvs[q], rsplits[q], p) for q in range(parts)])
             for p in range(parts)]
    outs = [hd.blocks_to_solution(backs[r], modes[r], g, ex, r) for r in range(parts)]
    return torch.cat(outs)


@pytest.mark.parametrize("parts,shape", [(2, (63, 63, 63)), (3, (127, 63, 50)),
                                         (8, (255, 255, 40)), (5, (31, 127, 23))])
def test_partitioned_mode_space_stages_bitwise(cuda, parts, shape):
    """The multi-GPU per-rank pipeline (mode-row exchange, TMA z-solve on y-slabs)
    reproduces the single-GPU one-call solve bit for bit."""
    import torch
    nx, ny, nz = shape
    g = hb.make_grid(hb.Domain(0, 1, 0, 1, 0, 1), nx, ny, nz)
    prof = hb.constant_profile(-20.0, g)
    F = torch.from_numpy(np.random.default_rng(parts).standard_normal((nz, ny, nx))).cuda()
    U = _emulated_partitioned(F, hb.SchemeKind.FOURTH_ORDER, prof, g, parts)
    plan = hb._native.get_plan(nx, ny, nz, F.device)
    hb.tridiag.device_coefficients(plan, hb.SchemeKind.FOURTH_ORDER, prof, g)
    ref = torch.empty_like(F)
    work = plan.workspace(0)
    hb._native.check(plan.lib.hfb_solve(plan.handle, hb._native.ptr(F), hb._native.ptr(ref),
                                        hb._native.ptr(work), plan.stream()), "solve")
    plan.fetch_status()
    assert torch.equal(U, ref)


def _nccl_worker(rank, world, port, q):
    import os
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("nccl", rank=rank, world_size=world)
    try:
        from paper_1912_03565_b200 import distributed as hd
        torch.cuda.set_device(0)
        g = hb.make_grid(hb.Domain(0, 1, 0, 1, 0, 1), 63, 63, 63)
        prof = hb.constant_profile(-20.0, g)
        F = torch.from_numpy(np.random.default_rng(1).standard_normal((63, 63, 63))).cuda()
        U = hd.solve_partitioned(F, hb.SchemeKind.FOURTH_ORDER, prof, g)
        u, _ = hb.solve_discrete(hb.Field3D(F.cpu().numpy()), hb.BoundaryData.zero(),
                                 hb.SchemeKind.FOURTH_ORDER, prof, g)
        q.put(float(np.abs(U.cpu().numpy() - u.values).max()))
    finally:
        dist.destroy_process_group()


def _a2a_worker(rank, world, port, q, shape):
    """One rank of solve_partitioned in its own process (all ranks on GPU 0): a gloo
    group, and all_to_all_single staged through host tensors (gloo has no CUDA
    all-to-all; NCCL refuses two ranks on one GPU) — everything else is the code
    path of a real multi-GPU run: plan_partition, chunked block transforms,
    chunk-ordered y-slab z-solve, split sizes."""
    import os
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1912_03565_b200 import distributed as hd
        torch.cuda.set_device(0)
        nx, ny, nz = shape
        g = hb.make_grid(hb.Domain(0, 1, 0, 1, 0, 1), nx, ny, nz)
        prof = hb.constant_profile(-20.0, g)
        F = torch.from_numpy(np.random.default_rng(3).standard_normal((nz, ny, nx))).cuda()
        z0, z1 = hb.plan_partition(nz, world)[rank]
        real_a2a = dist.all_to_all_single

        class Done:
            def wait(self):
                return True

        def staged(out, inp, output_split_sizes=None, input_split_sizes=None, group=None,
                   async_op=False):
            torch.cuda.synchronize()
            host_out = torch.empty(out.numel(), dtype=out.dtype)
            real_a2a(host_out, inp.cpu(), output_split_sizes, input_split_sizes, group=group)
            out.copy_(host_out)
            torch.cuda.synchronize()
            return Done() if async_op else None

        dist.all_to_all_single = staged
        fused = hd.fused_blocks(hb.make_exchange_plan(g, world))
        outs = []
        for _ in range(2):  # twice: buffers and plans reused
            U = hd.solve_partitioned(F[z0:z1].contiguous(), hb.SchemeKind.FOURTH_ORDER, prof, g,
                                     check=False)
            torch.cuda.synchronize()
            outs.append(U.cpu().numpy())
        hb._native.get_plan(nx, ny, nz, torch.device("cuda", 0)).fetch_status()
        assert np.array_equal(outs[0], outs[1])
        q.put((rank, outs[0], fused))
        dist.barrier()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,shape", [(2, (127, 127, 24)), (4, (127, 255, 19)),
                                         (3, (127, 127, 17))])
def test_solve_partitioned_processes_one_gpu(cuda, world, shape):
    """solve_partitioned with one PROCESS per rank (2 and 4 ranks: the fused block
    transforms; 3 ranks: the ragged geometry with the pack kernels), the exchange
    staged through the host: the concatenated slabs equal the one-call solve bit
    for bit."""
    import socket
    import torch
    import torch.multiprocessing as mp
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_a2a_worker, args=(r, world, port, q, shape))
             for r in range(world)]
    for p in procs:
        p.start()
    res = sorted((q.get(timeout=300) for _ in range(world)), key=lambda x: x[0])
    for p in procs:
        p.join(120)
    assert all(p.exitcode == 0 for p in procs)
    assert all(r[2] == (world != 3) for r in res)
    U = np.concatenate([r[1] for r in res])
    nx, ny, nz = shape
    g = hb.make_grid(hb.Domain(0, 1, 0, 1, 0, 1), nx, ny, nz)
    F = torch.from_numpy(np.random.default_rng(3).standard_normal((nz, ny, nx))).cuda()
    ref = _one_call(F, hb.SchemeKind.FOURTH_ORDER, hb.constant_profile(-20.0, g), g)
    assert np.array_equal(U, ref.cpu().numpy())


def test_solve_partitioned_nccl_single_rank(cuda):
    """solve_partitioned through a real NCCL communicator (one rank: this box has
    one GPU) against the one-call solve."""
    import socket
    import torch.multiprocessing as mp
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    p = ctx.Process(target=_nccl_worker, args=(0, 1, port, q))
    p.start()
    p.join(300)
    assert p.exitcode == 0
    assert q.get(timeout=10) == 0.0


def test_complex_rhs_sixth_and_convdiff_vs_reference(golden, cuda):
    """build_rhs with a complex 6th-order profile and with a complex convection
    gamma (row f3 with complex coefficients), then the complex solve."""
    src = wl.manufactured_source()
    g31 = wl.unit_grid(31)
    prof6 = hb.CoefficientProfile(k2=golden["z6_k2"], k2_z=golden["z6_k2z"],
                                  k2_zz=golden["z6_k2zz"])
    F6 = hb.build_rhs(hb.SchemeKind.SIXTH_ORDER, src, prof6, g31)
    assert np.iscomplexobj(F6.values)
    assert np.abs(F6.values - golden["zr6_F"]).max() <= 1e-15 * np.abs(golden["zr6_F"]).max()
    u6, _ = hb.solve_discrete(F6, hb.BoundaryData.zero(), hb.SchemeKind.SIXTH_ORDER, prof6, g31)
    assert rel_l2(u6.values, golden["zr6_U"]) < PARITY
    g15 = wl.unit_grid(15)
    pcd = hb.constant_profile(0.0, g15, gamma=-1.5 + 0.5j)
    Fcd = hb.build_rhs(hb.SchemeKind.CONVECTION_DIFFUSION_4, src, pcd, g15)
    assert np.abs(Fcd.values - golden["zrcd_F"]).max() <= 1e-15 * np.abs(golden["zrcd_F"]).max()
    ucd, _ = hb.solve_discrete(Fcd, hb.BoundaryData.zero(), hb.SchemeKind.CONVECTION_DIFFUSION_4,
                               pcd, g15)
    assert rel_l2(ucd.values, golden["zrcd_U"]) < PARITY


@pytest.mark.parametrize("shape", [(15, 15, 1), (15, 31, 2), (31, 15, 9), (4095, 15, 3),
                                   (15, 4095, 3), (2047, 63, 4), (63, 2047, 17), (127, 127, 65)])
@pytest.mark.parametrize("lean", [0, 1])
def test_one_call_edge_shapes_vs_oracle(cuda, shape, lean):
    """One-call solve (fast and lean layouts) at the edges of the engine: the
    smallest power-of-two lines (M = 16), M = 4096 (E = 32), M = 2048 (wide CTAs),
    1 and 2 levels, partial checkpoint chunks."""
    import torch
    nx, ny, nz = shape
    g = hb.make_grid(hb.Domain(0, 1, 0, 2, 0, 0.5), nx, ny, nz)
    prof = hb.constant_profile(7.0, g)
    F = np.random.default_rng(nx * 7 + ny + nz).standard_normal((nz, ny, nx))
    plan = hb._native.get_plan(nx, ny, nz, torch.device("cuda", 0))
    plan.set_workspace_mode(lean)
    try:
        u, _ = hb.solve_discrete(hb.Field3D(F), hb.BoundaryData.zero(), hb.SchemeKind.FOURTH_ORDER,
                                 prof, g)
    finally:
        plan.set_workspace_mode(0)
    ref = orc.solve(F, oracle_table("4", prof, g), *orc.mode_cosines(nx, ny), workers=4)
    assert rel_l2(u.values, ref) < PARITY


def _emulated_partitioned_chunked(F, scheme, prof, g, parts, chunks):
    """solve_partitioned's chunked schedule (per-chunk all-to-alls, the z-solve
    through the level table), every rank in one process, collectives emulated."""
    import torch
    from paper_1912_03565_b200 import distributed as hd
    ex = hb.make_exchange_plan(g, parts)
    ranges, level_plane = hd.chunk_layout(ex, chunks)
    zr = ex.partition.z_ranges
    slabs = [F[z0:z1].contiguous() for z0, z1 in zr]
    modes = []
    for r, (z0, z1) in enumerate(zr):
        tp = hb._native.get_plan(g.n_x, g.n_y, z1 - z0, F.device)
        ldm = int(tp.lib.hfb_modes_ld(tp.handle))
        modes.append(torch.empty((z1 - z0) * g.n_x * ldm, dtype=torch.float64, device=F.device))
    sends = [[hd.forward_chunk(slabs[r], modes[r], g, ex, r, *ranges[r][c]) for c in range(chunks)]
             for r in range(parts)]

    def piece(buf, sizes, q):
        off = sum(sizes[:q])
        return buf[off:off + sizes[q]]

    recvs = []
    for q in range(parts):
        blocks = []
        for c in range(chunks):
            for p in range(parts):
                blocks.append(piece(sends[p][c], hd.chunk_split_sizes(ex, ranges, p, c)[0], q))
        recvs.append(torch.cat(blocks))
    for q in range(parts):
        hd.solve_received_chunked(recvs[q], level_plane, scheme, prof, g, ex, q)
    outs = [torch.empty_like(s) for s in slabs]
    for p in range(parts):
        for c in range(chunks):
            # rank p's chunk c comes back from every q: the piece of q's y-slab
            # chunk-c region that p sent
            parts_back = []
            for q in range(parts):
                off_c = sum(sum(hd.chunk_split_sizes(ex, ranges, q, cc)[1]) for cc in range(c))
                rq = hd.chunk_split_sizes(ex, ranges, q, c)[1]
                region = recvs[q][off_c:off_c + sum(rq)]
                parts_back.append(piece(region, rq, p))
            hd.inverse_chunk(torch.cat(parts_back), modes[p], outs[p], g, ex, *ranges[p][c])
    return torch.cat(outs)


@pytest.mark.parametrize("parts,chunks,shape", [(2, 4, (63, 63, 63)), (3, 3, (127, 63, 50)),
                                                (8, 4, (255, 255, 40)), (4, 2, (31, 127, 9))])
def test_partitioned_chunked_stages_bitwise(cuda, parts, chunks, shape):
    """The overlapped (chunked) multi-GPU schedule reproduces the one-call solve
    bit for bit: chunk-ordered y-slabs, level table in the z-solve."""
    import torch
    nx, ny, nz = shape
    g = hb.make_grid(hb.Domain(0, 1, 0, 1, 0, 1), nx, ny, nz)
    prof = hb.constant_profile(-20.0, g)
    F = torch.from_numpy(np.random.default_rng(parts * 10 + chunks).standard_normal(
        (nz, ny, nx))).cuda()
    U = _emulated_partitioned_chunked(F, hb.SchemeKind.FOURTH_ORDER, prof, g, parts, chunks)
    plan = hb._native.get_plan(nx, ny, nz, F.device)
    hb.tridiag.device_coefficients(plan, hb.SchemeKind.FOURTH_ORDER, prof, g)
    ref = torch.empty_like(F)
    work = plan.workspace(0)
    hb._native.check(plan.lib.hfb_solve(plan.handle, hb._native.ptr(F), hb._native.ptr(ref),
                                        hb._native.ptr(work), plan.stream()), "solve")
    plan.fetch_status()
    assert torch.equal(U, ref)


def test_capi_argument_validation(cuda):
    """Error codes of the C-ABI entry points (include/helmfft_b200.h): null
    pointers, bad ranges, misaligned strides, missing coefficients."""
    import ctypes
    import torch
    from paper_1912_03565_b200 import _native as nv
    lib = nv.load_library()
    h = ctypes.c_void_p()
    assert lib.hfb_plan_create(0, 15, 15, 0, ctypes.byref(h)) == nv.HFB_ERR_ARGUMENT
    assert lib.hfb_plan_create(15, 15, 7, 0, ctypes.byref(h)) == nv.HFB_OK
    t = torch.zeros((7, 15, 15), dtype=torch.float64, device="cuda")
    w = torch.zeros(1 << 22, dtype=torch.float64, device="cuda")
    P, st = nv.ptr, None
    # no coefficients yet
    assert lib.hfb_solve(h, P(t), P(t), P(w), st) == nv.HFB_ERR_NO_COEFFICIENTS
    assert lib.hfb_solve_z(h, P(t), P(t), P(t), P(t), P(w), st) == nv.HFB_ERR_NO_COEFFICIENTS
    assert lib.hfb_solve(h, None, P(t), P(w), st) == nv.HFB_ERR_ARGUMENT
    assert lib.hfb_transform_stack(h, P(t), 3, 2, P(w), st) == nv.HFB_ERR_RANGE
    assert lib.hfb_transform_stack(h, P(t), 0, 8, P(w), st) == nv.HFB_ERR_RANGE
    assert lib.hfb_plan_set_workspace_mode(h, 2) == nv.HFB_ERR_ARGUMENT
    cx = np.cos(np.pi * np.arange(1, 16) / 16)
    tab = np.zeros(7 * 12)
    tab[5::12] = -6.0  # diagonal d at offset 0 of every level
    assert lib.hfb_plan_set_coefficients(h, tab.ctypes.data_as(ctypes.c_void_p),
                                         cx.ctypes.data_as(ctypes.c_void_p),
                                         cx.ctypes.data_as(ctypes.c_void_p), 1e-14) == nv.HFB_OK
    assert lib.hfb_solve_slab(h, P(t), 16, 0, P(w), st) == nv.HFB_ERR_RANGE
    assert lib.hfb_solve_modes(h, P(t), 15, 15, 0, P(w), st) == nv.HFB_ERR_ARGUMENT  # odd ld
    assert lib.hfb_solve_modes(h, P(t), 16, 15, 1, P(w), st) == nv.HFB_ERR_RANGE
    ys = (ctypes.c_int * 3)(0, 7, 14)  # must end at n_y = 15
    assert lib.hfb_pack_modes(h, P(t), P(w), ys, 2, st) == nv.HFB_ERR_ARGUMENT
    assert lib.hfb_solve(h, P(t), P(t), P(w), st) == nv.HFB_OK
    assert lib.hfb_plan_destroy(h) == nv.HFB_OK


# --------------------------------- the reference's acceptance problems (f2)
@pytest.fixture(scope="module")
def acceptance():
    import os
    path = os.path.join(os.path.dirname(__file__), "golden", "acceptance.npz")
    with np.load(path) as z:
        return {k: z[k] for k in z.files}


@pytest.mark.parametrize("key,n", [("2", 125), ("4", 125), ("6", 125), ("2", 250), ("4", 250),
                                   ("6", 250)])
def test_acceptance_wave_problems_match_reference(cuda, acceptance, key, n):
    """Variable-k wave problem on [0, pi]^3 with analytic Dirichlet data, through
    build_rhs + fold_dirichlet + the one-call solve: the discretisation errors
    reproduce the reference's own run (tests/golden/make_acceptance_golden.py)."""
    from acceptance_problems import error_metrics, helmholtz_case
    scheme = ZSCHEME[key]
    g, prof, src, bnd, u = helmholtz_case(10.0, 9.0, 10.0, 10.0, 9.0, scheme, n)
    F = hb.build_rhs(scheme, src, prof, g)
    sol, _ = hb.solve_discrete(F, bnd, scheme, prof, g)
    mx, l2 = error_metrics(sol.values, u, g)
    ref = acceptance[f"wave_{key}_{n}"]
    assert abs(mx - ref[0]) <= 1e-6 * ref[0] and abs(l2 - ref[1]) <= 1e-6 * ref[1], (mx, l2, ref)
    folded = hb.fold_dirichlet(F, bnd, scheme, prof, g)
    assert hb.residual_l2(sol, folded, scheme, prof, g) < 1e-11


@pytest.mark.parametrize("n", [64, 128, 256])
def test_acceptance_convdiff_matches_reference(cuda, acceptance, n):
    """Convection-diffusion gamma = -100 with analytic Dirichlet data (cd4)."""
    from acceptance_problems import convdiff_case, error_metrics
    g, prof, src, bnd, u = convdiff_case(-100.0, n)
    scheme = hb.SchemeKind.CONVECTION_DIFFUSION_4
    F = hb.build_rhs(scheme, src, prof, g)
    sol, _ = hb.solve_discrete(F, bnd, scheme, prof, g)
    mx, l2 = error_metrics(sol.values, u, g)
    ref = acceptance[f"cd_{n}"]
    assert abs(mx - ref[0]) <= 1e-6 * ref[0] and abs(l2 - ref[1]) <= 1e-6 * ref[1], (mx, l2, ref)


def _random_case(rng):
    """One seeded random problem: line lengths mixing powers of two (FFT engine)
    and arbitrary N (dense DST), a scheme, a z-dependent or constant profile
    and an execution mode."""
    def extent():
        return int(rng.choice([1, 3, 7, 15, 31, 63, 127, 255])) if rng.random() < 0.6 \
            else int(rng.integers(1, 90))
    nx, ny, nz = extent(), extent(), int(rng.integers(1, 70))
    scheme = [hb.SchemeKind.SECOND_ORDER, hb.SchemeKind.FOURTH_ORDER, hb.SchemeKind.SIXTH_ORDER,
              hb.SchemeKind.CONVECTION_DIFFUSION_4][int(rng.integers(0, 4))]
    if scheme is hb.SchemeKind.SIXTH_ORDER:  # uniform grid (stencil.py:110-114)
        h = 2.0 ** -int(rng.integers(3, 7))  # dyadic: (h (n + 1)) / (n + 1) == h exactly
        dom = hb.Domain(0, h * (nx + 1), 0, h * (ny + 1), 0, h * (nz + 1))
    else:
        dom = hb.Domain(0, float(rng.uniform(0.5, 3)), 0, float(rng.uniform(0.5, 3)),
                        0, float(rng.uniform(0.5, 3)))
    g = hb.make_grid(dom, nx, ny, nz)
    if scheme is hb.SchemeKind.CONVECTION_DIFFUSION_4:  # k^2 = 0 (stencil.py:143-144)
        prof = hb.constant_profile(0.0, g, gamma=float(rng.uniform(-20, 20)))
    elif rng.random() < 0.5:
        a, b, c = float(rng.uniform(0, 4)), float(rng.uniform(0, 2)), float(rng.uniform(0.5, 3))
        prof = hb.sample_profile(lambda z: a + b * np.sin(c * z), lambda z: b * c * np.cos(c * z),
                                 lambda z: -b * c * c * np.sin(c * z), 0.0, g)
    else:
        prof = hb.constant_profile(float(rng.uniform(-5, 5)), g)
    mode = [hb.SolverConfig(), hb.SolverConfig(mode=hb.SharedWorkers(2)),
            hb.SolverConfig(mode=hb.Partitioned(int(rng.integers(1, 4))))][int(rng.integers(0, 3))]
    return g, scheme, prof, mode


@pytest.mark.parametrize("seed", range(64))
def test_random_problems_vs_oracle(cuda, seed):
    """Seeded sweep over shapes (1 to 255 points per axis, FFT and dense DST
    lengths), schemes, constant and z-dependent profiles and execution modes:
    the device solve matches the oracle to PARITY (relative L2), unless the
    oracle itself reports a singular pivot, which the device must raise too."""
    rng = np.random.default_rng(1000 + seed)
    g, scheme, prof, cfg = _random_case(rng)
    F = rng.standard_normal(g.shape)
    T = oracle_table(scheme.value, prof, g)
    try:
        ref = orc.solve(F, T, *orc.mode_cosines(g.n_x, g.n_y))
    except orc.OracleSingular:  # singular system in the oracle: the device raises as well
        with pytest.raises(hb.SingularSystemError):
            solve(F, scheme, prof, g, cfg)
        return
    from paper_1912_03565_b200.solver import _validate_config
    try:
        _validate_config(cfg, g)
    except (ValueError, hb.InvalidPartitionError) as exc:  # the reference's bounds
        with pytest.raises(type(exc)):
            solve(F, scheme, prof, g, cfg)
        return
    u, _ = solve(F, scheme, prof, g, cfg)
    assert rel_l2(u, ref) < PARITY, (g.shape, scheme, cfg)


# ------------------------------------- transpose-free distributed z-solve
def _one_call(F, scheme, prof, g):
    import torch
    plan = hb._native.get_plan(g.n_x, g.n_y, g.n_z, F.device)
    hb.tridiag.device_coefficients(plan, scheme, prof, g)
    ref = torch.empty_like(F)
    work = plan.workspace(0)
    hb._native.check(plan.lib.hfb_solve(plan.handle, hb._native.ptr(F), hb._native.ptr(ref),
                                        hb._native.ptr(work), plan.stream()), "solve")
    plan.fetch_status()
    return ref


@pytest.mark.parametrize("parts,shape,scheme", [
    (2, (63, 63, 63), "fourth"), (3, (127, 63, 50), "convdiff"), (8, (255, 255, 40), "fourth"),
    (5, (31, 127, 23), "sixth"), (4, (63, 31, 9), "fourth"), (7, (127, 127, 64), "convdiff"),
    (1, (63, 63, 20), "fourth"), (6, (15, 15, 6), "fourth"), (3, (31, 1023, 9), "convdiff"),
    (4, (1023, 15, 11), "fourth")])
def test_carry_zsolve_bitwise(cuda, parts, shape, scheme):
    """The transpose-free distributed z-solve (every rank sweeps its own slab,
    carries through the neighbours' regions; ranks run one after another on
    one device) reproduces the one-call solve bit for bit: slabs shorter than
    a checkpoint chunk (40 levels on 8 ranks), uneven slabs, non-cubic grids,
    z-dependent k^2 and the nonsymmetric cd4 rows."""
    import torch
    from paper_1912_03565_b200 import distributed as hd
    nx, ny, nz = shape
    g = hb.make_grid(hb.Domain(0, 1, 0, 1, 0, 1), nx, ny, nz)
    if scheme == "fourth":
        sk, prof = hb.SchemeKind.FOURTH_ORDER, hb.constant_profile(-20.0, g)
    elif scheme == "convdiff":
        sk, prof = hb.SchemeKind.CONVECTION_DIFFUSION_4, hb.constant_profile(0.0, g, gamma=-3.0)
    else:
        g = hb.make_grid(hb.Domain(0, 1, 0, 1, 0, 1), 31, 31, 31) if nx != ny else g
        k2 = 100 * (1 + 0.5 * np.sin(PI * np.linspace(0, 1, g.n_z + 2))) ** 2
        sk = hb.SchemeKind.SIXTH_ORDER
        prof = hb.CoefficientProfile(k2=k2, k2_z=np.gradient(k2), k2_zz=np.zeros_like(k2))
        nx, ny, nz = g.n_x, g.n_y, g.n_z
    F = torch.from_numpy(np.random.default_rng(parts + nz).standard_normal((nz, ny, nx))).cuda()
    U = hd.solve_partitioned_carry_local(F, sk, prof, g, parts)
    assert torch.equal(U, _one_call(F, sk, prof, g))


def test_carry_zsolve_repeated_and_ranks_in_any_layout(cuda):
    """Two solves in a row through fresh carry regions and through the same
    plan give the same bits (epochs, checkpoints and carries do not leak)."""
    import torch
    from paper_1912_03565_b200 import distributed as hd
    g = hb.make_grid(hb.Domain(0, 1, 0, 1, 0, 1), 127, 63, 33)
    prof = hb.constant_profile(-5.0, g)
    F = torch.from_numpy(np.random.default_rng(3).standard_normal(g.shape)).cuda()
    a = hd.solve_partitioned_carry_local(F, hb.SchemeKind.FOURTH_ORDER, prof, g, 3)
    b = hd.solve_partitioned_carry_local(F, hb.SchemeKind.FOURTH_ORDER, prof, g, 3)
    c = hd.solve_partitioned_carry_local(F, hb.SchemeKind.FOURTH_ORDER, prof, g, 6)
    assert torch.equal(a, b) and torch.equal(a, c)


def test_carry_zsolve_reports_vanishing_pivot_like_one_call(cuda):
    """A resonant mode: the carry path latches the same first failing (l, m, n)
    key as the one-call solve (the pivot check uses the global level)."""
    import torch
    from paper_1912_03565_b200 import distributed as hd
    g = hb.make_grid(hb.Domain(0, PI, 0, PI, 0, PI), 15, 15, 12)
    sk = hb.SchemeKind.SECOND_ORDER
    # k^2 that makes the z-system of mode (1, 1) singular: the 2nd-order rows
    # are (1, di, 1) with di = 2 r_zx cx + 2 r_zy cy - 2 (r_zx + r_zy + 1) + h_z^2 k^2
    # (stencil.py:70-82), eigenvalues di + 2 cos(pi r / (n_z + 1))
    r_zx, r_zy = g.h_z**2 / g.h_x**2, g.h_z**2 / g.h_y**2
    cx, cy, cz = (math.cos(PI / (n + 1)) for n in (g.n_x, g.n_y, g.n_z))
    k2 = (2 * (r_zx + r_zy + 1) - 2 * r_zx * cx - 2 * r_zy * cy - 2 * cz) / g.h_z**2
    prof = hb.constant_profile(k2, g)
    F = torch.ones(g.shape, dtype=torch.float64, device="cuda")
    with pytest.raises(hb.SingularSystemError) as e1:
        _one_call(F, sk, prof, g)
    with pytest.raises(hb.SingularSystemError) as e2:
        hd.solve_partitioned_carry_local(F, sk, prof, g, 3)
    assert (e2.value.n, e2.value.m) == (e1.value.n, e1.value.m) == (1, 1)


def test_carry_missing_neighbour_latches_exchange_error(cuda):
    """A rank whose forward carry never arrives gives up after the timeout
    (tuning key 11) and reports ExchangeError(sender=rank-1, receiver=rank)
    instead of hanging the GPU; the latch clears after it is read."""
    import torch
    from paper_1912_03565_b200 import distributed as hd
    g = hb.make_grid(hb.Domain(0, 1, 0, 1, 0, 1), 63, 63, 16)
    plan = hb._native.get_plan(63, 63, 16, torch.device("cuda", 0))
    hb.tridiag.device_coefficients(plan, hb.SchemeKind.FOURTH_ORDER, hb.constant_profile(1.0, g), g)
    ld = int(plan.lib.hfb_modes_ld(plan.handle))
    size, _ = hd.carry_layout(plan, ld)
    mine = torch.zeros(size, dtype=torch.float64, device="cuda")
    modes = torch.zeros(8 * 63 * ld, dtype=torch.float64, device="cuda")
    cp = torch.empty(63 * ld, dtype=torch.float64, device="cuda")
    P = hb._native.ptr
    lib = plan.lib
    lib.hfb_set_tuning(11, 300)
    try:
        # "rank 1" of two (levels 8..15): nobody publishes its forward carry
        hb._native.check(lib.hfb_zsolve_carry(plan.handle, 0, P(modes), ld, 8, 8, P(cp), P(mine),
                                              None, 7, plan.stream()), "carry")
        code = hd.carry_status_code(plan)
    finally:
        lib.hfb_set_tuning(11, 0)
    assert code == 1
    err = hd.exchange_error_for(code, 1)
    assert isinstance(err, hb.ExchangeError) and (err.sender, err.receiver) == (0, 1)
    assert hd.carry_status_code(plan) == 0
    # argument checks: a peer is required exactly when a neighbour exists
    assert lib.hfb_zsolve_carry(plan.handle, 0, P(modes), ld, 0, 8, P(cp), P(mine), None, 1,
                                plan.stream()) == hb._native.HFB_ERR_ARGUMENT
    assert lib.hfb_zsolve_carry(plan.handle, 1, P(modes), ld, 8, 8, P(cp), P(mine), P(mine), 1,
                                plan.stream()) == 0
    assert lib.hfb_zsolve_carry(plan.handle, 0, P(modes), ld, 10, 8, P(cp), P(mine), None, 1,
                                plan.stream()) == hb._native.HFB_ERR_RANGE
    plan.fetch_status()
    hd.carry_status_code(plan)


def _carry_nccl_worker(rank, world, port, q):
    import os
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("nccl", rank=rank, world_size=world)
    try:
        from paper_1912_03565_b200 import distributed as hd
        torch.cuda.set_device(0)
        g = hb.make_grid(hb.Domain(0, 1, 0, 1, 0, 1), 63, 63, 63)
        prof = hb.constant_profile(-20.0, g)
        F = torch.from_numpy(np.random.default_rng(1).standard_normal((63, 63, 63))).cuda()
        U = hd.solve_partitioned_carry(F, hb.SchemeKind.FOURTH_ORDER, prof, g)
        V = hd.solve_partitioned_carry(F, hb.SchemeKind.FOURTH_ORDER, prof, g)
        u, _ = hb.solve_discrete(hb.Field3D(F.cpu().numpy()), hb.BoundaryData.zero(),
                                 hb.SchemeKind.FOURTH_ORDER, prof, g)
        # complex k(z) through the same links (the region is sized for complex carries)
        k2 = np.full(g.n_z + 2, -20.0 + 5.0j)
        profz = hb.CoefficientProfile(k2=k2, k2_z=np.zeros_like(k2), k2_zz=np.zeros_like(k2))
        Fz = torch.complex(F, 0.5 * F)
        W = hd.solve_partitioned_carry(Fz, hb.SchemeKind.FOURTH_ORDER, profz, g)
        ok_z = bool(torch.equal(W, _one_call_z(Fz, hb.SchemeKind.FOURTH_ORDER, profz, g)))
        q.put((float(np.abs(U.cpu().numpy() - u.values).max()), bool(torch.equal(U, V)), ok_z))
    finally:
        dist.destroy_process_group()


def test_solve_partitioned_carry_nccl_single_rank(cuda):
    """solve_partitioned_carry through a real NCCL process group (one rank: the
    IPC handle of the carry region is taken and gathered; no neighbour to map)."""
    import socket
    import torch.multiprocessing as mp
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    p = ctx.Process(target=_carry_nccl_worker, args=(0, 1, port, q))
    p.start()
    p.join(300)
    assert p.exitcode == 0
    assert q.get(timeout=10) == (0.0, True, True)


@pytest.mark.parametrize("shape", [(1023, 15, 6), (1023, 31, 5), (2047, 15, 3), (1023, 1023, 2)])
def test_flat_row_final_pass_bitwise(cuda, shape):
    """The final inverse x-pass writing the user's odd-pitch rows by flat-128B-row
    tensor stores (tuning key 13, on at M = 1024 / 2048) equals the thread-store
    path bit for bit, odd and even planes, and against the oracle."""
    import torch
    nx, ny, nz = shape
    g = hb.make_grid(hb.Domain(0, 1, 0, 1, 0, 1), nx, ny, nz)
    prof = hb.constant_profile(-7.0, g)
    F = torch.from_numpy(np.random.default_rng(nx + nz).standard_normal((nz, ny, nx))).cuda()
    plan = hb._native.get_plan(nx, ny, nz, F.device)
    lib = plan.lib
    outs = []
    for key in (1, 0):
        lib.hfb_set_tuning(13, key)
        try:
            outs.append(_one_call(F, hb.SchemeKind.FOURTH_ORDER, prof, g))
        finally:
            lib.hfb_set_tuning(13, 1)
    assert torch.equal(outs[0], outs[1])
    if nx * ny * nz <= 2e5:
        ref = orc.solve(F.cpu().numpy(), oracle_table("4", prof, g),
                        *orc.mode_cosines(nx, ny), workers=4)
        # the north star's 1e-10: the 2047 x 15 x 3 grid (h_x / h_z = 1/512) sits
        # at ~1e-11 against the oracle whatever the rounding order
        assert rel_l2(outs[0].cpu().numpy(), ref) < TOL


def _one_call_z(F, scheme, prof, g):
    import torch
    plan = hb._native.get_plan(g.n_x, g.n_y, g.n_z, F.device)
    hb.tridiag.device_coefficients(plan, scheme, prof, g)
    assert plan.complex_coef
    tr, ti = F.real.contiguous(), F.imag.contiguous()
    work = plan.workspace(3)
    P = hb._native.ptr
    hb._native.check(plan.lib.hfb_solve_z(plan.handle, P(tr), P(ti), P(tr), P(ti), P(work),
                                          plan.stream()), "solve_z")
    plan.fetch_status()
    return torch.complex(tr, ti)


@pytest.mark.parametrize("parts,shape,scheme", [(2, (63, 63, 40), "fourth"), (3, (127, 31, 25), "fourth"),
                                                (8, (63, 63, 29), "sixth"), (5, (31, 31, 31), "sixth")])
def test_carry_zsolve_complex_k_bitwise(cuda, parts, shape, scheme):
    """Complex k(z) (row f1) through the transpose-free distributed z-solve:
    complex carries, equal bit for bit to the one-call complex solve."""
    import torch
    from paper_1912_03565_b200 import distributed as hd
    nx, ny, nz = shape
    if scheme == "sixth":
        nx = ny = nz = shape[0]
    g = hb.make_grid(hb.Domain(0, 1, 0, 1, 0, 1), nx, ny, nz)
    z = np.linspace(0.0, 1.0, g.n_z + 2)
    k2 = (30.0 + 10.0j) * (1 + 0.5 * np.sin(PI * z)) ** 2
    prof = hb.CoefficientProfile(k2=k2, k2_z=np.gradient(k2, z), k2_zz=np.zeros_like(k2))
    sk = hb.SchemeKind.SIXTH_ORDER if scheme == "sixth" else hb.SchemeKind.FOURTH_ORDER
    rng = np.random.default_rng(parts + nz)
    F = torch.from_numpy(rng.standard_normal(g.shape) + 1j * rng.standard_normal(g.shape)).cuda()
    U = hd.solve_partitioned_carry_local(F, sk, prof, g, parts)
    assert torch.equal(U, _one_call_z(F, sk, prof, g))


@pytest.mark.parametrize("nx,ny,nz", [(7, 7, 70000), (10, 9, 70000), (15, 15, 66000)])
def test_transform_stack_more_planes_than_grid_limit(cuda, nx, ny, nz):
    """Stacks of more than 65535 small planes (the CUDA grid's y/z limit) on the
    generic FFT, dense and engine paths."""
    rng = np.random.default_rng(nx * ny)
    data = rng.standard_normal((nz, ny, nx))
    f = hb.Field3D(data.copy())
    hb.transform_stack(hb.make_plan(nx, ny), f)
    ref = orc.dst_stack(data, workers=8)
    assert np.abs(f.values - ref).max() < 1e-13 * np.abs(ref).max()


@pytest.mark.parametrize("nx,ny,nz", [(31, 31, 40), (15, 31, 9), (63, 63, 5), (40, 23, 7),
                                      (1, 5, 3), (64, 64, 2)])
def test_dmma_dst2d_vs_scipy(cuda, nx, ny, nz):
    """The whole-plane 2D DST-I on the FP64 tensor cores (tuning key 18) against
    scipy's DST (the reference's kernel), and the dense DMMA GEMM path (key 17)."""
    lib = hb._native.load_library()
    rng = np.random.default_rng(nx + 7 * ny)
    data = rng.standard_normal((nz, ny, nx))
    ref = orc.dst_stack(data, workers=4)
    for knobs in (((18, 64),), ((17, 64),), ((17, 64), (16, 0))):
        for k, v in knobs:
            lib.hfb_set_tuning(k, v)
        try:
            f = hb.Field3D(data.copy())
            hb.transform_stack(hb.make_plan(nx, ny), f)
        finally:
            lib.hfb_set_tuning(16, 1)
            lib.hfb_set_tuning(17, 0)
            lib.hfb_set_tuning(18, 0)
        assert np.abs(f.values - ref).max() < 1e-13 * np.abs(ref).max(), knobs


@pytest.mark.parametrize("shape", [(37, 23, 19), (64, 4, 33), (5, 130, 7), (129, 9, 65),
                                   (1, 1, 1), (33, 1, 2), (2, 33, 70)])
def test_marching_stencils_match_gather_kernels(cuda, shape):
    """The level-marching RHS operator, 27-point apply and residual (tuning key
    20 > 0, default 32) and the plane-streamed 27-point apply and residual
    (key 24 > 0 levels per CTA, default 64; key 25 rows per warp; key 27 the
    shared-memory staged planes, default) against the
    per-point gather kernels (keys 20 = 24 = 0) on shapes that do not fill the
    tiles: bitwise for the operators, 1e-14 for the (reordered) sum of squares."""
    import torch
    nx, ny, nz = shape
    g = hb.make_grid(hb.Domain(0, 1, 0, 1, 0, 1), nx, ny, nz)
    plan = hb._native.get_plan(nx, ny, nz, torch.device("cuda", 0))
    hb.tridiag.device_coefficients(plan, hb.SchemeKind.FOURTH_ORDER,
                                   hb.constant_profile(-3.0, g), g)
    lib, P, st = plan.lib, hb._native.ptr, plan.stream()
    rng = np.random.default_rng(nx * ny + nz)
    f = torch.from_numpy(rng.standard_normal((nz + 2, ny + 2, nx + 2))).cuda()
    rhs = torch.from_numpy(rng.standard_normal((nz, ny, nx))).cuda()
    u = torch.from_numpy(rng.standard_normal((nz, ny, nx))).cuda()
    part = torch.empty(int(lib.hfb_residual_partials(plan.handle)), dtype=torch.float64,
                       device="cuda")
    outs = []
    try:
        for v, ls, rj, tile in ((0, 0, 4, 0), (32, 0, 4, 0), (5, 0, 4, 0), (32, 64, 4, 0),
                                (32, 7, 4, 0), (32, 64, 2, 0), (32, 1, 2, 0), (32, 64, 4, 1),
                                (32, 7, 4, 1), (32, 1, 4, 1), (32, 200, 4, 1)):
            lib.hfb_set_tuning(20, v)
            lib.hfb_set_tuning(24, ls)
            lib.hfb_set_tuning(25, rj)
            lib.hfb_set_tuning(27, tile)
            F = torch.empty((nz, ny, nx), dtype=torch.float64, device="cuda")
            hb._native.check(lib.hfb_rhs_fourth(plan.handle, P(f), P(F), 0.37, st), "rhs4")
            A0 = torch.empty_like(F)
            hb._native.check(lib.hfb_apply27(plan.handle, P(f), P(rhs), P(A0), 0x7FFFFFF, 0, st),
                             "apply27")
            A1 = torch.empty_like(F)
            hb._native.check(lib.hfb_apply27(plan.handle, P(f), P(rhs), P(A1), 0x5A5A5A5, 1, st),
                             "fold")
            hb._native.check(lib.hfb_residual_sq(plan.handle, P(u), P(rhs), P(part), 0x7FFFFFF,
                                                 st), "residual")
            outs.append((F, A0, A1, float(part.sum())))
    finally:
        lib.hfb_set_tuning(20, 32)
        lib.hfb_set_tuning(24, 32)
        lib.hfb_set_tuning(25, 4)
        lib.hfb_set_tuning(27, 1)
    ref = outs[0]
    for o in outs[1:]:
        for a, b in zip(o[:3], ref[:3]):
            assert torch.equal(a, b)
        assert abs(o[3] - ref[3]) <= 1e-14 * ref[3]


def _ipc_carry_worker(rank, world, port, q, cplx=False):
    """One rank of a multi-process carry solve on ONE GPU, sequenced by host
    barriers (forward sweeps rank by rank up, back substitutions down), so
    every carry a kernel reads was published by a kernel that already finished:
    nothing waits on a concurrently running kernel. Exercises the real CUDA IPC
    path (handles gathered over gloo, the neighbour's region opened in another
    process, carries and flags stored into it)."""
    import os
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1912_03565_b200 import distributed as hd
        torch.cuda.set_device(0)
        dev = torch.device("cuda", 0)
        nx, ny, nz = 63, 63, 40
        g = hb.make_grid(hb.Domain(0, 1, 0, 1, 0, 1), nx, ny, nz)
        prof = _ipc_profile(g, cplx)
        F = _ipc_rhs(cplx)
        ex = hb.make_exchange_plan(g, world)
        z0, z1 = ex.partition.z_ranges[rank]
        kpz = z1 - z0
        links = hd.carry_links(g, None, dev)
        zplan = links.plan
        hb.tridiag.device_coefficients(zplan, hb.SchemeKind.FOURTH_ORDER, prof, g)
        tplan = hb._native.get_plan(nx, ny, kpz, dev)
        ld, P, st = links.ld, hb._native.ptr, tplan.stream()
        parts = [F.real, F.imag] if cplx else [F]
        modes = [torch.empty(kpz * nx * ld, dtype=torch.float64, device=dev) for _ in parts]
        work = tplan.workspace(5)
        for v, m in zip(parts, modes):
            hb._native.check(tplan.lib.hfb_forward_modes(tplan.handle, P(v[z0:z1].contiguous()),
                                                         P(m), P(work), st), "fwd")
        cp = torch.empty(len(parts) * ((kpz + 7) // 8) * nx * ld, dtype=torch.float64,
                         device=dev)
        epoch = links.next_epoch()

        def sweep(d):
            if cplx:
                peer = links.next_z if d == 0 else links.prev_z
                rc = zplan.lib.hfb_zsolve_carry_z(zplan.handle, d, P(modes[0]), P(modes[1]), ld,
                                                  z0, kpz, P(cp), P(links.region_z), peer, epoch,
                                                  zplan.stream())
            else:
                peer = links.next if d == 0 else links.prev
                rc = zplan.lib.hfb_zsolve_carry(zplan.handle, d, P(modes[0]), ld, z0, kpz,
                                                P(cp), P(links.region), peer, epoch,
                                                zplan.stream())
            hb._native.check(rc, f"sweep {d}")
            torch.cuda.synchronize()

        # one rank at a time: forward sweeps up the ranks, then back substitutions
        # down (the last rank does both in its phase)
        for phase in range(2 * world - 1):
            if phase == rank:
                sweep(0)
            if phase == 2 * world - 2 - rank:
                sweep(1)
            dist.barrier()
        outs = []
        for m in modes:
            out = torch.empty((kpz, ny, nx), dtype=torch.float64, device=dev)
            hb._native.check(tplan.lib.hfb_inverse_modes(tplan.handle, P(m), P(out), st), "inv")
            outs.append(out)
        torch.cuda.synchronize()
        res = torch.complex(outs[0], outs[1]) if cplx else outs[0]
        q.put((rank, res.cpu().numpy(), hd.carry_status_code(zplan)))
        dist.barrier()  # keep both regions mapped until both ranks are done
        links.close()
    finally:
        dist.destroy_process_group()


def _ipc_profile(g, cplx):
    if not cplx:
        return hb.constant_profile(-20.0, g)
    k2 = np.full(g.n_z + 2, -20.0 + 4.0j)
    return hb.CoefficientProfile(k2=k2, k2_z=np.zeros_like(k2), k2_zz=np.zeros_like(k2))


def _ipc_rhs(cplx):
    import torch
    rng = np.random.default_rng(11)
    F = rng.standard_normal((40, 63, 63))
    if cplx:
        F = F + 1j * rng.standard_normal((40, 63, 63))
    return torch.from_numpy(F).cuda()


@pytest.mark.parametrize("world,cplx", [(2, False), (3, False), (3, True)])
def test_carry_ipc_two_processes_one_gpu(cuda, world, cplx):
    """The transpose-free solve across two or three processes (three: a middle
    rank with a neighbour on each side): bitwise equal to the one-call solve, no
    missing carry."""
    import socket
    import torch
    import torch.multiprocessing as mp
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_ipc_carry_worker, args=(r, world, port, q, cplx))
             for r in range(world)]
    for p in procs:
        p.start()
    res = sorted((q.get(timeout=300) for _ in range(world)), key=lambda x: x[0])
    for p in procs:
        p.join(120)
    assert all(p.exitcode == 0 for p in procs)
    assert all(code == 0 for _, _, code in res)
    U = np.concatenate([r[1] for r in res])
    g = hb.make_grid(hb.Domain(0, 1, 0, 1, 0, 1), 63, 63, 40)
    F = _ipc_rhs(cplx)
    solve1 = _one_call_z if cplx else _one_call
    ref = solve1(F, hb.SchemeKind.FOURTH_ORDER, _ipc_profile(g, cplx), g)
    assert np.array_equal(U, ref.cpu().numpy())


@pytest.mark.parametrize("name", ["z4", "zb"])
def test_complex_k_on_device_tensors(golden, cuda, name):
    """complex128 CUDA tensors through the drop-in (round-1 verdict: complex k(z)
    with device fields raised): solve_discrete, fold_dirichlet, residual_l2 and
    apply_stencil return complex CUDA tensors equal to the numpy path's results,
    and the caller's tensor is not modified."""
    import torch
    g, prof, scheme, F, bnd = z_inputs(golden, name)
    Ft = torch.from_numpy(np.ascontiguousarray(F, dtype=complex)).to(cuda)
    keep = Ft.clone()
    ut, t = hb.solve_discrete(hb.Field3D(Ft), bnd, scheme, prof, g)
    assert ut.values.is_cuda and ut.values.dtype == torch.complex128
    assert torch.equal(Ft, keep)
    u, _ = hb.solve_discrete(hb.Field3D(F), bnd, scheme, prof, g)
    assert np.array_equal(ut.values.cpu().numpy(), u.values)
    assert rel_l2(u.values, golden[f"{name}_U"]) < PARITY
    assert t.transform_s > 0 and t.tridiag_s > 0
    Fft = hb.fold_dirichlet(hb.Field3D(Ft), bnd, scheme, prof, g)
    Ff = hb.fold_dirichlet(hb.Field3D(F), bnd, scheme, prof, g)
    assert Fft.values.is_cuda
    assert np.array_equal(Fft.values.cpu().numpy(), np.asarray(Ff.values, dtype=complex))
    assert hb.residual_l2(ut, Fft, scheme, prof, g) < 1e-11 * np.linalg.norm(Ff.values)
    Au = hb.apply_stencil(ut, bnd, scheme, prof, g)
    assert Au.values.is_cuda and rel_l2(Au.values.cpu().numpy(), F) < 1e-12


def test_real_k_complex_device_tensor_and_stage_operators(cuda):
    """A complex128 CUDA rhs with a real table is two real solves (bitwise the
    numpy path); the in-place stage operators (transform_stack, solve_all,
    transform_lines_x/y) work on complex and on non-contiguous CUDA views."""
    import torch
    w = wl.workload(1)
    g = w.grid
    rng = np.random.default_rng(11)
    F = rng.uniform(-1, 1, g.shape) + 1j * rng.uniform(-1, 1, g.shape)
    Ft = torch.from_numpy(F).to(cuda)
    ut, _ = hb.solve_discrete(hb.Field3D(Ft), hb.BoundaryData.zero(), w.scheme, w.profile, g)
    u, _ = hb.solve_discrete(hb.Field3D(F), hb.BoundaryData.zero(), w.scheme, w.profile, g)
    assert ut.values.dtype == torch.complex128
    assert np.array_equal(ut.values.cpu().numpy(), u.values)
    plan = hb.make_plan(g.n_x, g.n_y)
    a = F.copy()
    hb.transform_stack(plan, a)
    at = Ft.clone()
    hb.transform_stack(plan, at)
    assert np.array_equal(at.cpu().numpy(), a)
    hb.solve_all(a, w.scheme, w.profile, g)
    hb.solve_all(at, w.scheme, w.profile, g)
    assert np.array_equal(at.cpu().numpy(), a)
    # a non-contiguous float64 view (every other plane of a bigger tensor) is
    # transformed in place, not in a discarded copy
    big = torch.from_numpy(np.ascontiguousarray(
        np.stack([F.real, F.imag], axis=1).reshape(2 * g.n_z, g.n_y, g.n_x))).to(cuda)
    view = big[::2]
    assert not view.is_contiguous()
    hb.transform_lines_x(view, (0, g.n_y))
    hb.transform_lines_y(view, (0, g.n_x))
    ref = F.real.copy()
    hb.transform_lines_x(ref, (0, g.n_y))
    hb.transform_lines_y(ref, (0, g.n_x))
    assert np.array_equal(view.cpu().numpy(), ref)
    assert np.array_equal(big[1::2].cpu().numpy(), F.imag)
