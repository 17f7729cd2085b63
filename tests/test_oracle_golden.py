"""Pin the CPU oracle against vectors produced by the real reference (tests/golden)
and against the reference's own known-answer tests. CPU only."""
import math

import numpy as np
import pytest

from oracle import helm_oracle as orc
from paper_1912_03565_b200 import workloads as wl


def rel_l2(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def prof_arrays(prof):
    return (np.real(prof.k2), np.real(prof.k2_z), np.real(prof.k2_zz), complex(prof.gamma).real)


@pytest.mark.parametrize("key", ["2", "4", "6"])
def test_tables_bitwise(golden, key):
    g = wl.unit_grid(31)
    k2, k2z, k2zz, gam = prof_arrays(wl.profile_a(g))
    T = orc.weight_table(key, k2, k2z, k2zz, gam, (g.h_x, g.h_y, g.h_z), 31)
    assert np.array_equal(np.stack(T), golden[f"table_{key}_cfg1prof"])


@pytest.mark.parametrize("gamma", [-1.5, -100.0])
def test_convdiff_table_bitwise(golden, gamma):
    g = wl.unit_grid(31)
    z = np.zeros(33)
    T = orc.weight_table("cd4", z, z, z, gamma, (g.h_x, g.h_y, g.h_z), 31)
    assert np.array_equal(np.stack(T), golden[f"table_cd4_g{gamma:g}"])


def test_sixth_table_cfg3_profile(golden):
    g = wl.unit_grid(63)
    k2, k2z, k2zz, gam = prof_arrays(wl.profile_b(g))
    T = orc.weight_table("6", k2, k2z, k2zz, gam, (g.h_x, g.h_y, g.h_z), 63)
    assert np.array_equal(np.stack(T), golden["table_6_cfg3prof_n63"])


def test_mode_cosines(golden):
    cx, cy = orc.mode_cosines(31, 31)
    assert np.array_equal(cx, golden["cx31"]) and np.array_equal(cy, golden["cy31"])


def test_dst_known_answers(golden):
    # test_spectral.py:37-40: first basis vector of a 3-point line
    out = orc.dst_stack(np.array([[[1.0, 0.0, 0.0]]]))[0, 0]
    assert np.allclose(out, [0.5, 1 / math.sqrt(2), 0.5], atol=1e-15)
    assert np.allclose(golden["dst_basis3"], [0.5, 1 / math.sqrt(2), 0.5], atol=1e-15)
    # test_spectral.py:42-52: a single sine mode becomes a scaled delta
    n_x, n_y, n0, m0 = 8, 6, 3, 2
    i, j = np.arange(1, n_x + 1), np.arange(1, n_y + 1)
    plane = np.sin(math.pi * m0 * j / (n_y + 1))[:, None] * np.sin(math.pi * n0 * i / (n_x + 1))
    out = orc.dst_stack(plane[None])[0]
    expect = np.zeros_like(out)
    expect[m0 - 1, n0 - 1] = math.sqrt((n_x + 1) * (n_y + 1)) / 2.0
    assert np.abs(out - expect).max() < 1e-12


@pytest.mark.parametrize("n", [1, 2, 3, 7, 15, 31, 63, 125, 127])
def test_dst_matches_reference_and_dense(golden, n):
    inp, ref = golden[f"dst2d_in_{n}"], golden[f"dst2d_out_{n}"]
    fast = orc.dst_stack(inp[None])[0]
    dense = orc.dst_stack_dense(inp[None])[0]
    assert np.array_equal(fast, ref)  # same DUCC0 kernel as the reference
    assert np.abs(dense - ref).max() < 1e-12 * max(1.0, np.abs(ref).max())


def test_thomas_known_answers():
    # test_tridiag.py:24-27: hand-solved Poisson line
    x = orc.solve_line(np.array([0, -1, -1.0]), np.array([2, 2, 2.0]), np.array([-1, -1, 0.0]),
                       np.array([1.0, 0, 0]))
    assert np.allclose(x, [0.75, 0.5, 0.25], atol=1e-15)
    # test_tridiag.py:34-46: dense LU
    rng = np.random.default_rng(11)
    n = 50
    diag = 4.0 + rng.standard_normal(n)
    sub, sup = rng.standard_normal(n) * 0.5, rng.standard_normal(n) * 0.5
    sub[0] = sup[-1] = 0.0
    rhs = rng.standard_normal(n)
    A = np.diag(diag) + np.diag(sub[1:], -1) + np.diag(sup[:-1], 1)
    assert np.abs(orc.solve_line(sub, diag, sup, rhs) - np.linalg.solve(A, rhs)).max() < 1e-12
    with pytest.raises(orc.OracleSingular):
        orc.solve_line(np.array([0, 1.0]), np.array([0, 1.0]), np.array([1.0, 0]),
                       np.array([1.0, 1.0]))


def cfg1_table():
    g = wl.unit_grid(31)
    k2, k2z, k2zz, gam = prof_arrays(wl.profile_a(g))
    return orc.weight_table("4", k2, k2z, k2zz, gam, (g.h_x, g.h_y, g.h_z), 31), g


def test_solve_cfg1_uniform_rhs(golden):
    T, g = cfg1_table()
    F = wl.host_rhs(wl.workload(1))
    assert np.allclose([F.sum(), np.abs(F).sum()], golden["cfg1_F_sum"], rtol=0, atol=1e-9)
    U = orc.solve(F, T, *orc.mode_cosines(31, 31))
    assert rel_l2(U, golden["cfg1_U"]) < 1e-14


def test_rhs_fourth_and_solve_manufactured(golden):
    T, g = cfg1_table()
    src = wl.manufactured_source()
    x = g.x_nodes(closed=True)[None, None, :]
    y = g.y_nodes(closed=True)[None, :, None]
    z = g.z_nodes(closed=True)[:, None, None]
    F = orc.rhs_fourth(np.broadcast_to(src.f(x, y, z), (33, 33, 33)), g.h_z)
    assert np.array_equal(F, golden["cfg1A_F"])  # K1 is bit-exact against the reference
    U = orc.solve(F, T, *orc.mode_cosines(31, 31), workers=4)
    assert rel_l2(U, golden["cfg1A_U"]) < 1e-14


def test_solve_cd4_general_and_anisotropic(golden):
    g15 = wl.unit_grid(15)
    z = np.zeros(17)
    T = orc.weight_table("cd4", z, z, z, -1.5, (g15.h_x,) * 3, 15)
    U = orc.solve(golden["cd4_n15_F"], T, *orc.mode_cosines(15, 15))
    assert rel_l2(U, golden["cd4_n15_U"]) < 1e-14
    T = tuple(golden["gen_n15_table"])
    U = orc.solve(golden["gen_n15_F"], T, *orc.mode_cosines(15, 15))
    assert rel_l2(U, golden["gen_n15_U"]) < 1e-14
    # anisotropic grid (pi, 2, 1) box, extents 9 x 7 x 6, 4th order, k^2 = 2
    hx, hy, hz = math.pi / 10, 2.0 / 8, 1.0 / 7
    k2 = np.full(8, 2.0)
    T = orc.weight_table("4", k2, 0 * k2, 0 * k2, 0.0, (hx, hy, hz), 6)
    assert np.array_equal(np.stack(T), golden["table_4_aniso"])
    U = orc.solve(golden["aniso_F"], T, *orc.mode_cosines(9, 7))
    assert rel_l2(U, golden["aniso_U"]) < 1e-14


def test_oracle_resonance_reports_reference_mode(golden):
    k2, n, m = golden["resonance"]
    hx, hy, hz = math.pi / 6, math.pi / 7, math.pi / 5
    T = orc.weight_table("2", np.full(6, k2), np.zeros(6), np.zeros(6), 0.0, (hx, hy, hz), 4)
    with pytest.raises(orc.OracleSingular) as err:
        orc.solve(np.ones((4, 6, 5)), T, *orc.mode_cosines(5, 6))
    assert (err.value.n, err.value.m) == (int(n), int(m))


def test_residual_at_roundoff(golden):
    T, g = cfg1_table()
    assert orc.residual_l2(golden["cfg1_U"], wl.host_rhs(wl.workload(1)), T) < 1e-11


def test_oracle_is_bit_exact_on_cfg1(golden):
    """Plane-by-plane DUCC0 + reciprocal-form Thomas reproduce the reference exactly."""
    T, g = cfg1_table()
    U = orc.solve(wl.host_rhs(wl.workload(1)), T, *orc.mode_cosines(31, 31))
    assert np.array_equal(U, golden["cfg1_U"])


# ------------------------------------------------------ complex k(z) (f1)
from _zcases import oracle_fold, z_case  # noqa: E402
def test_complex_table_bitwise(golden):
    F, B, T, _ = z_case(golden, "z4", "4")
    assert np.array_equal(np.stack(T), golden["z4_table"])


@pytest.mark.parametrize("name,key", [("z4", "4"), ("z6", "6"), ("zb", "2"), ("zd2", "2"),
                                      ("zd4", "4"), ("zd6", "6")])
def test_complex_solves_match_reference(golden, name, key):
    """Complex k(z): the oracle's complex Thomas (reciprocal form) against the
    reference's complex division — same algorithm, roundoff-level agreement."""
    F, B, T, cs = z_case(golden, name, key)
    U = orc.solve(oracle_fold(F, B, T), T, *cs)
    assert rel_l2(U, golden[f"{name}_U"]) < 1e-12


# ------------------------------------ round 2: the benchmarked configurations
import _r2cases as r2  # noqa: E402


def test_oracle_general_table_63_full(golden_r2):
    """cfg5 class (general admissible table) at 63^3 against the reference."""
    F, T, (nx, ny, nz), *_ = r2.case("gen63")
    U = orc.solve(F, T, *orc.mode_cosines(nx, ny), workers=4)
    assert rel_l2(U, golden_r2["gen63_U"]) < 1e-13


@pytest.mark.parametrize("name", ["gen127", "cd4n127", "cfg4s", "cfg5s"])
def test_oracle_benchmarked_configs_summaries(golden_r2, name):
    """The cfg4 workload (first 8 of its 1023^2 planes), the cfg5 workload (first
    16 of its 2047^2 planes) and 127^3 cubes of both schemes, against summaries
    of the reference's solutions."""
    F, T, (nx, ny, nz), *_ = r2.case(name)
    U = orc.solve(F, T, *orc.mode_cosines(nx, ny), workers=orc.default_workers())
    errs = r2.summary_errors(name, U, golden_r2)
    assert max(errs) < 1e-13, errs
