"""The wavefront-fused z-solve (tuning key 21; measured slower, off by default —
DESIGN.md §8): forward elimination inside the y-pass, back substitution inside
the inverse y-pass, carries through L2 between the items of consecutive levels. It must equal the five-launch schedule (key 21 = 0) BIT FOR BIT — the
same expressions — on every shape class, and raise the same singular mode."""
import math

import numpy as np
import pytest

import paper_1912_03565_b200 as hb
from oracle import helm_oracle as orc
from paper_1912_03565_b200 import _native
from paper_1912_03565_b200.tridiag import device_coefficients

pytestmark = pytest.mark.gpu


def solve_with(key21, F, scheme, prof, g, cuda):
    import torch
    lib = _native.load_library()
    lib.hfb_set_tuning(21, key21)
    try:
        plan = _native.get_plan(g.n_x, g.n_y, g.n_z, cuda)
        device_coefficients(plan, scheme, prof, g)
        X = torch.from_numpy(np.ascontiguousarray(F)).to(cuda)
        Y = torch.empty_like(X)
        work = plan.workspace(0)
        _native.check(lib.hfb_solve(plan.handle, _native.ptr(X), _native.ptr(Y),
                                    _native.ptr(work), plan.stream()), "solve")
        plan.fetch_status()
        return Y.cpu().numpy()
    finally:
        lib.hfb_set_tuning(21, 0)


@pytest.mark.parametrize("nx,ny,nz", [(1023, 1023, 9), (511, 511, 20), (255, 511, 33),
                                      (2047, 1023, 5), (63, 1023, 17), (1023, 511, 1),
                                      (127, 1023, 2), (15, 511, 64)])
@pytest.mark.parametrize("scheme", ["cd4", "6", "table"])
def test_wave_equals_five_launch_schedule(cuda, nx, ny, nz, scheme):
    h = 1.0 / (max(nx, ny, nz) + 1)
    g = hb.make_grid(hb.Domain(0, h * (nx + 1), 0, h * (ny + 1), 0, h * (nz + 1)), nx, ny, nz)
    rng = np.random.default_rng(nx * 7 + ny * 3 + nz)
    F = rng.standard_normal(g.shape)
    if scheme == "cd4":
        sch, prof = hb.SchemeKind.CONVECTION_DIFFUSION_4, hb.constant_profile(0.0, g, gamma=-1.5)
    elif scheme == "6":
        z = g.z_nodes(closed=True)
        k2 = 400.0 * (1 + 0.3 * np.sin(2 * math.pi * z)) ** 2
        prof = hb.CoefficientProfile(k2=k2.astype(complex), k2_z=np.zeros_like(z, complex),
                                     k2_zz=np.zeros_like(z, complex))
        sch = hb.SchemeKind.SIXTH_ORDER
    else:
        from paper_1912_03565_b200 import workloads as wl
        sch, prof = wl.general_table(nz), hb.constant_profile(0.0, g)
    a = solve_with(1, F, sch, prof, g, cuda)
    b = solve_with(0, F, sch, prof, g, cuda)
    assert np.array_equal(a, b)
    if nx * ny * nz <= 4e6:
        T = (orc.weight_table(scheme, np.real(prof.k2), np.real(prof.k2_z), np.real(prof.k2_zz),
                              complex(prof.gamma).real, (g.h_x, g.h_y, g.h_z), nz)
             if scheme != "table" else (sch.A, sch.B, sch.C, sch.D))
        ref = orc.solve(F, T, *orc.mode_cosines(nx, ny), workers=8)
        assert np.linalg.norm(a - ref) / np.linalg.norm(ref) < 1e-10


def test_wave_repeat_solves_bitwise(cuda):
    """Level counters are reset per solve: repeated solves give the same bits."""
    g = hb.make_grid(hb.Domain(0, 1, 0, 1, 0, 1), 255, 511, 40)
    F = np.random.default_rng(1).standard_normal(g.shape)
    prof = hb.constant_profile(0.0, g, gamma=-1.5)
    outs = [solve_with(1, F, hb.SchemeKind.CONVECTION_DIFFUSION_4, prof, g, cuda) for _ in range(3)]
    assert np.array_equal(outs[0], outs[1]) and np.array_equal(outs[1], outs[2])


def test_wave_singular_mode_reported(cuda):
    """A resonant mode raises SingularSystemError with the same (n, m) as the
    five-launch schedule (first failing row l, then m, then n)."""
    g = hb.make_grid(hb.Domain(0, math.pi, 0, math.pi, 0, math.pi), 15, 511, 4)
    r_zx, r_zy = g.h_z**2 / g.h_x**2, g.h_z**2 / g.h_y**2
    cx, cy = orc.mode_cosines(15, 511)
    k2 = (2.0 * (r_zx + r_zy + 1.0) - 2.0 * r_zx * cx[1] - 2.0 * r_zy * cy[2]) / g.h_z**2
    prof = hb.constant_profile(k2, g)
    got = []
    for key in (1, 0):
        with pytest.raises(hb.SingularSystemError) as err:
            solve_with(key, np.ones(g.shape), hb.SchemeKind.SECOND_ORDER, prof, g, cuda)
        got.append((err.value.n, err.value.m))
    assert got[0] == got[1] == (2, 3)



@pytest.mark.parametrize("parts,shape", [(2, (127, 255, 40)), (3, (63, 511, 50)),
                                         (4, (255, 255, 64)), (8, (127, 127, 100)),
                                         (5, (1023, 1023, 20))])
def test_carry_protocol_live_cooperative(cuda, parts, shape):
    """The transpose-free multi-GPU z-solve's release/acquire protocol exercised
    LIVE: all virtual ranks' sweeps in one cooperative launch per direction
    (hfb_zsolve_carry_vranks), so consumer CTAs really spin while their producers
    run. Bit-identical to the one-call solve."""
    import torch
    from paper_1912_03565_b200 import distributed as hd
    nx, ny, nz = shape
    g = hb.make_grid(hb.Domain(0, 1, 0, 1, 0, 1), nx, ny, nz)
    prof = hb.constant_profile(0.0, g, gamma=-1.5)
    F = np.random.default_rng(parts * 31 + nz).standard_normal(g.shape)
    sch = hb.SchemeKind.CONVECTION_DIFFUSION_4
    one = solve_with(0, F, sch, prof, g, cuda)
    for _ in range(2):  # fresh regions and flags every call
        U = hd.solve_partitioned_carry_coop(torch.from_numpy(F).to(cuda), sch, prof, g, parts)
        assert np.array_equal(U.cpu().numpy(), one)
