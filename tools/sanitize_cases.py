"""Small solves that launch every hot kernel once, for compute-sanitizer runs
(SURVEY.md §5): racecheck / synccheck / memcheck on the mbarrier + TMA DST
engine (ROW, TLOAD, TRAN, flat-row tensor stores), the TMA and shared-memory
z-solves, the carry z-solve (virtual ranks in dependency order, one stream),
the DMMA whole-plane and batched transforms, the stencil kernels and the
complex path. Each case is checked against the oracle so a sanitizer run that
perturbs nothing still proves the kernels ran.

    compute-sanitizer --tool racecheck python tools/sanitize_cases.py
"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1912_03565_b200 as hb  # noqa: E402
from oracle import helm_oracle as orc  # noqa: E402
from paper_1912_03565_b200 import _native, distributed as hd, workloads as wl  # noqa: E402
from paper_1912_03565_b200.tridiag import device_coefficients  # noqa: E402

dev = torch.device("cuda", 0)
lib = _native.load_library()
worst = 0.0


def check(name, u, ref, tol=1e-10):
    global worst
    err = float(np.linalg.norm(np.asarray(u) - ref) / np.linalg.norm(ref))
    worst = max(worst, err)
    print(f"{name}: rel L2 {err:.2e}", flush=True)
    assert err < tol, name


def one_call(n_x, n_y, n_z, lean=False, inplace=False, tune=()):
    g = hb.make_grid(hb.Domain(0, 1, 0, 1, 0, 1), n_x, n_y, n_z)
    prof = hb.constant_profile(0.0, g, gamma=-1.5)
    F = np.random.default_rng(n_x + n_y + n_z).uniform(-1, 1, g.shape)
    for k, v in tune:
        lib.hfb_set_tuning(k, v)
    plan = _native.get_plan(n_x, n_y, n_z, dev)
    device_coefficients(plan, hb.SchemeKind.CONVECTION_DIFFUSION_4, prof, g)
    plan.set_workspace_mode(lean)
    X = torch.from_numpy(F).to(dev)
    Y = X if inplace else torch.empty_like(X)
    work = plan.workspace(0)
    _native.check(lib.hfb_solve(plan.handle, _native.ptr(X), _native.ptr(Y), _native.ptr(work),
                                plan.stream()), "solve")
    plan.fetch_status()
    plan.set_workspace_mode(False)
    z = np.zeros(n_z + 2)
    T = orc.weight_table("cd4", z, z, z, -1.5, (g.h_x, g.h_y, g.h_z), n_z)
    ref = orc.solve(F, T, *orc.mode_cosines(n_x, n_y), workers=4)
    check(f"one-call {n_x}x{n_y}x{n_z} lean={lean} inplace={inplace} tune={tune}",
          Y.cpu().numpy(), ref)
    for k, _ in tune:  # restore the defaults the library starts with
        lib.hfb_set_tuning(k, {19: 1}.get(k, 0))


def main():
    one_call(31, 31, 9)                            # DMMA 2D + shared-memory z-solve
    one_call(127, 127, 12, tune=((19, 0),))        # FFT engine ROW/TLOAD + TMA z-solve
    one_call(255, 127, 20)                         # flat-row tensor stores (odd pitch)
    one_call(255, 255, 6, lean=True, inplace=True)  # TRAN pass, lean in place
    one_call(2047, 63, 3)                          # M = 2048 column passes (256 threads)
    one_call(100, 36, 5)                           # dense (non power-of-two) DMMA products
    # carry z-solve, 3 virtual ranks in dependency order on one stream
    g = hb.make_grid(hb.Domain(0, 1, 0, 1, 0, 1), 63, 63, 30)
    prof = hb.constant_profile(0.0, g, gamma=-1.5)
    F = np.random.default_rng(3).uniform(-1, 1, g.shape)
    U = hd.solve_partitioned_carry_local(torch.from_numpy(F).to(dev),
                                         hb.SchemeKind.CONVECTION_DIFFUSION_4, prof, g, 3)
    z = np.zeros(32)
    T = orc.weight_table("cd4", z, z, z, -1.5, (g.h_x, g.h_y, g.h_z), 30)
    check("carry z-solve P=3", U.cpu().numpy(), orc.solve(F, T, *orc.mode_cosines(63, 63)))
    # stencil kernels: 4th-order RHS, fold with Dirichlet data, residual
    g = hb.make_grid(hb.Domain(0, 1, 0, 1, 0, 1), 30, 20, 10)
    prof = hb.constant_profile(3.0, g)
    rng = np.random.default_rng(5)
    B = hb.BoundaryData.from_array(rng.standard_normal((12, 22, 32)))
    rhs = hb.Field3D(rng.standard_normal(g.shape))
    u, _ = hb.solve_discrete(rhs, B, hb.SchemeKind.FOURTH_ORDER, prof, g)
    res = hb.residual_l2(u, hb.fold_dirichlet(rhs, B, hb.SchemeKind.FOURTH_ORDER, prof, g),
                         hb.SchemeKind.FOURTH_ORDER, prof, g)
    print(f"fold + solve + residual: {res:.2e}", flush=True)
    assert res < 1e-9
    # complex k(z)
    g = wl.unit_grid(15)
    k2 = (100.0 * (1 + 0.3j)) * np.ones(17)
    pz = hb.CoefficientProfile(k2=k2, k2_z=np.zeros(17, complex), k2_zz=np.zeros(17, complex))
    Fz = rng.standard_normal(g.shape) + 1j * rng.standard_normal(g.shape)
    uz, _ = hb.solve_discrete(hb.Field3D(Fz), hb.BoundaryData.zero(), hb.SchemeKind.FOURTH_ORDER,
                              pz, g)
    T = orc.weight_table("4", k2, np.zeros(17, complex), np.zeros(17, complex), 0.0,
                         (g.h_x, g.h_y, g.h_z), 15)
    check("complex k(z) 15^3", uz.values, orc.solve(Fz, T, *orc.mode_cosines(15, 15)))
    torch.cuda.synchronize()
    print(f"SANITIZE_CASES_OK worst rel L2 {worst:.2e}")


if __name__ == "__main__":
    main()
