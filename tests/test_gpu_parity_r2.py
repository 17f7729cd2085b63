"""Parity of the benchmarked configurations (round 2): cfg4 at its full 1023^3
through the bench's exact call, cfg5 on 2047^2 planes through the lean in-place
layout, and the general admissible table against the real reference.

All device work goes through the C-ABI. Tolerances: the north star's 1e-10
relative L2 against the oracle; against the reference's own summaries
(tests/golden/golden_r2.npz, make_golden_r2.py) the measured agreement is
~1e-14, asserted at 1e-11 (PARITY of test_gpu_parity.py).
"""
import os

import numpy as np
import pytest

import _r2cases as r2
import paper_1912_03565_b200 as hb
from oracle import helm_oracle as orc
from paper_1912_03565_b200 import _native, workloads as wl
from paper_1912_03565_b200.tridiag import device_coefficients

pytestmark = pytest.mark.gpu
TOL = 1e-10
PARITY = 1e-11


def rel_l2(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / np.linalg.norm(b))


def host_ram_gb():
    return os.sysconf("SC_PAGE_SIZE") * os.sysconf("SC_PHYS_PAGES") / 2**30


def test_cfg4_full_1023_bench_call(cuda):
    """cfg4 at its FULL 1023^3, exactly as bench.py times it: device-generated
    F (torch Philox, seed 4), hfb_solve into a separate U with the fast
    workspace, against the oracle on the same F (all host threads)."""
    import torch
    if host_ram_gb() < 80:
        pytest.fail(f"the 1023^3 oracle needs ~60 GB of host RAM; box has {host_ram_gb():.0f}")
    w = wl.workload(4)
    n = w.n
    lib = _native.load_library()
    plan = _native.get_plan(n, n, n, cuda)
    device_coefficients(plan, w.scheme, w.profile, w.grid)
    plan.set_workspace_mode(False)
    F = wl.device_rhs(w, cuda)
    U = torch.empty_like(F)
    work = plan.workspace(0)
    _native.check(lib.hfb_solve(plan.handle, _native.ptr(F), _native.ptr(U),
                                _native.ptr(work), plan.stream()), "solve")
    plan.fetch_status()
    del work
    Fh = F.cpu().numpy()
    Uh = U.cpu().numpy()
    del F, U
    torch.cuda.empty_cache()
    g = w.grid
    z = np.zeros(n + 2)
    T = orc.weight_table("cd4", z, z, z, -1.5, (g.h_x, g.h_y, g.h_z), n)
    ref = orc.solve(Fh, T, *orc.mode_cosines(n, n), workers=orc.default_workers())
    del Fh
    err = rel_l2(Uh, ref)
    print(f"cfg4 1023^3 full, bench call: rel L2 vs oracle {err:.3e}")
    assert err < TOL


def test_cfg5_slab_2047_lean_in_place(cuda, golden_r2):
    """cfg5 (general table, 2047^2 planes) on its first 16 planes through the
    layout the 2047^3 bench runs: lean workspace (hfb_plan_set_workspace_mode 1),
    in place (U = F). Against the oracle and the reference's summaries."""
    import torch
    F, T, (nx, ny, nz), scheme, prof, g = r2.case("cfg5s")
    lib = _native.load_library()
    plan = _native.get_plan(nx, ny, nz, cuda)
    device_coefficients(plan, scheme, prof, g)
    plan.set_workspace_mode(True)
    try:
        X = torch.from_numpy(F).to(cuda)
        work = plan.workspace(0)
        _native.check(lib.hfb_solve(plan.handle, _native.ptr(X), _native.ptr(X),
                                    _native.ptr(work), plan.stream()), "solve")
        plan.fetch_status()
        U = X.cpu().numpy()
    finally:
        plan.set_workspace_mode(False)
    ref = orc.solve(F, T, *orc.mode_cosines(nx, ny), workers=orc.default_workers())
    err = rel_l2(U, ref)
    errs = r2.summary_errors("cfg5s", U, golden_r2)
    print(f"cfg5 2047^2 x 16 lean in place: rel L2 vs oracle {err:.3e}; "
          f"vs reference summaries {errs}")
    assert err < TOL
    assert max(errs) < PARITY


def test_cfg5_slab_fast_layout_equals_lean(cuda):
    """The fast (two-volume) layout gives the same bits as the lean one at 2047^2."""
    import torch
    F, T, (nx, ny, nz), scheme, prof, g = r2.case("cfg5s")
    F = F[:9]
    g = r2.slab_grid(2047, 9)
    scheme = hb.StencilTable(*(t[:9] for t in T))
    out = []
    for lean in (False, True):
        plan = _native.get_plan(nx, ny, 9, cuda)
        device_coefficients(plan, scheme, r2.zero_profile(9), g)
        plan.set_workspace_mode(lean)
        X = torch.from_numpy(F.copy()).to(cuda)
        Y = torch.empty_like(X)
        work = plan.workspace(0)
        lib = _native.load_library()
        _native.check(lib.hfb_solve(plan.handle, _native.ptr(X), _native.ptr(Y),
                                    _native.ptr(work), plan.stream()), "solve")
        plan.fetch_status()
        plan.set_workspace_mode(False)
        out.append(Y.cpu().numpy())
    assert np.array_equal(out[0], out[1])


def test_general_table_63_full_vs_reference(cuda, golden_r2):
    F, T, _, scheme, prof, g = r2.case("gen63")
    u, _ = hb.solve_discrete(hb.Field3D(F), hb.BoundaryData.zero(), scheme, prof, g)
    err = rel_l2(u.values, golden_r2["gen63_U"])
    print(f"general table 63^3 vs reference: {err:.3e}")
    assert err < PARITY


@pytest.mark.parametrize("name", ["gen127", "cd4n127", "cfg4s"])
def test_benchmarked_schemes_vs_reference_summaries(cuda, golden_r2, name):
    F, T, (nx, ny, nz), scheme, prof, g = r2.case(name)
    u, _ = hb.solve_discrete(hb.Field3D(F), hb.BoundaryData.zero(), scheme, prof, g)
    errs = r2.summary_errors(name, u.values, golden_r2)
    ref = orc.solve(F, T, *orc.mode_cosines(nx, ny), workers=orc.default_workers())
    err = rel_l2(u.values, ref)
    print(f"{name}: vs oracle {err:.3e}, vs reference summaries {errs}")
    assert err < TOL
    assert max(errs) < PARITY


def test_cfg5_full_2047_residual(cuda):
    """cfg5 at its FULL 2047^3 (8.6e9 unknowns), the bench's lean in-place call:
    the relative residual ||A U - F|| / ||F|| of the 27-point system (the
    size-independent property; the 2047^3 oracle needs ~280 GB of host RAM).
    F (68.6 GB) is kept on the host across the solve, then re-uploaded next to U."""
    import torch
    if torch.cuda.get_device_properties(0).total_memory < 170e9 or host_ram_gb() < 120:
        pytest.fail("2047^3 needs a 180 GB B200 and >= 120 GB of host RAM")
    w = wl.workload(5)
    n = w.n
    lib = _native.load_library()
    plan = _native.get_plan(n, n, n, cuda)
    device_coefficients(plan, w.scheme, w.profile, w.grid)
    plan.set_workspace_mode(True)
    try:
        X = wl.device_rhs(w, cuda)
        nrm = float(torch.linalg.vector_norm(X).item())
        Fh = X.cpu()
        work = plan.workspace(0)
        _native.check(lib.hfb_solve(plan.handle, _native.ptr(X), _native.ptr(X),
                                    _native.ptr(work), plan.stream()), "solve")
        plan.fetch_status()
        del work
        torch.cuda.empty_cache()
    finally:
        plan.set_workspace_mode(False)
    Fd = Fh.to(cuda)
    del Fh
    res = hb.residual_l2(X, Fd, w.scheme, w.profile, w.grid)
    rel = res / nrm
    print(f"cfg5 2047^3 full, lean in place: relative residual {rel:.3e}")
    assert rel < 1e-12
    del X, Fd
    torch.cuda.empty_cache()


@pytest.mark.parametrize("shape,lean,inplace", [((1023, 1023, 9), False, False),
                                                ((255, 127, 20), False, False),
                                                ((255, 255, 6), True, True),
                                                ((2047, 63, 3), False, False),
                                                ((31, 31, 9), False, False),
                                                ((100, 36, 5), False, False)])
def test_guard_bands_untouched(cuda, shape, lean, inplace):
    """Out-of-bounds write check of the one-call solve (compute-sanitizer is closed
    on this pool): the input, output and workspace sit inside larger buffers whose
    guard bands (1 MiB before and after, NaN-filled) must come back unchanged,
    and the input must be unchanged when out of place."""
    import torch
    n_x, n_y, n_z = shape
    g = hb.make_grid(hb.Domain(0, 1, 0, 1, 0, 1), n_x, n_y, n_z)
    prof = hb.constant_profile(0.0, g, gamma=-1.5)
    lib = _native.load_library()
    plan = _native.get_plan(n_x, n_y, n_z, cuda)
    device_coefficients(plan, hb.SchemeKind.CONVECTION_DIFFUSION_4, prof, g)
    plan.set_workspace_mode(lean)
    try:
        G = 1 << 17  # doubles of guard band (1 MiB)
        vol = n_x * n_y * n_z
        F = np.random.default_rng(7).uniform(-1, 1, g.shape)
        fin = torch.full((vol + 2 * G,), float("nan"), dtype=torch.float64, device=cuda)
        fin[G:G + vol] = torch.from_numpy(F.ravel()).to(cuda)
        fout = fin if inplace else torch.full_like(fin, float("nan"))
        nws = int(lib.hfb_workspace_bytes(plan.handle, 0)) // 8
        ws = torch.full((nws + 2 * G,), float("nan"), dtype=torch.float64, device=cuda)
        X, Y, W = fin[G:G + vol], fout[G:G + vol], ws[G:G + nws]
        _native.check(lib.hfb_solve(plan.handle, _native.ptr(X), _native.ptr(Y), _native.ptr(W),
                                    plan.stream()), "solve")
        plan.fetch_status()
    finally:
        plan.set_workspace_mode(False)
    for buf in (fin, fout, ws):
        assert torch.isnan(buf[:G]).all() and torch.isnan(buf[-G:]).all()
    if not inplace:
        assert np.array_equal(X.cpu().numpy().reshape(g.shape), F)
    assert torch.isfinite(Y).all()


# ------------------------------------------- z-solve variants (round 2)
def _one_call(shape, scheme, seed, knobs, lean=False):
    """hfb_solve of a seeded F under tuning knobs; returns U on the host."""
    import torch
    nx, ny, nz = shape
    h = 1.0 / 64  # uniform spacing (the 6th-order scheme requires it)
    g = hb.make_grid(hb.Domain(0, (nx + 1) * h, 0, (ny + 1) * h, 0, (nz + 1) * h), nx, ny, nz)
    prof = hb.constant_profile(0.0, g, gamma=-1.5) if scheme == "cd4" else wl.profile_a(g)
    sk = hb.SchemeKind.CONVECTION_DIFFUSION_4 if scheme == "cd4" else hb.SchemeKind.SIXTH_ORDER
    lib = _native.load_library()
    plan = _native.get_plan(nx, ny, nz, torch.device("cuda", 0))
    device_coefficients(plan, sk, prof, g)
    plan.set_workspace_mode(lean)
    F = torch.from_numpy(np.random.default_rng(seed).standard_normal((nz, ny, nx))).cuda()
    U = F if lean else torch.empty_like(F)
    work = plan.workspace(0)
    try:
        for k, v in knobs:
            lib.hfb_set_tuning(k, v)
        _native.check(lib.hfb_solve(plan.handle, _native.ptr(F), _native.ptr(U),
                                    _native.ptr(work), plan.stream()), "solve")
        plan.fetch_status()
    finally:
        lib.hfb_set_tuning(23, 1)
        lib.hfb_set_tuning(26, 3)
        lib.hfb_set_tuning(28, 0)
        lib.hfb_set_tuning(30, 0)
        lib.hfb_set_tuning(31, 1)
        lib.hfb_set_tuning(19, 1)
        lib.hfb_set_tuning(29, 2)
    return U.cpu().numpy(), (F, sk, prof, g)


@pytest.mark.parametrize("shape", [(1023, 1023, 20), (255, 127, 9), (63, 300, 8), (33, 31, 1),
                                   (64, 513, 17), (127, 127, 300), (31, 600, 16)])
def test_zsolve_variants_bitwise(cuda, shape):
    """The one-call z-solve's variants are bitwise equal: the 3-stage TMA ring
    with dense x' rows (key 23 = 0, key 26 = 3) against sparse x' (key 23, x'
    stored once per 8-level chunk and recomputed in the back substitution) and
    the 4-stage ring (key 26 = 4), 128-mode blocks (key 28 = 1) and 16-level
    chunks with 3 or 2 stages (key 30 = 1, 2), and per-level eigenvalues for a
    z-invariant table (key 31 = 0; the cd4 cases here are z-invariant); shapes with n_z below, at and just above a
    chunk, partial mode blocks, many blocks per CTA; the small-n_z shared-memory
    kernel is switched off (key 19)."""
    scheme = "cd4" if shape[2] % 2 else "6"
    ref, _ = _one_call(shape, scheme, 7, [(19, 0), (23, 0), (26, 3)])
    for knobs in ([(19, 0), (23, 1), (26, 3)], [(19, 0), (23, 1), (26, 4)],
                  [(19, 0), (23, 0), (26, 4)], [(19, 0), (23, 1), (28, 1)],
                  [(19, 0), (23, 1), (30, 1)], [(19, 0), (23, 1), (30, 2)],
                  [(19, 0), (23, 0), (30, 2)], [(19, 0), (23, 1), (30, 1), (28, 1)],
                  [(19, 0), (23, 1), (31, 0)], [(19, 0), (23, 1), (31, 0), (30, 2)]):
        u, _ = _one_call(shape, scheme, 7, knobs)
        assert np.array_equal(u, ref), knobs


@pytest.mark.parametrize("shape", [(63, 127, 300), (255, 64, 257), (31, 600, 515)])
def test_checkpoint_cache_bitwise(cuda, shape):
    """Tuning key 32 (default on): the one-call z-solve keeps its cp checkpoints
    in a plan-owned array across solves with the same coefficients. Repeated
    solves (the second reads the cache), a change of chunk length or workspace
    layout (the cache is refilled) and a coefficient upload (the cache is
    invalidated) all give the bits of the uncached solve (key 32 = 0), on plans
    with n_z > 256 (below that the shared-memory z-solve needs no checkpoints)."""
    import torch
    nx, ny, nz = shape
    h = 1.0 / 64
    g = hb.make_grid(hb.Domain(0, (nx + 1) * h, 0, (ny + 1) * h, 0, (nz + 1) * h), nx, ny, nz)
    tables = [(hb.SchemeKind.SIXTH_ORDER, wl.profile_a(g)),
              (hb.SchemeKind.CONVECTION_DIFFUSION_4, hb.constant_profile(0.0, g, gamma=-1.5))]
    lib = _native.load_library()
    plan = _native.get_plan(nx, ny, nz, torch.device("cuda", 0))
    F = torch.from_numpy(np.random.default_rng(5).standard_normal((nz, ny, nx))).cuda()

    def solve(lean=False):
        plan.set_workspace_mode(lean)
        X = F.clone()
        U = X if lean else torch.empty_like(F)
        work = plan.workspace(0)
        work.fill_(0x7f)  # the workspace's own checkpoint planes are scratch either way
        _native.check(lib.hfb_solve(plan.handle, _native.ptr(X), _native.ptr(U),
                                    _native.ptr(work), plan.stream()), "solve")
        plan.fetch_status()
        return U.cpu().numpy()

    try:
        refs = {}
        for t, (sk, prof) in enumerate(tables):  # uncached references
            lib.hfb_set_tuning(32, 0)
            device_coefficients(plan, sk, prof, g)
            refs[t] = solve()
            refs[t, "lean"] = solve(lean=True)
        lib.hfb_set_tuning(32, 1)
        for t in (0, 1, 0):  # every upload invalidates what the last table cached
            device_coefficients(plan, *tables[t], g)
            assert np.array_equal(solve(), refs[t]), ("fill", t)
            assert np.array_equal(solve(), refs[t]), ("cached", t)
            lib.hfb_set_tuning(30, 1)  # 16-level chunks: other checkpoints, refilled
            assert np.array_equal(solve(), refs[t]), ("16-level chunks", t)
            assert np.array_equal(solve(), refs[t]), ("16-level chunks, cached", t)
            lib.hfb_set_tuning(30, 0)
            assert np.array_equal(solve(), refs[t]), ("8-level chunks again", t)
            assert np.array_equal(solve(lean=True), refs[t, "lean"]), ("lean layout", t)
            assert np.array_equal(solve(lean=True), refs[t, "lean"]), ("lean layout, cached", t)
            assert np.array_equal(solve(), refs[t]), ("fast layout again", t)
            _native.check(lib.hfb_plan_trim(plan.handle), "trim")  # cache freed, rebuilt
            assert np.array_equal(solve(), refs[t]), ("after hfb_plan_trim", t)
            assert np.array_equal(solve(), refs[t]), ("after hfb_plan_trim, cached", t)
    finally:
        lib.hfb_set_tuning(30, 0)
        lib.hfb_set_tuning(32, 1)
        plan.set_workspace_mode(False)


@pytest.mark.parametrize("shape,parts", [((127, 127, 16), 4), ((255, 511, 12), 8),
                                         ((1023, 1023, 8), 8), ((63, 63, 9), 2),
                                         ((2047, 511, 5), 4), ((511, 2047, 16), 8)])
def test_block_transforms_bitwise(cuda, shape, parts):
    """hfb_forward_blocks / hfb_inverse_blocks (the y-pass stores mode rows straight
    into the exchange blocks through a 5D tensor map; the inverse y-pass gathers
    its rows from the returned blocks) against forward_modes + pack_modes and
    unpack_modes + inverse_modes: the same bits in every valid block entry and in
    the solution planes, whole slabs and plane chunks, for every rank's slab."""
    import torch
    from paper_1912_03565_b200 import distributed as hd
    nx, ny, nz = shape
    g = hb.make_grid(hb.Domain(0, 1, 0, 1, 0, 1), nx, ny, nz)
    ex = hb.make_exchange_plan(g, parts)
    assert hd.fused_blocks(ex)
    rng = np.random.default_rng(17)
    kp = (ny + 1) // parts
    try:
        for rank in (0, parts - 1):
            z0, z1 = ex.partition.z_ranges[rank]
            kpz = z1 - z0
            if kpz == 0:
                continue
            slab = torch.from_numpy(rng.standard_normal((kpz, ny, nx))).cuda()
            back = torch.from_numpy(rng.standard_normal(kpz * nx * kp * parts)).cuda()

            def valid(buf, planes):  # drop the padding column of the last block
                return [buf.reshape(parts, planes, nx, kp)[q, :, :, :y1 - y0].cpu().numpy()
                        for q, (y0, y1) in enumerate(ex.partition.y_ranges)]

            res = {}
            for fused in (False, True):
                hd.FUSED_BLOCKS = fused
                send, modes = hd.forward_to_blocks(slab, g, ex, rank)
                out = hd.blocks_to_solution(back, modes, g, ex, rank)
                c0, c1 = kpz // 3, kpz  # a plane chunk through the chunked helpers
                m2 = torch.empty_like(modes)
                csend = hd.forward_chunk(slab, m2, g, ex, rank, c0, c1)
                cout = torch.zeros((kpz, ny, nx), dtype=torch.float64, device="cuda")
                hd.inverse_chunk(back[:(c1 - c0) * nx * kp * parts], m2, cout, g, ex, c0, c1)
                torch.cuda.synchronize()
                res[fused] = (valid(send, kpz), out.cpu().numpy(), valid(csend, c1 - c0),
                              cout.cpu().numpy())
            for a, b in zip(res[False], res[True]):
                if isinstance(a, list):
                    assert all(np.array_equal(x, y) for x, y in zip(a, b))
                else:
                    assert np.array_equal(a, b)
            assert np.isfinite(res[True][1]).all()
    finally:
        hd.FUSED_BLOCKS = True


def test_block_transforms_need_uniform_geometry(cuda):
    """Ragged exchange geometries (3 parts of 1023 modes) keep the pack path."""
    from paper_1912_03565_b200 import distributed as hd
    g = hb.make_grid(hb.Domain(0, 1, 0, 1, 0, 1), 1023, 1023, 9)
    assert not hd.fused_blocks(hb.make_exchange_plan(g, 3))
    assert hd.fused_blocks(hb.make_exchange_plan(g, 8))


@pytest.mark.parametrize("scheme", ["6", "cd4"])
def test_zsolve_default_vs_oracle(cuda, scheme):
    """The default z-solve (sparse x', guard-free interior chunks; for the
    z-invariant cd4 table the eigenvalues once per mode) against the oracle at a
    size that runs many blocks per CTA (1023^2 x 24; 6th order with k(z), cd4)."""
    u, (F, sk, prof, g) = _one_call((1023, 1023, 24), scheme, 11, [])
    T = orc.weight_table(scheme, np.real(prof.k2), np.real(prof.k2_z), np.real(prof.k2_zz),
                         np.real(prof.gamma), (g.h_x, g.h_y, g.h_z), g.n_z)
    ref = orc.solve(F.cpu().numpy(), T, *orc.mode_cosines(g.n_x, g.n_y),
                    workers=orc.default_workers())
    err = rel_l2(u, ref)
    print(f"default z-solve 1023^2 x 24 ({scheme}) vs oracle: {err:.3e}")
    assert err < TOL


@pytest.mark.parametrize("shape", [(1023, 1023, 9), (511, 255, 5), (2047, 2047, 3),
                                   (1023, 31, 17)])
def test_late_prefetch_bitwise(cuda, shape):
    """The DST passes' prefetch point (tuning key 29: before the batch, after
    its pre-processing for every pass, or for the flat-row-store passes only,
    the default) never changes a bit of the one-call solve."""
    ref, _ = _one_call(shape, "cd4", 3, [(29, 0)])
    for v in (1, 2):
        u, _ = _one_call(shape, "cd4", 3, [(29, v)])
        assert np.array_equal(u, ref), v
