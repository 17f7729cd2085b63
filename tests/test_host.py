"""Host-side logic of the drop-in package (no GPU): weight tables, partition and
exchange geometry, config validation, C-ABI table packing. Mirrors the
reference's test_stencil / test_solver structure."""
import math
import threading

import numpy as np
import pytest

import paper_1912_03565_b200 as hb
from paper_1912_03565_b200 import stencil, workloads as wl
from paper_1912_03565_b200.solver import _validate_config

PI = math.pi


@pytest.mark.parametrize("key,scheme", [("2", hb.SchemeKind.SECOND_ORDER),
                                        ("4", hb.SchemeKind.FOURTH_ORDER),
                                        ("6", hb.SchemeKind.SIXTH_ORDER)])
def test_tables_bitwise_equal_reference(golden, key, scheme):
    g = wl.unit_grid(31)
    T = hb.coefficient_table(scheme, wl.profile_a(g), g)
    assert all(t.dtype == np.float64 for t in T)
    assert np.array_equal(np.stack(T), golden[f"table_{key}_cfg1prof"])


@pytest.mark.parametrize("gamma", [-1.5, -100.0])
def test_convdiff_table_bitwise(golden, gamma):
    g = wl.unit_grid(31)
    T = hb.coefficient_table(hb.SchemeKind.CONVECTION_DIFFUSION_4,
                             hb.constant_profile(0.0, g, gamma=gamma), g)
    assert np.array_equal(np.stack(T), golden[f"table_cd4_g{gamma:g}"])


def test_sixth_table_cfg3_profile(golden):
    g = wl.unit_grid(63)
    T = hb.coefficient_table(hb.SchemeKind.SIXTH_ORDER, wl.profile_b(g), g)
    assert np.array_equal(np.stack(T), golden["table_6_cfg3prof_n63"])


def test_anisotropic_tables(golden):
    g = hb.make_grid(hb.Domain(0, PI, 0, 2.0, 0, 1.0), 9, 7, 6)
    p = hb.constant_profile(2.0, g)
    for key, s in (("2", hb.SchemeKind.SECOND_ORDER), ("4", hb.SchemeKind.FOURTH_ORDER)):
        assert np.array_equal(np.stack(hb.coefficient_table(s, p, g)), golden[f"table_{key}_aniso"])


def test_reference_scheme_objects_accepted():
    class Foreign:  # stands in for helmfft.SchemeKind.FOURTH_ORDER
        value = "4"
    g = wl.unit_grid(7)
    a = hb.coefficient_table(Foreign(), wl.profile_a(g), g)
    b = hb.coefficient_table(hb.SchemeKind.FOURTH_ORDER, wl.profile_a(g), g)
    assert all(np.array_equal(x, y) for x, y in zip(a, b))


def test_sixth_needs_uniform_grid():
    g = hb.make_grid(hb.Domain(0, 1, 0, 2, 0, 1), 4, 4, 4)
    with pytest.raises(hb.UnsupportedSchemeError):
        hb.coefficient_table(hb.SchemeKind.SIXTH_ORDER, hb.constant_profile(1.0, g), g)


def test_convdiff_needs_zero_k2():
    g = wl.unit_grid(5)
    with pytest.raises(ValueError):
        hb.coefficient_table(hb.SchemeKind.CONVECTION_DIFFUSION_4, hb.constant_profile(1.0, g), g)


def test_zero_row_sum_for_laplacian_schemes():
    """test_stencil.py:181-196: with k = 0 every row sums to zero (consistency)."""
    g = wl.unit_grid(9)
    for s in (hb.SchemeKind.SECOND_ORDER, hb.SchemeKind.FOURTH_ORDER, hb.SchemeKind.SIXTH_ORDER):
        for l in (1, 5, 9):
            assert abs(hb.coefficients_for(s, hb.constant_profile(0.0, g), g, l).row_sum()) < 1e-13


def test_general_table_is_diagonally_dominant():
    t = wl.general_table(64)
    off = 4 * np.abs(t.A).sum(1) + 2 * np.abs(t.B).sum(1) + 2 * np.abs(t.C).sum(1) \
        + np.abs(t.D[:, 0]) + np.abs(t.D[:, 2])
    assert np.allclose(t.D[:, 1], 1.5 * off)


def test_pack_table_layout_and_mask():
    g = wl.unit_grid(6)
    T = hb.coefficient_table(hb.SchemeKind.FOURTH_ORDER, wl.profile_a(g), g)
    packed = stencil.pack_table(T)
    assert packed.shape == (6 * 12,)
    l, k = 3, 2
    assert packed[l * 12 + k * 4:l * 12 + k * 4 + 4].tolist() == [T[i][l, k] for i in range(4)]
    mask = stencil.term_mask(T)
    # fourth order: corners only on the centre level, no x/y edges... check a few bits
    assert mask & (1 << (1 * 9 + 0)) and not mask & (1 << (0 * 9 + 0))
    assert mask & (1 << (0 * 9 + 8)) and mask & (1 << (2 * 9 + 4))


def test_pivot_threshold_matches_reference_rule():
    g = wl.unit_grid(8)
    T = hb.coefficient_table(hb.SchemeKind.FOURTH_ORDER, wl.profile_a(g), g)
    assert stencil.pivot_threshold(T) == 1e-14 * max(np.abs(t).max() for t in T)


# ------------------------------------------------------ partitions / exchange
def test_plan_partition_matches_reference_examples():
    assert [b - a for a, b in hb.plan_partition(10, 4)] == [3, 3, 2, 2]
    assert hb.plan_partition(8, 8) == [(i, i + 1) for i in range(8)]
    assert [b - a for a, b in hb.plan_partition(125, 2)] == [63, 62]
    assert [b - a for a, b in hb.plan_partition(1023, 8)] == [128] * 7 + [127]
    assert [b - a for a, b in hb.plan_partition(2047, 8)] == [256] * 7 + [255]
    for bad in ((4, 5), (4, 0)):
        with pytest.raises(hb.InvalidPartitionError):
            hb.plan_partition(*bad)


@pytest.mark.parametrize("parts", [2, 3, 4])
def test_exchange_plan_volume(parts):
    g = wl.unit_grid(9)
    ex = hb.make_exchange_plan(g, parts)
    z = [b - a for a, b in ex.partition.z_ranges]
    y = [b - a for a, b in ex.partition.y_ranges]
    for p in range(parts):
        for q in range(parts):
            assert ex.block_extents(p, q) == (9, y[q], z[p])
    assert ex.total_volume() == 9 ** 3


def _roundtrip(values, parts):
    nz, ny, nx = values.shape
    g = hb.make_grid(hb.Domain(0, 1, 0, 1, 0, 1), nx, ny, nz)
    ex = hb.make_exchange_plan(g, parts)
    mesh = hb.InProcessMesh(parts, timeout=10.0)
    out, slabs = np.empty_like(values), [None] * parts
    barrier = threading.Barrier(parts)

    def worker(p):
        z0, z1 = ex.partition.z_ranges[p]
        ys = hb.exchange_forward(ex, mesh.endpoint(p), p, values[z0:z1].copy())
        slabs[p] = ys.copy()
        barrier.wait()
        out[z0:z1] = hb.exchange_inverse(ex, mesh.endpoint(p), p, ys)

    th = [threading.Thread(target=worker, args=(p,)) for p in range(parts)]
    [t.start() for t in th]
    [t.join() for t in th]
    return out, slabs, ex


@pytest.mark.parametrize("parts", [2, 3, 4])
def test_exchange_roundtrip_and_transpose_oracle(parts):
    rng = np.random.default_rng(37)
    values = rng.standard_normal((8, 8, 5))
    out, slabs, ex = _roundtrip(values, parts)
    assert np.array_equal(out, values)
    for p, (y0, y1) in enumerate(ex.partition.y_ranges):
        assert np.array_equal(slabs[p], values[:, y0:y1, :])


def test_config_validation_mirrors_reference():
    g = wl.unit_grid(4)
    with pytest.raises(hb.InvalidPartitionError):
        _validate_config(hb.SolverConfig(mode=hb.SharedWorkers(5)), g)
    _validate_config(hb.SolverConfig(mode=hb.SharedWorkers(4),
                                     transform_parallelism=hb.PER_LINE_BATCH), g)
    with pytest.raises(hb.InvalidPartitionError):
        _validate_config(hb.SolverConfig(mode=hb.Partitioned(5)), g)
    with pytest.raises(hb.InvalidPartitionError):
        _validate_config(hb.SolverConfig(mode=hb.Partitioned(2, workers_per_part=3)), g)
    with pytest.raises(ValueError):
        _validate_config(hb.SolverConfig(transform_parallelism="per-point"), g)


def test_product_package_never_imports_the_oracle():
    import pathlib
    pkg = pathlib.Path(hb.__file__).parent
    for f in pkg.rglob("*.py"):
        text = f.read_text()
        assert "import oracle" not in text and "from oracle" not in text, f
        assert "helm_oracle" not in text, f


def test_no_gpu_means_no_solve():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    g = wl.unit_grid(3)
    with pytest.raises(hb.NativeUnavailableError):
        hb.solve_discrete(hb.Field3D(np.ones(g.shape)), hb.BoundaryData.zero(),
                          hb.SchemeKind.FOURTH_ORDER, hb.constant_profile(1.0, g), g)
