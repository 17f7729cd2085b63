"""Complex k(z) golden cases (tests/golden/make_golden.py),
shared by the oracle tests and the GPU parity tests."""
import math

import numpy as np

from oracle import helm_oracle as orc


def z_grid(name):
    if name == "zb":
        return (0.0, 1.0, 0.0, 2.0, 0.0, 0.5), (15, 31, 9)
    if name.startswith("zd"):
        return (0.0, math.pi, 0.0, math.pi, 0.0, math.pi), (6, 6, 6)
    return (0.0, 1.0, 0.0, 1.0, 0.0, 1.0), (31, 31, 31)


def z_case(golden, name, key):
    """(F, closed boundary box or None, oracle table, h, cosines) of a complex golden case."""
    dom, (nx, ny, nz) = z_grid(name)
    h = ((dom[1] - dom[0]) / (nx + 1), (dom[3] - dom[2]) / (ny + 1), (dom[5] - dom[4]) / (nz + 1))
    k2 = golden[f"{name}_k2"]
    k2z = golden.get(f"{name}_k2z", np.zeros_like(k2))
    k2zz = golden.get(f"{name}_k2zz", np.zeros_like(k2))
    T = orc.weight_table(key, k2, k2z, k2zz, 0.0, h, nz)
    if name in ("z4", "z6"):
        rng = np.random.default_rng(101 if name == "z4" else 102)
        F = rng.standard_normal((31, 31, 31)) + 1j * rng.standard_normal((31, 31, 31))
    else:
        F = golden[f"{name}_F"]
    B = golden.get(f"{name}_B")
    return F, B, T, orc.mode_cosines(nx, ny)


def oracle_fold(F, B, T):
    if B is None:
        return F
    ext = np.array(B, dtype=complex)
    ext[1:-1, 1:-1, 1:-1] = 0.0
    return F - orc.accumulate27(ext, T)


