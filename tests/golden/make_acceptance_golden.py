"""Reference metrics of its own acceptance problems (test_acceptance.py:68-92):
max error and relative L2 error against the analytic solution, and the
algebraic residual, for the variable-k wave problem (schemes 2/4/6 at
125^3 and 250^3) and convection-diffusion with gamma = -100 (64^3, 128^3,
256^3). Build container only (imports the real reference):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_acceptance_golden.py
"""
import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
import helmfft as hf  # noqa: E402
from helmfft.assembly import build_rhs, fold_dirichlet, residual_l2  # noqa: E402
from helmfft.problems import convdiff_problem, error_metrics, helmholtz_problem  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def run(problem):
    u, _ = hf.solve_with_timings(problem, hf.SolverConfig(mode=hf.SharedWorkers(8)))
    mx, l2 = error_metrics(u, problem.analytic, problem.grid)
    rhs = build_rhs(problem.scheme, problem.source, problem.profile, problem.grid)
    folded = fold_dirichlet(rhs, problem.boundary, problem.scheme, problem.profile, problem.grid)
    res = residual_l2(u, folded, problem.scheme, problem.profile, problem.grid)
    return [mx, l2, res]


out = {}
for key, scheme in (("2", hf.SchemeKind.SECOND_ORDER), ("4", hf.SchemeKind.FOURTH_ORDER),
                    ("6", hf.SchemeKind.SIXTH_ORDER)):
    for n in (125, 250):
        out[f"wave_{key}_{n}"] = np.array(run(helmholtz_problem(10.0, 9.0, 10.0, 10.0, 9.0,
                                                                scheme, n)))
        print(key, n, out[f"wave_{key}_{n}"], flush=True)
for n in (64, 128, 256):
    out[f"cd_{n}"] = np.array(run(convdiff_problem(-100.0, n)))
    print("cd", n, out[f"cd_{n}"], flush=True)
np.savez(os.path.join(HERE, "acceptance.npz"), **out)
