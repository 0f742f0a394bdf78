"""Small solves through every new kernel family for compute-sanitizer runs
(memcheck / racecheck): persistent half-length solve (all-on-chip and
three-vector layouts), half-length phase kernels, half-length four-step
engine, standalone operators."""
import os
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import oracle as O  # noqa: E402
import paper_2002_11978_b200 as P  # noqa: E402
from paper_2002_11978_b200 import workloads as WL  # noqa: E402


def solve(n, B):
    col, _, _ = O.ifl_column(1.5, 1.75, 1.0, n + 1)
    op = P.build_toeplitz(col)
    x, kx, fx, u0 = WL.instance_fields(n, 0, B)
    shift = 411.0
    kb = float(kx.mean())
    lev = P.LevelOperator(op, shift, kx)
    pc = P.build_preconditioner(col, shift, kb)
    rhs = fx + shift * u0
    xs, reps = P.solve_bicgstab(lev, pc, rhs, tol=1e-12)
    its = [r.iterations for r in (reps if isinstance(reps, list) else [reps])]
    y = P.toeplitz_matvec(op, rhs[0])
    z = P.precond_solve(pc, rhs[0])
    return its, float(np.linalg.norm(y)), float(np.linalg.norm(z))


for n, B in [(1024, 3), (512, 160), (4096, 2), (1 << 13, 1), (1 << 15, 2)]:
    print(n, B, solve(n, B), flush=True)
