"""B200-native FIDS per-time-step solve — a drop-in for the hot path of the
reference package `tsfrac` (arXiv 2002.11978).

Module layout and public names mirror tsfrac/__init__.py:11-63 for the
in-scope path (mesh, ifl, soe, toeplitz, krylov, scheme).  The reference's
manufactured problems and resolution couplings (out of scope, SURVEY §2 rows
11-12) live with the tests (tests/harness/) that re-run its acceptance gate.
Device work goes
through the C ABI in include/tsfrac_b200.h (libtsfrac_b200.so, sm_100a).
"""

from .ifl import IflDiscretization, build_ifl, normalization_constant
from .krylov import (KrylovReport, LevelOperator, MatrixFreeOperator, solve_bicgstab,
                     solve_cg, solve_dense)
from .mesh import GradedMesh, L1Weights, build_mesh, l1_weights
from .scheme import (FidsMarch, ProblemSpec, SeparableField, SolveReport, SolverOptions,
                     TimeStepSystem, run_dids, run_fids, run_fids_batched, select_solver)
from .soe import (FastHistory, SoeApproximation, SoeConstructionError, build_soe,
                  fast_caputo_rhs, fast_coefficients, history_push)
from .toeplitz import (CirculantPreconditioner, PreconditionerError, ToeplitzOperator,
                       build_preconditioner, build_toeplitz, precond_solve,
                       strang_first_column, toeplitz_matvec)

__version__ = "0.1.0"
