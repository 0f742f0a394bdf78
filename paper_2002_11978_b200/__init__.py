"""B200-native FIDS per-time-step solve — a drop-in for the hot path of the
reference package `tsfrac` (arXiv 2002.11978).

Module layout and public names mirror tsfrac/__init__.py:11-63 for the
in-scope path (mesh, ifl, soe, toeplitz, krylov, scheme) and the acceptance
harness inputs (problems, couplings).  Device work goes
through the C ABI in include/tsfrac_b200.h (libtsfrac_b200.so, sm_100a).
"""

from .couplings import m_from_n, n_from_m, rate, temporal_exponent
from .ifl import IflDiscretization, build_ifl, normalization_constant
from .krylov import (KrylovReport, LevelOperator, MatrixFreeOperator, solve_bicgstab,
                     solve_cg, solve_dense)
from .mesh import GradedMesh, L1Weights, build_mesh, l1_weights
from .scheme import (FidsMarch, ProblemSpec, SeparableField, SolveReport, SolverOptions,
                     TimeStepSystem, run_dids, run_fids, run_fids_batched, select_solver)
from .problems import (CASE_NAMES, ManufacturedCase, exact_ifl_of_bump, example_source,
                       hypergeom_terminating, make_case)
from .soe import (FastHistory, SoeApproximation, SoeConstructionError, build_soe,
                  fast_caputo_rhs, fast_coefficients, history_push)
from .toeplitz import (CirculantPreconditioner, PreconditionerError, ToeplitzOperator,
                       build_preconditioner, build_toeplitz, precond_solve,
                       strang_first_column, toeplitz_matvec)

__version__ = "0.1.0"
