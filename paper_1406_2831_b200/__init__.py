"""paper_1406_2831_b200 — B200-native recycling BiCGSTAB hot path.

Drop-in for the solver / recycle-space names of krecycle
(/root/reference/pkg/src/krecycle/__init__.py:33-52) that lie on the hot path
(SURVEY.md §8): the arithmetic runs in libkrb.so (hand-written sm_100a CUDA,
C ABI in include/krb.h).  Everything else in the reference (CLI, Matrix
Market I/O, problem generators, bi-Lanczos harness) is out of scope.
"""

from .device import prefetch_matrix
from .operators import CountingOperator, as_operator
from .recycling import (CapturedCycle, RecycleSpace, biorthonormalize,
                        project_initial, project_initial_dual, refresh_images)
from .solvers import (BREAKDOWN_OMEGA, BREAKDOWN_SECOND_KIND,
                      BREAKDOWN_SERIOUS, CONVERGED, MAX_ITN,
                      ConvergenceHistory, SolverConfig, bicgstab_solve,
                      bicgstab_solve_batch, rbicg_solve, rbicgstab_solve,
                      rbicgstab_solve_batch)
from .update import update_recycle_space
from .sparse import SparseMatrix
from .ilutp import (FactorizationError, IlutpFactors, SplitPreconditionedOperator,
                    apply_left, apply_left_h, apply_right, apply_right_h, ilutp_factor,
                    permutation_matrix, to_operator_coords)

__version__ = "0.1.0"

__all__ = [
    "CountingOperator", "as_operator",
    "CapturedCycle", "RecycleSpace", "biorthonormalize", "project_initial",
    "project_initial_dual", "refresh_images",
    "ConvergenceHistory", "SolverConfig", "bicgstab_solve", "rbicgstab_solve",
    "rbicg_solve", "update_recycle_space",
    "rbicgstab_solve_batch", "bicgstab_solve_batch",
    "CONVERGED", "MAX_ITN", "BREAKDOWN_SERIOUS", "BREAKDOWN_OMEGA",
    "BREAKDOWN_SECOND_KIND",
    "SparseMatrix", "prefetch_matrix",
    "FactorizationError", "IlutpFactors", "SplitPreconditionedOperator",
    "apply_left", "apply_left_h", "apply_right", "apply_right_h", "ilutp_factor",
    "permutation_matrix", "to_operator_coords",
]
