"""B200-native hot path of the blocked one-sided hyperbolic J-Jacobi
eigensolver (arXiv 1008.4166), drop-in for the reference package ``hjacobi``'s
``parallel_jacobi`` / ``run_solver`` / ``solve_hermitian`` entry points (every
variant).  Kernels: libhjb200.so (sm_100a); no CPU fallback.
"""

from .blocking import BlockPartition, greedy_partition, num_blocks, uniform_partition
from .core import EigenResult, as_matrix, as_signs
from .errors import (
    ChannelTimeoutError,
    DefinitenessError,
    HJacobiError,
    NonConvergenceError,
    PivotDefinitenessError,
    RankDeficiencyError,
    SingularMatrixError,
    StructuralError,
)
from .factorization import (FactoredForm, accept_external_factor, factorize_hermitian_indefinite,
                            order_by_inertia, scaled_condition, scaled_condition_factor)
from .matio import MatrixFormatError, read_matrix, read_matrix_pinned, read_signs, write_matrix, write_signs
from .sequential import BlockMessage, apply_rotation, block_oriented, full_block, jacobi_diagonalize
from .parallel import SolverConfig, parallel_jacobi
from .rotations import (HYPERBOLIC, IDENTITY, TRIGONOMETRIC, DiagInfo, PlaneRotation, Tolerances,
                        compute_plane_rotation, extract_eigen, orthogonality)
from .solve import SolveOptions, run_solver, solve_hermitian
from .strategies import MODULUS, ROUND_ROBIN, generate_sweep_schedule, normalize_strategy, steps_per_sweep

__version__ = "0.1.0"

__all__ = [
    "BlockPartition", "ChannelTimeoutError", "DefinitenessError", "DiagInfo", "EigenResult",
    "HJacobiError", "MODULUS", "NonConvergenceError", "PivotDefinitenessError", "ROUND_ROBIN",
    "RankDeficiencyError", "SingularMatrixError", "SolverConfig", "StructuralError", "Tolerances",
    "as_matrix", "as_signs", "extract_eigen", "orthogonality", "generate_sweep_schedule", "greedy_partition",
    "normalize_strategy", "num_blocks", "parallel_jacobi", "steps_per_sweep", "uniform_partition",
    "FactoredForm", "accept_external_factor", "factorize_hermitian_indefinite", "order_by_inertia",
    "scaled_condition", "SolveOptions", "run_solver", "solve_hermitian",
    "PlaneRotation", "compute_plane_rotation", "TRIGONOMETRIC", "HYPERBOLIC", "IDENTITY",
    "scaled_condition_factor", "MatrixFormatError", "read_matrix", "read_matrix_pinned", "read_signs",
    "write_matrix", "write_signs", "BlockMessage", "apply_rotation", "block_oriented", "full_block",
    "jacobi_diagonalize",
]
