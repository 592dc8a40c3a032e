"""B200-native unsmoothed-aggregation AMG (arXiv 1302.2547) -- setup/solve path.

Drop-in for the setup/solve subset of the reference package ``uaamg``
(/root/reference/pkg/src/uaamg/__init__.py:3-38): same names, signatures,
defaults and exception types.  All numerical work runs in hand-written
sm_100a CUDA kernels in ``libuaamg_b200.so`` (C ABI: include/uaamg_b200.h);
there is no CPU fallback.
"""

from .aggregation import (Aggregation, AggregationConfig, AggregationError, aggregate, compose,
                          quasi_random_scores, select_coarse_vertices, singleton_aggregation)
from .analysis import TwoLevelReport, hierarchy_report, q_energy_norm, reports_to_csv, two_level_rate
from .device import DeviceCSR
from .graph import GraphError, GraphProblem, assemble_laplacian, assemble_laplacian_device, generate_structured_grid
from .hierarchy import CoarseSolver, Hierarchy, Level, SetupError, detect_singular, galerkin_coarse, setup
from .solvers import (CycleSpec, NumericalError, Smoother, SolveReport, cycle, npcg_solve, prolongate_add,
                      restrict, smooth, smoother_inverse_diag)
from .reshaping import DisconnectedPair, PairTooLarge, reshape_sweep
from .sparse import SparseFormatError, SparseMatrix, squared_adjacency_pattern

__version__ = "0.1.0"

__all__ = [
    "Aggregation", "AggregationConfig", "AggregationError", "aggregate", "compose", "quasi_random_scores",
    "select_coarse_vertices", "singleton_aggregation",
    "CoarseSolver", "Hierarchy", "Level", "SetupError", "detect_singular", "galerkin_coarse", "setup",
    "CycleSpec", "NumericalError", "Smoother", "SolveReport", "cycle", "npcg_solve", "prolongate_add", "restrict",
    "smooth", "smoother_inverse_diag",
    "SparseMatrix", "SparseFormatError", "DeviceCSR", "squared_adjacency_pattern",
    "reshape_sweep", "DisconnectedPair", "PairTooLarge",
    "TwoLevelReport", "hierarchy_report", "q_energy_norm", "reports_to_csv", "two_level_rate",
    "GraphError", "GraphProblem", "assemble_laplacian", "assemble_laplacian_device", "generate_structured_grid",
    "__version__",
]
