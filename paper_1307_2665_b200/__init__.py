"""B200-native (sm_100a) build/solve hot path of the Gillman-Martinsson HPS direct solver.

Drop-in for the reference package's build/solve path (`hpsolve.grid`, `hpsolve.leafops`,
`hpsolve.solver`): same entry points, same arguments, same exceptions, and null-mode-invariant
results that match the reference. The arithmetic runs in hand-written CUDA (libhps_b200.so,
C ABI in include/hps_b200.h). There is no CPU fallback.
"""

from . import errors, grid, instrumentation, leafops, problems, solver  # noqa: F401
from .errors import ConfigError, LeafResonanceError, MergeResonanceError, SolverError  # noqa: F401
from .grid import BoxTree, GlobalNodeSet, Rectangle, build_tree  # noqa: F401
from .leafops import CoefficientField, LeafGeometry  # noqa: F401
from .solver import (Pipeline, SolverState, apply_global_dtn, boundary_flux_at, build,  # noqa: F401
                     gauge_fixed_solution, leaf_fields, memory_report, post_process, solve, solve_device)

__version__ = "0.1.0"
