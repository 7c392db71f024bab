"""B200-native kappa-cycle multigrid engine (arXiv 2010.00626).

Drop-in for the hot path of the reference package `kcycle`
(/root/reference/pkg/src/kcycle/__init__.py:18-88): the same solver API names
and signatures (ProblemSpec, CycleConfig, build_state, run_cycle,
kappa_cycle, solve_standalone, pcg_solve, bench_cycle, ...), backed by
hand-written sm_100a CUDA kernels behind the C-ABI of include/kcb200.h.
There is no CPU numerics fallback: importing the package without the built
library fails, and creating a state without an sm_100 GPU raises
CudaUnavailableError.
"""

from ._native import CudaError, CudaUnavailableError
from .cycle import (
    BREAKDOWN,
    CONVERGED,
    DIVERGED,
    MAX_CYCLES,
    BenchResult,
    CudaGridState,
    CycleConfig,
    CycleStats,
    DryState,
    GridState,
    SolveReport,
    bench_cycle,
    build_state,
    f_cycle,
    gamma_cycle,
    kappa_cycle,
    run_cycle,
    solve_standalone,
)
from . import costmodel
from .krylov import PcgConfig, pcg_solve
from .mesh import Coarsening, HierarchySpec, build_hierarchy
from .smoother import SmootherKind, SmootherSpec
from .stencil import ProblemSpec, Stencil9, galerkin_coarsen, operator_hierarchy, rotated_anisotropic_stencil

__version__ = "0.1.0"
