"""B200-native DFS spectral Poisson solver on the unit sphere (sm_100a).

The compute path is libsk_poisson.so (hand-written CUDA, C ABI declared in
include/sk_poisson.h); this package is the host-side mirror of the
reference's spherekit Poisson interface (poisson.hpp) on top of it.
"""
from .poisson import (  # noqa: F401
    AssembleReport, BenchRow, DeviceError, LowRankSphereFun, PivotBlock, Plan, PoissonProblem, PoissonSolution, ResidualReport,
    UnsupportedError, analyze_2d, assemble_poisson, bench_poisson, ge_step, integration_weights, pivot_search,
    precondition_error, residual,
    sample_dfs, sample_grid, size_error, solve, solve_grid, solve_grid_exact, structure_error, coefficients_from_half,
    rhs_coefficients)

__version__ = "0.2.0"
