"""B200-native (sm_100a) hot path of arXiv 1610.09146's `fdns` package.

The explicit 4th-order central-difference residual of the 3D compressible
Navier-Stokes equations (Taylor-Green vortex) in the paper's BL/RA/SN/SS
variants (plus RS), and the save-state RK3 update, as hand-written fp64 CUDA
kernels behind a C ABI (include/fdns_b200.h), with a Python host layer that
keeps the reference package's entry points:

    make_grid, PhysicalConstants, taylor_green_init, PLAN_NAMES, build_plan,
    ResidualEvaluator(...).evaluate, assemble_residual, RKScheme,
    rk_substep, advance_iteration, run, kinetic_energy_integral,
    enstrophy_integral, mean_density, make_collector

torch only owns device buffers and streams; there is no CPU fallback.
"""

from .mesh import (ConfigurationError, Field, Grid, halo_exchange,
                   live_field_count, make_grid, reduce_sum)
from .physics import (ConservativeState, PhysicalConstants, Residual,
                      SolverDivergenceError, eval_primitives_fused,
                      eval_primitives_grouped, heat_flux, skew_convective,
                      stress_tensor)
from .stencil import (cross_derivative, first_derivative, grid_weights,
                      make_weights, second_derivative)
from .plan import (PLAN_NAMES, KernelPlan, KernelSchedule, LoopGroup,
                   RaceViolation, ResidualEvaluator, assemble_residual,
                   build_plan, lower_plan, plan_storage,
                   validate_race_freedom, workarray_budget)
from .timeloop import (RK3_ALPHA, IterationState, RKScheme, RunReport,
                       advance_iteration, rk_substep, run)
from .diagnostics import (DiagnosticsRecord, conservation_sums,
                          enstrophy_integral, kinetic_energy_integral,
                          make_collector, mean_density, read_timeseries,
                          taylor_green_init, vorticity, write_timeseries)
from .decomp import Slab
from . import terms

__version__ = "0.1.0"
