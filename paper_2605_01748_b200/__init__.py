"""GATE max-min-fair traffic-engineering solver, B200-native (sm_100a).

Drop-in for the reference package `pathfair`'s solve path (see DESIGN.md and
INTEGRATION.md): the same entry points -- build_instance, solve, SolverConfig,
SolveResult, the per-step kernels and the projection -- executed by
hand-written CUDA kernels behind a C ABI (include/pf_b200.h).
"""

from .controller import (IterationTrace, Residuals, SolveResult, Solver, SolverConfig, SolverError, adapt_beta,
                         advance_alpha, check_convergence, compute_residuals, initialize_state, solve)
from .harness import gravity_demands, gravity_table, k_shortest_paths, random_topology
from .kernels import (KernelError, SolverState, det_diff_norm, solve_commodity_sums, solve_sum_equation,
                      update_duals, update_rate_suggestions, update_rates, update_slacks, utility)
from .metrics import dao_carry_rates, dao_evaluate, default_theta, optimality_from_sums
from .model import (FEAS_TOL, Commodity, CommodityTable, FlatPathSet, InputError, Instance, PathSet, Topology,
                    ViolationReport, build_instance, build_instance_flat, build_instance_raw, build_topology, commodity_sums,
                    edge_loads, edge_loads_from_pairs, validate_allocation, with_conditions)
from .projection import project, score_paths

__all__ = [
    "FEAS_TOL", "Commodity", "CommodityTable", "FlatPathSet", "InputError", "Instance", "IterationTrace",
    "KernelError", "PathSet", "Residuals", "SolveResult", "Solver", "SolverConfig", "SolverError", "SolverState",
    "Topology", "ViolationReport", "adapt_beta", "advance_alpha", "build_instance", "build_instance_flat", "build_instance_raw",
    "build_topology", "check_convergence", "commodity_sums", "compute_residuals", "default_theta",
    "det_diff_norm", "edge_loads", "edge_loads_from_pairs", "gravity_demands", "gravity_table",
    "initialize_state", "k_shortest_paths", "optimality_from_sums", "project", "random_topology", "score_paths",
    "solve", "solve_commodity_sums", "solve_sum_equation", "update_duals", "update_rate_suggestions",
    "update_rates", "update_slacks", "utility", "validate_allocation", "with_conditions",
    "dao_carry_rates", "dao_evaluate",
]
