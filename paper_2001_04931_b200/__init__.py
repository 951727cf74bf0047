"""B200-native Evolutionary MPC hot path (arXiv 2001.04931), drop-in for the
EMPC / knot-parameterization names of the reference package ``knotmpc``
(K/__init__.py:68-85)."""

from .closedloop import ClosedLoopFleet, Controller, SimResult, actual_cost, compute_metrics, run_closed_loop
from .dynamics import (
    ContinuousLinearModel,
    DiscreteLinearModel,
    NLinkArm,
    NLinkParams,
    Pendulum,
    PendulumParams,
    discretize,
    integrate,
    linearize,
)
from .empc import (
    BatchResult,
    CostModel,
    EmpcBatch,
    EmpcResult,
    EmpcSettings,
    Population,
    evaluate_cost,
    evolve_generation,
    init_population,
    solve_empc,
)
from .param import (
    KnotSchedule,
    KnotTrajectory,
    expand,
    expand_batch,
    input_at,
    interp_coeffs,
    interpolation_matrix,
    knot_spacing,
)
from .spec import MpcSpec

__version__ = "0.1.0"

__all__ = [
    "BatchResult", "ClosedLoopFleet", "Controller", "Pendulum", "PendulumParams", "SimResult", "actual_cost",
    "compute_metrics", "integrate", "run_closed_loop", "ContinuousLinearModel", "CostModel", "DiscreteLinearModel", "EmpcBatch", "EmpcResult",
    "EmpcSettings", "KnotSchedule", "KnotTrajectory", "MpcSpec", "NLinkArm", "NLinkParams", "Population",
    "discretize", "evaluate_cost", "evolve_generation", "expand", "expand_batch", "init_population", "input_at",
    "interp_coeffs", "interpolation_matrix", "knot_spacing", "linearize", "solve_empc",
]
