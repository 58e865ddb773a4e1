"""B200-native execution of the resource-aware layer-placement (RALP) training step.

The planner surface (`profile`, `find_split`, `volume_ralp`, `JobSpec`, ...)
mirrors the reference `ralp` package (pkg/src/ralp/__init__.py); the training
step itself runs in libralpb200.so (hand-written sm_100a kernels) driven
through the C ABI in include/ralpb.h.
"""
from .planner import *  # noqa: F401,F403
from .planner import __dict__ as _planner_ns
from .report import JobReport, StepBreakdown  # noqa: F401
from .scenario import (DEFAULT_CLUSTER, CapacityError, ClusterSpec, Placement, Scenario,  # noqa: F401
                       ScenarioError, SimReport, parse_scenario, run_scenario, simulate_run, simulate_step,
                       spread_placement)
from .executor import RankExecutor, run_job  # noqa: F401

# The reference package's surface (pkg/src/ralp/__init__.py:46-91) minus its consolidation study
# (simulate_consolidation / ConsolidationReport: a what-if of the network simulator, out of scope),
# plus the executor.
__all__ = [
    "CapacityError", "ClusterSpec", "DEFAULT_CLUSTER", "DescriptorError", "JobSpec", "LayerKind", "LayerSpec",
    "ModelError", "ModelGraph", "Placement", "ProfileReport", "ProfilerConfig", "Scenario", "ScenarioError",
    "ShapeMismatchError", "SimReport", "SkewnessMode", "SplitChoice", "StepBreakdown", "Strategy", "StrategyKind",
    "StrategyVolumes", "TensorShape", "UnknownModelError", "catalog_lookup", "catalog_names", "compare_strategies",
    "compute_load", "compute_skewness", "find_split", "gate_eligibility", "infer_layer", "parse_model",
    "parse_scenario", "profile", "serialize_model", "simulate_run", "simulate_step", "spread_placement",
    "volume_baseline", "volume_ralp", "volume_ring",
    "JobReport", "RankExecutor", "run_job", "run_scenario",
]

__version__ = "0.1.0"
