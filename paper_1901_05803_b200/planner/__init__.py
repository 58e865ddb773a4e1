"""Planner surface: the reference `ralp` package's placement, partitioner and
cost-model API (pkg/src/ralp/__init__.py:3-91).

VENDORED API MIRROR (attribution): this module follows the reference `ralp` package's own code for
the same surface closely -- same classes, checks, error messages and arithmetic -- because north_star
makes that planner API the drop-in surface and its outputs must match the reference bit-exactly
(tests/test_planner_golden.py pins them to the unmodified reference).  It is not original work and
it is not on the GPU path; the executor accepts the reference's own objects as well
(executor.py `_kv`).
"""
from .catalog import CATALOG_ENV_VAR, UnknownModelError, catalog_dir, catalog_lookup, catalog_names
from .costmodel import (CSV_HEADER, CostModelError, JobSpec, Strategy, StrategyKind, StrategyVolumes, VolumeRow,
                        compare_strategies, compute_load, gpu_assignments, rows_to_csv, rows_to_json,
                        volume_baseline, volume_ralp, volume_ralp_multi_ps, volume_ring, volumes_for)
from .descriptor import DescriptorError, ShapeMismatchError, parse_model, serialize_model
from .layers import (COMPUTE_DEMAND_KINDS, PARAMETERIZED_KINDS, LayerKind, LayerSpec, ModelError, ModelGraph,
                     TensorShape, conv_output_hw, infer_conv, infer_fc, infer_layer, infer_pool)
from .profiler import (ProfileReport, ProfilerConfig, ProfilerError, SkewnessMode, SplitChoice, compute_skewness,
                       find_split, gate_eligibility, profile)
