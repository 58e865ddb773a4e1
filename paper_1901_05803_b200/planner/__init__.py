"""Planner surface: the reference `ralp` package's placement, partitioner and
cost-model API (pkg/src/ralp/__init__.py:3-91), restated from scratch."""
from .catalog import CATALOG_ENV_VAR, UnknownModelError, catalog_dir, catalog_lookup, catalog_names
from .costmodel import (CSV_HEADER, CostModelError, JobSpec, Strategy, StrategyKind, StrategyVolumes, VolumeRow,
                        compare_strategies, compute_load, gpu_assignments, rows_to_csv, rows_to_json,
                        volume_baseline, volume_ralp, volume_ralp_multi_ps, volume_ring, volumes_for)
from .descriptor import DescriptorError, ShapeMismatchError, parse_model, serialize_model
from .layers import (COMPUTE_DEMAND_KINDS, PARAMETERIZED_KINDS, LayerKind, LayerSpec, ModelError, ModelGraph,
                     TensorShape, conv_output_hw, infer_conv, infer_fc, infer_layer, infer_pool)
from .profiler import (ProfileReport, ProfilerConfig, ProfilerError, SkewnessMode, SplitChoice, compute_skewness,
                       find_split, gate_eligibility, profile)
